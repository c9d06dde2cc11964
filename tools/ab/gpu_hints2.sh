#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_p2p.py tests/test_gpu_comm.py -q -p no:cacheprovider > gpurun_out/pytest_hints.log 2>&1
echo "pytest=$?" >> gpurun_out/status.txt
specs=()
for h in 0 1; do
  specs+=("SU3G_LINK_L2_HINTS=$h|--workload link --dtype f64")
  specs+=("SU3G_LINK_L2_HINTS=$h SU3G_LINK_MODE=fma|--workload link --dtype f64")
  specs+=("SU3G_LINK_L2_HINTS=$h|--workload link --dtype f32")
done
specs+=("X=1|--workload nn-weak --dtype f64" "X=1|--workload nn32 --dtype f64" "X=1|--workload dslash --dtype f64")
bash tools/gpu_ab_var.sh "${specs[@]}"
