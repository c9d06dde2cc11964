#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweeps.py -k "knobs" -q -p no:cacheprovider > gpurun_out/pytest_hints.log 2>&1
echo "pytest=$?" >> gpurun_out/status.txt
specs=()
for h in 0 1; do
  specs+=("SU3G_SWEEP_L2_HINTS=$h|--workload nn-weak --dtype f64")
  specs+=("SU3G_SWEEP_L2_HINTS=$h|--workload nn32 --dtype f64")
  specs+=("SU3G_SWEEP_L2_HINTS=$h|--workload dslash --dtype f32")
  specs+=("SU3G_SWEEP_L2_HINTS=$h|--workload dslash --dtype f64")
  specs+=("SU3G_SWEEP_L2_HINTS=$h|--workload nn-strong --dtype f64")
done
bash tools/gpu_ab_var.sh "${specs[@]}"
