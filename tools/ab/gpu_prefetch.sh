#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_comm.py -q -p no:cacheprovider -x > gpurun_out/pytest_pf.log 2>&1
echo "pytest=$?" >> gpurun_out/status.txt
specs=()
for pf in 0 1 2 4 8; do
  specs+=("SU3G_SWEEP_PREFETCH=$pf|--workload nn-weak --dtype f64")
  specs+=("SU3G_SWEEP_PREFETCH=$pf|--workload dslash --dtype f32")
  specs+=("SU3G_SWEEP_PREFETCH=$pf|--workload link --dtype f64")
  specs+=("SU3G_SWEEP_PREFETCH=$pf SU3G_LINK_MODE=fma|--workload link --dtype f64")
done
bash tools/gpu_ab_var.sh "${specs[@]}"
