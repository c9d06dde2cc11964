#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -k "link" -q -p no:cacheprovider -x > gpurun_out/pytest_tile.log 2>&1
echo "pytest=$?" >> gpurun_out/status.txt
bash tools/gpu_ab_var.sh "SU3G_LINK_VARIANT=0|--workload link --dtype f64" "SU3G_LINK_VARIANT=7|--workload link --dtype f64" "SU3G_LINK_VARIANT=0 SU3G_LINK_MODE=fma|--workload link --dtype f64" "SU3G_LINK_VARIANT=7 SU3G_LINK_MODE=fma|--workload link --dtype f64" "SU3G_LINK_VARIANT=0|--workload link --dtype f32" "SU3G_LINK_VARIANT=7|--workload link --dtype f32"
