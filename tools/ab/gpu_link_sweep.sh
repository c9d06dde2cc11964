#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sitebuffer.py tests/test_gpu_sweeps.py -k "sitebuffer or link or randomize or uniform or routines_run or complex_views or load_round" -q -p no:cacheprovider > gpurun_out/pytest_sb.log 2>&1
echo "pytest_sb=$?" >> gpurun_out/status.txt
specs=()
for m in exact fma; do for mb in 3 4 5 6; do for ec in 0 1; do specs+=("SU3G_LINK_MODE=$m SU3G_LINK_MINB=$mb SU3G_LINK_EARLY_C=$ec|--workload link --dtype f64"); done; done; done
for mb in 4 6 8; do for ec in 0 1; do specs+=("SU3G_LINK_MINB=$mb SU3G_LINK_EARLY_C=$ec|--workload link --dtype f32"); done; done
bash tools/gpu_ab_var.sh "${specs[@]}"
