#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
specs=()
for zc in 0 2 4 12 16 48; do for sa in 0 1; do specs+=("SU3G_LINK_MODE=exact SU3G_LINK_ZC=$zc SU3G_LINK_SMEM_A=$sa|--workload link --dtype f64"); done; done
for zc in 0 4 16; do for sa in 0 1; do specs+=("SU3G_LINK_MODE=fma SU3G_LINK_ZC=$zc SU3G_LINK_SMEM_A=$sa|--workload link --dtype f64"); done; done
bash tools/gpu_ab_var.sh "${specs[@]}"
python tools/prof_nn64.py > gpurun_out/prof_nn64_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_nn_sweep|k_nn_tma64|k_dslash' -c 6 \
      -o gpurun_out/prof_nn64 python tools/prof_nn64.py > gpurun_out/ncu_nn64.log 2>&1
echo "ncu=$?" >> gpurun_out/status.txt
