#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
specs=()
for m in exact fma; do for mb in 3 4; do for pb in 0 1; do
  specs+=("SU3G_LINK_MODE=$m SU3G_LINK_MINB=$mb SU3G_LINK_PREFETCH_B=$pb|--workload link --dtype f64")
done; done; done
for pb in 0 1; do specs+=("SU3G_LINK_PREFETCH_B=$pb|--workload link --dtype f32"); done
bash tools/gpu_ab_var.sh "${specs[@]}"
python tools/prof_targets.py > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_link_rows|k_dslash|k_nn_tma' -c 3 \
      -o gpurun_out/prof_final python tools/prof_targets.py > gpurun_out/ncu_final.log 2>&1
echo "ncu=$?" >> gpurun_out/status.txt
