#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for m in exact fma; do
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --mode $m"
$CMD > gpurun_out/plain_$m.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_nn_tma -s 30 -c 1 -o gpurun_out/prof_tma_$m $CMD > gpurun_out/ncu_tma_$m.log 2>&1
done
echo done
