#!/bin/bash
# Headline NN sweep (nn-weak f32, TMA t-walk): t-chunk length of the work items, 100-step runs.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do
for c in 0 8 4 2; do
  SU3G_NN_TMA_CHUNK=$c timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[chunk=$c] /" >> gpurun_out/chunk.txt
done; done
for c in 0 8; do
  SU3G_NN_TMA_CHUNK=$c ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_nn_tma -c 3 --csv python bench.py --steps 1 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/chunk_ncu_$c.csv 2>/dev/null
done
