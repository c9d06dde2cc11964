#!/bin/bash
# Small BASELINE configs (4096 / 65536 sites): CUDA-graph launches spread over concurrent branches.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for w in "routine:mult_su3_mat_vec --sites 4096" "routine:mult_su3_nn --sites 4096" "routine:mult_su3_mat_vec_sum_4dir --sites 65536"; do
for dt in f32 f64; do
for c in 1 2 4 8 16 32; do
  timeout 300 python bench.py --workload $w --dtype $dt --streams $c --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$w $dt streams=$c] /" >> gpurun_out/streams.txt
done; done; done
