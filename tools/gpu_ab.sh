#!/bin/bash
# A/B two library builds on the same box: tools/gpu_ab.sh <alt.so> "<bench args>" ...
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
ALT=$1; shift
for rep in 1 2; do
for args in "${@}"; do
  python bench.py $args --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[cur $args] /" >> gpurun_out/ab.txt
  SU3G_LIB=$ALT python bench.py $args --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[alt $args] /" >> gpurun_out/ab.txt
done; done
echo done
