#!/bin/bash
# Same-box A/B of two library builds (SU3G_LIB): tools/gpu_ab_lib.sh libA libB "<bench args>" ...
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
A=$1; B=$2; shift 2
for rep in 1 2 3; do
for args in "$@"; do
for lib in $A $B; do
  SU3G_LIB=$PWD/$lib timeout 300 python bench.py $args --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s|^|[$(basename $lib) $args] |" >> gpurun_out/ab_lib.txt
done; done; done
