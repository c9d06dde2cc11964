#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2 3; do
for spec in "SU3G_DSLASH_EO_HINTS=1|--workload dslash --dtype f64" "SU3G_DSLASH_EO_HINTS=0|--workload dslash --dtype f64" \
            "SU3G_DSLASH_EO_HINTS=1|--workload dslash --dtype f32" "SU3G_DSLASH_EO_HINTS=0|--workload dslash --dtype f32" \
            "SU3G_DSLASH_EO_HINTS=1|--workload dslash --dtype f32 --mode fma" "SU3G_DSLASH_EO_HINTS=0|--workload dslash --dtype f32 --mode fma"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  env $envs timeout 300 python bench.py $args --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$envs | $args] /" >> gpurun_out/abv_eoh.txt
done; done
