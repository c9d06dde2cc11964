#!/bin/bash
# A/B runtime variants (env knobs) on one box: tools/gpu_ab_var.sh "<ENV=val ...>|<bench args>" ...
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rep in 1 2; do
for spec in "${@}"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  env $envs python bench.py $args --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$envs | $args] /" >> gpurun_out/abv.txt
done; done
echo done
