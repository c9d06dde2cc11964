#!/bin/bash
# bench rows with env-var knobs: each argument is "ENV=val ... -- bench args"
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for spec in "${@}"; do
  envs="${spec%%--*}"; args="${spec#*--}"
  env $envs python bench.py $args --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$spec] /" >> gpurun_out/var2.txt
done
echo done
