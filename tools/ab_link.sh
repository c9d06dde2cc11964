#!/bin/bash
# link product: the link GPU tests, then a same-box A/B of link variants (FMA mode): tools/ab_link.sh [variants...]
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
VARS="${@:-5}"
timeout 900 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_guard.py -k "link" -q -x -p no:cacheprovider > gpurun_out/pytest_link.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
for rep in 1 2 3; do
for v in $VARS; do
  for w in "--workload link --mode fma" "--workload link --mode fma --dtype f32"; do
  env SU3G_LINK_VARIANT=$v timeout 300 python bench.py $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 | sed "s/^/[v$v $w] /" >> gpurun_out/ab.txt
  done
done; done
echo done
