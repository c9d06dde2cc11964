#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_nn_tma -c 1 -f -o gpurun_out/prof_nntma \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_nntma.log 2>&1
echo done
