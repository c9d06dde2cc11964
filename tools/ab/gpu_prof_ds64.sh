#!/bin/bash
# ncu --set full of the f64 dslash and the f64 generic NN kernels (one launch each).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dslash -c 1 -f -o gpurun_out/prof_ds64 \
  python bench.py --workload dslash --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_ds64.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_nn_sweep -c 1 -f -o gpurun_out/prof_nn64 \
  python bench.py --workload nn-weak --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_nn64.log 2>&1
echo done
