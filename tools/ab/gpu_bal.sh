#!/bin/bash
# Balanced work schedule of the TMA NN walk: tests + A/B on configs[2] (32^4) and the headline.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider -k "nn or dslash or slab" > gpurun_out/pytest_bal.log 2>&1
echo "pytest=$?" >> gpurun_out/bal.txt
for rep in 1 2; do
for b in -1 0 1; do
  SU3G_NN_TMA_BALANCED=$b timeout 300 python bench.py --workload nn32 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[nn32 bal=$b] /" >> gpurun_out/bal.txt
done
for b in -1 1; do
  SU3G_NN_TMA_BALANCED=$b timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[weak bal=$b] /" >> gpurun_out/bal.txt
  SU3G_NN_TMA_BALANCED=$b timeout 300 python bench.py --workload nn-strong --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[strong bal=$b] /" >> gpurun_out/bal.txt
  SU3G_NN_TMA_BALANCED=$b timeout 300 python bench.py --workload dslash --layout soa --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[dslash-soa bal=$b] /" >> gpurun_out/bal.txt
done; done
