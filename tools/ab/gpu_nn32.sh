#!/bin/bash
# configs[2] (32^4 f32 NN) and the headline: work-item chunk length x prologue L2 prefetch A/B.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider -k "nn" > gpurun_out/pytest_nn32.log 2>&1
echo "pytest=$?" >> gpurun_out/nn32.txt
for rep in 1 2; do
for pf in 1 0; do
for c in 0 16 8 4; do
  SU3G_NN_TMA_PROLOGUE_PREFETCH=$pf SU3G_NN_TMA_CHUNK=$c timeout 300 python bench.py --workload nn32 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[nn32 pf=$pf chunk=$c] /" >> gpurun_out/nn32.txt
done; done; done
for pf in 1 0; do for c in 0 8; do
  SU3G_NN_TMA_PROLOGUE_PREFETCH=$pf SU3G_NN_TMA_CHUNK=$c timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[weak pf=$pf chunk=$c] /" >> gpurun_out/nn32.txt
done; done
