#!/bin/bash
# NN-sweep kernel variants side by side (1 generic, 2 register walk, 3 TMA walk).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -q -x -p no:cacheprovider > gpurun_out/pytest_sweeps.log 2>&1
echo "pytest_sweeps=$?" >> gpurun_out/status.txt
for dt in f32 f64; do for var in 1 2 3; do for w in nn-weak nn32; do
  SU3G_NN_VARIANT=$var python bench.py --workload $w --dtype $dt --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/$dt var$var $w /" >> gpurun_out/variants.txt
done; done; done
echo done
