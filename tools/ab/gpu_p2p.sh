#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_p2p.py -q -p no:cacheprovider -x > gpurun_out/pytest_p2p.log 2>&1
echo "pytest_p2p=$?" >> gpurun_out/status.txt
for h in nccl p2p; do for dt in f32 f64; do
  timeout 300 python bench.py --workload nn-weak --dtype $dt --halo $h --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/nn_${h}_${dt}.json
done; done
echo done
