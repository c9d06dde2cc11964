#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for dt in f32 f64; do
  python bench.py --workload nn-weak --dtype $dt --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/e2e_nn_${dt}.json
done
python bench.py --workload nn-weak --halo p2p --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/e2e_nn_p2p.json
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/ref_arm.json
echo done
