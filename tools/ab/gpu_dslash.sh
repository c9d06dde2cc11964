#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -k "dslash or link" -q -p no:cacheprovider > gpurun_out/pytest_dslash.log 2>&1
echo "pytest_dslash=$?" >> gpurun_out/status.txt
for dt in f32 f64; do for m in exact fma; do
  python bench.py --workload dslash --dtype $dt --mode $m --steps 30 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/dslash_${dt}_${m}.json
done; done
python bench.py --workload link --dtype f64 --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/link_f64_default.json
SU3G_LINK_MODE=fma python bench.py --workload link --dtype f64 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/link_f64_fma.json
python bench.py --workload link --dtype f32 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/link_f32.json
echo done
