#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_routines.py -q -x -p no:cacheprovider > gpurun_out/pytest_routines.log 2>&1
echo "pytest_routines=$?" >> gpurun_out/status.txt
for dt in f32 f64; do for r in ${ROUTINES:-mult_su3_mat_vec_sum_4dir mult_adj_su3_mat_vec_4dir}; do
  python bench.py --workload routine:$r --dtype $dt --sites 16777216 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/$dt $r /" >> gpurun_out/routines.txt
done; done
echo done
