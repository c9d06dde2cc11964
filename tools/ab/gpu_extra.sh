#!/bin/bash
# Full GPU tests + smoke, then the extra-routine roofline rows and one e2e row.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_gpu=$?" >> gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke=$?" >> gpurun_out/status.txt
python tools/suite.py extra > gpurun_out/suite_extra.jsonl 2>&1
python bench.py --workload routine:sub_four_su3_vecs --sites 65536 --steps 50 --warmup 3 > gpurun_out/e2e_sub4.json 2>&1
python bench.py --workload routine:mult_adj_su3_mat_4vec --sites 65536 --steps 50 --warmup 3 > gpurun_out/e2e_4vec.json 2>&1
echo done
