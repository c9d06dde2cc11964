#!/bin/bash
# Full GPU test suite + targeted bench rows.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_gpu=$?" >> gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke=$?" >> gpurun_out/status.txt
for args in "${@}"; do
  python bench.py $args --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$args] /" >> gpurun_out/check.txt
done
echo done
