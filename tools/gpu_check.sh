#!/bin/bash
# Full GPU test suite + smoke + targeted bench rows: tools/gpu_check.sh "<bench args>" ...
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_gpu=$?" >> gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke=$?" >> gpurun_out/status.txt
for args in "${@}"; do
  python bench.py $args 2>>gpurun_out/check.err | tail -1 | sed "s/^/[$args] /" >> gpurun_out/check.txt
done
echo done
