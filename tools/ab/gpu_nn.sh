#!/bin/bash
# NN-sweep iteration: parity of the sweep kernels, bench lines, ncu of the walk kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -q -x -p no:cacheprovider > gpurun_out/pytest_sweeps.log 2>&1
echo "pytest_sweeps=$?" >> gpurun_out/status.txt
python tools/suite.py sweeps > gpurun_out/suite_sweeps.jsonl 2> gpurun_out/suite.err
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_default.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_nn_tma -s 30 -c 1 -o gpurun_out/prof_tma $CMD > gpurun_out/ncu_tma.log 2>&1
echo done
