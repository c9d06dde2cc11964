#!/bin/bash
# Round measurement pass: full GPU tests, smoke, the sanitizer driver (plain, then under compute-sanitizer
# memcheck / synccheck / racecheck on the su3g kernels), the whole suite, the bench
# default (20 and 100 steps), and the bench default's ncu launch list.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_gpu=$?" >> gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke=$?" >> gpurun_out/status.txt
timeout 600 python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1
echo "sanitize_plain=$?" >> gpurun_out/status.txt
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=4su3g --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "sanitize_$tool=$?" >> gpurun_out/status.txt
done
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench=$?" >> gpurun_out/status.txt
python bench.py --steps 100 --warmup 5 --no-e2e > gpurun_out/bench_100.json 2> gpurun_out/bench_100.err
python bench.py --dtype f64 --steps 100 --warmup 5 --no-e2e > gpurun_out/bench_100_f64.json 2>> gpurun_out/bench_100.err
python tools/suite.py configs routines extra sweeps > gpurun_out/suite_full.jsonl 2> gpurun_out/suite.err
echo "suite=$?" >> gpurun_out/status.txt
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu=$?" >> gpurun_out/status.txt
