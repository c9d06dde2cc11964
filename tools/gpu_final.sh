#!/bin/bash
# Round-end measurement pass: full GPU tests, smoke, the whole suite, the bench default's ncu launch list,
# and ncu --set full captures of the checkerboarded dslash.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_gpu=$?" >> gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke=$?" >> gpurun_out/status.txt
python tools/suite.py configs routines extra sweeps > gpurun_out/suite_full.jsonl 2> gpurun_out/suite.err
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench=$?" >> gpurun_out/status.txt
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu=$?" >> gpurun_out/status.txt
for dt in f64 f32; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_dslash_eo -c 1 -f -o gpurun_out/prof_dseo_$dt \
    python bench.py --workload dslash --dtype $dt --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_dseo_$dt.log 2>&1
  echo "ncu_dseo_$dt=$?" >> gpurun_out/status.txt
done
