#!/bin/bash
# Round measurement pass (one GPU): full GPU tests, smoke, the plain kernel driver, the whole suite, the
# bench default (20 and 100 steps, both dtypes), the reference arm, the bench default's ncu launch list,
# and one ncu --set full capture of every workload's dominant kernel (tools/prof_targets.py).
# compute-sanitizer is closed on this pool; tests/test_gpu_guard.py is the bounds check (in the pytest run).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_gpu=$?" >> gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke=$?" >> gpurun_out/status.txt
timeout 600 python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1
echo "sanitize_plain=$?" >> gpurun_out/status.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench=$?" >> gpurun_out/status.txt
python bench.py --dtype f64 --steps 20 --warmup 5 > gpurun_out/bench_default_f64.json 2>> gpurun_out/bench_default.err
python bench.py --steps 100 --warmup 5 --no-e2e --no-slab-probe > gpurun_out/bench_100.json 2> gpurun_out/bench_100.err
python bench.py --dtype f64 --steps 100 --warmup 5 --no-e2e --no-slab-probe > gpurun_out/bench_100_f64.json 2>> gpurun_out/bench_100.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "reference=$?" >> gpurun_out/status.txt
python tools/suite.py configs routines extra sweeps > gpurun_out/suite_full.jsonl 2> gpurun_out/suite.err
echo "suite=$?" >> gpurun_out/status.txt
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-slab-probe"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "ncu_launch=$?" >> gpurun_out/status.txt
python tools/prof_targets.py > gpurun_out/prof_targets_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_nn_ring|k_link|k_dslash' -c 8 \
      -o gpurun_out/prof_final python tools/prof_targets.py > gpurun_out/ncu_prof_final.log 2>&1
echo "ncu_full=$?" >> gpurun_out/status.txt
