cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest_gpu=$?" >> gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke=$?" >> gpurun_out/status.txt
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench=$?" >> gpurun_out/status.txt
for a in "--workload link --dtype f64" "--workload link --dtype f32" "--workload nn-weak --dtype f64" "--workload dslash --dtype f64" "--workload dslash --dtype f32"; do
python bench.py $a --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$a] /" >> gpurun_out/check.txt
done
