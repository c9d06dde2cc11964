# ring walks after the shared schedule helper: sweep GPU tests, then a same-box A/B of the columns schedule (dslash, NN, link)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_fullsize.py tests/test_gpu_guard.py -q -x -p no:cacheprovider > gpurun_out/pytest_sweeps.log 2>&1; echo "pytest_sweeps=$?" >> gpurun_out/status.txt
for rep in 1 2 3; do for c in 0 1; do for w in "--workload dslash" "--workload dslash --dtype f64" "--workload nn-weak" "--workload link --mode fma"; do
  SU3G_NN_RING_COLUMNS=$c timeout 300 python bench.py $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-slab-probe 2>>gpurun_out/abd.err | tail -1 | sed "s/^/[columns=$c $w] /" >> gpurun_out/abd.txt
done; done; done
