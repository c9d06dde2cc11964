# NN ring: the schedule tests, then a same-box A/B of the columns schedule on every NN workload
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_fullsize.py tests/test_gpu_guard.py -k "nn or config5 or ring" -q -x -p no:cacheprovider > gpurun_out/pytest_nn.log 2>&1; echo "pytest_nn=$?" >> gpurun_out/status.txt
for rep in 1 2 3; do for c in 0 1; do for w in "--workload nn-weak" "--workload nn-weak --dtype f64" "--workload nn-strong" "--workload nn-strong --dtype f64" "--workload nn32" "--workload nn32 --dtype f64"; do
  SU3G_NN_RING_COLUMNS=$c timeout 300 python bench.py $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-slab-probe 2>>gpurun_out/abn.err | tail -1 | sed "s/^/[columns=$c $w] /" >> gpurun_out/abn.txt
done; done; done
