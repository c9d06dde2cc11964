# link product rows gather: link GPU tests, then exact / FMA bench rows (f64, f32) x3
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_guard.py -k "link" -q -x -p no:cacheprovider > gpurun_out/pytest_link.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
for rep in 1 2 3; do for w in "--workload link" "--workload link --mode fma" "--workload link --dtype f32"; do
  SU3G_LINK_VARIANT=1 timeout 300 python bench.py $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 | sed "s/^/[rows $w] /" >> gpurun_out/abr.txt
done; done
