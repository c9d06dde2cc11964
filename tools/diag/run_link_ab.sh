# link product: link GPU tests, bench rows x3 (FMA f64 / f32, exact f32), optional ncu capture of k_link_fact: run_link_ab.sh [ncu-name]
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_guard.py -k "link" -q -x -p no:cacheprovider > gpurun_out/pytest_link.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
for rep in 1 2 3; do for w in "--workload link --mode fma" "--workload link --mode fma --dtype f32" "--workload link --dtype f32"; do
  timeout 300 python bench.py $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/ab.err | tail -1 | sed "s/^/[$w] /" >> gpurun_out/ab.txt
done; done
if [ -n "$1" ]; then
python tools/diag/prof_link.py 5:fma > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_link -c 1 -o gpurun_out/$1 python tools/diag/prof_link.py 5:fma > gpurun_out/ncu.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
fi
