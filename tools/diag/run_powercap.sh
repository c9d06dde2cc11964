# NN sweep headline under sustained load: 100-step runs, exact and FMA arithmetic, f32 and f64 (clocks and throttle reasons in each line)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for w in "--mode exact" "--mode fma" "--mode exact --dtype f64" "--mode fma --dtype f64"; do
  python bench.py $w --steps 100 --warmup 5 --no-e2e --no-cpu-baseline --no-slab-probe 2>>gpurun_out/pc.err | tail -1 | sed "s/^/[$w] /" >> gpurun_out/powercap.txt
done
