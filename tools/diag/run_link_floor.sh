# floors of k_link_fact: build libsu3g_ns.so / _nm.so / _nn.so first (make -C paper_1309_0551_b200/csrc BUILD=build_ns OUT=../lib/libsu3g_ns.so EXTRA=-DFACT_NOSTORE; _nm: -DFACT_NOMATH; _nn: both)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for rep in 1 2; do for lib in libsu3g.so libsu3g_ns.so libsu3g_nm.so libsu3g_nn.so; do for w in "--workload link --mode fma" "--workload link --mode fma --dtype f32"; do
SU3G_LIB=$PWD/paper_1309_0551_b200/lib/$lib timeout 300 python bench.py $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/x.err | tail -1 | sed "s|^|[$lib $w] |" >> gpurun_out/x.txt
done; done; done
