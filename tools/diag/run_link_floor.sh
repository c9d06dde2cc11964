# floors of k_link_fact: bench each library build given on the command line (default: all four floor builds).
# Build them first: make -C paper_1309_0551_b200/csrc BUILD=build_ns OUT=../lib/libsu3g_ns.so EXTRA=-DFACT_NOSTORE
#   _nm: -DFACT_NOMATH (data path only)   _nn: both   _nl: -DFACT_NOLOAD (compute only: slots never filled)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
LIBS="${@:-libsu3g.so libsu3g_ns.so libsu3g_nm.so libsu3g_nn.so libsu3g_nl.so}"
for rep in 1 2; do for lib in $LIBS; do for w in "--workload link --mode fma" "--workload link --mode fma --dtype f32"; do
[ -f paper_1309_0551_b200/lib/$lib ] || continue
SU3G_LIB=$PWD/paper_1309_0551_b200/lib/$lib timeout 300 python bench.py $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/x.err | tail -1 | sed "s|^|[$lib $w] |" >> gpurun_out/x.txt
done; done; done
echo done
