cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sweeps.py -k "ring" -q -x -p no:cacheprovider > gpurun_out/pytest_ring.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
for rep in 1 2; do
for spec in "SU3G_NN_VARIANT=3" "SU3G_NN_VARIANT=4 SU3G_NN_RING_CFG=0" "SU3G_NN_VARIANT=4 SU3G_NN_RING_CFG=1" "SU3G_NN_VARIANT=4 SU3G_NN_RING_CFG=2" "SU3G_NN_VARIANT=4 SU3G_NN_RING_CFG=3"; do
  for w in "--workload nn-weak" "--workload nn32"; do
  env $spec python bench.py $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/ab.err | tail -1 | sed "s/^/[$spec $w] /" >> gpurun_out/ab.txt
  done
done; done
