#!/bin/bash
# link-product ring walk: GPU tests, then same-box A/B against the rows gather kernel
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -k "link" -q -x -p no:cacheprovider > gpurun_out/pytest_link.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
for rep in 1 2; do
for spec in "SU3G_LINK_VARIANT=1" "SU3G_LINK_VARIANT=2"; do
  for w in "--workload link" "--workload link --mode fma" "--workload link --dtype f32"; do
  env $spec timeout 300 python bench.py $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-parity 2>>gpurun_out/ab.err | tail -1 | sed "s/^/[$spec $w] /" >> gpurun_out/ab.txt
  done
done; done
