#!/bin/bash
# Link product, 8x4x4 t-walk with U_3 through L2 (link_variant 10): parity tests, A/B, ncu.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider -k "link and (t-walk4 or t_walk4 or walk or config3)" > gpurun_out/pytest_tw4.log 2>&1
echo "pytest_tw4=$?" >> gpurun_out/status_tw4.txt
for spec in "SU3G_LINK_VARIANT=0|--workload link --dtype f64" "SU3G_LINK_VARIANT=10|--workload link --dtype f64" \
            "SU3G_LINK_VARIANT=0|--workload link --dtype f64 --mode fma" "SU3G_LINK_VARIANT=10|--workload link --dtype f64 --mode fma" \
            "SU3G_LINK_VARIANT=0|--workload link --dtype f32" "SU3G_LINK_VARIANT=10|--workload link --dtype f32" \
            "SU3G_LINK_VARIANT=10|--workload link --dtype f32 --mode fma" \
            "SU3G_LINK_VARIANT=10 SU3G_LINK_TW_CHUNK=12|--workload link --dtype f64" "SU3G_LINK_VARIANT=10 SU3G_LINK_TW_CHUNK=4|--workload link --dtype f64"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  env $envs timeout 300 python bench.py $args --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$envs | $args] /" >> gpurun_out/abv_tw4.txt
done
CMD="python bench.py --workload link --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
SU3G_LINK_VARIANT=10 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_link_tw4 -c 1 -f -o gpurun_out/prof_tw4 $CMD > gpurun_out/ncu_tw4.log 2>&1
echo "ncu=$?" >> gpurun_out/status_tw4.txt
