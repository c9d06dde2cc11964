#!/bin/bash
# Link product, three lanes per site (link_variant 9): parity tests, A/B against the rows kernel, one ncu capture.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider -k "link and (rows3 or config3)" > gpurun_out/pytest_r3.log 2>&1
echo "pytest_r3=$?" >> gpurun_out/status_r3.txt
for spec in "SU3G_LINK_VARIANT=0|--workload link --dtype f64" "SU3G_LINK_VARIANT=9|--workload link --dtype f64" \
            "SU3G_LINK_VARIANT=9 SU3G_LINK_ROWS3_MINB=5|--workload link --dtype f64" \
            "SU3G_LINK_VARIANT=9 SU3G_LINK_ROWS3_MINB=4|--workload link --dtype f64" \
            "SU3G_LINK_VARIANT=0|--workload link --dtype f64 --mode fma" "SU3G_LINK_VARIANT=9|--workload link --dtype f64 --mode fma" \
            "SU3G_LINK_VARIANT=9 SU3G_LINK_ROWS3_MINB=4|--workload link --dtype f64 --mode fma" \
            "SU3G_LINK_VARIANT=9|--workload link --dtype f32" "SU3G_LINK_VARIANT=9 SU3G_LINK_ROWS3_MINB=6|--workload link --dtype f32" \
            "SU3G_LINK_VARIANT=9|--workload link --dtype f32 --mode fma" \
            "SU3G_LINK_VARIANT=9 SU3G_LINK_ZC=4|--workload link --dtype f64" "SU3G_LINK_VARIANT=9 SU3G_LINK_ZC=48|--workload link --dtype f64"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  env $envs timeout 300 python bench.py $args --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$envs | $args] /" >> gpurun_out/abv_r3.txt
done
CMD="python bench.py --workload link --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
SU3G_LINK_VARIANT=9 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_link_rows3 -c 1 -f -o gpurun_out/prof_r3 $CMD > gpurun_out/ncu_r3.log 2>&1
echo "ncu=$?" >> gpurun_out/status_r3.txt
