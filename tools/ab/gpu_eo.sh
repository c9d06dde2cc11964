#!/bin/bash
# Checkerboarded dslash: parity tests, A/B against the SoA dslash kernels, DRAM bytes per launch.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider -k "eo or dslash" > gpurun_out/pytest_eo.log 2>&1
echo "pytest_eo=$?" >> gpurun_out/status_eo.txt
for spec in "|--workload dslash --dtype f64 --layout soa" "|--workload dslash --dtype f64 --layout eo" \
            "|--workload dslash --dtype f32 --layout soa" "|--workload dslash --dtype f32 --layout eo" \
            "SU3G_DSLASH_EO_ZC=4|--workload dslash --dtype f64" "SU3G_DSLASH_EO_ZC=16|--workload dslash --dtype f64" \
            "SU3G_DSLASH_EO_ZC=64|--workload dslash --dtype f64" "SU3G_DSLASH_EO_HINTS=0|--workload dslash --dtype f64" \
            "SU3G_DSLASH_EO_ZC=4|--workload dslash --dtype f32" "SU3G_DSLASH_EO_ZC=64|--workload dslash --dtype f32" \
            "|--workload dslash --dtype f64 --mode fma" "|--workload dslash --dtype f32 --mode fma"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  env $envs timeout 300 python bench.py $args --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$envs | $args] /" >> gpurun_out/abv_eo.txt
done
python bench.py --workload dslash --dtype f64 --steps 10 --warmup 3 > gpurun_out/bench_eo_f64.json 2>/dev/null
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for dt in f64 f32; do
timeout 300 ncu --metrics $M --clock-control none -k regex:k_dslash_eo -c 2 --csv python bench.py --workload dslash --dtype $dt --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null \
    | grep -E '"(dram|gpu__|lts)' | awk -F'","' -v t="eo $dt" '{printf "[%s] %s %s %s\n", t, $(NF-2), $(NF-1), $NF}' >> gpurun_out/eo_dram.txt
done
