#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for spec in "SU3G_LINK_TILED=1|--dtype f64" "SU3G_LINK_TILED=1 SU3G_LINK_CARVEOUT=0|--dtype f64" "SU3G_LINK_TILED=1 SU3G_LINK_CARVEOUT=30|--dtype f64" \
            "SU3G_LINK_TILED=1 SU3G_LINK_CARVEOUT=40|--dtype f64" "SU3G_LINK_TILED=1 SU3G_LINK_CARVEOUT=60|--dtype f64" "SU3G_LINK_TILED=1 SU3G_LINK_CARVEOUT=100|--dtype f64" \
            "SU3G_LINK_TILED=1 SU3G_LINK_CARVEOUT=40|--dtype f64 --mode fma" "SU3G_LINK_TILED=1 SU3G_LINK_CARVEOUT=40|--dtype f32"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  env $envs timeout 300 python bench.py --workload link $args --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$envs | $args] /" >> gpurun_out/tiled2.txt
done
SU3G_LINK_TILED=1 SU3G_LINK_CARVEOUT=40 timeout 600 ncu --metrics l1tex__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum,launch__shared_mem_config_size --clock-control none -k regex:k_link_rows -c 1 python bench.py --workload link --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tiled2.log 2>&1
