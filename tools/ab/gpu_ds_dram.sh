#!/bin/bash
# DRAM bytes per launch of the f64 dslash / NN generic kernels under L2-hint and z-chunk variants.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
run() {  # tag env... -- args
  tag=$1; shift
  env "$@" python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $ARGS > /dev/null 2>&1 || { echo "[$tag] plain run failed" >> gpurun_out/ds_dram.txt; return; }
  env "$@" timeout 300 ncu --metrics $M --clock-control none -k regex:"$KR" -c 2 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $ARGS 2>/dev/null \
    | grep -E '"(dram|gpu__|lts)' | awk -F'","' -v t="$tag" '{printf "[%s] %s %s %s\n", t, $(NF-2), $(NF-1), $NF}' >> gpurun_out/ds_dram.txt
}
ARGS="--workload dslash --dtype f64"; KR=k_dslash
run "ds64 default" SU3G_X=0
run "ds64 hints0" SU3G_SWEEP_L2_HINTS=0
run "ds64 zc4" SU3G_SWEEP_ZC=4
run "ds64 zc64" SU3G_SWEEP_ZC=64
ARGS="--workload nn-weak --dtype f64"; KR=k_nn_sweep
run "nn64 default" SU3G_X=0
ARGS="--workload dslash --dtype f32"; KR=k_
run "ds32 default" SU3G_X=0
echo done
