#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider -k "xw or slab_halo or multi_item or fma_mode" > gpurun_out/pytest_xw.log 2>&1
echo "pytest=$?" >> gpurun_out/xw.txt
for rep in 1 2; do
for spec in "SU3G_NN_XW=0|--workload nn-weak --dtype f64" "SU3G_NN_XW=1|--workload nn-weak --dtype f64" \
            "SU3G_NN_XW=0|--workload nn32 --dtype f64" "SU3G_NN_XW=1|--workload nn32 --dtype f64" \
            "SU3G_NN_XW=0|--workload nn-strong --dtype f64" "SU3G_NN_XW=1|--workload nn-strong --dtype f64" \
            "SU3G_NN_VARIANT=1|--workload nn-weak --dtype f32" "SU3G_NN_VARIANT=7|--workload nn-weak --dtype f32"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  env $envs timeout 300 python bench.py $args --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$envs | $args] /" >> gpurun_out/xw.txt
done; done
SU3G_NN_XW=1 timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_nn -c 1 python bench.py --workload nn-weak --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_xw.log 2>&1
SU3G_NN_XW=0 timeout 300 ncu --metrics dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum --clock-control none -k regex:k_nn -c 1 python bench.py --workload nn-weak --dtype f64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/ncu_xw.log 2>&1
