#!/bin/bash
# Link product TMA t-walk (link_variant 8): parity tests, A/B against the rows kernel, one ncu capture.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
(cd tools/ubench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fpipe fpipe.cu && ./fpipe) > gpurun_out/fpipe.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_sweeps.py -m gpu -q -x -p no:cacheprovider -k "link" > gpurun_out/pytest_tw.log 2>&1
echo "pytest_tw=$?" >> gpurun_out/status_tw.txt
for spec in "SU3G_LINK_VARIANT=0|--workload link --dtype f32" "SU3G_LINK_VARIANT=8|--workload link --dtype f32" \
            "SU3G_LINK_VARIANT=8 SU3G_LINK_MODE=fma|--workload link --dtype f32 --mode fma" \
            "SU3G_LINK_VARIANT=8 SU3G_LINK_TW_CHUNK=4|--workload link --dtype f32" \
            "SU3G_LINK_VARIANT=8 SU3G_LINK_TW_CHUNK=12|--workload link --dtype f32" \
            "SU3G_LINK_VARIANT=8 SU3G_LINK_TW_CHUNK=48|--workload link --dtype f32"; do
  envs="${spec%%|*}"; args="${spec#*|}"
  env $envs timeout 300 python bench.py $args --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[$envs | $args] /" >> gpurun_out/abv_tw.txt
done
CMD="python bench.py --workload link --dtype f32 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
SU3G_LINK_VARIANT=8 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_link_tw -c 1 -f -o gpurun_out/prof_tw $CMD > gpurun_out/ncu_tw.log 2>&1
echo "ncu=$?" >> gpurun_out/status_tw.txt
