#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py -k "runtime_geometries or tma or walk" -q -p no:cacheprovider > gpurun_out/pytest_geo.log 2>&1
echo "pytest=$?" >> gpurun_out/status.txt
specs=()
for d in 48,48,48,16 96,48,24,16 40,40,40,16 24,24,24,48 64,64,64,16; do specs+=("X=1|--workload nn-weak --dtype f32 --dims $d"); done
specs+=("SU3G_NN_VARIANT=2|--workload nn-weak --dtype f32 --dims 48,48,48,16")
bash tools/gpu_ab_var.sh "${specs[@]}"
