#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_routines.py -k "dslash or c_host or knobs" -q -p no:cacheprovider > gpurun_out/pytest_ds.log 2>&1
echo "pytest=$?" >> gpurun_out/status.txt
bash tools/gpu_ab_var.sh "X=1|--workload dslash --dtype f32" "X=1|--workload dslash --dtype f64" "X=1|--workload nn-weak --dtype f32"
