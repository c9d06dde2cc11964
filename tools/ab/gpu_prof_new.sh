#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_comm.py -q -p no:cacheprovider > gpurun_out/pytest_comm.log 2>&1
echo "pytest_comm=$?" >> gpurun_out/status.txt
python tools/prof_targets.py > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_link_rows|k_dslash' -s 1 -c 2 \
      -o gpurun_out/prof_new python tools/prof_targets.py > gpurun_out/ncu_new.log 2>&1
echo "ncu=$?" >> gpurun_out/status.txt
