#!/bin/bash
# One measurement pass on the GPU box: suite + ncu launch list + ncu full captures.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python tools/suite.py ${SUITE:-routines sweeps} > gpurun_out/suite.jsonl 2> gpurun_out/suite.err
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_nn_sweep -s 30 -c 1 -o gpurun_out/prof_nn $CMD > gpurun_out/ncu_nn.log 2>&1
CMD2="python bench.py --workload routine:mult_su3_nn --sites 16777216 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD2 > gpurun_out/plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_stream -s 3 -c 1 -o gpurun_out/prof_nn_routine $CMD2 > gpurun_out/ncu_routine.log 2>&1
CMD3="python bench.py --workload link --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD3 > gpurun_out/plain4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_link -s 3 -c 1 -o gpurun_out/prof_link $CMD3 > gpurun_out/ncu_link.log 2>&1
echo done
