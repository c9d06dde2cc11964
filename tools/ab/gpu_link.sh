#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for v in ${LINKV:-1 2 3}; do for m in fma exact; do
  SU3G_LINK_VARIANT=$v python bench.py --workload link --mode $m --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | sed "s/^/[var$v $m] /" >> gpurun_out/link.txt
done; done
CMD="python bench.py --workload link --mode fma --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_link.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_link -s 3 -c 1 -o gpurun_out/prof_link2 $CMD > gpurun_out/ncu_link2.log 2>&1
echo done
