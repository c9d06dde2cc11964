#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
specs=("SU3G_LINK_MODE=exact|--workload link --dtype f64" "SU3G_LINK_MODE=fma|--workload link --dtype f64" "SU3G_LINK_MODE=exact|--workload link --dtype f32")
for d in 64,64,64,16 62,64,64,16 64,62,62,16 60,60,60,16; do
  specs+=("X=1|--workload dslash --dtype f32 --dims $d")
  specs+=("X=1|--workload nn-weak --dtype f64 --dims $d")
  specs+=("X=1|--workload nn-weak --dtype f32 --dims $d")
done
bash tools/gpu_ab_var.sh "${specs[@]}"
