#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
specs=()
for zc in 0 4 16 32 64; do
  specs+=("SU3G_SWEEP_ZC=$zc|--workload nn-weak --dtype f64")
  specs+=("SU3G_SWEEP_ZC=$zc|--workload dslash --dtype f32")
  specs+=("SU3G_SWEEP_ZC=$zc|--workload dslash --dtype f64")
done
specs+=("SU3G_LINK_MODE=exact|--workload link --dtype f64" "SU3G_LINK_MODE=fma|--workload link --dtype f64" "SU3G_LINK_MODE=exact|--workload link --dtype f32")
bash tools/gpu_ab_var.sh "${specs[@]}"
