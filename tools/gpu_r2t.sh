#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2t}
for c in 2d_varcoef_f32 2d_elasticity_f32; do
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 6 -c 1 \
  -o gpurun_out/${T}_prof_${c} python bench.py --config $c --steps 5 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/${T}_ncu_${c}.log 2>&1
done
