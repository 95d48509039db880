#!/usr/bin/env bash
# ncu --set full of the 3D elasticity f32 and 2D var-coef f32 cell-array kernels (the two lowest 2^20 rows).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in 3d_elasticity_f32 2d_varcoef_f32; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 6 -c 1 \
    -o gpurun_out/r2bb_${cfg} python bench.py --config $cfg --steps 5 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/r2bb_${cfg}.log 2>&1
  ncu -i gpurun_out/r2bb_${cfg}.ncu-rep --page source --csv --print-source sass > gpurun_out/r2bb_${cfg}_src.csv 2>/dev/null
done
ls -la gpurun_out | grep r2bb
