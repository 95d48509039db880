#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2ap}
for c in 3d_varcoef_f64 3d_elasticity_f64 3d_elasticity_f32 2d_varcoef_f64; do
  for u in 8 16 24 32; do TXB_SCATTER_U=$u timeout 300 python tools/pipeline_bench.py $c | sed "s/^/U=$u /" >> gpurun_out/${T}_pipe.txt 2>&1; done
done
for u in 8 16 24 32; do TXB_SCATTER_U=$u timeout 300 python tools/pipeline_bench.py 3d_varcoef_f64 16777216 | sed "s/^/U=$u /" >> gpurun_out/${T}_pipe.txt 2>&1; done
