#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2w}
SWEEP_GRID="cells=96,128,192,256,288,384 inflight=48,72,96,128 dyn=1 pct=60 pf=-1" timeout 2400 python tools/sweep.py 3d_varcoef_f64 3d_varcoef_f32 2d_varcoef_f64 2d_varcoef_f32 2d_elasticity_f64 2d_elasticity_f32 3d_elasticity_f64 3d_elasticity_f32 > gpurun_out/${T}_sweep.jsonl 2>&1
