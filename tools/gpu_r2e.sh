#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2e}
SWEEP_GRID="cells=96,128,192,256 inflight=48,72,96,128 dyn=0,1 pct=0,30,60,90" timeout 2400 python tools/sweep.py 3d_varcoef_f64 3d_varcoef_f32 2d_varcoef_f64 2d_varcoef_f32 2d_elasticity_f64 2d_elasticity_f32 3d_elasticity_f64 3d_elasticity_f32 > gpurun_out/${T}_sweep.jsonl 2> gpurun_out/${T}_sweep.err
ls -la gpurun_out | grep ${T}
