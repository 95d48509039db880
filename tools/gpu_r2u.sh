#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2u}
SWEEP_GRID="cells=96,192,288 inflight=48,72,96,128 dyn=1 pct=0,40,60,80 pf=-1,8,16" timeout 1500 python tools/sweep.py 2d_varcoef_f32 2d_elasticity_f32 > gpurun_out/${T}_sweep.jsonl 2>&1
