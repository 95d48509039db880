#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2l}
scan() {
python - "$@" <<'PY'
import sys, json; sys.path.insert(0,'.'); import bench
for v in ('3d_varcoef_f64','3d_varcoef_f32','3d_elasticity_f64','2d_varcoef_f32'):
    print(json.dumps({"cfg": v, "env": sys.argv[1:], "tiled": bench.time_mesh(v, 200, 5, tiled=True)}), flush=True)
PY
}
for tc in 96 192; do TXB_TILE_CELLS=$tc scan tile=$tc >> gpurun_out/${T}_scan.jsonl 2>&1; done
for tc in 96 192; do TXB_TILE_CELLS=$tc TXB_TILED_DEBUG=3 scan tile=$tc,debug=3 >> gpurun_out/${T}_scan.jsonl 2>&1; done
TXB_TILE_CELLS=192 TXB_INFLIGHT_KB=32 scan tile=192,inflight=32 >> gpurun_out/${T}_scan.jsonl 2>&1
TXB_TILE_CELLS=192 TXB_INFLIGHT_KB=128 scan tile=192,inflight=128 >> gpurun_out/${T}_scan.jsonl 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_tiled_kernel -s 6 -c 1 \
  -o gpurun_out/${T}_prof_tiled_3dvar_f32 python tools/prof_mesh.py 3d_varcoef_f32 > gpurun_out/${T}_ncu_tiled.log 2>&1
