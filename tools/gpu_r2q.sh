#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2q}
scan() {
python - "$@" <<'PY'
import sys, json; sys.path.insert(0,'.'); import bench
for v in ('3d_varcoef_f64','3d_varcoef_f32','3d_elasticity_f32','2d_varcoef_f32'):
    print(json.dumps({"cfg": v, "env": sys.argv[1:], "tiled": bench.time_mesh(v, 200, 5, tiled=True)}), flush=True)
PY
}
scan default > gpurun_out/${T}_scan.jsonl 2>&1
for ns in 1000 20000 1000000; do TXB_TILED_SLEEP_NS=$ns TXB_TILED_CONSUMER_SLEEP_NS=$ns scan sleep_all=$ns >> gpurun_out/${T}_scan.jsonl 2>&1; done
TXB_TILED_SLEEP_NS=20000 scan sleep_pg=20000 >> gpurun_out/${T}_scan.jsonl 2>&1
TXB_TILED_CONSUMER_SLEEP_NS=20000 scan sleep_c=20000 >> gpurun_out/${T}_scan.jsonl 2>&1
TXB_TILED_SLEEP_NS=20000 TXB_TILED_CONSUMER_SLEEP_NS=20000 timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_tiled_kernel -s 6 -c 1 \
  -o gpurun_out/${T}_prof_tiled_3dvar_f32 python tools/prof_mesh.py 3d_varcoef_f32 > gpurun_out/${T}_ncu_tiled.log 2>&1
