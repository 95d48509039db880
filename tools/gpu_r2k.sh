#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2k}
scan() {
python - "$@" <<'PY'
import sys, json; sys.path.insert(0,'.'); import bench
for v in ('3d_varcoef_f64','3d_varcoef_f32','2d_varcoef_f32'):
    print(json.dumps({"cfg": v, "env": sys.argv[1:], "tiled": bench.time_mesh(v, 200, 5, tiled=True)}), flush=True)
PY
}
scan default > gpurun_out/${T}_scan.jsonl 2>&1
for d in 1 2 3; do TXB_TILED_DEBUG=$d scan debug=$d >> gpurun_out/${T}_scan.jsonl 2>&1; done
for kb in 32 64 128 160; do TXB_INFLIGHT_KB=$kb TXB_TILED_DEBUG=1 scan debug=1,inflight=$kb >> gpurun_out/${T}_scan.jsonl 2>&1; done
