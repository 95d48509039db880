#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2o}
timeout 900 python -m pytest tests/test_gpu_tiled.py -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
scan() {
python - "$@" <<'PY'
import sys, json; sys.path.insert(0,'.'); import bench
for v in ('3d_varcoef_f64','3d_varcoef_f32','3d_elasticity_f32','2d_varcoef_f32'):
    print(json.dumps({"cfg": v, "env": sys.argv[1:], "tiled": bench.time_mesh(v, 200, 5, tiled=True)}), flush=True)
PY
}
for ms in 8 12 16; do for tc in 128 256; do TXB_TILE_CELLS=$tc TXB_TILED_MAX_STAGES=$ms TXB_INFLIGHT_KB=256 scan tile=$tc,maxst=$ms,kb256 >> gpurun_out/${T}_scan.jsonl 2>&1; done; done
TXB_TILED_MAX_STAGES=16 TXB_INFLIGHT_KB=256 TXB_TILED_DEBUG=3 scan maxst16,kb256,debug3 >> gpurun_out/${T}_scan.jsonl 2>&1
scan default >> gpurun_out/${T}_scan.jsonl 2>&1
