#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2z}
timeout 900 python -m pytest tests/test_gpu_tiled.py -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
scan() {
python - "$@" <<'PY'
import sys, json; sys.path.insert(0,'.'); import bench
for v in ('3d_varcoef_f64','3d_varcoef_f32','3d_elasticity_f64','3d_elasticity_f32','2d_varcoef_f64','2d_varcoef_f32'):
    print(json.dumps({"cfg": v, "env": sys.argv[1:], "tiled": bench.time_mesh(v, 200, 5, tiled=True)}), flush=True)
PY
}
scan default > gpurun_out/${T}_scan.jsonl 2>&1
TXB_TILED_DEBUG=4 scan trust >> gpurun_out/${T}_scan.jsonl 2>&1
