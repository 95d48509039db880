#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2y}
timeout 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_mesh.py tests/test_gpu_residual_graph.py -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
scan() {
python - "$@" <<'PY'
import sys, json; sys.path.insert(0,'.'); import bench
for v in ('3d_varcoef_f64','3d_varcoef_f32','3d_elasticity_f64','3d_elasticity_f32','2d_varcoef_f64','2d_varcoef_f32'):
    for mode in ('tiled', 'given'):
        print(json.dumps({"cfg": v + ' ' + mode, "env": sys.argv[1:], "tiled": bench.time_mesh(v, 200, 5, tiled=mode == 'tiled', given_geometry=mode == 'given')}), flush=True)
PY
}
scan default > gpurun_out/${T}_scan.jsonl 2>&1
