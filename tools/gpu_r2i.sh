#!/usr/bin/env bash
# Round-2 session I: tiled kernel with the branch-free geometry; ring-depth / in-flight scan.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2i}
timeout 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_mesh.py -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
scan() {
python - "$@" <<'PY'
import sys, json; sys.path.insert(0,'.'); import bench
for v in ('3d_varcoef_f64','3d_varcoef_f32','3d_elasticity_f64','2d_varcoef_f64','2d_varcoef_f32'):
    print(json.dumps({"cfg": v, "env": sys.argv[1:], "tiled": bench.time_mesh(v, 200, 5, tiled=True)}), flush=True)
PY
}
scan default > gpurun_out/${T}_scan.jsonl 2>&1
for kb in 24 48 96; do TXB_INFLIGHT_KB=$kb scan inflight=$kb >> gpurun_out/${T}_scan.jsonl 2>&1; done
for st in 2 3 4; do TXB_STAGES=$st scan stages=$st >> gpurun_out/${T}_scan.jsonl 2>&1; done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_tiled_kernel -s 6 -c 1 \
  -o gpurun_out/${T}_prof_tiled_3dvar_f64 python tools/prof_mesh.py 3d_varcoef_f64 > gpurun_out/${T}_ncu_tiled.log 2>&1
ls -la gpurun_out | grep ${T}
