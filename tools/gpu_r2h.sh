#!/usr/bin/env bash
# Round-2 session H: tiled mesh kernel -- parity tests, mesh rows, ncu of the tiled kernel.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2h}
timeout 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_mesh.py -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python tools/mesh_rows.py 200 > gpurun_out/${T}_mesh_rows.jsonl 2> gpurun_out/${T}_mesh_rows.err
TXB_TILED_XPOSE=1 timeout 300 python -c "
import sys, json; sys.path.insert(0,'.'); import bench
for v in ('3d_varcoef_f64','3d_varcoef_f32','3d_elasticity_f64','2d_varcoef_f64'):
    print(v, 'xpose', bench.time_mesh(v, 200, 5, tiled=True))
" > gpurun_out/${T}_xpose.txt 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_tiled_kernel -s 6 -c 1 \
  -o gpurun_out/${T}_prof_tiled_3dvar_f64 python tools/prof_mesh.py 3d_varcoef_f64 > gpurun_out/${T}_ncu_tiled.log 2>&1
ls -la gpurun_out | grep ${T}
