#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2p}
scan() {
python - "$@" <<'PY'
import sys, json; sys.path.insert(0,'.'); import bench
for lg in (19, 20, 21, 22):
    for mode in ('tiled', 'given'):
        r = bench.time_mesh('3d_varcoef_f32', 100, 5, tiled=mode == 'tiled', given_geometry=mode == 'given', n_cells=1 << lg)
        print(json.dumps({"cfg": f"3d_varcoef_f32 2^{lg} {mode}", "env": sys.argv[1:], "tiled": r}), flush=True)
PY
}
scan default > gpurun_out/${T}_scan.jsonl 2>&1
TXB_TILED_DEBUG=3 scan debug3 >> gpurun_out/${T}_scan.jsonl 2>&1
TXB_PDL=0 scan nopdl >> gpurun_out/${T}_scan.jsonl 2>&1
