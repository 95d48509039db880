#!/usr/bin/env bash
# Tile size (cells per batch) of the tiled mesh kernel, per config, given / in-kernel geometry (graph-timed us).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for cfg in 3d_varcoef_f64 3d_varcoef_f32 3d_elasticity_f64 3d_elasticity_f32 2d_varcoef_f64 2d_varcoef_f32 2d_elasticity_f64; do
  case $cfg in 3d*) tiles="64 96 128 192";; *) tiles="96 192 288";; esac
  for tc in $tiles; do
    TXB_TILE_CELLS=$tc timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import bench
for given in (True, False):
    ms,_=bench.time_mesh('$cfg', 200, 5, given_geometry=given)
    print('$cfg', 'given' if given else 'inkernel', 'tile=$tc', round(ms*1e3,2), flush=True)
" 2>&1 | grep tile=
  done
done
