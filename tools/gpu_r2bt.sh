#!/usr/bin/env bash
# Diagnostic: tiled in-kernel geometry with / without the per-numerator range test (tune_libs/libtxb_diag.so, unsafe).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
cp paper_1607_04245_b200/libtxb.so /tmp/orig.so
for lib in default diag default diag; do
  cp tune_libs/libtxb_$lib.so paper_1607_04245_b200/libtxb.so
  timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench
for name in ('3d_varcoef_f64','3d_elasticity_f64','2d_varcoef_f64'):
    ms,_=bench.time_mesh(name, 200, 5)
    print('$lib', name, round(ms*1e3,2), flush=True)
" 2>&1 | grep -E "default|diag"
done
cp /tmp/orig.so paper_1607_04245_b200/libtxb.so
