#!/usr/bin/env bash
# e2e zero-copy host path: batch size (TXB_TARGET_CELLS) and in-flight bytes; ms per call.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for e in "X=1" "TXB_TARGET_CELLS=256" "TXB_TARGET_CELLS=512" "TXB_TARGET_CELLS=1024" "TXB_INFLIGHT_KB=160" "TXB_STATIC_PCT=100" "TXB_STATIC_PCT=0" "X=1"; do
  env $e timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import bench
for name in ('3d_varcoef_f64', '3d_varcoef_f32'):
    wl = bench.rank_workload(name, 0, 1)
    dt, h2d, d2h, _ = bench.time_e2e(wl, 30, 5)
    print('$e', name, round(dt / 30 * 1e3, 4), flush=True)
" 2>&1 | grep -E "^(X|TXB)"
done
