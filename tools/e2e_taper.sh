#!/usr/bin/env bash
# e2e host path: zero copy (default for pinned buffers) vs staged pieces with a tapering tail.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {
  env "$@" timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import bench
for name in ('3d_varcoef_f64', '3d_varcoef_f32', '3d_elasticity_f64'):
    wl = bench.rank_workload(name, 0, 1)
    dt, h2d, d2h, _ = bench.time_e2e(wl, 30, 5)
    print('$*', name, round(dt / 30 * 1e3, 4), flush=True)
" 2>&1 | grep -v Warn | tail -3
}
run TXB_HOST_ZERO_COPY=1
for pm in 16 32 64; do for tail in 1 2 4; do run TXB_HOST_ZERO_COPY=0 TXB_HOST_PIECE_MB=$pm TXB_HOST_TAIL_MB=$tail; done; done
run TXB_HOST_ZERO_COPY=1
