#!/usr/bin/env bash
# e2e host path for pinned buffers: DMA in (arrival flags, one kernel) vs zero copy; ms per call.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
run() {
  env "$@" timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import bench
for name in ('3d_varcoef_f64', '3d_varcoef_f32', '3d_elasticity_f64', '2d_varcoef_f64'):
    wl = bench.rank_workload(name, 0, 1)
    dt, h2d, d2h, _ = bench.time_e2e(wl, 30, 5)
    print('$*', name, round(dt / 30 * 1e3, 4), flush=True)
" 2>&1 | grep -v Warn | tail -4
}
run TXB_HOST_DMA=0
for pm in 8 16 32; do run TXB_HOST_DMA=1 TXB_HOST_PIECE_MB=$pm; done
run TXB_HOST_DMA=0
