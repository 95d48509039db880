#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_jit.py -m gpu -q --timeout 600 2>&1 | tail -1
python - <<'PY'
import json, sys, statistics
sys.path.insert(0, '.')
import bench
peak, _ = bench.peaks()
for name in ("3d_elasticity_f64", "3d_varcoef_f64", "3d_varcoef_f32", "2d_elasticity_f64", "3d_elasticity_f32"):
    _, bpc = bench.config_model(name)
    wl = bench.rank_workload(name, 0, 1)
    ns = bench.rotating_sets(bpc * wl["n"])
    us = [bench.time_device(wl, 200, 5, ns)[0] / 200 * 1e3 for _ in range(3)]
    m = statistics.median(us)
    print(json.dumps({"config": name, "us": round(m, 3), "frac": round(bpc * wl["n"] / (m * 1e-6) / 1e9 / peak, 4)}))
PY
