"""Static vs dynamic (cluster-launch-control) batch scheduling of the cell-array
kernel at the tuned defaults, per BASELINE configuration: python tools/dyn_scan.py"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

peak, _ = bench.peaks()
for name in ["3d_varcoef_f64", "3d_varcoef_f32", "2d_varcoef_f64", "2d_varcoef_f32", "2d_elasticity_f64",
             "2d_elasticity_f32", "3d_elasticity_f64", "3d_elasticity_f32", "2d_varcoef_f64_65536"]:
    _, bpc = bench.config_model(name)
    wl = bench.rank_workload(name, 0, 1)
    ns = bench.rotating_sets(bpc * wl["n"])
    for env in ({}, {"TXB_DYNAMIC": "1"}, {"TXB_DYNAMIC": "0"}, {"TXB_DYNAMIC": "1", "TXB_STATIC_PCT": "80"},
                {"TXB_DYNAMIC": "1", "TXB_STATIC_PCT": "40"}):
        os.environ.update(env)
        tot, _ = bench.time_device(wl, 200, 5, ns)
        for k in env:
            os.environ.pop(k)
        us = tot / 200 * 1e3
        print(json.dumps({"config": name, "env": env, "us": round(us, 3),
                          "frac": round(bpc * wl["n"] / (us * 1e-6) / 1e9 / peak, 4)}), flush=True)
    del wl
