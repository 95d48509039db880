"""Static share of the dynamic schedule (TXB_STATIC_PCT) x L2 prefetch depth for the
shortest 2^20-cell launches, 3 repetitions each: python tools/pct_scan.py"""
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

peak, _ = bench.peaks()
for name in ["2d_elasticity_f32", "2d_varcoef_f32", "3d_elasticity_f32"]:
    _, bpc = bench.config_model(name)
    wl = bench.rank_workload(name, 0, 1)
    ns = bench.rotating_sets(bpc * wl["n"])
    for pct in (30, 40, 50, 60, 70, 80):
        for pf in (-1, 8):
            os.environ["TXB_STATIC_PCT"] = str(pct)
            os.environ["TXB_PREFETCH_BATCHES"] = str(pf)
            us = [bench.time_device(wl, 200, 5, ns)[0] / 200 * 1e3 for _ in range(3)]
            m = statistics.median(us)
            print(json.dumps({"config": name, "pct": pct, "prefetch": pf, "us": round(m, 3),
                              "frac": round(bpc * wl["n"] / (m * 1e-6) / 1e9 / peak, 4)}), flush=True)
    for k in ("TXB_STATIC_PCT", "TXB_PREFETCH_BATCHES"):
        os.environ.pop(k, None)
    del wl
