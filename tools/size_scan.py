"""Per-launch time vs cell count (tuning aid): separates the fixed per-launch
cost (launch ramp + tail) from the streaming rate, t(n) = t0 + bytes(n) / BW.

python tools/size_scan.py [config ...]   -> one JSON line per (config, n), then a fit per config
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    configs = sys.argv[1:] or ["2d_varcoef_f32", "3d_varcoef_f32", "3d_varcoef_f64"]
    peak, _ = bench.peaks()
    for name in configs:
        dim, physics, dtype, _ = bench.CONFIGS[name]
        _, bpc = bench.config_model(name)
        xs, ys = [], []
        for lg in (18, 19, 20, 21, 22, 23):
            n = 1 << lg
            bench.CONFIGS["_scan"] = (dim, physics, dtype, n)
            wl = bench.rank_workload("_scan", 0, 1)
            n_sets = max(4, -(-3 * bench.L2_BYTES // (bpc * n)) + 1)
            steps = 400 if lg <= 20 else 100
            tot, _ = bench.time_device(wl, steps, 5, min(n_sets, 64))
            us = tot / steps * 1e3
            gbs = bpc * n / (us * 1e-6) / 1e9
            xs.append(bpc * n / 1e6)
            ys.append(us)
            print(json.dumps({"config": name, "log2_cells": lg, "us": round(us, 3), "gbs": round(gbs, 1),
                              "frac": round(gbs / peak, 3)}), flush=True)
            del wl
            torch.cuda.empty_cache()
        slope, t0 = np.polyfit(xs[2:], ys[2:], 1)  # fit on >= 2^20 cells
        print(json.dumps({"config": name, "fit_t0_us": round(float(t0), 3),
                          "fit_stream_gbs": round(1e3 / float(slope), 1)}), flush=True)


if __name__ == "__main__":
    main()
