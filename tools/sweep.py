"""Launch-parameter sweep of the integration kernel on one GPU (tuning aid).

python tools/sweep.py [config ...]   -> one line per (config, threads, smem target, stages)
Environment knobs read by libtxb per launch: TXB_TARGET_THREADS, TXB_SMEM_TARGET, TXB_STAGES.
"""
import itertools
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    configs = sys.argv[1:] or ["3d_varcoef_f64", "3d_varcoef_f32", "3d_elasticity_f64", "3d_elasticity_f32", "2d_varcoef_f32",
                               "2d_varcoef_f64", "2d_elasticity_f32"]
    peak, _ = bench.peaks()
    for name in configs:
        flops, bpc = bench.config_model(name)
        wl = bench.rank_workload(name, 0, 1)
        n_sets = max(4, -(-3 * bench.L2_BYTES // (bpc * wl["n"])) + 1)
        best = None
        knobs = os.environ.get("SWEEP_GRID", "cells=128,256 inflight=48,72 dyn=0,1 pct=50,75,90 pf=-1")
        kv = dict(x.split("=") for x in knobs.split())
        grid = [(int(c), int(i), int(dy), int(pc), int(pf)) for c in kv["cells"].split(",")
                for i in kv["inflight"].split(",") for dy in kv["dyn"].split(",")
                for pc in (kv["pct"].split(",") if dy == "1" else ["0"]) for pf in kv.get("pf", "-1").split(",")]
        for threads, smem, pdl, pct, pf in grid:
            os.environ["TXB_PREFETCH_BATCHES"] = str(pf)
            os.environ["TXB_STATIC_PCT"] = str(pct)
            os.environ["TXB_TARGET_CELLS"] = str(threads)
            os.environ["TXB_INFLIGHT_KB"] = str(smem)
            os.environ["TXB_DYNAMIC"] = str(pdl)
            try:
                tot, _ = bench.time_device(wl, 200, 5, n_sets)
            except Exception as exc:  # capacity etc.
                print(json.dumps({"config": name, "cells": threads, "smem_kb": smem, "error": str(exc)[:120]}))
                continue
            ms = tot / 200
            gbs = bpc * wl["n"] / (ms * 1e-3) / 1e9
            from paper_1607_04245_b200 import backend

            form = wl["form"]
            w = 4 if wl["dtype"] == "f32" else 8
            cfg = backend.launch_config(*backend.cuda_kernel(form, 1, wl["aux"], w), w, wl["dim"], 1,
                                        form.n_comp, wl["n"])
            rec = {"config": name, "cells": threads, "inflight_kb": smem, "dynamic": pdl, "static_pct": pct, "prefetch": pf, "gbs": round(gbs, 1),
                   "frac": round(gbs / peak, 3), "us": round(ms * 1e3, 2), **cfg}
            print(json.dumps(rec), flush=True)
            if best is None or gbs > best["gbs"]:
                best = rec
        print("BEST", json.dumps(best), flush=True)
        for k in ("TXB_TARGET_CELLS", "TXB_INFLIGHT_KB", "TXB_DYNAMIC", "TXB_STATIC_PCT", "TXB_PREFETCH_BATCHES"):
            os.environ.pop(k, None)
        del wl
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
