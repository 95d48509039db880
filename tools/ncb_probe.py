"""The reference's (N_bl, N_cb) decompositions run as given vs the tuned default on
the device (graph-timed integrate_cells chains, 2^20 cells): profiles/r2_decomposition.md.
Run from the repo root: python tools/ncb_probe.py"""
import sys, json, os
sys.path.insert(0, '.')
import numpy as np, torch, bench
import paper_1607_04245_b200 as txb
for name in ("3d_varcoef_f64", "3d_varcoef_f32", "2d_varcoef_f32"):
    _, bpc = bench.config_model(name)
    wl = bench.rank_workload(name, 0, 1)
    out = torch.empty_like(wl["coeffs"])
    geom = txb.CellGeometry(wl["inv"], wl["det"])
    for n_bl, n_cb in ((32, 0), (32, 1), (32, 8), (32, 64), (8, 8)):
        fn = lambda: txb.integrate_cells(wl["tab"], wl["rule"], geom, wl["coeffs"], wl["aux"], wl["form"], dtype=wl["dtype"], out=out, n_bl=n_bl, n_cb=n_cb)
        for _ in range(3): fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            for _ in range(50): fn()
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        print(json.dumps({"cfg": name, "n_bl": n_bl, "n_cb": n_cb, "us": round(us, 2)}))
