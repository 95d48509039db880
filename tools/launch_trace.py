"""Per-launch timeline of the integration kernel inside a graph-captured chain
(tuning aid): where the fixed per-launch cost t0 goes.

python tools/launch_trace.py [config] [launches]
Each launch's CTAs stamp %globaltimer at entry, after griddepcontrol.wait, at
their first ready batch (libtxb built with NVCC_EXTRA=-DTXB_TRACE_FIRST_BATCH
only; the stamp costs registers) and when their consumers finish
(txb_debug_trace).
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import ctypes

    import torch

    from paper_1607_04245_b200 import _lib, backend
    from paper_1607_04245_b200.physics import CellAux

    name = sys.argv[1] if len(sys.argv) > 1 else "3d_varcoef_f64"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    _, bpc = bench.config_model(name)
    wl = bench.rank_workload(name, 0, 1)
    n_sets = max(4, -(-3 * bench.L2_BYTES // (bpc * wl["n"])) + 1)
    width = 4 if wl["dtype"] == "f32" else 8
    kernel = backend.cuda_kernel(wl["form"], 1, wl["aux"], width)
    sets = []
    for _ in range(n_sets):
        aux = None if wl["aux"] is None else CellAux(wl["aux"].space, wl["aux"].values.clone())
        sets.append((wl["inv"].clone(), wl["det"].clone(), wl["coeffs"].clone(), aux, torch.empty_like(wl["coeffs"])))
    npdt = np.float32 if width == 4 else np.float64
    B, D, W = (np.ascontiguousarray(x, dtype=npdt) for x in (wl["tab"].basis, wl["tab"].basis_der, wl["rule"].weights))

    def launch(i):
        inv, det, co, aux, out = sets[i % n_sets]
        backend.run_cuda(kernel, B, D, W, inv, det, co, aux, out)

    for i in range(5):
        launch(i)
    torch.cuda.synchronize()
    cfg = backend.launch_config(*kernel, width, wl["dim"], 1, wl["form"].n_comp, wl["n"])
    grid = cfg["grid"]
    buf = torch.zeros(4 * grid * K, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    g = torch.cuda.CUDAGraph()
    L.txb_debug_trace(ctypes.c_void_p(buf.data_ptr()), buf.numel())
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for i in range(K):
            launch(i)
    L.txb_debug_trace(None, 0)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    buf.zero_()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = buf.cpu().numpy().reshape(K, grid, 4).astype(np.int64)
    ran = t[:, :, 0] > 0  # dynamic scheduling: CTAs cancelled by cluster launch control never run
    t0 = t[:, :, 0][ran].min()
    rows = []
    for k in range(K):
        s = t[k][ran[k]] - t0
        rows.append({"launch": k, "entry_first": int(s[:, 0].min()), "entry_last": int(s[:, 0].max()),
                     "wait_done_first": int(s[:, 1].min()), "wait_done_last": int(s[:, 1].max()),
                     "first_batch_med": int(np.median(s[:, 2])), "first_batch_last": int(s[:, 2].max()),
                     "done_first": int(s[:, 3].min()), "done_med": int(np.median(s[:, 3])), "done_last": int(s[:, 3].max())})
    for r in rows:
        print(json.dumps(r))
    steady = rows[2:-1]
    per = np.diff([r["done_last"] for r in rows[1:]]).mean()
    ideal = bpc * wl["n"] / 6545.9e9 * 1e9
    summary = {
        "config": name, "grid": grid, "ctas_run_per_launch": round(float(ran.sum(1).mean()), 1), "graph_us_per_launch": round(e0.elapsed_time(e1) / K * 1e3, 2),
        "period_ns": round(float(per), 1), "ideal_copy_peak_ns": round(ideal, 1),
        "wait_release_after_prev_done_ns": round(float(np.mean([rows[k]["wait_done_first"] - rows[k - 1]["done_last"] for k in range(2, K)])), 1),
        "first_batch_after_release_ns": round(float(np.mean([r["first_batch_med"] - r["wait_done_first"] for r in steady])), 1),
        "tail_ns(done_last-done_med)": round(float(np.mean([r["done_last"] - r["done_med"] for r in steady])), 1),
        "spread_ns(done_last-done_first)": round(float(np.mean([r["done_last"] - r["done_first"] for r in steady])), 1),
        "entry_before_prev_done_ns": round(float(np.mean([rows[k - 1]["done_last"] - rows[k]["entry_first"] for k in range(2, K)])), 1),
    }
    print("SUMMARY", json.dumps(summary))


if __name__ == "__main__":
    main()
