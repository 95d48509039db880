"""Host-buffer call with PAGEABLE numpy arrays (what a reference user passes) vs
pinned: ms per call of txb_integrate_cells_host, 3D var-coef f64, 2^20 cells."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    from paper_1607_04245_b200 import backend

    name = sys.argv[1] if len(sys.argv) > 1 else "3d_varcoef_f64"
    flops, _ = bench.config_model(name)
    wl = bench.rank_workload(name, 0, 1)
    tab, rule = wl["tab"], wl["rule"]
    npdt = np.float32 if wl["dtype"] == "f32" else np.float64
    B, D, W = (np.ascontiguousarray(x, dtype=npdt) for x in (tab.basis, tab.basis_der, rule.weights))
    kernel = backend.cuda_kernel(wl["form"], rule.n_q, wl["aux"], np.dtype(npdt).itemsize)
    from paper_1607_04245_b200.physics import CellAux
    for label in ("pageable", "pinned"):
        if label == "pageable":
            cp = lambda t: t.cpu().numpy().copy()  # noqa: E731
            out = np.empty(tuple(wl["coeffs"].shape), dtype=npdt)
        else:
            def cp(t):
                h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                h.copy_(t)
                return h.numpy()
            out = torch.empty(tuple(wl["coeffs"].shape), dtype=wl["coeffs"].dtype, pin_memory=True).numpy()
        inv, det, co = cp(wl["inv"]), cp(wl["det"]), cp(wl["coeffs"])
        aux = None if wl["aux"] is None else CellAux("p0", cp(wl["aux"].values))
        for _ in range(2):
            backend.run_cuda(kernel, B, D, W, inv, det, co, aux, out)
        t0 = time.perf_counter()
        for _ in range(10):
            backend.run_cuda(kernel, B, D, W, inv, det, co, aux, out)
        dt = (time.perf_counter() - t0) / 10
        print(json.dumps({"config": name, "buffers": label, "ms_per_call": round(dt * 1e3, 3),
                          "e2e_gflops": round(flops * wl["n"] / dt / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
