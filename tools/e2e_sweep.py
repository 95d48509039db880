"""Host-buffer (e2e) path tuning aid: pieces x streams of txb_integrate_cells_host.

python tools/e2e_sweep.py [config]   -> one JSON line per (piece MiB, slots)
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    name = sys.argv[1] if len(sys.argv) > 1 else "3d_varcoef_f64"
    flops, bpc = bench.config_model(name)
    wl = bench.rank_workload(name, 0, 1)
    # raw PCIe probes: pinned H2D / D2H of the step's bytes
    h = torch.empty(126 << 20, dtype=torch.uint8, pin_memory=True)
    d = torch.empty_like(h, device="cuda")
    for direction in ("h2d", "d2h"):
        src, dst = (h, d) if direction == "h2d" else (d, h)
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"probe": direction, "gbs": round(5 * h.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)}))
    for mb in (2, 4, 8, 16, 32):
        for slots in (2, 3, 4):
            os.environ["TXB_HOST_PIECE_MB"] = str(mb)
            os.environ["TXB_HOST_SLOTS"] = str(slots)
            dt, h2d, d2h, _ = bench.time_e2e(wl, 10, 2)
            gf = flops * wl["n"] * 10 / dt / 1e9
            print(json.dumps({"config": name, "piece_mb": mb, "slots": slots, "ms_per_step": round(dt / 10 * 1e3, 3),
                              "e2e_gflops": round(gf, 1), "h2d_gbs_effective": round(h2d * 10 / dt / 1e9, 1)}),
                  flush=True)


if __name__ == "__main__":
    main()
