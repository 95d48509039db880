"""Host-buffer (e2e) path modes of txb_integrate_cells_host, per configuration:
python tools/e2e_modes.py  -> one JSON line per (config, mode)
  TXB_HOST_MODE 0: DMA in (copy engine, growing pieces) + zero-copy out (default)
                1: zero copy (the kernel's bulk copies read mapped host memory)
                2: staged pieces over streams (the pageable-buffer path)"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    names = sys.argv[1:] or ["3d_varcoef_f64", "3d_varcoef_f32", "2d_varcoef_f64", "3d_elasticity_f64"]
    for name in names:
        flops, _ = bench.config_model(name)
        wl = bench.rank_workload(name, 0, 1)
        for rep in range(2):
            for mode in ("0", "1", "2"):
                os.environ["TXB_HOST_MODE"] = mode
                dt, h2d, d2h, _ = bench.time_e2e(wl, 10, 2)
                link = bench.h2d_link_gbs(h2d)
                print(json.dumps({"config": name, "mode": int(mode), "ms_per_step": round(dt / 10 * 1e3, 3),
                                  "e2e_gflops": round(flops * wl["n"] * 10 / dt / 1e9, 1),
                                  "frac_of_h2d_floor": round(h2d / link / 1e9 / (dt / 10), 3)}), flush=True)
        os.environ.pop("TXB_HOST_MODE", None)
        del wl


if __name__ == "__main__":
    main()
