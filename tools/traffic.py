"""DRAM traffic of ONE integration launch, write-back included (roofline.traffic).

A kernel-replay ncu capture sees only the DRAM writes that leave L2 while the
kernel runs: most of a 2^20-cell launch's element vectors are still dirty in
the 126 MB L2 when it ends, so the kernel-level dram__bytes_write.sum
under-counts the compulsory writes.  This tool measures reads and writes
separately:

  reads   kernel replay with --cache-control all (cold L2 before the launch):
          dram__bytes_read.sum of the integration kernel;
  writes  range replay over [integration launch; read-only 1 GiB sweep]: the
          sweep evicts every dirty line, so the range's dram__bytes_write.sum
          is the launch's complete write-back (the sweep itself writes
          nothing; a sweep-only range is measured as the baseline).

Usage (on the GPU box; both runs execute the same script):
  ncu --replay-mode range --metrics M --csv \
      --log-file gpurun_out/TAG_traffic_range.csv  python tools/traffic.py run
  ncu --profile-from-start off --cache-control all --clock-control none \
      -k regex:integrate --metrics M --csv \
      --log-file gpurun_out/TAG_traffic_kernel.csv python tools/traffic.py run
  python tools/traffic.py summarize TAG    # -> profiles/ncu_traffic.json,
                                           #    profiles/TAG_traffic.md
with M = dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum.
"""

from __future__ import annotations

import csv
import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

CONFIGS = ["3d_varcoef_f64", "3d_varcoef_f32", "2d_varcoef_f64", "2d_varcoef_f32", "2d_elasticity_f64",
           "2d_elasticity_f32", "3d_elasticity_f64", "3d_elasticity_f32"]
SWEEP_BYTES = 1 << 30
TO_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TO_NS = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}


def run(configs):
    import numpy as np
    import torch

    import bench
    from paper_1607_04245_b200 import backend

    torch.cuda.set_device(0)
    sweep = torch.ones(SWEEP_BYTES, dtype=torch.uint8, device="cuda")

    words = sweep.view(torch.int64)

    def flush():
        # read sweep with DEFAULT-policy loads (a torch reduction): it evicts --
        # writes back -- every dirty L2 line; evict-first (.cs) loads would only
        # recycle their own lines and leave the launch's outputs dirty in L2
        words.sum()

    for name in configs:
        wl = bench.rank_workload(name, 0, 1)
        width = 4 if wl["dtype"] == "f32" else 8
        kernel = backend.cuda_kernel(wl["form"], 1, wl["aux"], width)
        npdt = np.float32 if width == 4 else np.float64
        B, D, W = (np.ascontiguousarray(x, dtype=npdt) for x in (wl["tab"].basis, wl["tab"].basis_der,
                                                                  wl["rule"].weights))
        out = torch.empty_like(wl["coeffs"])

        def launch():
            backend.run_cuda(kernel, B, D, W, wl["inv"], wl["det"], wl["coeffs"], wl["aux"], out)

        launch()  # module load, attribute setup
        for _ in range(2):
            flush()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()  # range 1: the launch + the evicting sweep
        launch()
        flush()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        for _ in range(2):
            flush()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()  # range 2: the sweep alone (baseline)
        flush()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        print(json.dumps({"config": name, "cells": wl["n"]}), flush=True)
        del wl, out
        torch.cuda.empty_cache()


def _rows(path):
    """ncu --csv rows -> list of (id, metric, value in bytes or ns)."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 4]
    hdr = rows[0]
    iid, im, iv, iu = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        u = r[iu]
        v *= TO_B.get(u, TO_NS.get(u, 1.0))
        out.append((int(r[iid]), r[im], v))
    return out


def _by_id(rows):
    d = {}
    for i, m, v in rows:
        d.setdefault(i, {})[m] = v
    return [d[k] for k in sorted(d)]


def summarize(tag, configs):
    import bench

    rng = _by_id(_rows(REPO / "gpurun_out" / f"{tag}_traffic_range.csv"))
    ker = _by_id(_rows(REPO / "gpurun_out" / f"{tag}_traffic_kernel.csv"))
    assert len(rng) == 2 * len(configs) and len(ker) == len(configs), (len(rng), len(ker))
    res = {}
    md = [f"# DRAM traffic per launch, write-back included (`{tag}`, tools/traffic.py)", "",
          "reads: kernel replay, `--cache-control all`; writes: range replay over [launch; 1 GiB read-only "
          "sweep] minus the sweep-only range.  Algorithmic bytes = SURVEY.md §8(d) compulsory B/cell x cells.", "",
          "| config | cells | algorithmic MB | read MB | write MB | (read+write)/algorithmic | kernel-only write MB |"
          " sweep-only write MB |", "|---|---:|---:|---:|---:|---:|---:|---:|"]
    for k, name in enumerate(configs):
        n = bench.CONFIGS[name][3]
        _, bpc = bench.config_model(name)
        both, base = rng[2 * k], rng[2 * k + 1]
        rd = ker[k]["dram__bytes_read.sum"]
        wr = both["dram__bytes_write.sum"] - base["dram__bytes_write.sum"]
        alg = bpc * n
        res[name] = {"read_bytes_per_cell": rd / n, "write_bytes_per_cell": wr / n, "algorithmic_bytes_per_cell": bpc,
                     "ratio": (rd + wr) / alg, "kernel_only_write_bytes_per_cell": ker[k]["dram__bytes_write.sum"] / n,
                     "source": f"profiles/{tag}_traffic.md (tools/traffic.py)"}
        md.append(f"| {name} | {n} | {alg / 1e6:.2f} | {rd / 1e6:.2f} | {wr / 1e6:.2f} | {(rd + wr) / alg:.3f} | "
                  f"{ker[k]['dram__bytes_write.sum'] / 1e6:.2f} | {base['dram__bytes_write.sum'] / 1e6:.2f} |")
    out = {"how": "tools/traffic.py: reads from a cold-L2 kernel replay, writes from a range replay over the launch "
                  "and an evicting read-only sweep (write-back included)", "tag": tag, "configs": res}
    (REPO / "profiles" / "ncu_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    (REPO / "profiles" / f"{tag}_traffic.md").write_text("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "run"
    if mode == "run":
        run(sys.argv[2:] or CONFIGS)
    elif mode == "summarize":
        summarize(sys.argv[2], sys.argv[3:] or CONFIGS)
    else:
        raise SystemExit(__doc__)
