"""PCIe floor of the e2e call: pinned host <-> device copies of the headline's
bytes (126 MB in, 34 MB out per 2^20-cell 3D var-coef f64 call), H2D alone,
D2H alone, and both at once on two streams (copy engines, full duplex).
python tools/duplex_probe.py"""
import json
import time

import torch

H2D, D2H = 125_829_120, 33_554_432


def best(fn, reps=8):
    t = float("inf")
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        t = min(t, time.perf_counter() - t0)
    return t * 1e3


hs = torch.empty(H2D, dtype=torch.uint8, pin_memory=True)
hd = torch.empty(H2D, dtype=torch.uint8, device="cuda")
ds = torch.empty(D2H, dtype=torch.uint8, device="cuda")
dh = torch.empty(D2H, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        hd.copy_(hs, non_blocking=True)
    with torch.cuda.stream(s2):
        dh.copy_(ds, non_blocking=True)


r = {"h2d_ms": best(lambda: hd.copy_(hs, non_blocking=True)),
     "d2h_ms": best(lambda: dh.copy_(ds, non_blocking=True)),
     "duplex_ms": best(both)}
r["h2d_gbs"] = H2D / r["h2d_ms"] / 1e6
r["d2h_gbs"] = D2H / r["d2h_ms"] / 1e6
print(json.dumps({k: round(v, 3) for k, v in r.items()}))
