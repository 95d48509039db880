"""STREAM-like probe in a graph chain at small sizes (the per-launch floor of any kernel moving
the 2D var-coef f64 bytes): python tools/small_probe.py"""
import sys, json, ctypes
sys.path.insert(0, '.')
import torch, bench
from paper_1607_04245_b200 import _lib
L = _lib.lib()
for n in (65536, 1 << 18, 1 << 20):
    rb, wb = 72 * n, 24 * n
    sets = 16
    src = [torch.ones(rb // 8, dtype=torch.float64, device="cuda") for _ in range(sets)]
    dst = [torch.empty(wb // 8, dtype=torch.float64, device="cuda") for _ in range(sets)]
    s = torch.cuda.current_stream()
    def launch(i):
        rc = L.txb_stream_probe(ctypes.c_void_p(src[i % sets].data_ptr()), rb, ctypes.c_void_p(dst[i % sets].data_ptr()), wb,
                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, _lib.last_error()
    for i in range(20): launch(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for i in range(200): launch(i)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 200 * 1e3
    print(json.dumps({"cells": n, "bytes": rb + wb, "probe_us": round(us, 3), "gbs": round((rb + wb) / us / 1e3, 1)}))
