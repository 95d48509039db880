"""Two-pass scatter-add probe (tools/probes/sorted_scatter_probe.cu): permute the
element entries into slot-ordered runs, then sum each run (plain or staged in
shared memory), against the shipped gather walk (txb_scatter_add_slots).
python tools/sorted_scatter_probe.py [config] [cells]   (scalar configs)"""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import bench  # noqa: E402
sys.path.insert(0, str(HERE))
from pipeline_bench import graph_time  # noqa: E402


def main():
    import torch

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200 import _lib
    from paper_1607_04245_b200.mesh import _stream_ptr, build_incidence
    from paper_1607_04245_b200.workload import refine_for

    so_path = HERE / "probes" / "sorted_scatter_probe.so"
    subprocess.run(["nvcc", "-O3", "-fmad=false", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler",
                    "-fPIC", "-shared", "-o", str(so_path), str(HERE / "probes" / "sorted_scatter_probe.cu")],
                   check=True)
    P = ctypes.CDLL(str(so_path))
    P.probe_permute.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 4
    P.probe_runs.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 5
    name = sys.argv[1] if len(sys.argv) > 1 else "3d_varcoef_f64"
    dim, physics, dtype, n = bench.CONFIGS[name]
    if len(sys.argv) > 2:
        n = int(sys.argv[2])
    full = txb.generate_unit_simplex_mesh(dim, refine_for(dim, n))
    mesh = txb.Mesh(dim, full.vertices, np.ascontiguousarray(full.cells[:n]))
    tdt = torch.float32 if dtype == "f32" else torch.float64
    w = 4 if dtype == "f32" else 8
    cells = torch.from_numpy(mesh.cells).cuda()
    inc = build_incidence(mesh, cells)
    nb, nv = dim + 1, mesh.n_vertices
    ne = n * nb
    pos = torch.empty(ne, dtype=torch.int32, device="cuda")
    pos[inc.slot_incidence.long()] = torch.arange(ne, dtype=torch.int32, device="cuda")
    elem = torch.randn((n, nb), dtype=tdt, device="cuda")
    sorted_ = torch.empty(ne, dtype=tdt, device="cuda")
    out0 = torch.empty(nv, dtype=tdt, device="cuda")
    out1 = torch.empty_like(out0)
    out2 = torch.empty_like(out0)
    L = _lib.lib()
    st = lambda: _stream_ptr(torch)  # noqa: E731

    def shipped():
        L.txb_scatter_add_slots(w, nv, 1, inc.slot_offsets.data_ptr(), inc.slot_incidence.data_ptr(),
                                inc.slot_vertex.data_ptr(), elem.data_ptr(), out0.data_ptr(), st())

    def permute():
        P.probe_permute(w, ne, pos.data_ptr(), elem.data_ptr(), sorted_.data_ptr(), st())

    def runs(staged, out):
        P.probe_runs(w, staged, nv, inc.slot_offsets.data_ptr(), inc.slot_vertex.data_ptr(), sorted_.data_ptr(),
                     out.data_ptr(), st())

    res = {"config": name, "cells": n,
           "shipped_us": graph_time(shipped),
           "permute_us": graph_time(permute),
           "runs_us": graph_time(lambda: runs(0, out1)),
           "runs_staged_us": graph_time(lambda: runs(1, out2))}
    res["permute_plus_runs_staged_us"] = graph_time(lambda: (permute(), runs(1, out2)))
    torch.cuda.synchronize()
    iv = torch.int64 if w == 8 else torch.int32
    res["same_bits"] = bool(torch.equal(out0.view(iv), out1.view(iv)) and torch.equal(out0.view(iv), out2.view(iv)))
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
