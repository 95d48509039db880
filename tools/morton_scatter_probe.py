"""Would a space-filling-curve vertex order speed up the scatter-add?  The slot
order (vertices by first incident element row) puts thin slabs of vertices in
one CTA; a Morton order of the vertex coordinates puts compact blocks there, so
the 4 vertices of a cell more often share the CTA (and its L1).  Builds the
slot CSR for a given vertex order on the host (numpy), graph-times
txb_scatter_add_slots for: first-row order (shipped), Morton order, Morton
order of 2^k-vertex blocks kept in first-row order inside.  Same chains, same
bits.  python tools/morton_scatter_probe.py [config] [cells]"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent))
from pipeline_bench import graph_time  # noqa: E402


def morton(v, bits=10):
    lo, hi = v.min(0), v.max(0)
    q = np.minimum(((v - lo) / np.maximum(hi - lo, 1e-300) * (1 << bits)).astype(np.int64), (1 << bits) - 1)
    key = np.zeros(len(v), dtype=np.int64)
    d = v.shape[1]
    for b in range(bits):
        for k in range(d):
            key |= ((q[:, k] >> b) & 1) << (b * d + k)
    return key


def main():
    import torch

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200 import _lib
    from paper_1607_04245_b200.mesh import _stream_ptr, build_incidence
    from paper_1607_04245_b200.workload import PHYSICS, refine_for

    name = sys.argv[1] if len(sys.argv) > 1 else "3d_varcoef_f64"
    dim, physics, dtype, n = bench.CONFIGS[name]
    if len(sys.argv) > 2:
        n = int(sys.argv[2])
    factory, _ = PHYSICS[physics]
    nc = factory(dim).n_comp
    full = txb.generate_unit_simplex_mesh(dim, refine_for(dim, n))
    mesh = txb.Mesh(dim, full.vertices, np.ascontiguousarray(full.cells[:n]))
    tdt = torch.float32 if dtype == "f32" else torch.float64
    cells = torch.from_numpy(mesh.cells).cuda()
    nb = dim + 1
    inc = build_incidence(mesh, cells)
    off = inc.offsets.cpu().numpy()
    ind = inc.incidence.cpu().numpy()
    nv = mesh.n_vertices
    cnt = np.diff(off)

    def slots(order):
        so = np.zeros(nv + 1, dtype=np.int64)
        so[1:] = np.cumsum(cnt[order])
        # vectorised gather of every list in `order`
        starts = off[order]
        rep = np.repeat(starts - so[:-1], cnt[order])
        idx = np.arange(so[-1]) + rep
        return (torch.from_numpy(so).cuda(), torch.from_numpy(ind[idx].astype(np.int32)).cuda(),
                torch.from_numpy(order.astype(np.int32)).cuda())

    first = np.where(cnt > 0, ind[np.minimum(off[:-1], len(ind) - 1)], np.iinfo(np.int32).max)
    orders = {"first_row": np.argsort(first, kind="stable"),
              "morton": np.argsort(morton(mesh.vertices), kind="stable")}
    mk = morton(mesh.vertices)
    for blk in (256, 1024):
        # blocks of the Morton order, each walked in first-row order
        grp = np.empty(nv, dtype=np.int64)
        grp[np.argsort(mk, kind="stable")] = np.arange(nv) // blk
        orders[f"morton_blocks{blk}"] = np.lexsort((first, grp))
    elem = torch.randn((n, nb, nc), dtype=tdt, device="cuda")
    L = _lib.lib()
    res, ref = {}, None
    for k, order in orders.items():
        so, si, sv = slots(order)
        out = torch.empty(nv * nc, dtype=tdt, device="cuda")

        def scat():
            L.txb_scatter_add_slots(elem.element_size(), nv, nc, so.data_ptr(), si.data_ptr(), sv.data_ptr(),
                                    elem.data_ptr(), out.data_ptr(), _stream_ptr(torch))

        res[k + "_us"] = round(graph_time(scat), 2)
        torch.cuda.synchronize()
        bits = out.view(torch.int64 if dtype == "f64" else torch.int32).clone()
        ref = bits if ref is None else ref
        res[k + "_same_bits"] = bool(torch.equal(bits, ref))
    print(json.dumps({"config": name, "cells": n, **res}))


if __name__ == "__main__":
    main()
