"""Would a tile-permuted element layout speed up the scatter-add?  Element entries
(cell, b) re-laid out per tile in (vertex, cell) order -- the tile builder's sort
order -- so each vertex's entries are contiguous runs per tile; the slot CSR mapped
through the same permutation; graph-timed scatter, normal vs permuted layout
(same sums, same bits).  python tools/perm_scatter_probe.py [config] [cells]"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent))
from pipeline_bench import graph_time  # noqa: E402


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
    form = factory(dim)
    nc = form.n_comp
    full = txb.generate_unit_simplex_mesh(dim, refine_for(dim, n))
    mesh = txb.Mesh(dim, full.vertices, np.ascontiguousarray(full.cells[:n]))
    tdt = torch.float32 if dtype == "f32" else torch.float64
    cells = torch.from_numpy(mesh.cells).cuda()
    nb = dim + 1
    tile = 128 if dim == 3 else 192
    n_tiles = -(-n // tile)
    pad = n_tiles * tile - n
    keys = torch.cat([cells, torch.full((pad, nb), 1 << 40, dtype=torch.int64, device="cuda")]).view(n_tiles, tile * nb)
    pos = torch.arange(tile * nb, device="cuda", dtype=torch.int64)
    order = torch.argsort(keys * 2048 + pos, dim=1)
    rank = torch.empty_like(order)
    rank.scatter_(1, order, pos.expand(n_tiles, -1))
    P = (torch.arange(n_tiles, device="cuda").unsqueeze(1) * (tile * nb) + rank).view(-1)[: n * nb]
    inc = build_incidence(mesh, cells)
    elem = torch.randn((n, nb, nc), dtype=tdt, device="cuda")
    elem_p = torch.empty((n_tiles * tile * nb, nc), dtype=tdt, device="cuda")
    elem_p[P] = elem.view(-1, nc)
    inc_p = P[inc.slot_incidence.long()].to(torch.int32)
    out = torch.empty(mesh.n_vertices * nc, dtype=tdt, device="cuda")
    out_p = torch.empty_like(out)
    L = _lib.lib()

    def scat(e, si, o):
        L.txb_scatter_add_slots(e.element_size(), mesh.n_vertices, nc, inc.slot_offsets.data_ptr(), si.data_ptr(),
                                inc.slot_vertex.data_ptr(), e.data_ptr(), o.data_ptr(), _stream_ptr(torch))

    t0 = graph_time(lambda: scat(elem, inc.slot_incidence, out))
    t1 = graph_time(lambda: scat(elem_p, inc_p, out_p))
    torch.cuda.synchronize()
    same = bool(torch.equal(out.view(torch.int64 if dtype == "f64" else torch.int32),
                            out_p.view(torch.int64 if dtype == "f64" else torch.int32)))
    print(json.dumps({"config": name, "cells": n, "scatter_us": round(t0, 2), "scatter_permuted_us": round(t1, 2),
                      "same_bits": same}))


if __name__ == "__main__":
    main()
