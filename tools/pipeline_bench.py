"""Per-stage timing of the mesh-level residual pipeline (next rows of SURVEY §8f)
on one config: geometry, gather, integrate (cell arrays), fused mesh kernel with
and without given geometry, scatter-add (vertex order and slot order).
Graph-timed, 2^20 cells unless given.

python tools/pipeline_bench.py [config] [cells]
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def graph_time(fn, steps=50, warmup=3):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        for _ in range(steps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps * 1e3  # us


def main():
    import torch

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200.mesh import build_incidence
    from paper_1607_04245_b200.workload import PHYSICS, refine_for

    name = sys.argv[1] if len(sys.argv) > 1 else "3d_varcoef_f64"
    dim, physics, dtype, n = bench.CONFIGS[name]
    if len(sys.argv) > 2:
        n = int(sys.argv[2])
    factory, aux_space = PHYSICS[physics]
    form = factory(dim)
    full = txb.generate_unit_simplex_mesh(dim, refine_for(dim, n))
    mesh = txb.Mesh(dim, full.vertices, np.ascontiguousarray(full.cells[:n]))
    layout = txb.FieldLayout(form.n_comp)
    npdt = np.float32 if dtype == "f32" else np.float64
    tdt = torch.float32 if dtype == "f32" else torch.float64
    cells = torch.from_numpy(mesh.cells).cuda()
    verts = torch.from_numpy(np.ascontiguousarray(mesh.vertices)).cuda()
    glob = torch.from_numpy(np.random.default_rng(1).standard_normal(full.n_vertices * form.n_comp).astype(npdt)).cuda()
    aux = txb.CellAux("p0", torch.rand((n, 1), dtype=tdt, device="cuda") + 0.5) if aux_space == "p0" else None
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    geom64 = txb.compute_geometry(mesh, cells=cells, vertices=verts, device_out=True)
    geom = txb.CellGeometry(geom64.inv_jacobians.to(tdt), geom64.determinants.to(tdt))
    blocks = txb.gather_coefficients(mesh, layout, glob, cells=cells)
    out = torch.empty((n, dim + 1, form.n_comp), dtype=tdt, device="cuda")
    inc = build_incidence(mesh, cells)
    inc_plain = build_incidence(mesh, cells, slot_order=False)
    res = {}
    res["geometry_kernel_us"] = graph_time(lambda: txb.compute_geometry(mesh, cells=cells, device_out=True)) \
        if False else None  # (syncs on the orientation flag: not graph-capturable)
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        txb.compute_geometry(mesh, cells=cells, vertices=verts, device_out=True)
    torch.cuda.synchronize()
    res["geometry_kernel_us(wall, incl. flag sync)"] = (time.perf_counter() - t0) / 20 * 1e6
    res["gather_us"] = graph_time(lambda: txb.gather_coefficients(mesh, layout, glob, cells=cells))
    res["integrate_cells_us"] = graph_time(lambda: txb.integrate_cells(tab, rule, geom, blocks, aux, form,
                                                                       dtype=dtype, out=out))
    res["mesh_fused_given_geometry_us"] = graph_time(lambda: txb.integrate_mesh(
        mesh, layout, tab, rule, form, glob, aux, dtype=dtype, cell_geom=geom, cells=cells, vertices=verts, out=out,
        check_orientation=False))
    res["mesh_fused_geometry_us"] = graph_time(lambda: txb.integrate_mesh(
        mesh, layout, tab, rule, form, glob, aux, dtype=dtype, cells=cells, vertices=verts, out=out,
        check_orientation=False))
    resid = torch.empty(full.n_vertices * form.n_comp, dtype=tdt, device="cuda")
    res["scatter_us"] = graph_time(lambda: txb.scatter_add_element_vectors(mesh, layout, out, incidence=inc))
    res["scatter_vertex_order_us"] = graph_time(
        lambda: txb.scatter_add_element_vectors(mesh, layout, out, incidence=inc_plain))
    print(json.dumps({"config": name, "cells": n, **{k: (round(v, 2) if v else v) for k, v in res.items()}}))


if __name__ == "__main__":
    main()
