"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

  compute-sanitizer --tool racecheck python tools/sanitize_workload.py

Covers the ahead-of-time integration kernel (all forms, f32/f64, n_q 1-3,
static and dynamic batch scheduling, ragged tails, unaligned buffers), the
fused mesh kernels (given geometry; in-kernel geometry per cell and over
tiles with per-tile vertex tables), gather, incidence build,
scatter-add, geometry, the run-time compiled kernel (cell arrays and mesh entry
points) and the halo pack/assemble.
Every result is checked against the oracle so a sanitizer run is also a
parity run.  Test/tuning infrastructure: uses oracle/ as the checker.
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


QUICK = os.environ.get("SANITIZE_QUICK", "0") == "1"  # fewer sizes (racecheck is ~100x slower)


def main():
    import torch

    import paper_1607_04245_b200 as txb
    from oracle import oracle, user_forms
    from paper_1607_04245_b200 import halo
    from paper_1607_04245_b200.physics import CellAux

    dev = lambda x, dt=np.float64: torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).cuda()  # noqa: E731
    checks = 0
    for dim in (2, 3):
        for physics, fc, am in (("varcoef_p0", 1, 1), ("varcoef_p1", 1, 2), ("elasticity", 2, 0), ("poisson", 0, 0)):
            for n in ((1, 37, 600) if QUICK else (1, 37, 2000, 40_000)):
                _, inv, det, co, aux = oracle.workload(dim, physics, n, seed=n)
                for n_q in ((1, 3) if QUICK else (1, 2, 3)):
                    B, D, W = oracle.p1_tables(dim, min(n_q, 2))
                    if n_q == 3:
                        rng = np.random.default_rng(3)
                        B, D, W = rng.uniform(0, 1, (3, dim + 1)), rng.uniform(-1, 1, (3, dim + 1, dim)), rng.uniform(0.1, 0.5, 3)
                    for dt in (np.float64, np.float32):
                        out = torch.full(co.shape, float("nan"), dtype=torch.float64 if dt == np.float64 else torch.float32,
                                         device="cuda")
                        ax = None if aux is None else CellAux("p0" if am == 1 else "p1", dev(aux, dt))
                        for n_cb in (0, 3):  # dynamic (default) and the paper's static chunks
                            txb.run_cuda((fc, am), B, D, W, dev(inv, dt), dev(det, dt), dev(co, dt), ax, out, n_cb=n_cb)
                            torch.cuda.synchronize()
                            ref = oracle.integrate(fc, am, B, D, W, inv, det, co, aux, dt)
                            assert out.cpu().numpy().tobytes() == ref.tobytes(), (dim, physics, n, n_q, dt, n_cb)
                            checks += 1
    # unaligned buffers (global-load fallback)
    _, inv, det, co, aux = oracle.workload(3, "varcoef_p0", 999, seed=5)
    B, D, W = oracle.p1_tables(3)
    raw = torch.empty(999 * 9 + 1, dtype=torch.float64, device="cuda")
    iv = raw[1:].view(999, 3, 3)
    iv.copy_(dev(inv))
    out = torch.empty((999, 4, 1), dtype=torch.float64, device="cuda")
    txb.run_cuda((1, 1), B, D, W, iv, dev(det), dev(co), CellAux("p0", dev(aux)), out)
    torch.cuda.synchronize()
    assert out.cpu().numpy().tobytes() == oracle.integrate(1, 1, B, D, W, inv, det, co, aux).tobytes()
    checks += 1

    # mesh-level: geometry, gather, incidence + scatter, fused mesh kernel, halo
    for dim, refine in ((2, 20), (3, 6)):
        mesh = txb.generate_unit_simplex_mesh(dim, refine)
        for form in (txb.poisson_varcoef_form(dim), txb.elasticity_form(dim)):
            layout = txb.FieldLayout(form.n_comp)
            rule = txb.quadrature_rule(dim, 1)
            tab = txb.tabulate(dim, rule)
            glob = np.random.default_rng(1).standard_normal(layout.global_size(mesh))
            aux = CellAux("p0", np.random.default_rng(2).uniform(0.5, 1.5, (mesh.n_cells, 1))) if form.n_aux else None
            res, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=4, n_cb=2)
            g = txb.compute_geometry(mesh, device_out=True)
            res2, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=4, n_cb=2,
                                               cell_geom=g)
            inv, det = oracle.geometry(mesh.vertices, mesh.cells)
            elem = oracle.integrate(1 if form.n_aux else 2, 1 if form.n_aux else 0, tab.basis, tab.basis_der,
                                    rule.weights, inv, det, oracle.gather(mesh.cells, glob, form.n_comp),
                                    None if aux is None else aux.values)
            want = oracle.scatter_add(mesh.cells, elem, mesh.n_vertices)
            assert res.tobytes() == want.tobytes() and res2.tobytes() == want.tobytes()
            blocks = txb.gather_coefficients(mesh, layout, glob)
            assert blocks.tobytes() == oracle.gather(mesh.cells, glob, form.n_comp).tobytes()
            # two emulated ranks through the halo plan
            got = np.zeros_like(want)
            box = {}
            for r in (1, 0):
                plan = halo.build_halo_plan(mesh.cells, mesh.n_vertices, r, 2, 16)

                def ex(recv, send, rs, ss, r=r):
                    if r == 1:
                        box["m"] = send.clone()
                    else:
                        recv.copy_(box["m"])

                ids, vals, _ = txb.integrate_partitioned(mesh, layout, tab, rule, form, glob, aux, rank=r, world=2,
                                                         exchange=ex, plan=plan)
                got.reshape(-1, form.n_comp)[ids] = vals.cpu().numpy().reshape(-1, form.n_comp)
            assert got.tobytes() == want.tobytes()
            checks += 4

    # tiled mesh kernel (geometry + gather from per-tile vertex tables): shuffled numbering (uint16 local
    # indices), partial last tile, both basis phases (midpoint in-lane, two-point transposed), P1 aux,
    # an unaligned aux base (global-memory aux path), f32 and f64
    rng = np.random.default_rng(12)
    base = txb.generate_unit_simplex_mesh(3, 5)
    perm = rng.permutation(base.n_vertices)
    smesh = txb.Mesh(3, np.ascontiguousarray(base.vertices[np.argsort(perm)]),
                     np.ascontiguousarray(perm[base.cells][rng.permutation(base.n_cells)][:700]))
    for m in (smesh, txb.generate_unit_simplex_mesh(2, 13)):
        dim = m.dim
        form = txb.poisson_varcoef_form(dim)
        glob = rng.standard_normal(m.n_vertices)
        nodal = rng.uniform(0.5, 1.5, (m.n_vertices, 1))[m.cells]
        inv, det = oracle.geometry(m.vertices, m.cells)
        for rule in (txb.quadrature_rule(dim, 1), txb.two_point_rule(dim)):
            tab = txb.tabulate(dim, rule)
            for dt, tdt in ((np.float64, torch.float64), (np.float32, torch.float32)):
                raw = torch.empty(nodal.size + 1, dtype=tdt, device="cuda")
                av = raw[1:].view(nodal.shape)
                av.copy_(dev(nodal, dt))
                out = txb.integrate_mesh(m, txb.FieldLayout(1), tab, rule, form, dev(glob, dt), CellAux("p1", av),
                                         dtype="f64" if dt == np.float64 else "f32")
                torch.cuda.synchronize()
                ref = oracle.integrate(1, 2, tab.basis, tab.basis_der, rule.weights, inv, det,
                                       oracle.gather(m.cells, glob, 1), nodal, dt)
                assert out.cpu().numpy().tobytes() == ref.tobytes(), (dim, rule.n_q, dt)
                checks += 1

    # run-time compiled user forms
    for name in user_forms.SPECS:
        s = user_forms.spec(name, 3)
        f = user_forms.make_form(txb.user_form, name, 3)
        n = 5000
        rng = np.random.default_rng(9)
        jac = np.eye(3) + 0.2 * rng.uniform(-1, 1, (n, 3, 3))
        inv, det = np.linalg.inv(jac), np.linalg.det(jac)
        co = rng.standard_normal((n, 4, s["n_comp"]))
        aux = None
        if s["aux"]:
            shape = (n, s["n_aux"]) if s["aux"] == "p0" else (n, 4, s["n_aux"])
            aux = CellAux(s["aux"], rng.uniform(0.5, 1.5, shape))
        B, D, W = oracle.p1_tables(3, 2)
        k = txb.cuda_kernel(f, 2, aux, 8)
        out = torch.empty((n, 4, s["n_comp"]), dtype=torch.float64, device="cuda")
        txb.run_cuda(k, B, D, W, dev(inv), dev(det), dev(co), None if aux is None else CellAux(aux.space, dev(aux.values)),
                     out)
        torch.cuda.synchronize()
        ref = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], B, D, W, inv, det, co,
                                     None if aux is None else aux.values)
        assert out.cpu().numpy().tobytes() == ref.tobytes(), name
        checks += 1
        # the same form on a mesh: the mesh entry point (geometry + gather in-kernel) + scatter-add
        mesh = txb.generate_unit_simplex_mesh(3, 3)
        layout = txb.FieldLayout(s["n_comp"])
        glob = rng.standard_normal(layout.global_size(mesh))
        maux = None
        if s["aux"]:
            shape = (mesh.n_cells, s["n_aux"]) if s["aux"] == "p0" else (mesh.n_cells, 4, s["n_aux"])
            maux = CellAux(s["aux"], rng.uniform(0.5, 1.5, shape))
        rule = txb.quadrature_rule(3, 1)
        tab = txb.tabulate(3, rule)
        res, _ = txb.integrate_transposed(mesh, layout, tab, rule, f, glob, maux, n_bl=8, n_cb=2,
                                          shared_mem_limit=None)
        minv, mdet = oracle.geometry(mesh.vertices, mesh.cells)
        elem = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], tab.basis,
                                      tab.basis_der, rule.weights, minv, mdet,
                                      oracle.gather(mesh.cells, glob, s["n_comp"]),
                                      None if maux is None else maux.values)
        assert res.tobytes() == oracle.scatter_add(mesh.cells, elem, mesh.n_vertices).tobytes(), name
        checks += 1
    print(f"sanitize_workload: {checks} checks bit-identical to the oracle", flush=True)


if __name__ == "__main__":
    os.environ.setdefault("TXB_PDL", "1")
    main()
