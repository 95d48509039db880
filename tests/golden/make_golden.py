"""Generate the golden fixtures that pin the oracle and the CUDA lane.

TEST INFRASTRUCTURE.  Runs ONLY in the build container, where the reference
(`/root/reference/pkg/src/txfem`, read-only) is importable and its compiled
lane has been built into `oracle/_ref/` by `oracle/build_ref.sh`.  The GPU box
never runs this: it only reads the committed outputs

  tests/golden/small_cases.npz   full inputs + outputs for small problems
  tests/golden/big_hashes.json   sha256 of inputs/outputs for BASELINE configs
  tests/golden/user_cases.npz    user physics forms (f0, several aux fields,
                                 grad a; oracle/user_forms.py) through the
                                 reference's python lane, f64 and f32
  tests/golden/residual_cases.npz  mesh-level residuals of the reference's own
                                 txfem.integrate_transposed (executor.py:161-267):
                                 f32 / f64, remainder cells n_r > 0 (float64
                                 + cast in the reference), every shipped form,
                                 midpoint and two-point rules, perturbed
                                 meshes with shuffled numbering
  tests/golden/residual_hashes.json  sha256 of larger integrate_transposed
                                 residuals (84k-cell 3D meshes)

Every output here comes from the reference itself:
  * ``ref_f64``  txfem.reference.integrate_reference (reference.py:40-112)
  * ``cy_f64`` / ``cy_f32``  the reference's compiled lane
    _kernels_cy.integrate_cells (_kernels_cy.pyx:37-123), marshalled exactly
    like txfem.backend.run_compiled (backend.py:55-87).

Input conventions follow the reference tests and CLI:
  * Kuhn meshes (mesh.py:81-147) + compute_geometry (mesh.py:150-190);
  * N(0,1) global coefficients from default_rng(seed), gathered
    (tests/conftest.py:27-28, cli.py:79-81, mesh.py:202-217);
  * P0 kappa ~ U[0.5,1.5) from default_rng(seed+1) (cli.py:96-99);
    P1 kappa nodal U[0.5,1.5) from default_rng(seed+2) (tests/conftest.py:37-40);
  * random near-identity Jacobians J = I + 0.2 U(-1,1)
    (tests/test_executor.py:273-280).

Usage:  python tests/golden/make_golden.py [user|residual]   (only user_cases.npz / the residual goldens)
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REPO / "oracle" / "_ref"))

import txfem  # noqa: E402  (reference package, read-only)
from txfem.mesh import CellGeometry, Mesh  # noqa: E402
from txfem.physics import CellAux  # noqa: E402

import _kernels_cy  # noqa: E402  (reference compiled lane, built by oracle/build_ref.sh)

OUT = Path(__file__).resolve().parent

FORMS = {
    "poisson": (txfem.poisson_form, None),
    "varcoef_p0": (txfem.poisson_varcoef_form, "p0"),
    "varcoef_p1": (txfem.poisson_varcoef_form, "p1"),
    "elasticity": (txfem.elasticity_form, None),
}
FORM_CODE = {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}
AUX_MODE = {None: 0, "p0": 1, "p1": 2}


def run_compiled(form, tab, rule, inv_j, det_j, coeffs, aux, dtype):
    """backend.run_compiled (backend.py:55-87) on inputs cast once to dtype
    (executor._device_arrays, executor.py:77-90)."""
    dt = np.dtype(dtype)
    B = np.ascontiguousarray(tab.basis, dtype=dt)
    D = np.ascontiguousarray(tab.basis_der, dtype=dt)
    W = np.ascontiguousarray(rule.weights, dtype=dt)
    ij = np.ascontiguousarray(inv_j, dtype=dt)
    dj = np.ascontiguousarray(det_j, dtype=dt)
    co = np.ascontiguousarray(coeffs, dtype=dt)
    aux_const = np.empty((0, 0), dtype=dt)
    aux_nodal = np.empty((0, 0, 0), dtype=dt)
    mode = AUX_MODE[None if aux is None else aux.space]
    if mode == 1:
        aux_const = np.ascontiguousarray(aux.values, dtype=dt)
    elif mode == 2:
        aux_nodal = np.ascontiguousarray(aux.values, dtype=dt)
    out = np.empty(co.shape, dtype=dt)
    _kernels_cy.integrate_cells(
        FORM_CODE[form.name], mode, B, D, W, ij, dj, co, aux_const, aux_nodal, out
    )
    return out


def kuhn_problem(dim, refine, form, aux_space, rule, seed):
    mesh = txfem.generate_unit_simplex_mesh(dim, refine)
    layout = txfem.FieldLayout(n_comp=form.n_comp)
    geom = txfem.compute_geometry(mesh)
    coeffs = txfem.gather_coefficients(
        mesh, layout, np.random.default_rng(seed).standard_normal(layout.global_size(mesh))
    )
    aux = None
    if aux_space == "p0":
        aux = CellAux("p0", np.random.default_rng(seed + 1).uniform(0.5, 1.5, (mesh.n_cells, 1)))
    elif aux_space == "p1":
        nodal = np.random.default_rng(seed + 2).uniform(0.5, 1.5, (mesh.n_vertices, 1))
        aux = CellAux("p1", nodal[mesh.cells])
    return geom.inv_jacobians, geom.determinants, coeffs, aux


def randj_problem(dim, n, form, aux_space, seed):
    rng = np.random.default_rng(seed)
    jac = np.broadcast_to(np.eye(dim), (n, dim, dim)).copy()
    jac += 0.2 * rng.uniform(-1.0, 1.0, jac.shape)
    det = np.linalg.det(jac)
    assert (det > 0).all()
    inv = np.linalg.inv(jac)
    n_b = dim + 1
    coeffs = rng.standard_normal((n, n_b, form.n_comp))
    aux = None
    if aux_space == "p0":
        aux = CellAux("p0", rng.uniform(0.5, 1.5, (n, 1)))
    elif aux_space == "p1":
        aux = CellAux("p1", rng.uniform(0.5, 1.5, (n, n_b, 1)))
    return np.ascontiguousarray(inv), np.ascontiguousarray(det), coeffs, aux


def small_cases():
    arrays = {}
    index = []
    for dim, refine in ((2, 6), (3, 3)):
        for fname, (factory, aux_space) in FORMS.items():
            form = factory(dim)
            for rname, rule in (("q1", txfem.quadrature_rule(dim, 1)), ("q2", txfem.two_point_rule(dim))):
                tab = txfem.tabulate(dim, rule)
                for family in ("kuhn", "randj"):
                    seed = 100 * dim + 7 * len(index) + 3
                    if family == "kuhn":
                        inv, det, coeffs, aux = kuhn_problem(dim, refine, form, aux_space, rule, seed)
                    else:
                        inv, det, coeffs, aux = randj_problem(dim, 97, form, aux_space, seed)
                    ref = txfem.integrate_reference(tab, rule, CellGeometry(inv, det), form, coeffs, aux)
                    cy64 = run_compiled(form, tab, rule, inv, det, coeffs, aux, np.float64)
                    cy32 = run_compiled(form, tab, rule, inv, det, coeffs, aux, np.float32)
                    # The reference's own lanes agree bitwise in f64 (tests/test_backends.py).
                    assert np.array_equal(cy64.view(np.uint64), ref.view(np.uint64)), (dim, fname, rname, family)
                    name = f"{dim}d_{fname}_{rname}_{family}"
                    index.append(name)
                    arrays[f"{name}/basis"] = tab.basis
                    arrays[f"{name}/basis_der"] = tab.basis_der
                    arrays[f"{name}/weights"] = rule.weights
                    arrays[f"{name}/inv_j"] = inv
                    arrays[f"{name}/det_j"] = det
                    arrays[f"{name}/coeffs"] = coeffs
                    if aux is not None:
                        arrays[f"{name}/aux"] = aux.values
                    arrays[f"{name}/ref_f64"] = ref
                    arrays[f"{name}/cy_f32"] = cy32
                    meta = dict(dim=dim, form=form.name, aux=aux_space, n_q=rule.n_q, n_comp=form.n_comp)
                    arrays[f"{name}/meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    return arrays


# ---- BASELINE.json configs: too big to commit, pinned by hash -------------------

BIG = [
    # (name, dim, physics, n_cells)  — BASELINE.json configs[0..3]
    ("2d_varcoef_p0_65536", 2, "varcoef_p0", 65536),
    ("3d_varcoef_p0_1048576", 3, "varcoef_p0", 1 << 20),
    ("2d_elasticity_1048576", 2, "elasticity", 1 << 20),
    ("3d_elasticity_1048576", 3, "elasticity", 1 << 20),
]
BIG_SEED = 1234  # cli.py RunConfig.seed default


def refine_for(dim, n_cells):
    r = 1
    while (2 * r * r if dim == 2 else 6 * r ** 3) < n_cells:
        r += 1
    return r


def big_workload(dim, physics, n_cells, seed=BIG_SEED):
    """Kuhn mesh sliced to exactly n_cells (cells are independent), reference
    geometry, seeded gathered coefficients and P0 kappa (cli._problem)."""
    factory, aux_space = FORMS[physics]
    form = factory(dim)
    full = txfem.generate_unit_simplex_mesh(dim, refine_for(dim, n_cells))
    mesh = Mesh(dim=dim, vertices=full.vertices, cells=full.cells[:n_cells])
    layout = txfem.FieldLayout(n_comp=form.n_comp)
    geom = txfem.compute_geometry(mesh)
    glob = np.random.default_rng(seed).standard_normal(layout.global_size(full))
    coeffs = txfem.gather_coefficients(mesh, layout, glob)
    aux = None
    if aux_space == "p0":
        aux = CellAux("p0", np.random.default_rng(seed + 1).uniform(0.5, 1.5, (full.n_cells, 1))[:n_cells])
    return form, geom.inv_jacobians, geom.determinants, coeffs, aux


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def big_hashes():
    out = {}
    for name, dim, physics, n in BIG:
        form, inv, det, coeffs, aux = big_workload(dim, physics, n)
        rule = txfem.quadrature_rule(dim, 1)
        tab = txfem.tabulate(dim, rule)
        ref = txfem.integrate_reference(tab, rule, CellGeometry(inv, det), form, coeffs, aux)
        cy64 = run_compiled(form, tab, rule, inv, det, coeffs, aux, np.float64)
        cy32 = run_compiled(form, tab, rule, inv, det, coeffs, aux, np.float32)
        assert np.array_equal(cy64, ref)
        full = txfem.generate_unit_simplex_mesh(dim, refine_for(dim, n))
        entry = {
            "dim": dim, "physics": physics, "n_cells": n, "seed": BIG_SEED,
            "refine": refine_for(dim, n),
            "mesh": {"vertices": sha(full.vertices), "cells": sha(full.cells)},
            "inputs_f64": {"inv_j": sha(inv), "det_j": sha(det), "coeffs": sha(coeffs)},
            "ref_f64": sha(ref),
            "cy_f32": sha(cy32),
            "ref_f64_absmax": float(np.abs(ref).max()),
            "cy_f32_sum": float(cy32.astype(np.float64).sum()),
        }
        if aux is not None:
            entry["inputs_f64"]["aux"] = sha(aux.values)
        out[name] = entry
        print(name, "done", flush=True)
    return out


# ---- user physics (run-time compiled lane) ---------------------------------------

def user_cases():
    """Every spec of oracle/user_forms.py, built with the REFERENCE's user_form,
    integrated by the reference's python lane (_kernels_py.integrate_cells,
    _kernels_py.py:20-110) on inputs cast once to the run dtype."""
    from txfem import _kernels_py
    from txfem.physics import user_form as ref_user_form

    sys.path.insert(0, str(REPO))
    from oracle import user_forms

    arrays, index = {}, []
    for dim, refine in ((2, 5), (3, 2)):
        for sname in user_forms.SPECS:
            spec = user_forms.spec(sname, dim)
            form = user_forms.make_form(ref_user_form, sname, dim)
            rng_tab = np.random.default_rng(17 * dim + len(sname))
            rules = [("q1", *_tables(txfem.quadrature_rule(dim, 1), dim)),
                     ("q2", *_tables(txfem.two_point_rule(dim), dim)),
                     ("q3rand", rng_tab.uniform(0, 1, (3, dim + 1)), rng_tab.uniform(-1, 1, (3, dim + 1, dim)),
                      rng_tab.uniform(0.1, 0.5, 3))]
            for rname, B, D, W in rules:
                for family in ("kuhn", "randj"):
                    seed = 1000 + 100 * dim + 7 * len(index)
                    pform = FORMS["poisson"][0](dim) if spec["n_comp"] == 1 else FORMS["elasticity"][0](dim)
                    if family == "kuhn":
                        mesh = txfem.generate_unit_simplex_mesh(dim, refine)
                        inv, det, coeffs, _ = kuhn_problem(dim, refine, pform, None, None, seed)
                        n = mesh.n_cells
                    else:
                        n = 61
                        inv, det, coeffs, _ = randj_problem(dim, n, pform, None, seed)
                    aux = None
                    rng = np.random.default_rng(seed + 5)
                    if spec["aux"] == "p0":
                        aux = CellAux("p0", rng.uniform(0.5, 1.5, (n, spec["n_aux"])))
                    elif spec["aux"] == "p1":
                        if family == "kuhn":
                            nodal = rng.uniform(0.5, 1.5, (mesh.n_vertices, spec["n_aux"]))
                            aux = CellAux("p1", np.ascontiguousarray(nodal[mesh.cells]))
                        else:
                            aux = CellAux("p1", rng.uniform(0.5, 1.5, (n, dim + 1, spec["n_aux"])))
                    name = f"{dim}d_{sname}_{rname}_{family}"
                    index.append(name)
                    for dt, tag in ((np.float64, "py_f64"), (np.float32, "py_f32")):
                        c = lambda a: np.ascontiguousarray(a, dtype=dt)  # noqa: E731
                        out = np.empty((n, dim + 1, spec["n_comp"]), dtype=dt)
                        ax = None if aux is None else CellAux(aux.space, c(aux.values))
                        _kernels_py.integrate_cells(form, c(B), c(D), c(W), c(inv), c(det), c(coeffs), ax, out)
                        arrays[f"{name}/{tag}"] = out
                    arrays[f"{name}/basis"] = B
                    arrays[f"{name}/basis_der"] = D
                    arrays[f"{name}/weights"] = W
                    arrays[f"{name}/inv_j"] = inv
                    arrays[f"{name}/det_j"] = det
                    arrays[f"{name}/coeffs"] = coeffs
                    if aux is not None:
                        arrays[f"{name}/aux"] = aux.values
                    meta = dict(dim=dim, spec=sname, aux=spec["aux"], n_q=int(B.shape[0]), n_comp=spec["n_comp"])
                    arrays[f"{name}/meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    return arrays


RESIDUAL_FORMS = ["poisson", "varcoef_p0", "varcoef_p1", "elasticity"]


def residual_problem(dim, refine, physics, seed):
    """A perturbed Kuhn mesh with a shuffled vertex numbering and cell order,
    N(0,1) global coefficients, the form's aux (reference conventions)."""
    rng = np.random.default_rng(seed)
    base = txfem.generate_unit_simplex_mesh(dim, refine)
    perm = rng.permutation(base.n_vertices)
    verts = base.vertices[np.argsort(perm)] + (0.15 / refine) * rng.uniform(-1, 1, base.vertices.shape)
    cells = perm[base.cells][rng.permutation(base.n_cells)]
    mesh = Mesh(dim=dim, vertices=np.ascontiguousarray(verts), cells=np.ascontiguousarray(cells))
    factory, aux_space = FORMS[physics]
    form = factory(dim)
    layout = txfem.FieldLayout(n_comp=form.n_comp)
    glob = rng.standard_normal(layout.global_size(mesh))
    aux = None
    if aux_space == "p0":
        aux = CellAux("p0", rng.uniform(0.5, 1.5, (mesh.n_cells, 1)))
    elif aux_space == "p1":
        aux = CellAux("p1", rng.uniform(0.5, 1.5, (mesh.n_vertices, 1))[mesh.cells])
    return mesh, form, layout, glob, aux


def residual_cases():
    """integrate_transposed of the reference (default lane: compiled) with
    n_bl / n_cb chosen so n mod N_chunk > 0."""
    arrays, index = {}, []
    for dim, refine in ((2, 9), (3, 4)):
        for physics in RESIDUAL_FORMS:
            for n_q in (1, 2):
                seed = 100 * dim + 10 * RESIDUAL_FORMS.index(physics) + n_q
                mesh, form, layout, glob, aux = residual_problem(dim, refine, physics, seed)
                rule = txfem.quadrature_rule(dim, 1) if n_q == 1 else txfem.two_point_rule(dim)
                tab = txfem.tabulate(dim, rule)
                n_bl, n_cb = 5, 3
                g = txfem.derive_execution_geometry(dim, tab.n_b, form.n_comp, rule.n_q, n_bl, n_cb, mesh.n_cells)
                assert g.n_r > 0 and g.n_chunks > 0
                name = f"{dim}d_{physics}_q{n_q}"
                for dt in ("f64", "f32"):
                    res, trace = txfem.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=n_bl,
                                                            n_cb=n_cb, dtype=dt, shared_mem_limit=None)
                    assert trace.remainder_cells == g.n_r
                    arrays[f"{name}/res_{dt}"] = res
                arrays[f"{name}/vertices"] = mesh.vertices
                arrays[f"{name}/cells"] = mesh.cells
                arrays[f"{name}/glob"] = glob
                if aux is not None:
                    arrays[f"{name}/aux"] = aux.values
                meta = dict(dim=dim, physics=physics, n_q=n_q, n_bl=n_bl, n_cb=n_cb, n_r=g.n_r,
                            span=g.n_chunks * g.n_chunk, aux=None if aux is None else aux.space)
                arrays[f"{name}/meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
                index.append(name)
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    return arrays


def residual_hashes():
    """Larger residuals by hash: 3D refine 24 (82,944 cells), seeded as
    residual_problem, midpoint rule, n_bl = 32 / n_cb = 7 (n_r > 0)."""
    out = {}
    for physics in ("varcoef_p0", "elasticity"):
        mesh, form, layout, glob, aux = residual_problem(3, 24, physics, 7)
        rule = txfem.quadrature_rule(3, 1)
        tab = txfem.tabulate(3, rule)
        g = txfem.derive_execution_geometry(3, tab.n_b, form.n_comp, 1, 32, 7, mesh.n_cells)
        ent = {"n_cells": mesh.n_cells, "n_r": g.n_r, "inputs": sha(np.concatenate(
            [mesh.vertices.ravel(), mesh.cells.ravel().astype(np.float64), glob]
            + ([aux.values.ravel()] if aux is not None else [])))}
        for dt in ("f64", "f32"):
            res, _ = txfem.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=32, n_cb=7,
                                                dtype=dt, shared_mem_limit=None)
            ent[dt] = sha(res)
        out[f"3d_{physics}_refine24"] = ent
    return out


def _tables(rule, dim):
    tab = txfem.tabulate(dim, rule)
    return tab.basis, tab.basis_der, rule.weights


def main():
    if sys.argv[1:] == ["residual"]:
        np.savez_compressed(OUT / "residual_cases.npz", **residual_cases())
        (OUT / "residual_hashes.json").write_text(json.dumps(residual_hashes(), indent=1) + "\n")
        print("wrote", OUT / "residual_cases.npz", OUT / "residual_hashes.json")
        return
    if sys.argv[1:] == ["user"]:
        np.savez_compressed(OUT / "user_cases.npz", **user_cases())
        print("wrote", OUT / "user_cases.npz")
        return
    np.savez_compressed(OUT / "user_cases.npz", **user_cases())
    arrays = small_cases()
    np.savez_compressed(OUT / "small_cases.npz", **arrays)
    (OUT / "big_hashes.json").write_text(json.dumps(big_hashes(), indent=1) + "\n")
    np.savez_compressed(OUT / "residual_cases.npz", **residual_cases())
    (OUT / "residual_hashes.json").write_text(json.dumps(residual_hashes(), indent=1) + "\n")
    print("wrote", OUT / "small_cases.npz", OUT / "big_hashes.json", OUT / "residual_cases.npz")


if __name__ == "__main__":
    main()
