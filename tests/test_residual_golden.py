"""Mesh-level residuals against the reference's OWN integrate_transposed.

tests/golden/residual_cases.npz and residual_hashes.json hold residuals the
reference produced (txfem.integrate_transposed, executor.py:161-267, default
lane) on perturbed, renumbered Kuhn meshes with remainder cells n_r > 0 --
which the reference integrates in float64 and casts (executor.py:258-264) --
for every shipped form, the midpoint and two-point rules, f32 and f64
(tests/golden/make_golden.py).  Bar: bit-identical in BOTH precisions.

* CPU: the oracle's residual (geometry -> gather -> integrate in the run
  precision, float64 remainder, np.add.at order) is pinned to them.
* GPU: integrate_transposed of this framework -- in-kernel geometry and given
  geometry -- reproduces them bit for bit.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, bitwise_equal, rel_err
from oracle import oracle

NPZ = np.load(GOLDEN / "residual_cases.npz")
NAMES = json.loads(bytes(NPZ["index"]).decode())
HASHES = json.loads((GOLDEN / "residual_hashes.json").read_text())
FC = {"poisson": 0, "varcoef_p0": 1, "varcoef_p1": 1, "elasticity": 2}


def case(name):
    meta = json.loads(bytes(NPZ[f"{name}/meta"]).decode())
    aux = NPZ[f"{name}/aux"] if f"{name}/aux" in NPZ.files else None
    return meta, NPZ[f"{name}/vertices"], NPZ[f"{name}/cells"], NPZ[f"{name}/glob"], aux


def oracle_residual(meta, verts, cells, glob, aux, npdt):
    dim = meta["dim"]
    n_comp = dim if meta["physics"] == "elasticity" else 1
    B, D, W = oracle.p1_tables(dim, meta["n_q"])
    inv, det = oracle.geometry(verts, cells)
    am = {None: 0, "p0": 1, "p1": 2}[meta["aux"]]
    elem = oracle.integrate_with_remainder(FC[meta["physics"]], am, B, D, W, inv, det,
                                           oracle.gather(cells, glob, n_comp), aux, npdt, meta["span"])
    return oracle.scatter_add(cells, elem, verts.shape[0])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("name", NAMES)
def test_oracle_pinned_to_reference_residuals(name, dtype):
    meta, verts, cells, glob, aux = case(name)
    assert meta["n_r"] > 0
    npdt = np.float64 if dtype == "f64" else np.float32
    got = oracle_residual(meta, verts, cells, glob, aux, npdt)
    assert bitwise_equal(got, NPZ[f"{name}/res_{dtype}"])


def test_oracle_f32_remainder_matters():
    """The golden f32 residuals really depend on the float64 remainder: an
    all-f32 evaluation differs from them (so the GPU test below pins it)."""
    differs = 0
    for name in NAMES:
        meta, verts, cells, glob, aux = case(name)
        m = dict(meta, span=cells.shape[0])  # no remainder: every cell in f32
        differs += not bitwise_equal(oracle_residual(m, verts, cells, glob, aux, np.float32),
                                     NPZ[f"{name}/res_f32"])
    assert differs >= len(NAMES) // 2


# ----------------------------------------------------------------------------- GPU
def _txb_problem(name):
    import paper_1607_04245_b200 as txb

    meta, verts, cells, glob, aux = case(name)
    dim = meta["dim"]
    factory = {"poisson": txb.poisson_form, "varcoef_p0": txb.poisson_varcoef_form,
               "varcoef_p1": txb.poisson_varcoef_form, "elasticity": txb.elasticity_form}[meta["physics"]]
    form = factory(dim)
    rule = txb.quadrature_rule(dim, 1) if meta["n_q"] == 1 else txb.two_point_rule(dim)
    mesh = txb.Mesh(dim, verts, cells)
    ax = None if aux is None else txb.CellAux(meta["aux"], aux)
    return txb, meta, mesh, form, rule, txb.tabulate(dim, rule), txb.FieldLayout(form.n_comp), glob, ax


@pytest.mark.gpu
@pytest.mark.parametrize("given", [False, True])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("name", NAMES)
def test_integrate_transposed_reproduces_reference_residual(name, dtype, given):
    txb, meta, mesh, form, rule, tab, layout, glob, aux = _txb_problem(name)
    cg = None
    if given:
        inv, det = oracle.geometry(mesh.vertices, mesh.cells)
        cg = txb.CellGeometry(inv, det)
    res, trace = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=meta["n_bl"],
                                          n_cb=meta["n_cb"], dtype=dtype, shared_mem_limit=None, cell_geom=cg)
    want = NPZ[f"{name}/res_{dtype}"]
    assert trace.remainder_cells == meta["n_r"]
    assert rel_err(res, NPZ[f"{name}/res_f64"]) <= (1e-5 if dtype == "f32" else 1e-12)
    assert bitwise_equal(res, want)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("key", sorted(HASHES))
def test_integrate_transposed_reference_residual_hashes(key, dtype):
    import paper_1607_04245_b200 as txb

    physics = key.split("_")[1]
    ent = HASHES[key]
    rng = np.random.default_rng(7)  # residual_problem(3, 24, physics, 7) of make_golden.py
    base = txb.generate_unit_simplex_mesh(3, 24)
    perm = rng.permutation(base.n_vertices)
    verts = base.vertices[np.argsort(perm)] + (0.15 / 24) * rng.uniform(-1, 1, base.vertices.shape)
    cells = perm[base.cells][rng.permutation(base.n_cells)]
    mesh = txb.Mesh(3, np.ascontiguousarray(verts), np.ascontiguousarray(cells))
    form = txb.poisson_varcoef_form(3) if physics == "varcoef" else txb.elasticity_form(3)
    layout = txb.FieldLayout(form.n_comp)
    glob = rng.standard_normal(layout.global_size(mesh))
    aux = txb.CellAux("p0", rng.uniform(0.5, 1.5, (mesh.n_cells, 1))) if form.n_aux else None
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    inputs = np.concatenate([mesh.vertices.ravel(), mesh.cells.ravel().astype(np.float64), glob]
                            + ([aux.values.ravel()] if aux is not None else []))
    assert sha(inputs) == ent["inputs"]
    rule = txb.quadrature_rule(3, 1)
    res, _ = txb.integrate_transposed(mesh, layout, txb.tabulate(3, rule), rule, form, glob, aux, n_bl=32,
                                      n_cb=7, dtype=dtype, shared_mem_limit=None)
    assert sha(res) == ent[dtype]
