"""Device gather / scatter-add / geometry vs the oracle, bitwise."""

import numpy as np
import pytest

from conftest import bitwise_equal
from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1607_04245_b200 as txb  # noqa: E402


@pytest.mark.parametrize("dim,n", [(2, 50), (3, 12)])
def test_geometry_bitwise(dim, n):
    mesh = txb.generate_unit_simplex_mesh(dim, n)
    g = txb.compute_geometry(mesh)
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    assert bitwise_equal(g.inv_jacobians, inv) and bitwise_equal(g.determinants, det)
    # perturbed (non-grid) vertices
    rng = np.random.default_rng(1)
    v = mesh.vertices + 0.1 / n * rng.uniform(-1, 1, mesh.vertices.shape)
    m2 = txb.Mesh(dim, v, mesh.cells)
    g2 = txb.compute_geometry(m2)
    inv2, det2 = oracle.geometry(v, mesh.cells)
    assert bitwise_equal(g2.inv_jacobians, inv2) and bitwise_equal(g2.determinants, det2)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("seed", [0, 1])
def test_geometry_division_on_random_simplices(dim, seed):
    """2^20 random simplices over 12 decades of scale and arbitrary shapes: the
    device's reciprocal + two-correction quotient (DetDivider) equals numpy's
    correctly rounded x / det for every one of the 9.4 M (3D) entries."""
    rng = np.random.default_rng(seed)
    n = 1 << 20
    scale = 10.0 ** rng.uniform(-6, 6, (n, 1, 1))
    x = rng.uniform(-1, 1, (n, dim + 1, dim)) * scale
    x[: n // 8] = np.round(x[: n // 8] * 64) / 64  # lattice-like cells: exact zeros and small integers
    verts = x.reshape(-1, dim)
    cells = np.arange(n * (dim + 1), dtype=np.int64).reshape(n, dim + 1)
    with np.errstate(divide="ignore", invalid="ignore"):  # degenerate draws are dropped below
        _, det = oracle.geometry(verts, cells)
        flip = det < 0  # orient every simplex positively (swap two vertices)
        cells[flip, 1], cells[flip, 2] = cells[flip, 2].copy(), cells[flip, 1].copy()
        keep = np.nonzero(oracle.geometry(verts, cells)[1] > 0)[0]
    cells = np.ascontiguousarray(cells[keep])
    m = txb.Mesh(dim, verts, cells)
    g = txb.compute_geometry(m)
    inv, det = oracle.geometry(verts, cells)
    assert bitwise_equal(g.determinants, det)
    assert bitwise_equal(g.inv_jacobians, inv)


@pytest.mark.parametrize("n_comp", [1, 2, 3])
def test_gather_and_scatter_bitwise(n_comp):
    mesh = txb.generate_unit_simplex_mesh(3, 9)
    layout = txb.FieldLayout(n_comp)
    g = np.random.default_rng(2).standard_normal(layout.global_size(mesh))
    blocks = txb.gather_coefficients(mesh, layout, g)
    assert bitwise_equal(blocks, oracle.gather(mesh.cells, g, n_comp))
    elem = np.random.default_rng(3).standard_normal((mesh.n_cells, 4, n_comp))
    for dt in (np.float64, np.float32):
        e = elem.astype(dt)
        assert bitwise_equal(txb.scatter_add_element_vectors(mesh, layout, e),
                             oracle.scatter_add(mesh.cells, e, mesh.n_vertices))


@pytest.mark.parametrize("case", ["kuhn3d", "shuffled", "isolated", "empty_mesh"])
@pytest.mark.parametrize("n_comp", [1, 3])
def test_slot_order_scatter_bitwise(case, n_comp):
    """The slot-ordered scatter (vertices visited by first element row) and the
    vertex-ordered one give the oracle's np.add.at sums bit for bit; the slot
    order is a permutation, each slot carries its vertex's list unchanged."""
    from paper_1607_04245_b200.mesh import build_incidence

    mesh = txb.generate_unit_simplex_mesh(3, 7)
    cells, nv = mesh.cells, mesh.n_vertices
    rng = np.random.default_rng(4)
    if case == "shuffled":  # random vertex numbering and cell order
        perm = rng.permutation(nv)
        cells = perm[cells][rng.permutation(len(cells))]
    elif case == "isolated":  # vertices no cell touches sit between used ones
        cells = cells * 3 + 1
        nv = nv * 3 + 2
    elif case == "empty_mesh":
        cells = cells[:0]
    m = txb.Mesh(3, np.zeros((nv, 3)), np.ascontiguousarray(cells))
    layout = txb.FieldLayout(n_comp)
    cells_dev = torch.from_numpy(m.cells).cuda()
    plain, slots = build_incidence(m, cells_dev, slot_order=False), build_incidence(m, cells_dev)
    sv = slots.slot_vertex[:nv].cpu().numpy()
    assert np.array_equal(np.sort(sv), np.arange(nv))
    so, si = slots.slot_offsets.cpu().numpy(), slots.slot_incidence.cpu().numpy()
    po, pi = plain.offsets.cpu().numpy(), plain.incidence.cpu().numpy()
    for t in rng.choice(nv, min(nv, 200), replace=False):
        v = sv[t]
        assert np.array_equal(si[so[t]:so[t + 1]], pi[po[v]:po[v + 1]])
    first = [pi[po[v]] if po[v + 1] > po[v] else np.iinfo(np.int64).max for v in sv]
    assert all(a <= b for a, b in zip(first, first[1:]))
    for dt in (np.float64, np.float32):
        e = rng.standard_normal((m.n_cells, 4, n_comp)).astype(dt)
        want = oracle.scatter_add(m.cells, e, nv)
        assert bitwise_equal(txb.scatter_add_element_vectors(m, layout, e, incidence=slots), want)
        assert bitwise_equal(txb.scatter_add_element_vectors(m, layout, e, incidence=plain), want)


def test_scatter_multiplicity_oracle():
    """scatter_add(gather(one-hot)) counts cells per vertex (SPEC mesh invariants)."""
    mesh = txb.generate_unit_simplex_mesh(2, 7)
    layout = txb.FieldLayout(1)
    ones = txb.gather_coefficients(mesh, layout, np.ones(mesh.n_vertices))
    counts = txb.scatter_add_element_vectors(mesh, layout, ones)
    np.testing.assert_array_equal(counts, np.bincount(mesh.cells.ravel(), minlength=mesh.n_vertices))


# ---- fused mesh kernel (txb_integrate_mesh): geometry + gather + cast + integrate ----

import hashlib  # noqa: E402

from conftest import BIG  # noqa: E402

FORMS = [(txb.poisson_form, None), (txb.poisson_varcoef_form, "p0"), (txb.poisson_varcoef_form, "p1"),
         (txb.elasticity_form, None)]


def _mesh_problem(dim, n, factory, aux_space, seed, perturb=True):
    mesh = txb.generate_unit_simplex_mesh(dim, n)
    if perturb:  # non-grid vertices, still positively oriented
        rng = np.random.default_rng(seed)
        mesh = txb.Mesh(dim, mesh.vertices + 0.15 / n * rng.uniform(-1, 1, mesh.vertices.shape), mesh.cells)
    form = factory(dim)
    glob = np.random.default_rng(seed + 1).standard_normal(mesh.n_vertices * form.n_comp)
    aux = None
    if aux_space == "p0":
        aux = txb.CellAux("p0", np.random.default_rng(seed + 2).uniform(0.5, 1.5, (mesh.n_cells, 1)))
    elif aux_space == "p1":
        nodal = np.random.default_rng(seed + 3).uniform(0.5, 1.5, (mesh.n_vertices, 1))
        aux = txb.CellAux("p1", nodal[mesh.cells])
    return mesh, form, glob, aux


def _oracle_elem(mesh, form, glob, aux, rule, npdt):
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    blocks = oracle.gather(mesh.cells, glob, form.n_comp)
    tab = txb.tabulate(mesh.dim, rule)
    fc = {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}[form.name]
    am = {None: 0, "p0": 1, "p1": 2}[None if aux is None else aux.space]
    return oracle.integrate(fc, am, tab.basis, tab.basis_der, rule.weights, inv, det, blocks,
                            None if aux is None else aux.values, npdt), (inv, det)


@pytest.mark.parametrize("dim,n", [(2, 23), (3, 7)])
@pytest.mark.parametrize("factory,aux_space", FORMS)
def test_fused_mesh_kernel_bitwise(dim, n, factory, aux_space):
    mesh, form, glob, aux = _mesh_problem(dim, n, factory, aux_space, seed=5 * dim + n)
    layout = txb.FieldLayout(form.n_comp)
    for rule in (txb.quadrature_rule(dim, 1), txb.two_point_rule(dim)):
        tab = txb.tabulate(dim, rule)
        for dtype, npdt, tdt in (("f64", np.float64, torch.float64), ("f32", np.float32, torch.float32)):
            ref, (inv, det) = _oracle_elem(mesh, form, glob, aux, rule, npdt)
            g = torch.from_numpy(glob.astype(npdt)).cuda()
            out = txb.integrate_mesh(mesh, layout, tab, rule, form, g, aux, dtype=dtype)
            assert bitwise_equal(out.cpu().numpy(), ref), (dtype, rule.n_q, "geometry from vertices")
            out = txb.integrate_mesh(mesh, layout, tab, rule, form, g, aux, dtype=dtype,
                                     cell_geom=txb.CellGeometry(inv, det))
            assert bitwise_equal(out.cpu().numpy(), ref), (dtype, rule.n_q, "given geometry")
            for n_bl in (1, 5, 32):
                out = txb.integrate_mesh(mesh, layout, tab, rule, form, g, aux, dtype=dtype, n_bl=n_bl)
                assert bitwise_equal(out.cpu().numpy(), ref), (dtype, rule.n_q, n_bl)


def test_fused_mesh_kernel_unaligned_connectivity():
    mesh, form, glob, aux = _mesh_problem(3, 6, txb.poisson_varcoef_form, "p0", seed=9)
    rule = txb.quadrature_rule(3, 1)
    ref, _ = _oracle_elem(mesh, form, glob, aux, rule, np.float64)
    buf = torch.empty(mesh.cells.size + 1, dtype=torch.int64, device="cuda")
    cells = buf[1:].view(mesh.cells.shape)  # 8-byte aligned, not 16: direct global path
    cells.copy_(torch.from_numpy(mesh.cells))
    out = txb.integrate_mesh(mesh, txb.FieldLayout(1), txb.tabulate(3, rule), rule, form,
                             torch.from_numpy(glob).cuda(), aux, dtype="f64", cells=cells)
    assert bitwise_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("tiled", ["0", "1"])
def test_fused_mesh_kernel_elasticity_coefficient_alignment(dim, dtype, offset, tiled, monkeypatch):
    """Given geometry, elasticity: the coefficient gathers pair a vertex's
    components (16/8-byte loads, even and odd vertices) when the global vector
    is pair-aligned, scalar loads when it is not — same bits either way (and
    through the tiled kernel, TXB_TILED=1, whose gatherer copies scalars)."""
    monkeypatch.setenv("TXB_TILED", tiled)
    mesh, form, glob, aux = _mesh_problem(dim, 6 if dim == 3 else 20, txb.elasticity_form, None, seed=21 + dim)
    rule = txb.quadrature_rule(dim, 1)
    npdt = np.float64 if dtype == "f64" else np.float32
    tdt = torch.float64 if dtype == "f64" else torch.float32
    tab = txb.tabulate(dim, rule)
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    ref = oracle.integrate(2, 0, tab.basis, tab.basis_der, rule.weights, inv, det,
                           oracle.gather(mesh.cells, glob, dim), None, npdt)
    buf = torch.empty(glob.size + offset, dtype=tdt, device="cuda")
    g = buf[offset:]
    g.copy_(torch.from_numpy(glob.astype(npdt)))
    geom = txb.CellGeometry(torch.from_numpy(inv.astype(npdt)).cuda(), torch.from_numpy(det.astype(npdt)).cuda())
    out = txb.integrate_mesh(mesh, txb.FieldLayout(dim), tab, rule, form, g, None, dtype=dtype, cell_geom=geom)
    assert bitwise_equal(out.cpu().numpy(), ref)


def test_fused_mesh_kernel_orientation_error():
    mesh = txb.Mesh(3, np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1]]),
                    np.array([[0, 1, 2, 3], [0, 1, 2, 4]]))
    rule = txb.quadrature_rule(3, 1)
    with pytest.raises(txb.OrientationError, match="cell 1"):
        txb.integrate_mesh(mesh, txb.FieldLayout(1), txb.tabulate(3, rule), rule, txb.poisson_form(3),
                           torch.zeros(5, dtype=torch.float64, device="cuda"), None)


@pytest.mark.parametrize("name", sorted(BIG))
def test_fused_mesh_kernel_baseline_configs_by_hash(name):
    """BASELINE configs[0..3] straight from the Kuhn mesh: bit-identical to the reference."""
    e = BIG[name]
    from paper_1607_04245_b200.workload import PHYSICS, refine_for

    factory, aux_space = PHYSICS[e["physics"]]
    form = factory(e["dim"])
    full = txb.generate_unit_simplex_mesh(e["dim"], refine_for(e["dim"], e["n_cells"]))
    mesh = txb.Mesh(e["dim"], full.vertices, np.ascontiguousarray(full.cells[:e["n_cells"]]))
    glob = np.random.default_rng(e["seed"]).standard_normal(full.n_vertices * form.n_comp)
    aux = None
    if aux_space == "p0":
        aux = txb.CellAux("p0", np.random.default_rng(e["seed"] + 1).uniform(0.5, 1.5, (full.n_cells, 1))[:e["n_cells"]])
    rule = txb.quadrature_rule(e["dim"], 1)
    for dtype, key, npdt in (("f64", "ref_f64", np.float64), ("f32", "cy_f32", np.float32)):
        out = txb.integrate_mesh(mesh, txb.FieldLayout(form.n_comp), txb.tabulate(e["dim"], rule), rule, form,
                                 torch.from_numpy(glob.astype(npdt)).cuda(), aux, dtype=dtype)
        torch.cuda.synchronize()
        assert hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest() == e[key], (name, dtype)


# ---- randomised mesh-level residuals (integrate_transposed end to end) ----

from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402


@settings(max_examples=30, deadline=None, suppress_health_check=list(HealthCheck))
@given(dim=st.integers(2, 3), refine=st.integers(1, 9), form_i=st.integers(0, 3), dtype=st.sampled_from(["f64", "f32"]),
       given_geom=st.booleans(), two_point=st.booleans(), seed=st.integers(0, 2 ** 31 - 1))
def test_random_mesh_residual_bitwise(dim, refine, form_i, dtype, given_geom, two_point, seed):
    """integrate_transposed on a Kuhn mesh with a random vertex numbering and
    cell order (the gathers, the slot order and the incidence see arbitrary
    index patterns): fused mesh kernel (in-kernel or given geometry) +
    slot-ordered scatter-add, bit-identical to the oracle's geometry -> gather
    -> integrate -> np.add.at."""
    rng = np.random.default_rng(seed)
    base = txb.generate_unit_simplex_mesh(dim, refine if dim == 3 else 3 * refine)
    perm = rng.permutation(base.n_vertices)
    inv_perm = np.argsort(perm)
    verts = np.ascontiguousarray(base.vertices[inv_perm])  # new vertex i = old vertex inv_perm[i]
    cells = np.ascontiguousarray(perm[base.cells][rng.permutation(base.n_cells)])
    mesh = txb.Mesh(dim, verts, cells)
    factory, aux_space = FORMS[form_i]
    form = factory(dim)
    layout = txb.FieldLayout(form.n_comp)
    rule = txb.two_point_rule(dim) if two_point else txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    glob = rng.standard_normal(layout.global_size(mesh))
    aux = None
    if aux_space == "p0":
        aux = txb.CellAux("p0", rng.uniform(0.5, 1.5, (mesh.n_cells, 1)))
    elif aux_space == "p1":
        aux = txb.CellAux("p1", rng.uniform(0.5, 1.5, (mesh.n_vertices, 1))[mesh.cells])
    npdt = np.float64 if dtype == "f64" else np.float32
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    cg = txb.CellGeometry(inv, det) if given_geom else None
    res, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=8, n_cb=2, dtype=dtype,
                                      shared_mem_limit=None, cell_geom=cg)
    fc = {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}[form.name]
    am = {None: 0, "p0": 1, "p1": 2}[aux_space]
    g = txb.derive_execution_geometry(dim, tab.n_b, form.n_comp, rule.n_q, 8, 2, mesh.n_cells)
    elem = oracle.integrate_with_remainder(fc, am, tab.basis, tab.basis_der, rule.weights, inv, det,
                                           oracle.gather(mesh.cells, glob, form.n_comp),
                                           None if aux is None else aux.values, npdt, g.n_chunks * g.n_chunk)
    want = oracle.scatter_add(mesh.cells, elem, mesh.n_vertices)
    assert bitwise_equal(res, want)
