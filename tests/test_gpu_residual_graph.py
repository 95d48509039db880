"""ResidualGraph: integrate_transposed captured once into a CUDA graph, replayed
per residual -- the same bits as the eager call for every form / dtype / rule,
across replays with different global vectors, for given and in-kernel
geometry, a run-time compiled form and a non-standard tabulation."""

import numpy as np
import pytest

from conftest import bitwise_equal

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1607_04245_b200 as txb  # noqa: E402

FORMS = [(txb.poisson_form, None), (txb.poisson_varcoef_form, "p0"), (txb.poisson_varcoef_form, "p1"),
         (txb.elasticity_form, None)]


def _problem(dim, n, factory, aux_space, seed):
    rng = np.random.default_rng(seed)
    mesh = txb.generate_unit_simplex_mesh(dim, n)
    mesh = txb.Mesh(dim, mesh.vertices + 0.1 / n * rng.uniform(-1, 1, mesh.vertices.shape), mesh.cells)
    form = factory(dim)
    aux = None
    if aux_space == "p0":
        aux = txb.CellAux("p0", rng.uniform(0.5, 1.5, (mesh.n_cells, 1)))
    elif aux_space == "p1":
        aux = txb.CellAux("p1", rng.uniform(0.5, 1.5, (mesh.n_vertices, 1))[mesh.cells])
    return mesh, form, aux, rng


@pytest.mark.parametrize("dim,n", [(2, 17), (3, 6)])
@pytest.mark.parametrize("factory,aux_space", FORMS)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("two_point", [False, True])
def test_graph_replays_match_eager(dim, n, factory, aux_space, dtype, two_point):
    mesh, form, aux, rng = _problem(dim, n, factory, aux_space, seed=dim * 10 + n)
    layout = txb.FieldLayout(form.n_comp)
    rule = txb.two_point_rule(dim) if two_point else txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    kw = dict(n_bl=8, n_cb=3, dtype=dtype, shared_mem_limit=None)  # n_r > 0: the f32 remainder path too
    g = txb.ResidualGraph(mesh, layout, tab, rule, form, aux, **kw)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    for it in range(3):
        glob = torch.from_numpy(rng.standard_normal(layout.global_size(mesh))).to("cuda", tdt)
        want, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, **kw)
        got = g(glob)
        assert bitwise_equal(got.cpu().numpy(), want.cpu().numpy()), it
    # numpy input, out= copy
    gh = rng.standard_normal(layout.global_size(mesh))
    want, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, gh, aux, **kw)
    out = torch.empty_like(g.residual)
    g(gh, out=out)
    assert bitwise_equal(out.cpu().numpy(), want)
    # in place: the solver writes graph.glob and replays without a copy
    g.glob.copy_(torch.from_numpy(gh * 0.5))
    want, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, gh * 0.5, aux, **kw)
    assert bitwise_equal(g().cpu().numpy(), want)
    assert bitwise_equal(g(g.glob).cpu().numpy(), want)


def test_graph_given_geometry_and_nonstandard_tables():
    mesh, form, aux, rng = _problem(3, 5, txb.poisson_varcoef_form, "p0", seed=3)
    layout = txb.FieldLayout(1)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    geom = txb.compute_geometry(mesh)
    kw = dict(n_bl=8, n_cb=2, dtype="f64", shared_mem_limit=None)
    glob = rng.standard_normal(mesh.n_vertices)
    g = txb.ResidualGraph(mesh, layout, tab, rule, form, aux, cell_geom=geom, **kw)
    want, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, cell_geom=geom, **kw)
    assert bitwise_equal(g(glob).cpu().numpy(), want)
    # scaled reference gradients: not the standard P1 tables -> the unfused path, geometry computed once
    tab2 = txb.Tabulation(dim=tab.dim, n_b=tab.n_b, basis=tab.basis, basis_der=tab.basis_der * 2.0)
    g2 = txb.ResidualGraph(mesh, layout, tab2, rule, form, aux, **kw)
    want2, _ = txb.integrate_transposed(mesh, layout, tab2, rule, form, glob, aux, **kw)
    assert bitwise_equal(g2(glob).cpu().numpy(), want2)


@pytest.mark.parametrize("name", ["reaction", "advect"])
def test_graph_user_form(name):
    """A run-time compiled form (f0, P1 aux fields with gradients): the NVRTC
    mesh entry point inside the graph."""
    from oracle import user_forms

    form = user_forms.make_form(txb.user_form, name, 3)
    s = user_forms.spec(name, 3)
    mesh, _, _, rng = _problem(3, 5, txb.poisson_form, None, seed=4)
    layout = txb.FieldLayout(form.n_comp)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    aux = None
    if s["aux"] == "p1":
        aux = txb.CellAux("p1", rng.uniform(0.5, 1.5, (mesh.n_cells, 4, s["n_aux"])))
    elif s["aux"] == "p0":
        aux = txb.CellAux("p0", rng.uniform(0.5, 1.5, (mesh.n_cells, s["n_aux"])))
    kw = dict(n_bl=8, n_cb=2, dtype="f64", shared_mem_limit=None)
    g = txb.ResidualGraph(mesh, layout, tab, rule, form, aux, **kw)
    for _ in range(2):
        glob = rng.standard_normal(layout.global_size(mesh))
        want, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, **kw)
        assert bitwise_equal(g(glob).cpu().numpy(), want)


def test_graph_orientation_error_at_construction():
    mesh = txb.Mesh(3, np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1]]),
                    np.array([[0, 1, 2, 3], [0, 1, 2, 4]]))
    rule = txb.quadrature_rule(3, 1)
    with pytest.raises(txb.OrientationError):
        txb.ResidualGraph(mesh, txb.FieldLayout(1), txb.tabulate(3, rule), rule, txb.poisson_form(3), None,
                          n_bl=8, n_cb=1, shared_mem_limit=None)


def test_graph_shape_check():
    mesh, form, aux, rng = _problem(2, 5, txb.poisson_form, None, seed=1)
    rule = txb.quadrature_rule(2, 1)
    g = txb.ResidualGraph(mesh, txb.FieldLayout(1), txb.tabulate(2, rule), rule, form, None, n_bl=8, n_cb=1,
                          shared_mem_limit=None)
    with pytest.raises(txb.ShapeError):
        g(np.zeros(mesh.n_vertices + 1))


def test_graph_survives_cache_eviction():
    """The graph keeps the device mesh data it captured alive: evaluating other
    meshes (which evicts the module caches), invalidating them and churning the
    allocator does not change its residual."""
    mesh, form, aux, rng = _problem(3, 6, txb.poisson_varcoef_form, "p0", seed=8)
    layout = txb.FieldLayout(1)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    kw = dict(n_bl=8, n_cb=3, dtype="f64", shared_mem_limit=None)
    glob = rng.standard_normal(mesh.n_vertices)
    g = txb.ResidualGraph(mesh, layout, tab, rule, form, aux, **kw)
    want = g(glob).cpu().numpy().copy()
    other, f2, a2, _ = _problem(3, 7, txb.poisson_varcoef_form, "p0", seed=9)
    txb.integrate_transposed(other, layout, tab, rule, f2, rng.standard_normal(other.n_vertices), a2, **kw)
    txb.invalidate_mesh_cache()
    torch.cuda.empty_cache()
    junk = [torch.full((1 << 20,), 7.0, dtype=torch.float64, device="cuda") for _ in range(8)]
    assert bitwise_equal(g(glob).cpu().numpy(), want)
    del junk
