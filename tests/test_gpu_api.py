"""Reference-API behaviour of the CUDA lane (txfem/executor.py, tests/test_executor.py)."""

import numpy as np
import pytest

from conftest import TOL, bitwise_equal, rel_err
from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1607_04245_b200 as txb  # noqa: E402
from paper_1607_04245_b200.errors import CapacityError, ShapeError  # noqa: E402
from paper_1607_04245_b200.mesh import CellGeometry  # noqa: E402

FORMS = {"poisson": txb.poisson_form, "poisson_varcoef": txb.poisson_varcoef_form,
         "elasticity": txb.elasticity_form}


def make_problem(dim, factory, n, seed=0, rule=None):
    form = factory(dim)
    mesh = txb.generate_unit_simplex_mesh(dim, n)
    layout = txb.FieldLayout(n_comp=form.n_comp)
    rule = rule or txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    coeffs = np.random.default_rng(seed).standard_normal(layout.global_size(mesh))
    return form, mesh, layout, rule, tab, CellGeometry(inv, det), coeffs


def oracle_residual(mesh, layout, tab, rule, form, geom, coeffs, aux, dtype=np.float64, span=None):
    """The reference's residual: lane cells [0, span) in ``dtype``, remainder
    cells in float64 then cast (executor.py:258-264), np.add.at assembly."""
    blocks = oracle.gather(mesh.cells, coeffs, form.n_comp)
    fc = {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}[form.name]
    am = {None: 0, "p0": 1, "p1": 2}[None if aux is None else aux.space]
    elem = oracle.integrate_with_remainder(fc, am, tab.basis, tab.basis_der, rule.weights, geom.inv_jacobians,
                                           geom.determinants, blocks, None if aux is None else aux.values, dtype,
                                           mesh.n_cells if span is None else span)
    return oracle.scatter_add(mesh.cells, elem, mesh.n_vertices)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("name", list(FORMS))
def test_integrate_transposed_matches_oracle_residual(dim, name):
    form, mesh, layout, rule, tab, geom, coeffs = make_problem(dim, FORMS[name], 6 if dim == 3 else 20, seed=3)
    aux = None
    if form.n_aux:
        aux = txb.CellAux("p0", np.random.default_rng(4).uniform(0.5, 1.5, (mesh.n_cells, 1)))
    for dtype, npdt in (("f64", np.float64), ("f32", np.float32)):
        res, trace = txb.integrate_transposed(mesh, layout, tab, rule, form, coeffs, aux, n_bl=3, n_cb=2,
                                              dtype=dtype, cell_geom=geom)
        assert res.dtype == npdt
        ref64 = oracle_residual(mesh, layout, tab, rule, form, geom, coeffs, aux)
        assert rel_err(res, ref64) <= TOL[dtype]
        span = trace.geom.n_chunks * trace.geom.n_chunk
        assert bitwise_equal(res, oracle_residual(mesh, layout, tab, rule, form, geom, coeffs, aux, npdt, span))
        assert trace.remainder_cells == trace.geom.n_r


def test_integrate_transposed_computes_geometry_on_device():
    form, mesh, layout, rule, tab, geom, coeffs = make_problem(3, txb.elasticity_form, 5, seed=8)
    res, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, coeffs, n_bl=4, n_cb=2, dtype="f64")
    assert bitwise_equal(res, oracle_residual(mesh, layout, tab, rule, form, geom, coeffs, None))


def test_affine_field_zero_interior_residual():
    form, mesh, layout, rule, tab, geom, _ = make_problem(2, txb.poisson_form, 8)
    v = mesh.vertices
    u = 2.0 * v[:, 0] + 3.0 * v[:, 1] + 1.0
    res, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, u, n_bl=4, n_cb=2, dtype="f64",
                                      cell_geom=geom)
    assert np.abs(res[txb.interior_vertex_mask(mesh)]).max() <= 1e-12


def test_constant_coefficients_exact_zero():
    form, mesh, layout, rule, tab, geom, _ = make_problem(2, txb.poisson_form, 4)
    res, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, np.ones(layout.global_size(mesh)),
                                      n_bl=2, n_cb=2, dtype="f32", cell_geom=geom)
    assert (res == 0).all()


def test_execute_chunk_on_reference_triangle_copies():
    geom = txb.derive_execution_geometry(2, 3, 1, 1, 1, 2, 6)
    cells = CellGeometry(np.broadcast_to(np.eye(2), (6, 2, 2)).copy(), np.ones(6))
    coeffs = np.zeros((6, 3, 1))
    coeffs[:, 1, 0] = 1.0
    rule = txb.quadrature_rule(2, 1)
    elem, trace = txb.execute_chunk(geom, txb.tabulate(2, rule), rule, cells, coeffs, None, txb.poisson_form(2))
    for c in range(6):
        np.testing.assert_array_equal(elem[c, :, 0], [-0.5, 0.5, 0.0])
    assert len(trace.batches) == 2


def test_vector_two_point_chunk_zero_ulp():
    geom = txb.derive_execution_geometry(2, 3, 2, 2, 2, 1, 12)
    rng = np.random.default_rng(7)
    jac = np.eye(2) + 0.2 * rng.uniform(-1, 1, (12, 2, 2))
    cells = CellGeometry(np.linalg.inv(jac), np.linalg.det(jac))
    coeffs = np.random.default_rng(8).standard_normal((12, 3, 2))
    rule = txb.two_point_rule(2)
    tab = txb.tabulate(2, rule)
    elem, _ = txb.execute_chunk(geom, tab, rule, cells, coeffs, None, txb.elasticity_form(2))
    ref = oracle.integrate(2, 0, tab.basis, tab.basis_der, rule.weights, cells.inv_jacobians,
                           cells.determinants, coeffs)
    assert bitwise_equal(elem, ref)


def test_errors():
    form, mesh, layout, rule, tab, geom, coeffs = make_problem(2, txb.poisson_form, 4)
    with pytest.raises(CapacityError) as exc:
        txb.integrate_transposed(mesh, layout, tab, rule, form, coeffs, n_bl=8, n_cb=2, dtype="f64",
                                 shared_mem_limit=256, cell_geom=geom)
    assert exc.value.limit_bytes == 256
    with pytest.raises(ValueError, match="reference CPU lane"):
        txb.integrate_transposed(mesh, layout, tab, rule, form, coeffs, n_bl=2, n_cb=2, backend="compiled",
                                 cell_geom=geom)
    with pytest.raises(txb.ConfigurationError):
        txb.integrate_transposed(mesh, layout, tab, rule, form, coeffs, n_bl=400, n_cb=2, cell_geom=geom)
    with pytest.raises(txb.MissingAuxiliaryError):
        txb.integrate_transposed(mesh, layout, tab, rule, txb.poisson_varcoef_form(2), coeffs, n_bl=2,
                                 n_cb=2, cell_geom=geom)
    with pytest.raises(ShapeError):
        geom6 = txb.derive_execution_geometry(2, 3, 1, 1, 1, 2, 6)
        txb.execute_chunk(geom6, tab, rule, CellGeometry(geom.inv_jacobians[:4], geom.determinants[:4]),
                          np.zeros((4, 3, 1)), None, form)


def test_orientation_error_names_the_cell():
    mesh = txb.Mesh(2, np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [2.0, 0.0]]),
                    np.array([[0, 1, 2], [0, 1, 3]]))
    with pytest.raises(txb.OrientationError, match="cell 1"):
        txb.compute_geometry(mesh)


def test_integrate_transposed_orientation_error_names_the_cell():
    """The mesh-level call raises the reference's OrientationError for a
    degenerate / negatively oriented cell (the in-kernel geometry's flag is
    read once after the scatter-add is queued)."""
    mesh = txb.Mesh(3, np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [0, 0, -1], [1, 1, 1]]),
                    np.array([[0, 1, 2, 3], [0, 1, 2, 5], [0, 1, 2, 4]]))
    rule = txb.quadrature_rule(3, 1)
    with pytest.raises(txb.OrientationError, match="cell 2"):
        txb.integrate_transposed(mesh, txb.FieldLayout(1), txb.tabulate(3, rule), rule, txb.poisson_form(3),
                                 np.ones(6), None, n_bl=4, n_cb=2, shared_mem_limit=None)


@pytest.mark.parametrize("paper", ["0", "1"])
def test_reference_decomposition_is_a_model_parameter(paper, monkeypatch):
    """The caller's (N_bl, N_cb) shape the geometry, checks and trace; the
    device runs its tuned schedule unless TXB_PAPER_DECOMPOSITION=1 -- the
    element vectors and the residual are the same bits either way."""
    monkeypatch.setenv("TXB_PAPER_DECOMPOSITION", paper)
    form, mesh, layout, rule, tab, geom, coeffs = make_problem(3, txb.poisson_varcoef_form, 5)
    kappa = txb.CellAux("p0", np.random.default_rng(3).uniform(0.5, 1.5, (mesh.n_cells, 1)))
    glob = np.random.default_rng(4).standard_normal(mesh.n_vertices)
    res, trace = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, kappa, n_bl=16, n_cb=8,
                                          dtype="f64", shared_mem_limit=None)
    g = txb.derive_execution_geometry(3, 4, 1, 1, 16, 8, mesh.n_cells)
    assert trace.remainder_cells == g.n_r
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    elem = oracle.integrate(1, 1, tab.basis, tab.basis_der, rule.weights, inv, det,
                            oracle.gather(mesh.cells, glob, 1), kappa.values)
    assert bitwise_equal(res, oracle.scatter_add(mesh.cells, elem, mesh.n_vertices))


def test_integrate_transposed_from_threads():
    """The reference's callers run the lane from a thread pool (executor.py:228-239);
    here eight threads share the process's mesh / incidence / tile caches and
    the pinned staging of numpy inputs, each integrating its own mesh and
    coefficient vector (numpy in, numpy out; in-kernel and given geometry,
    f64 and f32): every residual bit-identical to the oracle's."""
    from concurrent.futures import ThreadPoolExecutor

    jobs = []
    for k in range(16):
        dim = 2 if k % 2 else 3
        size = 30 if k == 0 else (40 if dim == 2 else 8) + k % 3  # k = 0: 162,000 tets
        form, mesh, layout, rule, tab, geom, coeffs = make_problem(dim, FORMS["poisson_varcoef"], size, seed=k)
        # >= 1 MiB of kappa for some: the pinned-staging H2D path
        aux = txb.CellAux("p0", np.random.default_rng(100 + k).uniform(0.5, 1.5, (mesh.n_cells, 1)))
        jobs.append((form, mesh, layout, rule, tab, geom, coeffs, aux, "f32" if k % 4 == 3 else "f64", k % 3 == 0))

    def run(job):
        form, mesh, layout, rule, tab, geom, coeffs, aux, dtype, given = job
        res, trace = txb.integrate_transposed(mesh, layout, tab, rule, form, coeffs, aux, n_bl=4, n_cb=2,
                                              dtype=dtype, cell_geom=geom if given else None)
        return res, trace

    with ThreadPoolExecutor(8) as ex:
        results = list(ex.map(run, jobs * 2))
    for (form, mesh, layout, rule, tab, geom, coeffs, aux, dtype, _), (res, trace) in zip(jobs * 2, results):
        npdt = np.float32 if dtype == "f32" else np.float64
        span = trace.geom.n_chunks * trace.geom.n_chunk
        assert bitwise_equal(res, oracle_residual(mesh, layout, tab, rule, form, geom, coeffs, aux, npdt, span))
