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


def test_scatter_multiplicity_oracle():
    """scatter_add(gather(one-hot)) counts cells per vertex (SPEC mesh invariants)."""
    mesh = txb.generate_unit_simplex_mesh(2, 7)
    layout = txb.FieldLayout(1)
    ones = txb.gather_coefficients(mesh, layout, np.ones(mesh.n_vertices))
    counts = txb.scatter_add_element_vectors(mesh, layout, ones)
    np.testing.assert_array_equal(counts, np.bincount(mesh.cells.ravel(), minlength=mesh.n_vertices))
