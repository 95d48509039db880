"""Property test of the mesh-level residual (integrate_transposed: geometry +
gather + integration + deterministic scatter-add on the device) over random
meshes: perturbed Kuhn meshes of random size, random vertex numbering, random
cell order and subsets, every shipped form and aux space, f32 / f64, midpoint
and two-point rules, the tiled and the per-cell fused kernel, in-kernel and
given geometry.  Every residual must equal the reference's (oracle: float64
geometry cast once, lane cells in the run precision, remainder cells float64
then cast, np.add.at assembly -- executor.py:161-267) bit for bit."""

import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from conftest import bitwise_equal
from oracle import oracle

pytestmark = pytest.mark.gpu

import paper_1607_04245_b200 as txb  # noqa: E402

FORMS = [(txb.poisson_form, None), (txb.poisson_varcoef_form, "p0"), (txb.poisson_varcoef_form, "p1"),
         (txb.elasticity_form, None)]


@settings(max_examples=int(os.environ.get("TXB_HYPOTHESIS_EXAMPLES", 60)), deadline=None,
          suppress_health_check=list(HealthCheck))
@given(dim=st.integers(2, 3), refine=st.integers(1, 9), form_i=st.integers(0, 3), dtype=st.sampled_from(["f64", "f32"]),
       two_point=st.booleans(), shuffle=st.booleans(), keep=st.floats(0.3, 1.0), tiled=st.booleans(),
       given_geom=st.booleans(), n_bl=st.integers(1, 12), n_cb=st.integers(1, 4), seed=st.integers(0, 2 ** 16))
def test_random_mesh_residual_bitwise(dim, refine, form_i, dtype, two_point, shuffle, keep, tiled, given_geom, n_bl,
                                      n_cb, seed):
    os.environ["TXB_TILED"] = "1" if tiled else "0"
    try:
        rng = np.random.default_rng(seed)
        n = refine * (4 if dim == 2 else 1) + 1
        base = txb.generate_unit_simplex_mesh(dim, n)
        verts = base.vertices + 0.1 / n * rng.uniform(-1, 1, base.vertices.shape)  # a tenth of the spacing
        cells = base.cells
        if shuffle:
            perm = rng.permutation(base.n_vertices)
            verts = verts[np.argsort(perm)]
            cells = perm[cells][rng.permutation(len(cells))]
        cells = np.ascontiguousarray(cells[: max(1, int(len(cells) * keep))])
        mesh = txb.Mesh(dim, np.ascontiguousarray(verts), cells)
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
        inv, det = oracle.geometry(mesh.vertices, mesh.cells)
        geom = txb.CellGeometry(inv, det)
        res, trace = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=n_bl, n_cb=n_cb,
                                              dtype=dtype, shared_mem_limit=None,
                                              cell_geom=geom if given_geom else None)
        npdt = np.float32 if dtype == "f32" else np.float64
        span = trace.geom.n_chunks * trace.geom.n_chunk
        fc = {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}[form.name]
        am = {None: 0, "p0": 1, "p1": 2}[aux_space]
        elem = oracle.integrate_with_remainder(fc, am, tab.basis, tab.basis_der, rule.weights, inv, det,
                                               oracle.gather(mesh.cells, glob, form.n_comp),
                                               None if aux is None else aux.values, npdt, span)
        want = oracle.scatter_add(mesh.cells, elem, mesh.n_vertices)
        assert bitwise_equal(res, want)
    finally:
        os.environ.pop("TXB_TILED", None)
