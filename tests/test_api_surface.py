"""The reference's public names (txfem/__init__.py) are importable from this
package, so ``import paper_1607_04245_b200 as txfem`` is a drop-in; the only
absences are the virtual-device simulator (out of scope)."""

import numpy as np
import pytest

import paper_1607_04245_b200 as txb

REFERENCE_NAMES = [
    "active_backend", "compiled_available", "KernelSource", "generate_kernel_source", "BatchCounters",
    "ChunkTrace", "ExecutionTrace", "model_batch_counters", "shared_image_bytes", "QuadratureRule", "Tabulation",
    "p1_basis", "quadrature_rule", "tabulate", "two_point_rule", "CapacityError", "CodegenError",
    "ConfigurationError", "DomainError", "InvalidDimensionError", "MissingAuxiliaryError", "OrientationError",
    "ShapeError", "UnsupportedOrderError", "execute_chunk", "integrate_transposed", "scalar_dtype", "CellGeometry",
    "FieldLayout", "Mesh", "compute_geometry", "dump_mesh", "gather_coefficients", "generate_unit_simplex_mesh",
    "interior_vertex_mask", "scatter_add_element_vectors", "PerfEstimate", "balance", "build_estimate",
    "predict_bandwidth_bound", "shared_memory_bytes", "traffic_and_flops", "CellAux", "PhysicsForm", "PointState",
    "elasticity_form", "poisson_form", "poisson_varcoef_form", "user_form", "assemble_residual",
    "integrate_reference", "ExecutionGeometry", "derive_execution_geometry", "__version__",
]
OUT_OF_SCOPE = {"TaskRecord", "simulate_chunk"}  # the virtual-device simulator (device.py:230-398)


@pytest.mark.parametrize("name", REFERENCE_NAMES)
def test_reference_name_exported(name):
    assert hasattr(txb, name), name


def test_lane_reporting():
    assert txb.active_backend() == "cuda"
    assert txb.compiled_available() is False  # the reference's CPU lane is not part of this framework


def test_integrate_reference_validates_like_the_reference():
    dim = 2
    tab = txb.tabulate(dim, txb.quadrature_rule(dim, 1))
    geom = txb.CellGeometry(np.tile(np.eye(2), (3, 1, 1)), np.ones(3))
    with pytest.raises(txb.ShapeError):
        txb.integrate_reference(tab, txb.quadrature_rule(dim, 1), geom, txb.poisson_form(dim), np.zeros((3, 2, 1)))
    with pytest.raises(txb.MissingAuxiliaryError):
        txb.integrate_reference(tab, txb.quadrature_rule(dim, 1), geom, txb.poisson_varcoef_form(dim),
                                np.zeros((3, 3, 1)))


@pytest.mark.gpu
def test_integrate_reference_bitwise_on_the_gpu():
    from oracle import oracle

    for dim, physics, fc in ((3, "varcoef_p0", 1), (2, "elasticity", 2)):
        _, inv, det, coeffs, aux = oracle.workload(dim, physics, 5000, seed=9)
        rule = txb.quadrature_rule(dim, 1)
        tab = txb.tabulate(dim, rule)
        form = txb.poisson_varcoef_form(dim) if fc == 1 else txb.elasticity_form(dim)
        ax = None if aux is None else txb.CellAux("p0", aux)
        got = txb.integrate_reference(tab, rule, txb.CellGeometry(inv, det), form, coeffs, ax)
        want = oracle.integrate(fc, 1 if aux is not None else 0, tab.basis, tab.basis_der, rule.weights, inv, det,
                                coeffs, aux, np.float64)
        assert isinstance(got, np.ndarray) and got.dtype == np.float64
        assert got.tobytes() == want.tobytes()
