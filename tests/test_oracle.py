"""The CPU oracle is pinned to the reference itself (tests/golden/, produced
by tests/golden/make_golden.py from txfem.integrate_reference and the
reference's compiled lane).  CPU-only."""

import hashlib

import numpy as np
import pytest

from conftest import BIG, SMALL_CASES, bitwise_equal
from oracle import oracle


@pytest.mark.parametrize("case", SMALL_CASES, ids=lambda c: c.name)
def test_oracle_f64_bitwise_matches_integrate_reference(case):
    out = oracle.integrate(case.form_code, case.aux_mode, case.basis, case.basis_der, case.weights,
                           case.inv_j, case.det_j, case.coeffs, case.aux, np.float64)
    assert bitwise_equal(out, case.ref_f64)


@pytest.mark.parametrize("case", SMALL_CASES, ids=lambda c: c.name)
def test_oracle_f32_bitwise_matches_reference_compiled_lane(case):
    out = oracle.integrate(case.form_code, case.aux_mode, case.basis, case.basis_der, case.weights,
                           case.inv_j, case.det_j, case.coeffs, case.aux, np.float32)
    assert bitwise_equal(out, case.cy_f32)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", sorted(BIG))
def test_oracle_reproduces_baseline_configs_by_hash(name):
    """BASELINE.json configs[0..3] at full size: inputs and outputs, bit for bit."""
    e = BIG[name]
    full, inv, det, coeffs, aux = oracle.workload(e["dim"], e["physics"], e["n_cells"], e["seed"])
    assert _sha(full.vertices) == e["mesh"]["vertices"]
    assert _sha(full.cells) == e["mesh"]["cells"]
    assert _sha(inv) == e["inputs_f64"]["inv_j"]
    assert _sha(det) == e["inputs_f64"]["det_j"]
    assert _sha(coeffs) == e["inputs_f64"]["coeffs"]
    if aux is not None:
        assert _sha(aux) == e["inputs_f64"]["aux"]
    form_code = 2 if e["physics"] == "elasticity" else 1
    aux_mode = 1 if aux is not None else 0
    B, D, W = oracle.p1_tables(e["dim"])
    out64 = oracle.integrate(form_code, aux_mode, B, D, W, inv, det, coeffs, aux, np.float64)
    assert _sha(out64) == e["ref_f64"]
    out32 = oracle.integrate(form_code, aux_mode, B, D, W, inv, det, coeffs, aux, np.float32)
    assert _sha(out32) == e["cy_f32"]


def test_known_answers_reference_triangle():
    """u = x on the reference triangle -> (-1/2, 1/2, 0) (tests/test_reference.py:28-43)."""
    B, D, W = oracle.p1_tables(2)
    inv = np.eye(2)[None]
    det = np.ones(1)
    out = oracle.integrate(0, 0, B, D, W, inv, det, np.array([[[0.0], [1.0], [0.0]]]))
    np.testing.assert_array_equal(out[0, :, 0], [-0.5, 0.5, 0.0])
    co = np.zeros((1, 3, 2))
    co[0, 1, 0] = 1.0
    out = oracle.integrate(2, 0, B, D, W, inv, det, co)
    np.testing.assert_array_equal(out[0], [[-0.5, 0.0], [0.5, 0.0], [0.0, 0.0]])


def test_constant_field_gives_exact_zero():
    """Constant coefficients on a Kuhn mesh -> exactly 0 (tests/test_reference.py:21-25)."""
    for dim in (2, 3):
        B, D, W = oracle.p1_tables(dim)
        _, inv, det, coeffs, _ = oracle.workload(dim, "poisson", 300)
        out = oracle.integrate(0, 0, B, D, W, inv, det, np.ones_like(coeffs))
        assert (out == 0).all()


def test_scatter_oracle_matches_np_add_at():
    rng = np.random.default_rng(3)
    cells = rng.integers(0, 40, size=(200, 3))
    elem = rng.standard_normal((200, 3, 2))
    ref = np.zeros((40, 2))
    np.add.at(ref, cells.ravel(), elem.reshape(-1, 2))
    assert bitwise_equal(oracle.scatter_add(cells, elem, 40), ref.ravel())


@pytest.mark.skipif(oracle.ref_lane() is None, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("case", SMALL_CASES[:8], ids=lambda c: c.name)
def test_reference_lane_from_oracle_ref_matches_golden(case):
    lane = oracle.ref_lane()
    for dt, key in ((np.float64, "ref_f64"), (np.float32, "cy_f32")):
        c = lambda a: np.ascontiguousarray(a, dtype=dt)  # noqa: E731
        out = np.empty(case.coeffs.shape, dtype=dt)
        oracle.ref_integrate(lane, case.form_code, case.aux_mode, c(case.basis), c(case.basis_der),
                             c(case.weights), c(case.inv_j), c(case.det_j), c(case.coeffs),
                             c(case.aux) if case.aux is not None else None, out)
        assert bitwise_equal(out, getattr(case, key))


# ---- user physics: the numpy-lane restatement is pinned to the reference's python lane ----
from conftest import USER_CASES  # noqa: E402


@pytest.mark.parametrize("case", USER_CASES, ids=lambda c: c.name)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_oracle_forms_bitwise_matches_reference_python_lane(case, dtype):
    from oracle import user_forms

    s = user_forms.spec(case.spec, case.dim)
    dt = np.float64 if dtype == "f64" else np.float32
    out = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], case.basis,
                                 case.basis_der, case.weights, case.inv_j, case.det_j, case.coeffs, case.aux, dt)
    assert bitwise_equal(out, case.py_f64 if dtype == "f64" else case.py_f32)


def test_oracle_forms_reproduces_shipped_forms():
    """The generic restatement with the shipped f1 equals the C oracle bit for bit."""
    import paper_1607_04245_b200 as txb

    for case in SMALL_CASES:
        factory = {"poisson": txb.poisson_form, "poisson_varcoef": txb.poisson_varcoef_form,
                   "elasticity": txb.elasticity_form}[case.form]
        f = factory(case.dim)
        out = oracle.integrate_forms(f.f1_many, None, False, case.aux_space, case.basis, case.basis_der,
                                     case.weights, case.inv_j, case.det_j, case.coeffs, case.aux, np.float64)
        assert bitwise_equal(out, case.ref_f64), case.name
