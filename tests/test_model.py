"""Schedule and performance-model closed forms (txfem/schedule.py,
perf_model.py, device.py:147-227; tests/test_schedule.py, test_perf_model.py)."""

from fractions import Fraction

import pytest
from hypothesis import given, settings, strategies as st

import paper_1607_04245_b200 as txb
from paper_1607_04245_b200.perf_model import compulsory_bytes_per_cell, flops_per_cell
from paper_1607_04245_b200.trace import batch_loaded_bytes, shared_image_bytes


@settings(max_examples=300, deadline=None)
@given(dim=st.integers(2, 3), n_comp=st.integers(1, 3), n_q=st.integers(1, 8), n_bl=st.integers(1, 40),
       n_cb=st.integers(1, 16), n=st.integers(0, 10 ** 6))
def test_schedule_identities(dim, n_comp, n_q, n_bl, n_cb, n):
    n_b = dim + 1
    try:
        g = txb.derive_execution_geometry(dim, n_b, n_comp, n_q, n_bl, n_cb, n)
    except txb.ConfigurationError:
        assert n_b * n_q * n_bl * n_comp > 1024
        return
    assert g.n_bs == n_b * n_q and g.n_bc == g.n_bs * n_bl and g.n_t == g.n_bc * n_comp
    assert g.n_chunk == n_cb * g.n_bc and g.n_chunks * g.n_chunk + g.n_r == n and 0 <= g.n_r < g.n_chunk
    assert g.n_sqc * n_b == g.n_bs and g.n_sbc * n_q == g.n_bs and g.n_cbc == n_bl * n_q
    assert g.block_threads * n_bl == g.n_t


def test_paper_balance_2d_poisson():
    # 132 bytes and 246 flops per batch of one 3-cell block -> 41/22 (tests/test_perf_model.py:50-54)
    g = txb.derive_execution_geometry(2, 3, 1, 1, 1, 1, 3)
    assert txb.traffic_and_flops(g, 4) == (132, 246)
    assert txb.balance(g) == Fraction(41, 22)
    g = txb.derive_execution_geometry(2, 3, 2, 1, 1, 1, 3)
    assert txb.balance(g) == Fraction(41, 28)


def test_shared_image_and_eq6():
    g = txb.derive_execution_geometry(2, 3, 1, 1, 1, 1, 3)
    assert shared_image_bytes(g, 4, True) == 168
    assert shared_image_bytes(g, 4, False) < 168
    m, mc = txb.shared_memory_bytes(g, 4, True)
    assert m == 168 and mc == Fraction(168, 3)


@pytest.mark.parametrize("dim,n_comp,s,aux,expected", [(3, 1, 8, "p0", 152), (3, 1, 4, "p0", 76),
                                                       (2, 1, 8, "p0", 96), (2, 2, 4, None, 68),
                                                       (3, 3, 8, None, 272), (2, 2, 8, None, 136)])
def test_compulsory_bytes_match_survey_table(dim, n_comp, s, aux, expected):
    assert compulsory_bytes_per_cell(dim, n_comp, s, aux) == expected


def test_compulsory_equals_eq6_plus_aux_for_scalar_p1():
    for dim in (2, 3):
        g = txb.derive_execution_geometry(dim, dim + 1, 1, 1, 1, 1, dim + 1)
        eq6 = batch_loaded_bytes(g, 8) // g.n_bc
        assert eq6 + 8 == compulsory_bytes_per_cell(dim, 1, 8, "p0")


def test_eq7_flops_per_cell():
    g3 = txb.derive_execution_geometry(3, 4, 1, 1, 1, 1, 4)
    g2 = txb.derive_execution_geometry(2, 3, 1, 1, 1, 1, 3)
    e3 = txb.derive_execution_geometry(3, 4, 3, 1, 1, 1, 4)
    e2 = txb.derive_execution_geometry(2, 3, 2, 1, 1, 1, 3)
    assert (flops_per_cell(g3), flops_per_cell(g2), flops_per_cell(e3), flops_per_cell(e2)) == (206, 82, 618, 164)


def test_model_counters_structure():
    g = txb.derive_execution_geometry(2, 3, 1, 1, 2, 2, 24)
    c = txb.model_batch_counters(g, txb.poisson_varcoef_form(2), 8, txb.CellAux("p1", __import__("numpy").ones((1, 3, 1))))
    assert c.barriers == 1 and c.model_flops == txb.traffic_and_flops(g, 8)[1]
    assert c.bytes_loaded == txb.traffic_and_flops(g, 8)[0]
