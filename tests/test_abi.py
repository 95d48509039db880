"""C ABI surface, CPU-only: libtxb.so loads, exports every function
include/txb.h declares, and its host-side logic (capability probe, launch
geometry, argument validation) behaves like the reference's seam
(txfem/backend.py:38-52, schedule.py:86-90).  No kernel is launched."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1607_04245_b200 import _lib, backend
import paper_1607_04245_b200 as txb

HEADER = Path(__file__).resolve().parents[1] / "include" / "txb.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(txb_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    names = declared_functions()
    assert len(names) >= 10
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert _lib.lib().txb_abi_version() == 1


def test_library_is_sm100a_only():
    blob = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in blob


@pytest.mark.parametrize("dtype", [4, 8])
def test_query_coverage_matches_compiled_kernel(dtype):
    q = _lib.lib().txb_query
    for dim in (2, 3):
        for n_q in range(1, 9):
            assert q(0, 0, dtype, dim, n_q, 1) == 0
            assert q(1, 1, dtype, dim, n_q, 1) == 0
            assert q(1, 2, dtype, dim, n_q, 1) == 0
            assert q(2, 0, dtype, dim, n_q, dim) == 0
        assert q(0, 0, dtype, dim, 9, 1) != 0       # n_q > MAX_QUAD
        assert q(1, 0, dtype, dim, 1, 1) != 0       # var-coef needs aux
        assert q(0, 1, dtype, dim, 1, 1) != 0       # poisson takes no aux
        assert q(2, 0, dtype, dim, 1, 1) != 0       # elasticity needs n_comp == dim
        assert q(3, 0, dtype, dim, 1, 1) != 0       # unknown form
    assert q(0, 0, dtype, 4, 1, 1) != 0
    assert q(0, 0, 2, 3, 1, 1) != 0


def test_cuda_kernel_mirrors_reference_probe():
    f = txb.poisson_varcoef_form(3)
    assert backend.cuda_kernel(f, 1, txb.CellAux("p0", np.ones((4, 1)))) == (1, 1)
    assert backend.cuda_kernel(f, 1, txb.CellAux("p1", np.ones((4, 4, 1)))) == (1, 2)
    # outside the ahead-of-time coverage (n_aux != 1): the run-time compiled lane
    # takes it, where the reference would fall back to its python lane
    assert isinstance(backend.cuda_kernel(f, 1, txb.CellAux("p0", np.ones((4, 2)))), backend.JitKernel)
    assert backend.cuda_kernel(txb.elasticity_form(2), 1, None) == (2, 0)
    assert backend.cuda_kernel(txb.poisson_form(2), 9, None) is None


def test_launch_geometry_follows_the_paper_decomposition():
    cfg = backend.launch_config(1, 1, 8, 3, 1, 1, 1 << 20, n_bl=32)
    assert cfg["n_bc"] == 32 * 4 and cfg["n_t"] == 128 and cfg["n_bl"] == 32
    cfg = backend.launch_config(2, 0, 4, 3, 2, 3, 1000, n_bl=5, n_cb=3)
    assert cfg["n_bc"] == 5 * 4 * 2 and cfg["n_t"] == 5 * 4 * 2 * 3 and cfg["n_cb"] == 3
    assert 2 <= cfg["stages"] <= 8 and cfg["smem_bytes"] <= 227 * 1024
    default = backend.launch_config(1, 1, 8, 3, 1, 1, 1 << 20)
    assert default["n_bc"] % 32 == 0


def test_thread_limit_is_a_configuration_error():
    with pytest.raises(txb.ConfigurationError, match="thread block needs"):
        backend.launch_config(2, 0, 8, 3, 1, 3, 100, n_bl=100)  # 100*4*3 = 1200 > 1024


def test_shape_errors_before_any_device_work():
    B = np.ones((1, 4)); D = np.ones((1, 4, 3)); W = np.ones(1)
    with pytest.raises(txb.ShapeError):
        backend.run_cuda((0, 0), B, D, W, np.ones((5, 3, 3)), np.ones(5), np.ones((4, 4, 1)), None,
                         np.ones((5, 4, 1)))
    with pytest.raises(txb.ShapeError):
        backend.run_cuda((1, 1), B, D, W, np.ones((5, 3, 3)), np.ones(5), np.ones((5, 4, 1)),
                         txb.CellAux("p0", np.ones((4, 1))), np.ones((5, 4, 1)))
    with pytest.raises(TypeError):
        backend.run_cuda((0, 0), B, D, W, np.ones((5, 3, 3), np.float32), np.ones(5), np.ones((5, 4, 1)), None,
                         np.ones((5, 4, 1)))


def test_error_codes_map_to_reference_exceptions():
    L = _lib.lib()
    rc = L.txb_integrate_cells(0, 0, 8, 3, 3, 1, 1, 10, None, None, None, None, None, None, None, None, 0, 0, None)
    assert rc == _lib.TXB_E_SHAPE  # n_b != dim + 1
    with pytest.raises(txb.ShapeError):
        _lib.check(rc)
    with pytest.raises(ValueError, match="unavailable"):
        _lib.check(L.txb_query(9, 0, 8, 3, 1, 1))
    rc = L.txb_integrate_cells(0, 0, 8, 3, 4, 1, 1, 10, None, None, None, None, None, None, None, None, 0, 0, None)
    assert rc == _lib.TXB_E_ARG  # tables missing
    assert "basis" in _lib.last_error()
