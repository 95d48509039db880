import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def rel_err(result, reference):
    """max|r - ref| / max|ref| — the reference metric (cli.py:102-105, tests/conftest.py:13-15)."""
    reference = np.asarray(reference, dtype=np.float64)
    scale = max(float(np.max(np.abs(reference))) if reference.size else 0.0, 1e-300)
    if reference.size == 0:
        return 0.0
    return float(np.max(np.abs(np.asarray(result, dtype=np.float64) - reference))) / scale


# Tolerances of BASELINE.json north_star: relative 1e-5 (f32), 1e-12 (f64).
TOL = {"f32": 1e-5, "f64": 1e-12}


def bitwise_equal(a, b) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


class GoldenCase:
    def __init__(self, npz, name):
        self.name = name
        meta = json.loads(bytes(npz[f"{name}/meta"]).decode())
        self.dim, self.form, self.aux_space = meta["dim"], meta["form"], meta["aux"]
        self.n_q, self.n_comp = meta["n_q"], meta["n_comp"]
        for key in ("basis", "basis_der", "weights", "inv_j", "det_j", "coeffs", "ref_f64", "cy_f32"):
            setattr(self, key, npz[f"{name}/{key}"])
        self.aux = npz[f"{name}/aux"] if f"{name}/aux" in npz.files else None

    @property
    def form_code(self):
        return {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}[self.form]

    @property
    def aux_mode(self):
        return {None: 0, "p0": 1, "p1": 2}[self.aux_space]


def load_small_cases():
    npz = np.load(GOLDEN / "small_cases.npz")
    names = json.loads(bytes(npz["index"]).decode())
    return [GoldenCase(npz, n) for n in names]


def load_big_hashes():
    return json.loads((GOLDEN / "big_hashes.json").read_text())


SMALL_CASES = load_small_cases()
BIG = load_big_hashes()


class UserCase:
    """A user-physics golden problem (tests/golden/user_cases.npz): inputs and
    the reference python lane's f64 / f32 outputs for an oracle/user_forms spec."""

    def __init__(self, npz, name):
        self.name = name
        meta = json.loads(bytes(npz[f"{name}/meta"]).decode())
        self.dim, self.spec, self.aux_space = meta["dim"], meta["spec"], meta["aux"]
        self.n_q, self.n_comp = meta["n_q"], meta["n_comp"]
        for key in ("basis", "basis_der", "weights", "inv_j", "det_j", "coeffs", "py_f64", "py_f32"):
            setattr(self, key, npz[f"{name}/{key}"])
        self.aux = npz[f"{name}/aux"] if f"{name}/aux" in npz.files else None


def load_user_cases():
    npz = np.load(GOLDEN / "user_cases.npz")
    names = json.loads(bytes(npz["index"]).decode())
    return [UserCase(npz, n) for n in names]


USER_CASES = load_user_cases()
