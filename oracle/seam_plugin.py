"""pytest plugin for the seam run (tests/test_reference_seam.py): counts the
B200-lane calls of the patched reference (txfem.backend.run_cuda) and writes
the count to $TXFEM_SEAM_COUNT at session end.  TEST INFRASTRUCTURE ONLY."""

import os

_calls = {"n": 0}


def pytest_configure(config):
    import txfem.backend as b

    if hasattr(b, "run_cuda"):
        inner = b.run_cuda

        def counted(*a, **k):
            _calls["n"] += 1
            return inner(*a, **k)

        b.run_cuda = counted


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("TXFEM_SEAM_COUNT")
    if path:
        with open(path, "w") as f:
            f.write(str(_calls["n"]))
