"""compute-sanitizer over every kernel family (tools/sanitize_workload.py):
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory
hazards of the bulk-copy + mbarrier ring, the warp-scope transposition),
synccheck.  The workload checks every result against the oracle too."""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


@pytest.mark.skipif(shutil.which("compute-sanitizer") is None, reason="compute-sanitizer not on PATH")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_kernels_are_sanitizer_clean(tool):
    env = dict(os.environ, SANITIZE_QUICK="1")
    r = subprocess.run(["compute-sanitizer", "--tool", tool, "--error-exitcode", "9", sys.executable,
                        str(REPO / "tools" / "sanitize_workload.py")], cwd=REPO, env=env, capture_output=True,
                       text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "bit-identical to the oracle" in out
    assert "0 errors" in out, out[-3000:]
