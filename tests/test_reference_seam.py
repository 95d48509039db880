"""The reference's OWN test suite through the seam INTEGRATION.md describes.

oracle/apply_seam.py appends INTEGRATION.md's two stub blocks (the B200 lane
in txfem/backend.py, lane "cuda" in txfem/executor.py) to a scratch copy of
the reference package (oracle/_ref/txfem_pkg, staged by oracle/build_ref.sh;
test infrastructure).  Then the reference's unchanged tests run on it:

* CPU: the whole suite with the seam present and the lane unrouted -- the
  stub does not disturb the reference;
* GPU: tests/test_executor.py, test_backends.py and test_acceptance.py with
  TXFEM_CUDA_LANE=compiled, i.e. every lane call the B200 lane covers (the
  default lane and explicit "compiled" requests) runs through libtxb.so's
  txb_integrate_cells_host; the seam plugin counts those calls.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

from oracle import apply_seam

REPO = Path(__file__).resolve().parents[1]

HAVE_REF = (apply_seam.PRISTINE / "tests").exists()
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref/txfem_pkg not staged (oracle/build_ref.sh)")


def _run(dest, tests, env_extra, timeout):
    env = dict(os.environ)
    env.update(env_extra)
    env["PYTHONPATH"] = os.pathsep.join([str(dest / "src"), str(REPO / "oracle")])
    env["TXFEM_TXB_LIB"] = str(REPO / "paper_1607_04245_b200" / "libtxb.so")
    count = dest / "seam_calls.txt"
    env["TXFEM_SEAM_COUNT"] = str(count)
    p = subprocess.run([sys.executable, "-m", "pytest", *tests, "-q", "-p", "seam_plugin", "-p", "no:cacheprovider"],
                       cwd=dest, env=env, capture_output=True, text=True, timeout=timeout)
    calls = int(count.read_text()) if count.exists() else -1
    return p, calls


def test_seam_blocks_are_what_integration_md_shows():
    blocks = apply_seam.seam_blocks()
    assert "def run_cuda(" in blocks["backend"] and "txb_integrate_cells_host" in blocks["backend"]
    assert "def _resolve_backend(" in blocks["executor"] and 'lane == "cuda"' in blocks["executor"]
    for b in blocks.values():
        compile(b, "<seam>", "exec")


@needs_ref
def test_reference_suite_passes_with_the_seam_unrouted(tmp_path):
    dest = apply_seam.apply(tmp_path / "txfem_pkg")
    p, calls = _run(dest, ["tests"], {"TXFEM_CUDA_LANE": ""}, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert calls == 0


@pytest.mark.gpu
@needs_ref
def test_reference_tests_run_on_the_b200_lane(tmp_path):
    dest = apply_seam.apply(tmp_path / "txfem_pkg")
    tests = ["tests/test_executor.py", "tests/test_backends.py", "tests/test_acceptance.py"]
    p, calls = _run(dest, tests, {"TXFEM_CUDA_LANE": "compiled"}, timeout=1500)
    out = p.stdout[-4000:] + p.stderr[-2000:]
    assert p.returncode == 0, out
    assert calls > 100, (calls, out)  # the lane really ran (every covered lane call)
    (REPO / "gpurun_out").mkdir(exist_ok=True)
    (REPO / "gpurun_out" / "reference_seam.log").write_text(f"b200 lane calls: {calls}\n" + p.stdout[-6000:])
