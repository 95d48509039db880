"""In-tree builds: the product library (nvcc, sm_100a) and the test oracle.

``build_library()``  -> paper_1607_04245_b200/libtxb.so   (product)
``build_oracle()``   -> oracle/libtxb_oracle.so            (test infrastructure)
                        oracle/_ref/_kernels_cy*.so        (reference's own lane,
                        only where /root/reference exists; see oracle/build_ref.sh)
"""

from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libtxb.so"
SOURCES = [CSRC / "txb_integrate.cu", CSRC / "txb_integrate_mesh.cu", CSRC / "txb_mesh.cu"]
HEADERS = [CSRC / "txb_common.cuh", CSRC / "txb_kernels.cuh", REPO / "include" / "txb.h"]

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    # the kernels already use _rn intrinsics; this keeps any plain expression
    # from being contracted into FMA as well (reference: -ffp-contract=off)
    "-fmad=false",
]


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Compile each translation unit in parallel (they share no device code),
    then link the shared library."""
    if force or _stale(LIB, SOURCES + HEADERS):
        nvcc = os.environ.get("NVCC", "nvcc")
        objdir = PKG / "build_obj"
        objdir.mkdir(exist_ok=True)
        procs = []
        for src in SOURCES:
            obj = objdir / (src.stem + ".o")
            cmd = [nvcc, *[f for f in NVCC_FLAGS if f != "-shared"], f"-I{REPO / 'include'}", "-c", "-o", str(obj),
                   str(src)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            procs.append((subprocess.Popen(cmd), cmd))
        for p, cmd in procs:
            if p.wait() != 0:
                raise subprocess.CalledProcessError(p.returncode, cmd)
        objs = [str(objdir / (s.stem + ".o")) for s in SOURCES]
        subprocess.run([nvcc, "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-o", str(LIB), *objs], check=True)
    return LIB


def build_oracle(force: bool = False) -> Path:
    src = REPO / "oracle" / "txb_oracle.c"
    out = REPO / "oracle" / "libtxb_oracle.so"
    if force or _stale(out, [src]):
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", str(out), str(src)],
                       check=True)
    ref_script = REPO / "oracle" / "build_ref.sh"
    if Path("/root/reference/pkg/src/txfem/_kernels_cy.pyx").exists() and ref_script.exists():
        ref_dir = REPO / "oracle" / "_ref"
        if force or not any(ref_dir.glob("_kernels_cy*.so")):
            subprocess.run(["bash", str(ref_script)], check=True)
    return out
