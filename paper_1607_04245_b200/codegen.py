"""Run-time kernel assembly (txfem/codegen.py:50-256) on the CUDA lane.

The reference assembles OpenCL kernel TEXT around a form's source strings and
never compiles it (codegen.py:1-10).  Here the same inputs produce the CUDA
translation unit that the run-time lane actually compiles (NVRTC, sm_100a)
and launches (csrc/txb_jit.cu): ``KernelSource.text`` is that unit,
``entry_name`` its kernel, and ``kernel`` the compiled handle, ready for
``backend.run_cuda``.  Errors follow the reference (CodegenError for a bad
scalar, missing source strings, or a form/geometry mismatch).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import CodegenError
from .physics import CellAux, PhysicsForm
from .schedule import ExecutionGeometry

__all__ = ["KernelSource", "generate_kernel_source"]

_SCALARS = {"f32": 4, "f64": 8}


@dataclass(frozen=True)
class KernelSource:
    text: str
    entry_name: str
    specialization: tuple  # (dim, n_b, n_comp, n_q, n_bl, scalar type name)
    kernel: object = None  # backend.JitKernel


def generate_kernel_source(geom: ExecutionGeometry, form: PhysicsForm, scalar: str = "f32", tab=None,
                           weights: Optional[np.ndarray] = None, aux_space: Optional[str] = None) -> KernelSource:
    """Assemble and compile the integration kernel for one (geometry, form,
    scalar) combination (codegen.py:50-97).  ``aux_space`` ("p0"/"p1") selects
    the auxiliary layout for forms with n_aux > 0 (default "p0").  Identical
    inputs yield byte-identical text (and the memoised kernel)."""
    from . import backend

    if scalar not in _SCALARS:
        raise CodegenError(f"scalar must be 'f32' or 'f64', got {scalar!r}")
    if not form.source_f1:
        raise CodegenError(f"form {form.name!r} carries no f1 source string")
    if form.has_f0 and not form.source_f0:
        raise CodegenError(f"form {form.name!r} has f0 but no f0 source string")
    if form.dim != geom.dim or form.n_comp != geom.n_comp:
        raise CodegenError("form and execution geometry disagree on dim or components")
    if tab is not None and weights is None:
        raise CodegenError("explicit tabulation needs explicit weights")
    aux = None
    if form.n_aux:
        space = aux_space or "p0"
        shape = (1, form.n_aux) if space == "p0" else (1, geom.n_b, form.n_aux)
        aux = CellAux(space, np.zeros(shape))
    try:
        k = backend.jit_kernel(form, geom.n_q, aux, _SCALARS[scalar])
    except ValueError as exc:
        if isinstance(exc, CodegenError):
            raise
        raise CodegenError(str(exc)) from exc
    ctype = "float" if scalar == "f32" else "double"
    return KernelSource(text=k.source, entry_name="txb_jit_integrate",
                        specialization=(geom.dim, geom.n_b, geom.n_comp, geom.n_q, geom.n_bl, ctype), kernel=k)
