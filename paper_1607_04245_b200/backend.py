"""The CUDA lane: capability probe and kernel call.

Mirrors txfem/backend.py:38-87 — ``compiled_kernel``/``run_compiled`` become
``cuda_kernel``/``run_cuda`` over the C ABI (include/txb.h).  Form codes and
aux modes are the reference's (backend.py:26-27).  There is no CPU lane and
no fallback: when the library or the device is missing, the call raises.

Two kinds of kernel come back from ``cuda_kernel``:
  * ``(form_code, aux_mode)`` — a shipped form inside the ahead-of-time
    kernel's coverage (the reference's compiled-lane coverage);
  * a ``JitKernel`` — every other form with source text (user forms, f0,
    several auxiliary fields, grad a): its f1/f0 source compiled at run time
    by NVRTC (txb_jit_compile), where the reference would fall back to its
    numpy lane (executor.py:93-106).

``run_cuda`` accepts either
  * CUDA torch tensors (device-resident; async on the current torch stream,
    via ``txb_integrate_cells``), or
  * numpy arrays (the reference's own calling convention; host->device copies,
    kernel and device->host copy pipelined inside ``txb_integrate_cells_host``).
``out`` is caller-allocated and fully overwritten, like the Cython lane.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from .errors import CodegenError, CudaLaneError, ShapeError
from .physics import CellAux, PhysicsForm

__all__ = ["cuda_available", "active_backend", "cuda_kernel", "run_cuda", "launch_config", "jit_kernel",
           "JitKernel", "FORM_CODES", "AUX_MODES"]

FORM_CODES = {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}
AUX_MODES = {None: 0, "p0": 1, "p1": 2}
MAX_DIM, MAX_BASIS, MAX_COMPONENTS, MAX_QUAD = 3, 4, 3, 8


def cuda_available() -> bool:
    try:
        _lib.lib()
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def active_backend() -> str:
    return "cuda"


def compiled_available() -> bool:
    """The reference's question (backend.py:30-31): is ITS compiled CPU lane
    here?  Never -- this framework's lane is "cuda" (cuda_available())."""
    return False


class JitKernel:
    """A run-time compiled integration kernel (process-lifetime handle)."""

    __slots__ = ("handle", "form_name", "dtype_bytes", "dim", "n_q", "n_comp", "n_aux", "aux_mode", "has_f0")

    def __init__(self, handle, form, dtype_bytes, n_q, n_aux, aux_mode):
        self.handle = handle
        self.form_name, self.dim, self.n_comp, self.has_f0 = form.name, form.dim, form.n_comp, form.has_f0
        self.dtype_bytes, self.n_q, self.n_aux, self.aux_mode = dtype_bytes, n_q, n_aux, aux_mode

    @property
    def source(self) -> str:
        """The generated translation unit (the counterpart of codegen.KernelSource.text)."""
        return _lib.lib().txb_jit_source(ctypes.c_void_p(self.handle)).decode()

    @property
    def cubin(self) -> bytes:
        """The sm_100a cubin NVRTC produced (inspect with cuobjdump -sass / -res-usage)."""
        L = _lib.lib()
        n = L.txb_jit_cubin(ctypes.c_void_p(self.handle), None, 0)
        buf = ctypes.create_string_buffer(n)
        L.txb_jit_cubin(ctypes.c_void_p(self.handle), buf, n)
        return buf.raw

    @property
    def log(self) -> str:
        return _lib.lib().txb_jit_log(ctypes.c_void_p(self.handle)).decode()

    def __repr__(self):
        return (f"JitKernel({self.form_name!r}, dim={self.dim}, n_q={self.n_q}, n_comp={self.n_comp}, "
                f"n_aux={self.n_aux}, aux_mode={self.aux_mode}, f0={self.has_f0}, s={self.dtype_bytes})")


def jit_kernel(form: PhysicsForm, n_q: int, aux: Optional[CellAux], dtype_bytes: int = 8) -> JitKernel:
    """Compile ``form``'s source text for this configuration (NVRTC, no device
    needed; memoised on the generated text).  Raises CodegenError when the
    form has no source or it does not compile, ValueError when the
    configuration is outside the run-time kernel's coverage."""
    if not form.source_f1:
        raise CodegenError(f"form {form.name!r} carries no f1 source string")
    if form.has_f0 and not form.source_f0:
        raise CodegenError(f"form {form.name!r} has f0 but no f0 source string")
    n_aux = 0 if aux is None else aux.n_aux
    mode = AUX_MODES[None if aux is None else aux.space]
    h = ctypes.c_void_p()
    rc = _lib.lib().txb_jit_compile(form.name.encode(), form.source_f1.encode(),
                                    form.source_f0.encode() if form.has_f0 else None, dtype_bytes, form.dim,
                                    n_q, form.n_comp, n_aux, mode, 1 if form.uses_grad_a else 0, ctypes.byref(h))
    _lib.check(rc, "txb_jit_compile")
    return JitKernel(h.value, form, dtype_bytes, n_q, n_aux, mode)


def cuda_kernel(form: PhysicsForm, n_q: int, aux: Optional[CellAux], dtype_bytes: int = 8):
    """The kernel that integrates ``form`` on the CUDA lane, or None.

    ``(form_code, aux_mode)`` when the ahead-of-time kernel covers the
    configuration — the coverage of backend.compiled_kernel (backend.py:38-52);
    otherwise a run-time compiled ``JitKernel`` for forms with source text;
    None when neither applies."""
    code = FORM_CODES.get(form.name)
    aot = code is not None and not form.has_f0 and not form.uses_grad_a
    if form.dim > MAX_DIM or form.n_comp > MAX_COMPONENTS or form.dim + 1 > MAX_BASIS or n_q > MAX_QUAD:
        return None
    if aux is not None and (aux.n_aux != 1 or form.n_aux != 1):
        aot = False
    if aot:
        mode = AUX_MODES[None if aux is None else aux.space]
        if _lib.lib().txb_query(code, mode, dtype_bytes, form.dim, n_q, form.n_comp) == 0:
            return code, mode
    if not form.source_f1:
        return None
    try:
        return jit_kernel(form, n_q, aux, dtype_bytes)
    except ValueError as exc:
        if isinstance(exc, CodegenError):
            raise
        return None


def launch_config(form_code: int, aux_mode: int, dtype_bytes: int, dim: int, n_q: int, n_comp: int,
                  n_cells: int, n_bl: int = 0, n_cb: int = 0) -> dict:
    """Launch geometry the library would use (n_bc, n_t, stages, smem, grid, n_bl, n_cb)."""
    vals = [ctypes.c_int(0) for _ in range(7)]
    _lib.check(_lib.lib().txb_launch_config(form_code, aux_mode, dtype_bytes, dim, n_q, n_comp, n_cells,
                                            n_bl, n_cb, *[ctypes.byref(v) for v in vals]),
               "txb_launch_config")
    keys = ("n_bc", "n_t", "stages", "smem_bytes", "grid", "n_bl", "n_cb")
    return {k: v.value for k, v in zip(keys, vals)}


def _host_table(x, dt) -> np.ndarray:
    if not isinstance(x, np.ndarray):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(x, dtype=dt)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def run_cuda(kernel, basis, basis_der, weights, inv_j, det_j, coeffs, aux: Optional[CellAux], out,
             *, n_bl: int = 0, n_cb: int = 0, stream=None) -> None:
    """Integrate every cell of the span into ``out`` (backend.run_compiled)."""
    if isinstance(kernel, JitKernel):
        return _run_jit(kernel, basis, basis_der, weights, inv_j, det_j, coeffs, aux, out, n_bl=n_bl, n_cb=n_cb,
                        stream=stream)
    form_code, aux_mode = kernel
    n = int(det_j.shape[0])
    n_q, n_b = int(basis.shape[0]), int(basis.shape[1])
    d = int(basis_der.shape[2])
    n_comp = int(out.shape[2])
    dt = np.dtype(str(coeffs.dtype).replace("torch.", ""))
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise TypeError(f"coeffs must be float32 or float64, got {coeffs.dtype}")
    # shape checks (the Cython lane would fail on mismatched memoryviews)
    if tuple(inv_j.shape) != (n, d, d) or tuple(coeffs.shape) != (n, n_b, n_comp) or \
            tuple(out.shape) != (n, n_b, n_comp):
        raise ShapeError(
            f"inconsistent spans: inv_j {tuple(inv_j.shape)}, det_j ({n},), coeffs {tuple(coeffs.shape)}, "
            f"out {tuple(out.shape)}")
    aux_vals = None
    if aux_mode:
        aux_vals = aux.values
        want = (n, 1) if aux_mode == 1 else (n, n_b, 1)
        if tuple(aux_vals.shape) != want:
            raise ShapeError(f"aux values have shape {tuple(aux_vals.shape)}, expected {want}")
    arrays = [inv_j, det_j, coeffs, out] + ([aux_vals] if aux_vals is not None else [])
    for a in arrays:
        if str(a.dtype).replace("torch.", "") != dt.name:
            raise TypeError("all per-cell arrays must share one floating dtype")
    B, D, W = _host_table(basis, dt), _host_table(basis_der, dt), _host_table(weights, dt)
    L = _lib.lib()
    args = (form_code, aux_mode, dt.itemsize, d, n_b, n_q, n_comp, n,
            B.ctypes.data, D.ctypes.data, W.ctypes.data)
    if _is_torch(out):
        import torch

        for a in arrays:
            if not a.is_cuda:
                raise ValueError("device path needs CUDA tensors for every per-cell array")
        if not out.is_contiguous():
            raise ValueError("out must be a contiguous CUDA tensor (it is written in place)")
        # inputs: contiguous views (a copy only if needed), as run_compiled's
        # np.ascontiguousarray (backend.py:76-84)
        inv_j, det_j, coeffs = inv_j.contiguous(), det_j.contiguous(), coeffs.contiguous()
        if aux_vals is not None:
            aux_vals = aux_vals.contiguous()
        s = stream if stream is not None else torch.cuda.current_stream()
        rc = L.txb_integrate_cells(*args, inv_j.data_ptr(), det_j.data_ptr(), coeffs.data_ptr(),
                                   aux_vals.data_ptr() if aux_vals is not None else None,
                                   out.data_ptr(), n_bl, n_cb, ctypes.c_void_p(s.cuda_stream))
        _lib.check(rc, "txb_integrate_cells")
        return
    # host (numpy) path
    if not (out.flags.c_contiguous and out.flags.writeable):
        raise ValueError("out must be a writeable C-contiguous array")
    host = [np.ascontiguousarray(a) for a in (inv_j, det_j, coeffs)]
    av = np.ascontiguousarray(aux_vals) if aux_vals is not None else None
    try:
        import torch

        if not torch.cuda.is_available():
            raise CudaLaneError("the CUDA lane needs a CUDA device")
    except ImportError as exc:  # pragma: no cover
        raise CudaLaneError("torch is required to select the CUDA device") from exc
    rc = L.txb_integrate_cells_host(*args, host[0].ctypes.data, host[1].ctypes.data, host[2].ctypes.data,
                                    av.ctypes.data if av is not None else None, out.ctypes.data,
                                    n_bl, n_cb)
    _lib.check(rc, "txb_integrate_cells_host")


def _run_jit(kernel: JitKernel, basis, basis_der, weights, inv_j, det_j, coeffs, aux, out, *, n_bl, n_cb, stream):
    """run_cuda for a run-time compiled kernel: device tensors directly; numpy
    buffers are staged through the device (H2D, launch, D2H)."""
    n = int(det_j.shape[0])
    n_q, n_b = int(basis.shape[0]), int(basis.shape[1])
    d = int(basis_der.shape[2])
    dt = np.dtype(str(coeffs.dtype).replace("torch.", ""))
    if dt.itemsize != kernel.dtype_bytes:
        raise TypeError(f"kernel compiled for {kernel.dtype_bytes}-byte scalars, arrays are {dt}")
    if (n_q, d, int(out.shape[2])) != (kernel.n_q, kernel.dim, kernel.n_comp):
        raise ShapeError(f"kernel compiled for n_q={kernel.n_q}, dim={kernel.dim}, n_comp={kernel.n_comp}")
    nc = kernel.n_comp
    if tuple(inv_j.shape) != (n, d, d) or tuple(coeffs.shape) != (n, n_b, nc) or tuple(out.shape) != (n, n_b, nc):
        raise ShapeError(
            f"inconsistent spans: inv_j {tuple(inv_j.shape)}, det_j ({n},), coeffs {tuple(coeffs.shape)}, "
            f"out {tuple(out.shape)}")
    aux_vals = None
    if kernel.aux_mode:
        aux_vals = aux.values
        want = (n, kernel.n_aux) if kernel.aux_mode == 1 else (n, n_b, kernel.n_aux)
        if tuple(aux_vals.shape) != want:
            raise ShapeError(f"aux values have shape {tuple(aux_vals.shape)}, expected {want}")
    arrays = [inv_j, det_j, coeffs, out] + ([aux_vals] if aux_vals is not None else [])
    for a in arrays:
        if str(a.dtype).replace("torch.", "") != dt.name:
            raise TypeError("all per-cell arrays must share one floating dtype")
    B, D, W = _host_table(basis, dt), _host_table(basis_der, dt), _host_table(weights, dt)
    import torch

    if not torch.cuda.is_available():
        raise CudaLaneError("the CUDA lane needs a CUDA device")
    host = not _is_torch(out)
    if host:
        if not (out.flags.c_contiguous and out.flags.writeable):
            raise ValueError("out must be a writeable C-contiguous array")
        dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda")  # noqa: E731
        inv_d, det_d, co_d = dev(inv_j), dev(det_j), dev(coeffs)
        aux_d = dev(aux_vals) if aux_vals is not None else None
        out_d = torch.empty(tuple(out.shape), dtype=co_d.dtype, device="cuda")
    else:
        for a in arrays:
            if not a.is_cuda:
                raise ValueError("device path needs CUDA tensors for every per-cell array")
        if not out.is_contiguous():
            raise ValueError("out must be a contiguous CUDA tensor (it is written in place)")
        inv_d, det_d, co_d = inv_j.contiguous(), det_j.contiguous(), coeffs.contiguous()
        aux_d = aux_vals.contiguous() if aux_vals is not None else None
        out_d = out
    s = stream if stream is not None else torch.cuda.current_stream()
    rc = _lib.lib().txb_jit_integrate(ctypes.c_void_p(kernel.handle), n, B.ctypes.data, D.ctypes.data,
                                      W.ctypes.data, inv_d.data_ptr(), det_d.data_ptr(), co_d.data_ptr(),
                                      aux_d.data_ptr() if aux_d is not None else None, out_d.data_ptr(),
                                      n_bl, n_cb, ctypes.c_void_p(s.cuda_stream))
    _lib.check(rc, "txb_jit_integrate")
    if host:
        out[...] = out_d.cpu().numpy()
