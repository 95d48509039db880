"""Batch-integration API of the reference (txfem/executor.py:117-267) on the
CUDA lane.

* ``execute_chunk``  — integrate exactly one chunk.
* ``integrate_transposed`` — mesh-level driver: gather (E),
  element integration, deterministic scatter-add (E^T), all on the device.
* ``integrate_cells`` — the span call without the chunk bookkeeping, for
  device-resident callers (bench.py, multi-GPU ranks).

Differences from the reference, all deliberate:
  * the only lane is ``"cuda"`` (``backend=None`` selects it); ``"compiled"``,
    ``"python"`` and ``"simulated"`` are the reference's CPU lanes and raise
    ValueError here; ``log_tasks`` (the virtual-device task log) is an audit
    tool of the simulated device and is not available;
  * remainder cells (n mod N_chunk) are integrated in float64 and cast, as
    the reference does (executor.py:258-264), but by the float64 CUDA
    kernels (bit-identical to integrate_reference): the f32 residual equals
    the reference's bit for bit (tests/test_residual_golden.py);
  * ``jobs`` is accepted and has no effect on the result -- the reference's
    thread pool over chunks (executor.py:228-239) produces the same bits as
    its single call, and here one launch covers every chunk;
  * the caller's (N_bl, N_cb) define the execution geometry, its checks and
    the modelled trace exactly as in the reference, while the kernels run
    their B200-tuned batches (the same bits; _kernel_decomposition).
"""

from __future__ import annotations

import os
import weakref
from dataclasses import replace
from typing import Optional, Union

import numpy as np

from . import backend as _backend
from .element import QuadratureRule, Tabulation
from .errors import CapacityError, ShapeError
from .mesh import (CellGeometry, FieldLayout, Mesh, _stream_ptr, build_incidence, compute_geometry,
                   gather_coefficients, scatter_add_element_vectors)
from .physics import CellAux, PhysicsForm
from .schedule import DEFAULT_THREAD_LIMIT, ExecutionGeometry, derive_execution_geometry
from .trace import ChunkTrace, ExecutionTrace, model_batch_counters, shared_image_bytes

__all__ = ["DEFAULT_SHARED_MEM_LIMIT", "scalar_dtype", "execute_chunk", "integrate_transposed",
           "integrate_cells", "integrate_mesh", "integrate_partitioned", "invalidate_mesh_cache",
           "integrate_reference"]

DEFAULT_SHARED_MEM_LIMIT = 48 * 1024
_DTYPE_NAMES = {"f32": np.float32, "f64": np.float64}


def scalar_dtype(spec) -> np.dtype:
    """'f32'/'f64' or a float dtype -> np.dtype (executor.py:53-63)."""
    if isinstance(spec, str):
        try:
            return np.dtype(_DTYPE_NAMES[spec])
        except KeyError:
            raise ValueError(f"scalar must be 'f32' or 'f64', got {spec!r}") from None
    dt = np.dtype(spec)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError(f"scalar must be float32 or float64, got {dt}")
    return dt


def _check_capacity(geom: ExecutionGeometry, width: int, needs_f0: bool, limit: Optional[int]):
    """The reference's shared-memory budget check (executor.py:66-74), on the
    paper's image model, so callers see the same CapacityError behaviour."""
    required = shared_image_bytes(geom, width, needs_f0)
    if limit is not None and required > limit:
        raise CapacityError(
            f"shared-memory image needs {required} bytes, budget is {limit} "
            f"(n_bl={geom.n_bl}, scalar width {width})", required_bytes=required, limit_bytes=limit)


def _resolve_backend(requested: Optional[str], form: PhysicsForm, n_q: int, aux, width: int):
    """executor.py:93-106 with the lane set {"cuda"}."""
    if requested not in (None, "cuda"):
        if requested in ("compiled", "python", "simulated"):
            raise ValueError(f"backend {requested!r} is a reference CPU lane; this framework runs 'cuda'")
        raise ValueError(f"unknown backend {requested!r}")
    kernel = _backend.cuda_kernel(form, n_q, aux, width)
    if kernel is None:
        raise ValueError("cuda backend requested but unavailable for this configuration")
    return kernel


_CUDA_OK = False  # torch.cuda.is_available() seen True once (it does not flip back within a process)


def _torch():
    global _CUDA_OK
    import torch

    if not _CUDA_OK:
        if not torch.cuda.is_available():
            from .errors import CudaLaneError

            raise CudaLaneError("the CUDA lane needs a CUDA device")
        _CUDA_OK = True
    return torch


_PINNED_H2D_MIN_BYTES = 1 << 20


def _h2d(a: np.ndarray, torch):
    """numpy -> CUDA.  Arrays of >= 1 MiB go through a pinned staging block
    (torch's multi-threaded host copy, then an asynchronous DMA; the caching
    host allocator keeps the block until the copy has run): a pageable
    cudaMemcpy of the ~8 MB P0 kappa of a 2^20-cell mesh took 0.46 ms on the
    B200 box, staged 0.2 ms (tools/api_breakdown.py)."""
    t = torch.from_numpy(a)
    if a.nbytes < _PINNED_H2D_MIN_BYTES:
        return t.to("cuda")
    staged = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    staged.copy_(t)
    return staged.to("cuda", non_blocking=True)


def _dev(x, torch, dt):
    """Cast once to the configured scalar (executor._device_arrays, executor.py:77-90) and
    place on the device."""
    tdt = torch.float32 if dt == np.float32 else torch.float64
    if isinstance(x, np.ndarray):
        return _h2d(np.ascontiguousarray(x, dtype=dt), torch)
    return x.to(device="cuda", dtype=tdt).contiguous()


def integrate_cells(tab: Tabulation, rule: QuadratureRule, cell_geom: CellGeometry, coeffs,
                    aux: Optional[CellAux], form: PhysicsForm, *, dtype="f64", out=None,
                    n_bl: int = 0, n_cb: int = 0, stream=None):
    """Element vectors for every cell of the span on the CUDA lane.

    CUDA tensors in -> CUDA tensor out (async on the current stream); numpy in
    -> numpy out (host path).  ``n_bl``/``n_cb`` <= 0 pick the tuned defaults.
    """
    dt = scalar_dtype(dtype)
    form.require_aux(aux)
    n = cell_geom.n_cells
    if int(coeffs.shape[0]) != n or (aux is not None and int(aux.values.shape[0]) != n):
        raise ShapeError(f"per-cell arrays disagree: geometry {n} cells, coefficients {coeffs.shape[0]}")
    kernel = _resolve_backend(None, form, rule.n_q, aux, dt.itemsize)
    host = isinstance(coeffs, np.ndarray)
    if host:
        inv = np.ascontiguousarray(cell_geom.inv_jacobians, dtype=dt)
        det = np.ascontiguousarray(cell_geom.determinants, dtype=dt)
        co = np.ascontiguousarray(coeffs, dtype=dt)
        ax = None if aux is None else CellAux(aux.space, np.ascontiguousarray(aux.values, dtype=dt))
        res = out if out is not None else np.empty((n, tab.n_b, form.n_comp), dtype=dt)
    else:
        torch = _torch()
        inv, det, co = (_dev(x, torch, dt) for x in (cell_geom.inv_jacobians, cell_geom.determinants, coeffs))
        ax = None if aux is None else CellAux(aux.space, _dev(aux.values, torch, dt))
        res = out if out is not None else torch.empty((n, tab.n_b, form.n_comp), dtype=co.dtype, device="cuda")
    _backend.run_cuda(kernel, tab.basis, tab.basis_der, rule.weights, inv, det, co, ax, res,
                      n_bl=n_bl, n_cb=n_cb, stream=stream)
    return res


def integrate_reference(tab: Tabulation, rule: QuadratureRule, geom: CellGeometry, form: PhysicsForm, coeffs,
                        aux: Optional[CellAux] = None):
    """The reference's float64 oracle entry point (reference.py:40-112) with
    its contract -- (n, n_b, n_comp) float64 element vectors, inputs cast to
    float64, ShapeError on inconsistent spans -- computed by the float64 CUDA
    kernels, which reproduce integrate_reference bit for bit (shipped forms
    on the ahead-of-time kernels, user forms on the run-time compiled ones).
    numpy in -> numpy out; CUDA tensors in -> CUDA tensor out."""
    n = geom.n_cells
    shape = (n, tab.n_b, form.n_comp)
    if tuple(int(x) for x in coeffs.shape) != shape:
        raise ShapeError(f"coefficients have shape {tuple(coeffs.shape)}, expected {shape}")
    form.require_aux(aux)
    if aux is not None and int(aux.values.shape[0]) != n:
        raise ShapeError(f"auxiliary data covers {aux.values.shape[0]} cells, expected {n}")
    return integrate_cells(tab, rule, geom, coeffs, aux, form, dtype="f64")


def _kernel_decomposition(n_bl: int, n_cb: int):
    """(N_bl, N_cb) handed to the kernels by the reference-API calls.  The
    caller's decomposition shapes the execution geometry, its checks
    (ConfigurationError, CapacityError) and the modelled trace exactly as in
    the reference; the device schedule does not change a single bit of the
    result (tests/test_gpu_parity.py decomposition grid), so by default the
    kernels run their B200-tuned batches with dynamic scheduling -- the
    reference's own defaults (N_bl 16, N_cb 8: 64-cell batches in static
    8-batch chunks) cost 1.2-3x on this device (tools/ncb_probe.py).
    TXB_PAPER_DECOMPOSITION=1 launches the requested decomposition as is."""
    if os.environ.get("TXB_PAPER_DECOMPOSITION", "0") != "0":
        return n_bl, n_cb
    return 0, 0


def execute_chunk(geom: ExecutionGeometry, tab: Tabulation, rule: QuadratureRule, cell_geom: CellGeometry,
                  coeffs, aux: Optional[CellAux], form: PhysicsForm, *, dtype="f64", chunk_index: int = 0,
                  shared_mem_limit: Optional[int] = DEFAULT_SHARED_MEM_LIMIT, log_tasks: bool = False,
                  backend: Optional[str] = None):
    """Integrate exactly one chunk of cells (executor.py:117-158)."""
    dt = scalar_dtype(dtype)
    if cell_geom.n_cells != geom.n_chunk or int(coeffs.shape[0]) != geom.n_chunk:
        raise ShapeError(f"chunk slice covers {cell_geom.n_cells} cells, expected {geom.n_chunk}")
    form.require_aux(aux)
    _check_capacity(geom, dt.itemsize, form.has_f0, shared_mem_limit)
    if log_tasks:
        raise ValueError("log_tasks is a simulated-device audit feature; not available on the cuda lane")
    _resolve_backend(backend, form, geom.n_q, aux, dt.itemsize)
    k_bl, k_cb = _kernel_decomposition(geom.n_bl, geom.n_cb)
    elem = integrate_cells(tab, rule, cell_geom, coeffs, aux, form, dtype=dt, n_bl=k_bl, n_cb=k_cb)
    per_batch = model_batch_counters(geom, form, dt.itemsize, aux)
    trace = ChunkTrace(chunk_index=chunk_index, batches=[replace(per_batch) for _ in range(geom.n_cb)])
    return elem, trace


# Device copies of the last mesh's static data (connectivity, vertices, the
# vertex incidence CSR), reused across residual evaluations of the same mesh
# arrays on the same device.  Keyed on array identity + device + a sampled
# fingerprint of the contents (64 rows: catches typical in-place mesh motion
# for free); a caller that mutates a mesh in place in some other way calls
# invalidate_mesh_cache().
_INCIDENCE_CACHE: dict = {}
_MESH_CACHE: dict = {}


def invalidate_mesh_cache() -> None:
    """Drop every cached device copy of mesh data (connectivity, vertices,
    incidence, partitions): the next call re-uploads and re-validates."""
    _INCIDENCE_CACHE.clear()
    _MESH_CACHE.clear()
    _PART_CACHE.clear()
    _TILE_CACHE.clear()
    _ORIENTED.clear()


_FP_ROWS: dict = {}


def _fingerprint(a: np.ndarray) -> bytes:
    rows = a.shape[0]
    if rows == 0:
        return b""
    idx = _FP_ROWS.get(rows)
    if idx is None:  # the 64 sampled rows of an array of this length (memoised: per-call host cost)
        idx = np.unique(np.linspace(0, rows - 1, min(rows, 64)).astype(np.int64))
        if len(_FP_ROWS) > 256:
            _FP_ROWS.clear()
        _FP_ROWS[rows] = idx
    return a[idx].tobytes()


def _device_index(torch) -> int:
    return torch.cuda.current_device()


def _check_connectivity(mesh: Mesh):
    """0 <= cells < n_vertices, once per upload (the reference's numpy fancy
    indexing raises IndexError on a bad id; the kernels would read out of
    bounds)."""
    c = mesh.cells
    if c.size and (int(c.min()) < 0 or int(c.max()) >= mesh.n_vertices):
        raise IndexError(f"cell connectivity holds vertex ids outside [0, {mesh.n_vertices})")


def _incidence_for(mesh: Mesh, cells_dev):
    import torch

    key = (id(mesh.cells), mesh.cells.shape, mesh.n_vertices, _device_index(torch), _fingerprint(mesh.cells))
    hit = _INCIDENCE_CACHE.get(key)
    if hit is not None and hit[0] is mesh.cells:
        return hit[1]
    inc = build_incidence(mesh, cells_dev)
    _INCIDENCE_CACHE.clear()
    _INCIDENCE_CACHE[key] = (mesh.cells, inc)
    return inc


def _mesh_on_device(mesh: Mesh, torch):
    """(cells int64, vertices float64) CUDA tensors of ``mesh``, uploaded once."""
    key = (id(mesh.cells), id(mesh.vertices), mesh.cells.shape, mesh.vertices.shape, _device_index(torch),
           _fingerprint(mesh.cells), _fingerprint(mesh.vertices))
    hit = _MESH_CACHE.get(key)
    if hit is not None and hit[0] is mesh.cells and hit[1] is mesh.vertices:
        return hit[2], hit[3]
    _check_connectivity(mesh)
    cells = torch.from_numpy(np.ascontiguousarray(mesh.cells, dtype=np.int64)).to("cuda")
    verts = torch.from_numpy(np.ascontiguousarray(mesh.vertices, dtype=np.float64)).to("cuda")
    _MESH_CACHE.clear()
    _MESH_CACHE[key] = (mesh.cells, mesh.vertices, cells, verts)
    return cells, verts


# Cached device connectivity tensors (weakly, by id) whose mesh passed the
# orientation check (every detJ > 0) in a checked call: their later residuals
# skip the flag read-back, so a device-resident call stays asynchronous.  An
# entry dies with its tensor (a new upload is checked again).
_ORIENTED = weakref.WeakValueDictionary()


def _orientation_verified(cells_dev) -> bool:
    return _ORIENTED.get(id(cells_dev)) is cells_dev


def _mark_oriented(cells_dev) -> None:
    _ORIENTED[id(cells_dev)] = cells_dev


_PART_CACHE: dict = {}
_PART_CACHE_SIZE = 8


def _partition_on_device(mesh: Mesh, lo: int, hi: int, torch):
    """(cells[lo:hi] int64, vertices float64) CUDA tensors of one rank's cell
    range, uploaded once per (mesh arrays, range, device)."""
    key = (id(mesh.cells), id(mesh.vertices), mesh.cells.shape, mesh.vertices.shape, lo, hi, _device_index(torch),
           _fingerprint(mesh.cells), _fingerprint(mesh.vertices))
    hit = _PART_CACHE.get(key)
    if hit is not None and hit[0] is mesh.cells and hit[1] is mesh.vertices:
        return hit[2], hit[3]
    _check_connectivity(Mesh(mesh.dim, mesh.vertices, mesh.cells[lo:hi]))
    cells = torch.from_numpy(np.ascontiguousarray(mesh.cells[lo:hi], dtype=np.int64)).to("cuda")
    verts = torch.from_numpy(np.ascontiguousarray(mesh.vertices, dtype=np.float64)).to("cuda")
    while len(_PART_CACHE) >= _PART_CACHE_SIZE:  # several ranks may share a process (peer-group emulation)
        _PART_CACHE.pop(next(iter(_PART_CACHE)))
    _PART_CACHE[key] = (mesh.cells, mesh.vertices, cells, verts)
    return cells, verts


def integrate_transposed(mesh: Mesh, layout: FieldLayout, tab: Tabulation, rule: QuadratureRule,
                         form: PhysicsForm, coeffs_global, aux: Optional[CellAux] = None, *, n_bl: int,
                         n_cb: int, dtype: Union[str, np.dtype] = "f64", jobs: int = 1,
                         shared_mem_limit: Optional[int] = DEFAULT_SHARED_MEM_LIMIT,
                         thread_limit: int = DEFAULT_THREAD_LIMIT, log_tasks: bool = False,
                         backend: Optional[str] = None, cell_geom: Optional[CellGeometry] = None,
                         check_orientation: bool = True):
    """Global residual with the transposed schedule (executor.py:161-267).

    Returns (residual, trace): residual is a numpy vector in the configured
    scalar (a CUDA tensor if ``coeffs_global`` is one).  ``check_orientation``
    (extension): False skips the detJ <= 0 read-back of the in-kernel
    geometry (one host sync) -- for a mesh already checked (ResidualGraph)."""
    dt = scalar_dtype(dtype)
    geom = derive_execution_geometry(mesh.dim, tab.n_b, form.n_comp, rule.n_q, n_bl, n_cb, mesh.n_cells,
                                     thread_limit=thread_limit)
    form.require_aux(aux)
    _check_capacity(geom, dt.itemsize, form.has_f0, shared_mem_limit)
    if log_tasks:
        raise ValueError("log_tasks is a simulated-device audit feature; not available on the cuda lane")
    kernel = _resolve_backend(backend, form, rule.n_q, aux, dt.itemsize)
    if aux is not None and int(aux.values.shape[0]) != mesh.n_cells:
        raise ShapeError(f"auxiliary data covers {aux.values.shape[0]} cells, expected {mesh.n_cells}")
    n_bl, n_cb = _kernel_decomposition(n_bl, n_cb)  # (geom above keeps the caller's decomposition)
    torch = _torch()
    host_out = isinstance(coeffs_global, np.ndarray) or not hasattr(coeffs_global, "is_cuda")
    cells_dev, verts_dev = _mesh_on_device(mesh, torch)
    glob = coeffs_global if not host_out else np.asarray(coeffs_global, dtype=np.float64)
    glob_dev = _dev(glob, torch, dt)
    aux_dev = None if aux is None else CellAux(aux.space, _dev(aux.values, torch, dt))

    # the orientation of an uploaded mesh is checked once (one host sync), not per residual
    check = check_orientation and not _orientation_verified(cells_dev)
    if _mesh_fusable(tab, rule) and not isinstance(kernel, _backend.JitKernel):
        # geometry + gather + cast + integrate in one kernel (csrc/txb_integrate_tiled.cu / _mesh.cu)
        elem = integrate_mesh(mesh, layout, tab, rule, form, glob_dev, aux_dev, dtype=dt, cell_geom=cell_geom,
                              cells=cells_dev, vertices=verts_dev, n_bl=n_bl, check_orientation=check)
        if check and cell_geom is None:
            _mark_oriented(cells_dev)
    elif (isinstance(kernel, _backend.JitKernel) and os.environ.get("TXB_JIT_MESH", "1") != "0" and
          (cell_geom is None or _tiled_enabled(mesh, rule))):
        # run-time compiled form, fused the same way (csrc/txb_jit_kernel.cuh, mesh entry points; given
        # geometry through the tiled entry point)
        elem = _jit_mesh(kernel, mesh, tab, rule, form, glob_dev, aux_dev, dt, cells_dev, verts_dev, n_bl,
                         check and cell_geom is None, cell_geom=cell_geom)
        if check and cell_geom is None:
            _mark_oriented(cells_dev)
    else:
        if cell_geom is None:
            cell_geom = compute_geometry(mesh, cells=cells_dev, vertices=verts_dev, device_out=True)
        blocks = gather_coefficients(mesh, layout, glob_dev, cells=cells_dev)
        elem = integrate_cells(
            tab, rule, CellGeometry(_dev(cell_geom.inv_jacobians, torch, dt), _dev(cell_geom.determinants, torch, dt)),
            blocks, aux_dev, form, dtype=dt, n_bl=n_bl, n_cb=n_cb)
    if geom.n_r and dt == np.float32:
        # executor.py:258-264: the remainder cells (n mod N_chunk) are integrated
        # in float64 and cast -- here by the float64 kernels (bit-identical to
        # integrate_reference), so the f32 residual equals the reference's bits
        span = geom.n_chunks * geom.n_chunk
        elem[span:] = _remainder_f64(mesh, layout, tab, rule, form, kernel, glob, aux, cell_geom, cells_dev,
                                     verts_dev, span, n_bl, check).to(elem.dtype)
    residual = scatter_add_element_vectors(mesh, layout, elem, incidence=_incidence_for(mesh, cells_dev))

    trace = ExecutionTrace.uniform(geom, dt.itemsize, model_batch_counters(geom, form, dt.itemsize, aux),
                                   remainder_cells=geom.n_r)
    if host_out:
        residual = residual.cpu().numpy()
    return residual, trace




_FUSABLE: dict = {}


def _remainder_f64(mesh: Mesh, layout: FieldLayout, tab: Tabulation, rule: QuadratureRule, form: PhysicsForm,
                   kernel, glob, aux: Optional[CellAux], cell_geom: Optional[CellGeometry], cells_dev, verts_dev,
                   span: int, n_bl: int, check_orientation: bool = True):
    """Element vectors of cells [span, n) in float64 (a CUDA tensor): the
    reference's remainder path (integrate_reference on float64 geometry,
    coefficients and aux, executor.py:258-264) on the float64 kernels."""
    torch = _torch()
    f64 = np.dtype(np.float64)
    n = mesh.n_cells
    sub = Mesh(mesh.dim, mesh.vertices, mesh.cells[span:])
    cells = cells_dev[span:]
    g64 = _dev(glob, torch, f64)
    a64 = None if aux is None else CellAux(aux.space, _dev(aux.values[span:n], torch, f64))
    cg = None
    if cell_geom is not None:
        cg = CellGeometry(_dev(cell_geom.inv_jacobians[span:n], torch, f64),
                          _dev(cell_geom.determinants[span:n], torch, f64))
    k64 = _resolve_backend(None, form, rule.n_q, aux, 8)
    if _mesh_fusable(tab, rule) and not isinstance(k64, _backend.JitKernel):
        return integrate_mesh(sub, layout, tab, rule, form, g64, a64, dtype=f64, cell_geom=cg, cells=cells,
                              vertices=verts_dev, n_bl=n_bl, check_orientation=check_orientation)
    if isinstance(k64, _backend.JitKernel) and cg is None and os.environ.get("TXB_JIT_MESH", "1") != "0":
        return _jit_mesh(k64, sub, tab, rule, form, g64, a64, f64, cells, verts_dev, n_bl, check_orientation)
    if cg is None:
        cg = compute_geometry(sub, cells=cells, vertices=verts_dev, device_out=True)
    blocks = gather_coefficients(sub, layout, g64, cells=cells)
    return integrate_cells(tab, rule, CellGeometry(_dev(cg.inv_jacobians, torch, f64), _dev(cg.determinants, torch, f64)),
                           blocks, a64, form, dtype=f64, n_bl=n_bl)


def _check_aux_shape(aux, n_cells: int, n_b: int, form: PhysicsForm):
    """The full shape of a CellAux's values: (n, n_aux) for p0, (n, n_b, n_aux)
    for p1 -- the reference's memoryviews reject anything else
    (_kernels_cy.pyx:37-49); the fused kernels would read out of bounds."""
    if aux is None:
        return
    want = (n_cells, form.n_aux) if aux.space == "p0" else (n_cells, n_b, form.n_aux)
    got = tuple(int(x) for x in aux.values.shape)
    if got != want:
        raise ShapeError(f"{aux.space} auxiliary values have shape {got}, expected {want}")


def _jit_mesh(kernel, mesh: Mesh, tab: Tabulation, rule: QuadratureRule, form: PhysicsForm, glob_dev, aux_dev, dt,
              cells_dev, verts_dev, n_bl: int, check_orientation: bool = True, out=None, cell_geom=None):
    """Element vectors of a run-time compiled form straight from the mesh
    (txb_jit_integrate_mesh: float64 geometry + gather in-kernel, any
    tabulation).  Raises OrientationError for a cell with detJ <= 0."""
    import ctypes

    from . import _lib
    from .errors import OrientationError

    torch = _torch()
    n = mesh.n_cells
    _check_aux_shape(aux_dev, n, tab.n_b, form)
    if int(glob_dev.numel()) != mesh.n_vertices * form.n_comp:
        raise ShapeError(f"global vector has {glob_dev.numel()} entries, expected {mesh.n_vertices * form.n_comp}")
    res = out if out is not None else torch.empty((n, tab.n_b, form.n_comp), dtype=glob_dev.dtype, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda") if check_orientation else None
    B, D, W = (np.ascontiguousarray(x, dtype=dt) for x in (tab.basis, tab.basis_der, rule.weights))
    av = None if aux_dev is None else aux_dev.values.contiguous()
    inv = det = None
    if cell_geom is not None:  # (tiled path only: the caller's geometry, cast once to the run precision)
        inv, det = _dev(cell_geom.inv_jacobians, torch, dt), _dev(cell_geom.determinants, torch, dt)
        bad = None
    if n > 0 and _tiled_enabled(mesh, rule):
        # per-tile vertex tables (the tiled kernel's design, run-time compiled form)
        tiles = cell_tiles(cells_dev, mesh.dim, default_tile_cells(mesh.dim, rule.n_q, inv is not None,
                                                                   np.dtype(dt).itemsize))
        rc = _lib.lib().txb_jit_integrate_mesh_tiled(
            ctypes.c_void_p(kernel.handle), n, mesh.n_vertices, B.ctypes.data, D.ctypes.data, W.ctypes.data,
            verts_dev.data_ptr(), tiles.tile_cells, tiles.records.data_ptr(), tiles.vrec, tiles.local.data_ptr(),
            tiles.local_bytes, glob_dev.data_ptr(), None if inv is None else inv.data_ptr(),
            None if det is None else det.data_ptr(), None if av is None else av.data_ptr(), res.data_ptr(),
            None if bad is None else bad.data_ptr(), _stream_ptr(torch))
        _lib.check(rc, "txb_jit_integrate_mesh_tiled")
    else:
        rc = _lib.lib().txb_jit_integrate_mesh(ctypes.c_void_p(kernel.handle), n, mesh.n_vertices, B.ctypes.data,
                                               D.ctypes.data, W.ctypes.data, verts_dev.data_ptr(),
                                               cells_dev.data_ptr(), glob_dev.data_ptr(),
                                               None if av is None else av.data_ptr(), res.data_ptr(),
                                               None if bad is None else bad.data_ptr(), n_bl, _stream_ptr(torch))
        _lib.check(rc, "txb_jit_integrate_mesh")
    if bad is not None:
        i = int(bad.item())
        if i >= 0:
            raise OrientationError(f"cell {i} is degenerate or negatively oriented")
    return res


def _mesh_fusable(tab: Tabulation, rule: QuadratureRule) -> bool:
    """The fused mesh kernel needs the standard P1 reference gradients (what
    element.tabulate produces for every rule) and n_q <= 2.  Memoised per
    tabulation object (tables are not mutated in place)."""
    if rule.n_q > 2:
        return False
    hit = _FUSABLE.get(id(tab))
    if hit is not None and hit[0] is tab:
        return hit[1]
    D = np.asarray(tab.basis_der, dtype=np.float64)
    want = np.vstack([-np.ones((1, tab.dim)), np.eye(tab.dim)])
    ok = all(np.array_equal(D[q], want) for q in range(D.shape[0]))
    if len(_FUSABLE) > 64:
        _FUSABLE.clear()
    _FUSABLE[id(tab)] = (tab, ok)
    return ok


class CellTiles:
    """A mesh's cells cut into tiles of ``tile_cells`` consecutive cells, each
    with the ascending list of its distinct vertices (``records``, int32, stride
    ``vrec``: [count, 0, 0, 0, ids...]) and every cell's 4 local indices into
    it (``local``, uint8 or uint16): the per-mesh input of the tiled kernel
    (csrc/txb_integrate_tiled.cu).  Built on the device by txb_tile_counts +
    txb_tile_build (one host sync: the largest count sizes the records)."""

    def __init__(self, cells_dev, dim: int, tile_cells: int):
        from . import _lib

        torch = _torch()
        n = int(cells_dev.shape[0])
        self.tile_cells = tile_cells
        self.n_tiles = -(-n // tile_cells)
        counts = torch.zeros(max(1, self.n_tiles), dtype=torch.int32, device=cells_dev.device)
        s = _stream_ptr(torch)
        _lib.check(_lib.lib().txb_tile_counts(dim, n, cells_dev.data_ptr(), tile_cells, counts.data_ptr(), s),
                   "txb_tile_counts")
        if self.n_tiles and int(counts.min().item()) < 0:
            raise IndexError("cell connectivity holds vertex ids outside [0, 2^31) (tiled mesh kernel)")
        self.max_count = int(counts.max().item()) if self.n_tiles else 0
        self.vrec = 4 + max(4, -(-self.max_count // 4) * 4)
        self.local_bytes = 1 if self.max_count <= 256 else 2
        self.records = torch.zeros(max(1, self.n_tiles) * self.vrec, dtype=torch.int32, device=cells_dev.device)
        self.local = torch.zeros(max(1, self.n_tiles) * tile_cells * 4 * self.local_bytes, dtype=torch.uint8,
                                 device=cells_dev.device)
        _lib.check(_lib.lib().txb_tile_build(dim, n, cells_dev.data_ptr(), tile_cells, self.vrec, self.local_bytes,
                                             self.records.data_ptr(), self.local.data_ptr(), s), "txb_tile_build")
        self.mean_count = float(counts.double().mean().item()) if self.n_tiles else 0.0


_TILE_CACHE: dict = {}
_TILE_CACHE_SIZE = 32


def default_tile_cells(dim: int, n_q: int, given_geometry: bool = False, dtype_bytes: int = 8) -> int:
    """Cells per tile (= per batch) of the tiled kernel: 3D 128 (midpoint) / 64
    (two points), 2D 192 / 96 -- multiples of n_b * n_q and of the warp slice
    32 / n_q, at most 6 slices (4-6 consumer warps).  The caller's float64
    geometry (80 / 40 B per cell streamed with the batch) runs best on half
    those tiles at the midpoint rule (3D var-coef 25.7 -> 23.4 us, 2D
    elasticity 21.2 -> 19.6 us at 2^20 cells; profiles/r2_tiled.md).
    TXB_TILE_CELLS overrides."""
    env = os.environ.get("TXB_TILE_CELLS")
    if env:
        return int(env)
    half = given_geometry and dtype_bytes == 8 and n_q == 1
    if dim == 3:
        return (64 if half else 128) if n_q == 1 else 64
    return (96 if half else 192) if n_q == 1 else 96


def cell_tiles(cells_dev, dim: int, tile_cells: int) -> CellTiles:
    """The CellTiles of a device connectivity tensor, built once per (memory
    range, tile size, device) and cached (the tensor is kept alive with them,
    so the address cannot be reused; a view of the same range hits the same
    entry).  An in-place modification through torch bumps the tensor's version
    and rebuilds the tables; writes through raw pointers are not seen (the
    mesh caches above hand out fresh tensors when the host mesh changes)."""
    # (torch's in-place version counter: a connectivity tensor modified in place by torch ops misses)
    key = (cells_dev.data_ptr(), tuple(cells_dev.shape), tuple(cells_dev.stride()), cells_dev.device.index,
           tile_cells, cells_dev._version)
    hit = _TILE_CACHE.get(key)
    if hit is not None:  # (the cached tensor keeps that memory alive: same key, same storage; views match too)
        return hit[1]
    tiles = CellTiles(cells_dev, dim, tile_cells)
    size = lambda e: (e[0].numel() * e[0].element_size() + e[1].records.numel() * 4  # noqa: E731
                      + e[1].local.numel())
    budget = int(os.environ.get("TXB_TILE_CACHE_MB", "4096")) << 20
    entry = (cells_dev, tiles)
    # bounded: at most _TILE_CACHE_SIZE entries and TXB_TILE_CACHE_MB of tables + the connectivity
    # they keep alive (oldest first out)
    while _TILE_CACHE and (len(_TILE_CACHE) >= _TILE_CACHE_SIZE or
                           sum(size(e) for e in _TILE_CACHE.values()) + size(entry) > budget):
        _TILE_CACHE.pop(next(iter(_TILE_CACHE)))
    _TILE_CACHE[key] = entry
    return tiles


def _tiled_enabled(mesh: Mesh, rule: QuadratureRule) -> bool:
    """The tiled kernel takes the geometry-in-kernel mesh calls (TXB_TILED=0
    keeps the per-cell fused kernel): int32 vertex ids, n_q <= 2."""
    return os.environ.get("TXB_TILED", "1") != "0" and mesh.n_vertices < (1 << 31) and rule.n_q <= 2


def integrate_mesh(mesh: Mesh, layout: FieldLayout, tab: Tabulation, rule: QuadratureRule, form: PhysicsForm,
                   coeffs_global, aux: Optional[CellAux] = None, *, dtype="f64", cell_geom=None, cells=None,
                   vertices=None, out=None, n_bl: int = 0, check_orientation: bool = True):
    """Element vectors straight from the mesh on the device: the reference's
    compute_geometry -> gather_coefficients -> cast -> integrate_cells
    (executor.py:194-212) fused into one kernel (txb_integrate_mesh).

    ``coeffs_global``: (n_vertices * n_comp) CUDA tensor in the run dtype.
    ``cell_geom``: None (geometry from the vertices, float64) or given geometry.
    ``cells`` / ``vertices``: optional device copies of the connectivity and
    coordinates (uploaded from ``mesh`` otherwise).
    Returns a CUDA tensor (n_cells, n_b, n_comp).  Raises OrientationError
    naming the first cell with detJ <= 0 (a host sync) when the geometry is
    computed and ``check_orientation``."""
    import ctypes

    from . import _lib
    from .errors import OrientationError

    torch = _torch()
    dt = scalar_dtype(dtype)
    form.require_aux(aux)
    kernel = _resolve_backend(None, form, rule.n_q, aux, dt.itemsize)
    if isinstance(kernel, _backend.JitKernel):
        raise ValueError(f"the fused mesh kernel covers the shipped forms; form {form.name!r} runs through "
                         "integrate_transposed (geometry -> gather -> run-time compiled integration)")
    n = mesh.n_cells
    _check_aux_shape(aux, n, tab.n_b, form)
    if cells is None:
        _check_connectivity(mesh)  # (caller-provided device connectivity is the caller's contract)
    C = cells if cells is not None else torch.from_numpy(np.ascontiguousarray(mesh.cells, dtype=np.int64)).cuda()
    X = vertices if vertices is not None else \
        torch.from_numpy(np.ascontiguousarray(mesh.vertices, dtype=np.float64)).cuda()
    g = _dev(coeffs_global, torch, dt)
    if int(g.numel()) != mesh.n_vertices * form.n_comp:
        raise ShapeError(f"global vector has {g.numel()} entries, expected {mesh.n_vertices * form.n_comp}")
    inv = det = None
    if cell_geom is not None:
        inv, det = _dev(cell_geom.inv_jacobians, torch, dt), _dev(cell_geom.determinants, torch, dt)
    av = None if aux is None else _dev(aux.values, torch, dt)
    res = out if out is not None else torch.empty((n, tab.n_b, form.n_comp), dtype=g.dtype, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda") if cell_geom is None and check_orientation else None
    B, D, W = (np.ascontiguousarray(x, dtype=dt) for x in (tab.basis, tab.basis_der, rule.weights))
    ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    tiles = None
    if n > 0 and _tiled_enabled(mesh, rule):
        tiles = cell_tiles(C, mesh.dim, default_tile_cells(mesh.dim, rule.n_q, inv is not None, dt.itemsize))
    if tiles is not None:
        # (geometry +) gather from per-tile vertex tables (csrc/txb_integrate_tiled.cu)
        rc = _lib.lib().txb_integrate_mesh_tiled(
            kernel[0], kernel[1], dt.itemsize, mesh.dim, rule.n_q, form.n_comp, n, mesh.n_vertices,
            B.ctypes.data, D.ctypes.data, W.ctypes.data, X.data_ptr(), tiles.tile_cells, tiles.records.data_ptr(),
            tiles.vrec, tiles.local.data_ptr(), tiles.local_bytes, g.data_ptr(), ptr(inv), ptr(det), ptr(av),
            res.data_ptr(), ptr(bad), _stream_ptr(torch))
        _lib.check(rc, "txb_integrate_mesh_tiled")
    else:
        rc = _lib.lib().txb_integrate_mesh(
            kernel[0], kernel[1], dt.itemsize, mesh.dim, rule.n_q, form.n_comp, n, mesh.n_vertices,
            B.ctypes.data, D.ctypes.data, W.ctypes.data, X.data_ptr(), C.data_ptr(), g.data_ptr(), ptr(inv),
            ptr(det), ptr(av), res.data_ptr(), ptr(bad), n_bl, _stream_ptr(torch))
        _lib.check(rc, "txb_integrate_mesh")
    if bad is not None:
        i = int(bad.item())
        if i >= 0:
            raise OrientationError(f"cell {i} is degenerate or negatively oriented")
    return res


class ResidualGraph:
    """``integrate_transposed`` for one fixed (mesh, layout, tabulation, rule,
    form, aux, dtype) captured ONCE into a CUDA graph: every later residual
    evaluation is a copy of the global vector into the graph's input buffer
    and one graph replay (fused mesh kernel, f32 remainder cells, deterministic
    scatter-add) -- no per-call Python dispatch, argument checks, cache
    lookups or launch overhead (the device-resident call's ~0.1 ms host floor,
    DESIGN.md §7).  For GPU-resident solver loops (Newton / Krylov iterations
    over a static mesh).  Same bits as integrate_transposed.

    The constructor runs one eager call (uploads and caches the mesh's device
    data, builds the incidence and tile tables, compiles a run-time form, and
    checks orientation -- OrientationError is raised there), then captures.
    The mesh, aux and tabulation are frozen at construction (aux is copied);
    build a new ResidualGraph after changing them.

    ``graph(coeffs_global)`` -> the residual, a CUDA tensor owned by the graph
    and overwritten by the next call (pass ``out=`` to copy it out).
    ``coeffs_global``: CUDA tensor or numpy array of layout.global_size(mesh)
    entries (held in float64, cast to the run dtype inside the graph).  A
    solver that writes the graph's own input buffer ``graph.glob`` in place
    calls ``graph()`` (or passes ``graph.glob``): no copy, one replay.
    One caller at a time: the input and residual buffers are the graph's own
    (not thread-safe; replays are ordered on the caller's current stream)."""

    def __init__(self, mesh: Mesh, layout: FieldLayout, tab: Tabulation, rule: QuadratureRule, form: PhysicsForm,
                 aux: Optional[CellAux] = None, *, n_bl: int, n_cb: int, dtype="f64",
                 cell_geom: Optional[CellGeometry] = None, **kwargs):
        torch = _torch()
        dt = scalar_dtype(dtype)
        tdt = torch.float32 if dt == np.float32 else torch.float64
        self.dtype = dt
        self.n = layout.global_size(mesh)
        # float64 input buffer (and aux copy) whatever the run precision: the f32 lane reads it cast once (in the graph),
        # the f32 run's float64 remainder cells read it as given -- as integrate_transposed does with a
        # float64 global vector (executor.py:258-264); an f32 input is copied in exactly
        self.glob = torch.zeros(self.n, dtype=torch.float64, device="cuda")
        del tdt
        self.aux = None if aux is None else CellAux(aux.space, _dev(aux.values, torch, np.dtype(np.float64)).clone())
        if cell_geom is not None:
            cell_geom = CellGeometry(_dev(cell_geom.inv_jacobians, torch, dt).clone(),
                                     _dev(cell_geom.determinants, torch, dt).clone())
        call = dict(n_bl=n_bl, n_cb=n_cb, dtype=dt, cell_geom=cell_geom, **kwargs)
        self._args = (mesh, layout, tab, rule, form)
        kernel = _resolve_backend(kwargs.get("backend"), form, rule.n_q, aux, dt.itemsize)
        if cell_geom is None and not isinstance(kernel, _backend.JitKernel) and not _mesh_fusable(tab, rule):
            # the unfused path's geometry call synchronises (its orientation check): geometry once, here
            cells_dev, verts_dev = _mesh_on_device(mesh, torch)
            g = compute_geometry(mesh, cells=cells_dev, vertices=verts_dev, device_out=True)
            call["cell_geom"] = CellGeometry(_dev(g.inv_jacobians, torch, dt), _dev(g.determinants, torch, dt))
        self._call = call  # the graph reads these device tensors (given / precomputed geometry): keep them alive
        # eager warm-up (caches, tables, compilation, the orientation check)
        _, self.trace = integrate_transposed(*self._args, self.glob, self.aux, **call)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(self.graph, stream=side):
                self.residual, _ = integrate_transposed(*self._args, self.glob, self.aux, check_orientation=False,
                                                        **call)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        # the graph holds raw pointers into the cached device mesh data (connectivity, vertices, incidence,
        # tile tables): keep THIS mesh's tensors alive past any later eviction from the module caches
        cells_dev, verts_dev = _mesh_on_device(mesh, torch)
        lo = cells_dev.data_ptr()
        hi = lo + cells_dev.numel() * cells_dev.element_size()
        self._keep = [cells_dev, verts_dev, _incidence_for(mesh, cells_dev),
                      [t for k, t in _TILE_CACHE.items() if lo <= k[0] < hi]]

    def __call__(self, coeffs_global=None, out=None):
        torch = _torch()
        if coeffs_global is not None and not (hasattr(coeffs_global, "data_ptr") and
                                              coeffs_global.data_ptr() == self.glob.data_ptr()):
            if isinstance(coeffs_global, np.ndarray) or not hasattr(coeffs_global, "is_cuda"):
                src = torch.from_numpy(np.ascontiguousarray(coeffs_global, dtype=np.float64))
            else:
                src = coeffs_global
            if int(src.numel()) != self.n:
                raise ShapeError(f"global vector has {src.numel()} entries, expected {self.n}")
            self.glob.copy_(src.reshape(-1), non_blocking=False)
        # (None, or the graph's own input buffer: the caller wrote graph.glob in place -- no copy)
        self.graph.replay()
        if out is not None:
            out.copy_(self.residual)
            return out
        return self.residual


def integrate_partitioned(mesh: Mesh, layout: FieldLayout, tab: Tabulation, rule: QuadratureRule,
                          form: PhysicsForm, coeffs_global, aux: Optional[CellAux] = None, *, rank: int,
                          world: int, exchange=None, dtype="f64", plan=None, align: int = 256, n_bl: int = 0,
                          peer=None, check: bool = True):
    """One rank's share of integrate_transposed for the contiguous cell-range
    partition over ``world`` ranks (shard.cell_range): integrate the rank's
    cells on its GPU, then the halo exchange + assembly of halo.py.

    Returns (owned_vertex_ids (numpy, in the plan's slot order),
    owned_residual (CUDA tensor (n_owned * n_comp,)), plan).  Placing every
    rank's owned entries at their vertex ids reproduces the reference
    residual (executor.py:266, np.add.at order) bit for bit.  ``exchange``: halo.all_to_all_exchange() under torch.distributed
    (None for world == 1).  ``plan``: a cached halo.build_halo_plan result.
    ``peer``: a halo.PeerHalo — the exchange over peer memory (txb_halo_put /
    txb_halo_assemble) instead of ``exchange``; its plan is used.  With
    ``check`` (default) a failed exchange raises CudaLaneError here (one host
    sync); ``check=False`` keeps the call asynchronous -- then call
    ``peer.check()`` before trusting the result (a failed epoch's owned
    entries are NaN, never silently stale)."""
    from . import halo

    torch = _torch()
    dt = scalar_dtype(dtype)
    form.require_aux(aux)
    if peer is not None:
        plan = peer.plan
    if plan is None:
        plan = halo.build_halo_plan(mesh.cells, mesh.n_vertices, rank, world, align)
    lo, hi = plan.lo, plan.hi
    n_b, nc = tab.n_b, form.n_comp
    sub = Mesh(mesh.dim, mesh.vertices, np.ascontiguousarray(mesh.cells[lo:hi]))
    tdt = torch.float32 if dt == np.float32 else torch.float64
    recv_rows = 0 if peer is not None else plan.n_recv  # the peer path receives into its window
    buf = torch.empty((plan.n_local_rows + recv_rows, nc), dtype=tdt, device="cuda")
    elem = buf[:plan.n_local_rows].view(hi - lo, n_b, nc)
    if hi > lo:
        kernel = _resolve_backend(None, form, rule.n_q, aux, dt.itemsize)
        glob_dev = _dev(coeffs_global, torch, dt)
        aux_dev = None if aux is None else CellAux(aux.space, _dev(aux.values[lo:hi], torch, dt))
        cells_dev, verts_dev = _partition_on_device(mesh, lo, hi, torch)
        if _mesh_fusable(tab, rule) and not isinstance(kernel, _backend.JitKernel):
            # orientation checked on the first residual of this uploaded range only (one host sync)
            check_o = not _orientation_verified(cells_dev)
            integrate_mesh(sub, layout, tab, rule, form, glob_dev, aux_dev, dtype=dt, cells=cells_dev,
                           vertices=verts_dev, out=elem, n_bl=n_bl, check_orientation=check_o)
            if check_o:
                _mark_oriented(cells_dev)
        elif isinstance(kernel, _backend.JitKernel) and os.environ.get("TXB_JIT_MESH", "1") != "0":
            # run-time compiled form: its (tiled) mesh entry point, as integrate_transposed
            check_o = not _orientation_verified(cells_dev)
            _jit_mesh(kernel, sub, tab, rule, form, glob_dev, aux_dev, dt, cells_dev, verts_dev, n_bl, check_o,
                      out=elem)
            if check_o:
                _mark_oriented(cells_dev)
        else:
            g = compute_geometry(sub, cells=cells_dev, vertices=verts_dev, device_out=True)
            blocks = gather_coefficients(sub, layout, glob_dev, cells=cells_dev)
            integrate_cells(tab, rule, CellGeometry(_dev(g.inv_jacobians, torch, dt), _dev(g.determinants, torch, dt)),
                            blocks, aux_dev, form, dtype=dt, out=elem, n_bl=n_bl)
    if peer is not None:
        owned = peer.exchange_assemble(buf)
        if check:
            torch.cuda.current_stream().synchronize()
            peer.check()
    else:
        owned = halo.assemble_owned(plan, buf, nc, exchange)
    return plan.owned, owned.reshape(-1), plan
