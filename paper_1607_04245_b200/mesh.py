"""Meshes and the data movement either side of the integration kernel.

* ``generate_unit_simplex_mesh`` — Kuhn/Freudenthal meshes of the unit
  square/cube (txfem/mesh.py:81-147): the synthetic-input producer, host
  numpy, identical cell order and coordinates to the reference.
* ``compute_geometry``, ``gather_coefficients``, ``scatter_add_element_vectors``
  — the reference's host steps (mesh.py:150-234) executed by the CUDA library
  (csrc/txb_mesh.cu).  They accept numpy arrays (returning numpy, a host round
  trip) or CUDA torch tensors (staying on the device).  All three are
  bit-identical to the reference: same expression order, and a deterministic
  CSR scatter in ascending cell order instead of float atomics.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import TextIO

import numpy as np

from . import _lib
from .errors import InvalidDimensionError, ShapeError

__all__ = [
    "Mesh", "CellGeometry", "FieldLayout", "generate_unit_simplex_mesh", "compute_geometry",
    "gather_coefficients", "scatter_add_element_vectors", "interior_vertex_mask", "dump_mesh",
    "VertexIncidence", "build_incidence",
]

# (axis permutation, parity) of the six Kuhn tetrahedra of a cube
_CUBE_PERMS = (((0, 1, 2), 1), ((0, 2, 1), -1), ((1, 0, 2), -1), ((1, 2, 0), 1), ((2, 0, 1), 1),
               ((2, 1, 0), -1))


@dataclass(frozen=True)
class Mesh:
    dim: int
    vertices: np.ndarray  # (n_vertices, dim) float64
    cells: np.ndarray  # (n_cells, dim + 1) int64

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def n_cells(self) -> int:
        return self.cells.shape[0]


@dataclass(frozen=True)
class CellGeometry:
    inv_jacobians: object  # (n_cells, d, d) row-major; numpy or CUDA tensor
    determinants: object  # (n_cells,)

    @property
    def n_cells(self) -> int:
        return int(self.determinants.shape[0])


@dataclass(frozen=True)
class FieldLayout:
    """Interleaved global layout: entry v*n_comp + c is component c at vertex v."""

    n_comp: int = 1

    def global_size(self, mesh: Mesh) -> int:
        return mesh.n_vertices * self.n_comp


def generate_unit_simplex_mesh(dim: int, n: int) -> Mesh:
    """2 n^2 triangles / 6 n^3 positively oriented tetrahedra on a regular grid."""
    if dim not in (2, 3):
        raise InvalidDimensionError(f"dim must be 2 or 3, got {dim}")
    if n < 1:
        raise ValueError(f"need at least one subdivision per axis, got {n}")
    ticks = np.linspace(0.0, 1.0, n + 1)
    m = n + 1
    if dim == 2:
        iy, ix = np.divmod(np.arange(m * m), m)
        vertices = np.column_stack([ticks[ix], ticks[iy]])
        sy, sx = np.divmod(np.arange(n * n, dtype=np.int64), n)  # squares, x fastest
        v00 = sy * m + sx
        v10, v01 = v00 + 1, v00 + m
        v11 = v01 + 1
        cells = np.stack([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)], 1)
        return Mesh(2, vertices, cells.reshape(-1, 3))
    idx = np.arange(m ** 3)
    vertices = np.column_stack([ticks[idx % m], ticks[(idx // m) % m], ticks[idx // (m * m)]])
    cube = np.arange(n ** 3, dtype=np.int64)
    corner = np.column_stack([cube // (n * n), (cube // n) % n, cube % n])  # x slowest, z fastest
    tets = np.empty((n ** 3, 6, 4), dtype=np.int64)
    eye = np.eye(3, dtype=np.int64)
    for t, (perm, parity) in enumerate(_CUBE_PERMS):
        p1 = corner + eye[perm[0]]
        p2 = p1 + eye[perm[1]]
        p3 = p2 + eye[perm[2]]
        path = (corner, p1, p2, p3) if parity > 0 else (corner, p1, p3, p2)
        for k, pt in enumerate(path):
            tets[:, t, k] = (pt[:, 2] * m + pt[:, 1]) * m + pt[:, 0]
    return Mesh(3, vertices, tets.reshape(-1, 4))


def interior_vertex_mask(mesh: Mesh, tol: float = 1e-12) -> np.ndarray:
    v = mesh.vertices
    return ~((np.abs(v) < tol) | (np.abs(v - 1.0) < tol)).any(axis=1)


def dump_mesh(mesh: Mesh, stream: TextIO) -> None:
    stream.write(f"{mesh.dim} {mesh.n_vertices} {mesh.n_cells}\n")
    for v in mesh.vertices:
        stream.write(" ".join(f"{x:.17g}" for x in v) + "\n")
    for c in mesh.cells:
        stream.write(" ".join(str(int(i)) for i in c) + "\n")


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

_CUDA_OK = False  # torch.cuda.is_available() seen True once


def _torch():
    global _CUDA_OK
    import torch

    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise _lib.CudaLaneError("the CUDA lane needs a CUDA device (torch.cuda.is_available() is False)")
        _CUDA_OK = True
    return torch


def _stream_ptr(torch):
    # current_stream(<int device>) skips torch's device-index resolution of the
    # no-argument form (a few us per call on the mesh-level path)
    return ctypes.c_void_p(torch.cuda.current_stream(torch.cuda.current_device()).cuda_stream)


def _to_device(x, torch, dtype=None):
    if isinstance(x, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(x))
        if dtype is not None:
            t = t.to(dtype)
        return t.to("cuda", non_blocking=False), True
    t = x if dtype is None else x.to(dtype)
    if not t.is_cuda:
        t = t.to("cuda")
        return t.contiguous(), True
    return t.contiguous(), False


def compute_geometry(mesh: Mesh, *, cells=None, vertices=None, device_out: bool = False) -> CellGeometry:
    """Inverse Jacobians (J's k-th column = v_{k+1} - v_0) and detJ on the
    device, float64, cofactor formulas of mesh.py:150-190.  Raises
    OrientationError naming the first cell with detJ <= 0.  ``cells`` /
    ``vertices``: optional device copies (int64 / float64) of the mesh arrays."""
    torch = _torch()
    d = mesh.dim
    X = vertices if vertices is not None else \
        _to_device(np.ascontiguousarray(mesh.vertices, dtype=np.float64), torch)[0]
    C = cells if cells is not None else _to_device(np.ascontiguousarray(mesh.cells, dtype=np.int64), torch)[0]
    n = int(C.shape[0])
    inv = torch.empty((n, d, d), dtype=torch.float64, device="cuda")
    det = torch.empty((n,), dtype=torch.float64, device="cuda")
    bad = ctypes.c_int64(-1)
    rc = _lib.lib().txb_compute_geometry(d, n, X.data_ptr(), C.data_ptr(), inv.data_ptr(),
                                         det.data_ptr(), ctypes.byref(bad), _stream_ptr(torch))
    if rc == _lib.TXB_E_ORIENTATION:
        i = int(bad.value)
        from .errors import OrientationError

        raise OrientationError(
            f"cell {i} is degenerate or negatively oriented (detJ = {float(det[i])!r})")
    _lib.check(rc, "txb_compute_geometry")
    if device_out:
        return CellGeometry(inv, det)
    return CellGeometry(inv.cpu().numpy(), det.cpu().numpy())


def gather_coefficients(mesh: Mesh, layout: FieldLayout, global_vec, *, cells=None):
    """Per-cell blocks out[c][b][k] = global[cells[c][b]*n_comp + k] (mesh.py:202-217).
    numpy in -> numpy out; CUDA tensor in -> CUDA tensor out."""
    torch = _torch()
    expected = layout.global_size(mesh)
    if tuple(global_vec.shape) != (expected,):
        raise ShapeError(f"global vector has shape {tuple(global_vec.shape)}, expected ({expected},)")
    host = isinstance(global_vec, np.ndarray)
    if host and global_vec.dtype not in (np.float32, np.float64):
        global_vec = global_vec.astype(np.float64)
    g, _ = _to_device(global_vec, torch)
    C = cells if cells is not None else _to_device(np.ascontiguousarray(mesh.cells, dtype=np.int64), torch)[0]
    n = int(C.shape[0])
    out = torch.empty((n, mesh.dim + 1, layout.n_comp), dtype=g.dtype, device="cuda")
    _lib.check(_lib.lib().txb_gather_coefficients(g.element_size(), n, mesh.dim + 1, layout.n_comp,
                                                  C.data_ptr(), g.data_ptr(), out.data_ptr(),
                                                  _stream_ptr(torch)), "txb_gather_coefficients")
    return out.cpu().numpy() if host else out


@dataclass
class VertexIncidence:
    """vertex -> (cell*n_b + b) CSR, entries in ascending cell order (device).
    ``slot_*``: the same lists in slot order (vertices by first element row,
    txb_build_scatter_order) — what the scatter walks; None = vertex order."""

    offsets: object
    incidence: object
    n_vertices: int
    n_cells: int
    slot_offsets: object = None
    slot_incidence: object = None
    slot_vertex: object = None


def build_scatter_order(inc: VertexIncidence) -> VertexIncidence:
    """Attach the slot-ordered CSR to ``inc`` (device, one sort over the vertices)."""
    torch = _torch()
    L = _lib.lib()
    nv = inc.n_vertices
    n_entries = int(inc.incidence.numel()) if inc.n_cells else 0
    slot_offsets = torch.empty((nv + 1,), dtype=torch.int64, device="cuda")
    slot_inc = torch.empty((max(n_entries, 1),), dtype=torch.int32, device="cuda")
    slot_vertex = torch.empty((max(nv, 1),), dtype=torch.int32, device="cuda")
    scratch = torch.empty((max(int(L.txb_scatter_order_scratch_bytes(nv)), 16),), dtype=torch.uint8, device="cuda")
    _lib.check(L.txb_build_scatter_order(nv, n_entries, inc.offsets.data_ptr(), inc.incidence.data_ptr(),
                                         slot_offsets.data_ptr(), slot_inc.data_ptr(), slot_vertex.data_ptr(),
                                         scratch.data_ptr(), _stream_ptr(torch)), "txb_build_scatter_order")
    inc.slot_offsets, inc.slot_incidence, inc.slot_vertex = slot_offsets, slot_inc, slot_vertex
    return inc


def build_incidence(mesh: Mesh, cells=None, *, slot_order: bool = True) -> VertexIncidence:
    torch = _torch()
    C = cells if cells is not None else _to_device(np.ascontiguousarray(mesh.cells, dtype=np.int64), torch)[0]
    n, n_b, nv = int(C.shape[0]), mesh.dim + 1, mesh.n_vertices
    L = _lib.lib()
    offsets = torch.empty((nv + 1,), dtype=torch.int64, device="cuda")
    inc = torch.empty((max(n * n_b, 1),), dtype=torch.int32, device="cuda")
    scratch = torch.empty((max(int(L.txb_incidence_scratch_bytes(n, n_b, nv)), 16),), dtype=torch.uint8,
                          device="cuda")
    _lib.check(L.txb_build_incidence(n, n_b, nv, C.data_ptr(), offsets.data_ptr(), inc.data_ptr(),
                                     scratch.data_ptr(), _stream_ptr(torch)), "txb_build_incidence")
    res = VertexIncidence(offsets, inc, nv, n)
    return build_scatter_order(res) if slot_order else res


def scatter_add_element_vectors(mesh: Mesh, layout: FieldLayout, elem_vecs, *, incidence=None):
    """Sum per-cell blocks into the global vector in ascending cell order
    (mesh.py:220-234), bit-identical to np.add.at.  numpy in -> numpy out."""
    torch = _torch()
    expected = (mesh.n_cells, mesh.dim + 1, layout.n_comp)
    if tuple(elem_vecs.shape) != expected:
        raise ShapeError(f"element vectors have shape {tuple(elem_vecs.shape)}, expected {expected}")
    host = isinstance(elem_vecs, np.ndarray)
    e, _ = _to_device(elem_vecs, torch)
    inc = incidence if incidence is not None else build_incidence(mesh)
    out = torch.empty((mesh.n_vertices * layout.n_comp,), dtype=e.dtype, device="cuda")
    if mesh.n_cells == 0:
        out.zero_()
    elif inc.slot_vertex is not None:
        _lib.check(_lib.lib().txb_scatter_add_slots(e.element_size(), mesh.n_vertices, layout.n_comp,
                                                    inc.slot_offsets.data_ptr(), inc.slot_incidence.data_ptr(),
                                                    inc.slot_vertex.data_ptr(), e.data_ptr(), out.data_ptr(),
                                                    _stream_ptr(torch)), "txb_scatter_add_slots")
    else:
        _lib.check(_lib.lib().txb_scatter_add(e.element_size(), mesh.n_vertices, layout.n_comp,
                                              inc.offsets.data_ptr(), inc.incidence.data_ptr(), e.data_ptr(),
                                              out.data_ptr(), _stream_ptr(torch)), "txb_scatter_add")
    return out.cpu().numpy() if host else out
