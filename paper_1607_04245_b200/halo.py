"""Partitioned global assembly with a halo exchange.

The reference assembles the residual with ``np.add.at`` over ALL cells in
ascending cell order (txfem/mesh.py:220-234, executor.py:266; SPEC.md:94
requires that order for bit-reproducibility).  With the cells partitioned
into contiguous ranges over P ranks (shard.cell_range), a vertex on a
partition boundary collects element-vector entries from several ranks.

Ownership and order.  Vertex v is OWNED by the lowest rank that touches it.
Because the cell ranges ascend with the rank, v's contributions in ascending
cell order are: the owner's own entries, then those of each higher rank in
rank order.  The owner therefore receives the other ranks' RAW entries (not
partial sums) and continues its chain with them in (rank, cell) order — the
reference's sequential sum, bit for bit, with ONE exchange step regardless of
how many ranks share a vertex.

Data path per rank (all on the device, nothing allocated by the library):
  buf = [ local element rows (n_local_cells * N_b) | received rows ]  (n_comp wide)
  1. integration writes the local rows            (integrate_mesh / integrate_cells)
  2. pack: gather the rows owed to lower ranks     (txb_gather_coefficients, n_b = 1)
  3. exchange: all_to_all_single(buf[recv], packed) (NCCL over NVLink; gloo on CPU)
  4. assemble: owned residual = CSR chain over [own rows, received rows]
                                                     (txb_scatter_add)
The plan (ownership, send lists, CSR) is computed once per mesh and
partition on the host from the connectivity; every rank derives the same
plan independently, so no metadata is exchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .shard import all_ranges

__all__ = ["HaloPlan", "build_halo_plan", "assemble_owned", "all_to_all_exchange"]


@dataclass
class HaloPlan:
    rank: int
    world: int
    n_b: int
    lo: int                      # owned cell range [lo, hi)
    hi: int
    n_vertices: int              # global vertex count
    owned: np.ndarray            # (n_owned,) global ids of the vertices this rank owns, ascending
    offsets: np.ndarray          # (n_owned + 1,) int64 CSR over owned vertices
    incidence: np.ndarray        # (nnz,) int32 rows of buf, (rank, cell) ascending per vertex
    send_rows: np.ndarray        # (n_send,) int64 local rows owed to lower ranks, peers ascending
    send_counts: list            # rows per peer
    recv_counts: list            # rows per peer
    _dev: dict = field(default_factory=dict, repr=False)

    @property
    def n_local_rows(self) -> int:
        return (self.hi - self.lo) * self.n_b

    @property
    def n_recv(self) -> int:
        return int(sum(self.recv_counts))

    @property
    def n_send(self) -> int:
        return int(sum(self.send_counts))

    def device_arrays(self, torch):
        """Device copies of the index arrays (uploaded once)."""
        if not self._dev:
            self._dev = {
                "offsets": torch.from_numpy(self.offsets).cuda(),
                "incidence": torch.from_numpy(np.ascontiguousarray(self.incidence)).cuda()
                if self.incidence.size else torch.zeros(1, dtype=torch.int32, device="cuda"),
                "send_rows": torch.from_numpy(self.send_rows).cuda()
                if self.send_rows.size else torch.zeros(1, dtype=torch.int64, device="cuda"),
            }
        return self._dev


def vertex_owners(cells: np.ndarray, n_vertices: int, world: int, align: int = 256) -> np.ndarray:
    """owner[v] = lowest rank whose cell range touches v (world if untouched)."""
    cells = np.asarray(cells)
    n, n_b = cells.shape
    his = np.array([hi for _, hi in all_ranges(n, world, align)], dtype=np.int64)
    inc_v = cells.ravel()
    uniq, first = np.unique(inc_v, return_index=True)  # first occurrence = lowest cell (ravel is cell-major)
    owner = np.full(n_vertices, world, dtype=np.int64)
    owner[uniq] = np.searchsorted(his, first // n_b, side="right")
    return owner


def build_halo_plan(cells: np.ndarray, n_vertices: int, rank: int, world: int, align: int = 256,
                    owner: Optional[np.ndarray] = None) -> HaloPlan:
    """The assembly plan of ``rank`` for the contiguous-range partition of
    ``cells`` (n_cells, N_b) over ``world`` ranks (boundaries on ``align``)."""
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    n, n_b = cells.shape
    ranges = all_ranges(n, world, align)
    lo, hi = ranges[rank]
    his = np.array([h for _, h in ranges], dtype=np.int64)
    if owner is None:
        owner = vertex_owners(cells, n_vertices, world, align)
    inc_v = cells.ravel()

    # every contribution to a vertex this rank owns, ordered by (vertex, cell)
    idx = np.nonzero(owner[inc_v] == rank)[0]                 # incidence positions cell*n_b + b
    idx = idx[np.argsort(inc_v[idx], kind="stable")]           # stable: cells stay ascending per vertex
    sv = inc_v[idx]
    srank = np.searchsorted(his, idx // n_b, side="right")
    owned, counts = np.unique(sv, return_counts=True)
    offsets = np.zeros(owned.size + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    rows = np.empty(idx.size, dtype=np.int64)
    mine = srank == rank
    rows[mine] = idx[mine] - lo * n_b
    recv_counts = [0] * world
    base = (hi - lo) * n_b
    for s in range(rank + 1, world):
        sel = np.nonzero(srank == s)[0]
        recv_counts[s] = int(sel.size)
        rows[sel] = base + np.arange(sel.size)
        base += sel.size
    if rows.size and rows.max() >= 2 ** 31:
        raise ValueError("halo plan rows exceed the int32 incidence range")

    # entries of this rank's cells owed to lower ranks, per peer in (vertex, cell) order
    ipos = np.arange(lo * n_b, hi * n_b, dtype=np.int64)
    ov = owner[inc_v[ipos]]
    send_rows, send_counts = [], [0] * world
    for p in range(rank):
        sel = ipos[ov == p]
        sel = sel[np.argsort(inc_v[sel], kind="stable")]
        send_rows.append(sel - lo * n_b)
        send_counts[p] = int(sel.size)
    send = np.concatenate(send_rows) if send_rows else np.zeros(0, dtype=np.int64)
    return HaloPlan(rank, world, n_b, lo, hi, n_vertices, owned, offsets, rows.astype(np.int32), send,
                    send_counts, recv_counts)


def all_to_all_exchange(group=None) -> Callable:
    """The exchange step over torch.distributed (NCCL for CUDA tensors)."""
    import torch.distributed as dist

    def exchange(recv, send, recv_splits, send_splits):
        dist.all_to_all_single(recv, send, recv_splits, send_splits, group=group)

    return exchange


def assemble_owned(plan: HaloPlan, buf, n_comp: int, exchange: Optional[Callable] = None):
    """Owned-vertex residual (n_owned, n_comp) from ``buf`` — a CUDA tensor
    (n_local_rows + n_recv, n_comp) whose first n_local_rows rows hold this
    rank's element vectors.  ``exchange(recv, send, recv_splits, send_splits)``
    moves the halo rows (all_to_all_exchange(); may be None when world == 1).
    Asynchronous on the current stream apart from the exchange's own ordering."""
    import ctypes

    import torch

    from . import _lib

    if tuple(buf.shape) != (plan.n_local_rows + plan.n_recv, n_comp):
        raise ValueError(f"buf must be ({plan.n_local_rows + plan.n_recv}, {n_comp}), got {tuple(buf.shape)}")
    dev = plan.device_arrays(torch)
    L = _lib.lib()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    s = buf.element_size()
    if plan.world > 1:
        send = torch.empty((max(plan.n_send, 1), n_comp), dtype=buf.dtype, device=buf.device)
        if plan.n_send:
            _lib.check(L.txb_gather_coefficients(s, plan.n_send, 1, n_comp, dev["send_rows"].data_ptr(),
                                                 buf.data_ptr(), send.data_ptr(), stream), "halo pack")
        if exchange is None:
            raise ValueError("world > 1 needs an exchange")
        exchange(buf[plan.n_local_rows:].reshape(-1), send[:plan.n_send].reshape(-1),
                 [c * n_comp for c in plan.recv_counts], [c * n_comp for c in plan.send_counts])
    out = torch.empty((max(plan.owned.size, 1), n_comp), dtype=buf.dtype, device=buf.device)
    if plan.owned.size:
        _lib.check(L.txb_scatter_add(s, plan.owned.size, n_comp, dev["offsets"].data_ptr(),
                                     dev["incidence"].data_ptr(), buf.data_ptr(), out.data_ptr(), stream),
                   "halo assemble")
    return out[:plan.owned.size]
