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
     The owned vertices are listed in SLOT order (first own element row
     ascending), so the assembly reads the element rows in memory order;
     the ids come back with the residual.
The plan (ownership, send lists, CSR) is computed once per mesh and
partition on the host from the connectivity; every rank derives the same
plan independently, so no metadata is exchanged.

Peer-memory variant (``PeerHalo``, csrc/txb_halo.cu): steps 2-4 without NCCL
— ``txb_halo_put`` stores the owed rows straight into the owner's window (a
device buffer shared by CUDA IPC handle; P2P stores over NVLink) and raises
an epoch flag there; ``txb_halo_assemble`` waits on the flags and runs the same
CSR chain over [local rows | window rows].  Same plan, same bits.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .shard import all_ranges

__all__ = ["HaloPlan", "build_halo_plan", "assemble_owned", "all_to_all_exchange", "PeerHalo",
           "local_peer_group", "distributed_peer_halo", "peer_send_layout"]


@dataclass
class HaloPlan:
    rank: int
    world: int
    n_b: int
    lo: int                      # owned cell range [lo, hi)
    hi: int
    n_vertices: int              # global vertex count
    owned: np.ndarray            # (n_owned,) global ids of the vertices this rank owns, in slot order
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
    # Slot order: visit the owned vertices by their first row (always one of
    # this rank's own element rows, in cell order) so that neighbouring
    # assembly threads read neighbouring element rows (mesh.build_scatter_order;
    # the reference's 3D unit mesh numbers vertices and cells in different
    # orders).  Each chain is moved whole, so the sums do not change.
    if owned.size:
        perm = np.argsort(rows[offsets[:-1]], kind="stable")
        owned, counts = owned[perm], counts[perm]
        new_offsets = np.zeros_like(offsets)
        np.cumsum(counts, out=new_offsets[1:])
        src = np.repeat(offsets[:-1][perm] - new_offsets[:-1], counts) + np.arange(rows.size, dtype=np.int64)
        rows, offsets = rows[src], new_offsets

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


# ---------------------------------------------------------------------------
# Peer-memory exchange (txb_halo_put / txb_halo_assemble): the same plan, the
# same chain, without NCCL — each rank stores its owed rows straight into the
# owner's window (P2P over NVLink within a node) and the owner's assembly
# kernel waits on per-sender epoch flags.
# ---------------------------------------------------------------------------

def slot_bytes(n_recv: int, n_comp: int, dtype_bytes: int) -> int:
    """Bytes of one receive slot (txb_halo_window_bytes = 2048 + 2 slots)."""
    return (max(n_recv, 1) * n_comp * dtype_bytes + 255) // 256 * 256


def peer_send_layout(plan: HaloPlan, recv_counts_of: list):
    """Where this rank's owed rows land: for each send row, the destination
    rank and its row in that rank's receive slot.  ``recv_counts_of[p]`` is
    rank p's plan.recv_counts; rank p's slot holds the rows of senders
    s = p+1.. in ascending order, each sender's rows in (vertex, cell) order —
    the order p's CSR expects (build_halo_plan)."""
    r = plan.rank
    peers, dsts = [], []
    o = 0
    for p in range(plan.world):
        c = plan.send_counts[p]
        if not c:
            continue
        base = int(sum(recv_counts_of[p][:r]))
        if recv_counts_of[p][r] != c:
            raise ValueError(f"rank {r} owes {c} rows to rank {p}, which expects {recv_counts_of[p][r]}")
        peers.append(np.full(c, p, dtype=np.int32))
        dsts.append(base + np.arange(c, dtype=np.int64))
        o += c
    send_peer = np.concatenate(peers) if peers else np.zeros(0, dtype=np.int32)
    send_dst = np.concatenate(dsts) if dsts else np.zeros(0, dtype=np.int64)
    out_peers = np.array([p for p in range(plan.world) if plan.send_counts[p]], dtype=np.int32)
    in_peers = np.array([s for s in range(plan.world) if plan.recv_counts[s]], dtype=np.int32)
    return send_peer, send_dst, out_peers, in_peers


class PeerHalo:
    """One rank's peer-memory halo exchange.  Build with ``local_peer_group``
    (all ranks in this process: tests, single-GPU emulation) or
    ``distributed_peer_halo`` (one process per GPU, windows shared by CUDA
    IPC handle).  ``exchange_assemble(rows)`` is one residual evaluation."""

    def __init__(self, plan: HaloPlan, n_comp: int, dtype_bytes: int, windows: list, recv_counts_of: list,
                 on_close=None):
        import torch

        self.plan, self.n_comp, self.dtype_bytes = plan, n_comp, dtype_bytes
        self.epoch = 0
        self.window = windows[plan.rank]
        self._on_close = on_close
        send_peer, send_dst, out_peers, in_peers = peer_send_layout(plan, recv_counts_of)
        dev = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt) if len(a) else  # noqa: E731
                                             np.zeros(1, dtype=dt)).cuda()
        self._d = {
            "send_rows": dev(plan.send_rows, np.int64), "send_peer": dev(send_peer, np.int32),
            "send_dst": dev(send_dst, np.int64), "out_peers": dev(out_peers, np.int32),
            "in_peers": dev(in_peers, np.int32),
            "windows": dev(np.array(windows, dtype=np.uint64).view(np.int64), np.int64),  # device void*[world]
            "slot_bytes": dev(np.array([slot_bytes(sum(rc), n_comp, dtype_bytes) for rc in recv_counts_of],
                                       dtype=np.int64), np.int64),
        }
        self.n_out, self.n_in = int(out_peers.size), int(in_peers.size)
        self.my_slot = slot_bytes(plan.n_recv, n_comp, dtype_bytes)

    def _check_rows(self, rows):
        plan, nc, s = self.plan, self.n_comp, self.dtype_bytes
        if tuple(rows.shape) != (plan.n_local_rows, nc) or rows.element_size() != s or not rows.is_contiguous():
            raise ValueError(f"rows must be a contiguous ({plan.n_local_rows}, {nc}) tensor of {s}-byte scalars")

    def exchange_assemble(self, rows):
        """rows: CUDA tensor (n_local_rows, n_comp) — this rank's element rows.
        Put (txb_halo_put) then assemble.  Returns the owned-vertex residual
        (n_owned, n_comp).  Asynchronous."""
        import ctypes

        import torch

        from . import _lib

        plan, nc, s = self.plan, self.n_comp, self.dtype_bytes
        self._check_rows(rows)
        self.epoch += 1
        d = self._d
        L = _lib.lib()
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        _lib.check(L.txb_halo_put(s, nc, plan.rank, plan.world, plan.n_send, ptr(d["send_rows"]), ptr(d["send_peer"]),
                                  ptr(d["send_dst"]), ptr(rows), ptr(d["windows"]), ptr(d["slot_bytes"]),
                                  ptr(d["out_peers"]), self.n_out, self.epoch, stream), "txb_halo_put")
        return self.assemble(rows)

    def assemble(self, rows):
        """The assembly half of the current epoch (its put already issued by
        exchange_assemble).  Returns the owned-vertex residual (n_owned, n_comp)."""
        import ctypes

        import torch

        from . import _lib

        plan, nc, s = self.plan, self.n_comp, self.dtype_bytes
        self._check_rows(rows)
        d = self._d
        dc = plan.device_arrays(torch)
        L = _lib.lib()
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        ptr = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        out = torch.empty((max(plan.owned.size, 1), nc), dtype=rows.dtype, device=rows.device)
        _lib.check(L.txb_halo_assemble(s, nc, plan.rank, plan.world, plan.owned.size, ptr(dc["offsets"]),
                                       ptr(dc["incidence"]), plan.n_local_rows, ptr(rows), ptr(d["windows"]),
                                       self.my_slot, ptr(d["in_peers"]), self.n_in, self.epoch, ptr(out), stream),
                   "txb_halo_assemble")
        return out[:plan.owned.size]

    def check(self) -> None:
        """Raise if a put or an assembly of this rank failed (host sync).  The
        error is sticky: once failed, the window never acks again."""
        import ctypes

        from . import _lib
        from .errors import CudaLaneError

        e = ctypes.c_int(0)
        _lib.check(_lib.lib().txb_halo_window_error(ctypes.c_void_p(self.window), ctypes.byref(e)))
        if e.value:
            what = {1: "timed out waiting for a peer's ack (its put skipped the stores and poisoned its flag)",
                    2: "timed out waiting for a peer's rows", 3: "a peer's put failed (poisoned flag)"}
            raise CudaLaneError(f"halo exchange on rank {self.plan.rank}: {what.get(e.value, e.value)}; the owned "
                                f"residual of the failed epoch is NaN (TXB_HALO_TIMEOUT_MS)")

    def close(self) -> None:
        if self._on_close is not None:
            self._on_close()
            self._on_close = None


def _alloc_window(n_recv: int, n_comp: int, dtype_bytes: int, ipc: bool):
    import ctypes

    from . import _lib

    L = _lib.lib()
    w = ctypes.c_void_p()
    handle = ctypes.create_string_buffer(64) if ipc else None
    _lib.check(L.txb_halo_window_alloc(L.txb_halo_window_bytes(n_recv, n_comp, dtype_bytes), ctypes.byref(w),
                                       handle), "txb_halo_window_alloc")
    return w.value, (handle.raw if ipc else None)


def local_peer_group(plans: list, n_comp: int, dtype_bytes: int) -> list:
    """PeerHalo objects for ALL ranks in this process (one device): tests and
    single-GPU emulation.  Launch every rank's exchange in rank-independent
    order on one stream: puts only wait for acks of two epochs back."""
    from . import _lib

    windows = [_alloc_window(p.n_recv, n_comp, dtype_bytes, False)[0] for p in plans]
    recv_counts_of = [p.recv_counts for p in plans]

    def free():
        for w in windows:
            _lib.lib().txb_halo_window_free(w)

    group = [PeerHalo(p, n_comp, dtype_bytes, windows, recv_counts_of) for p in plans]
    group[0]._on_close = free
    return group


def distributed_peer_halo(plan: HaloPlan, n_comp: int, dtype_bytes: int, group=None) -> PeerHalo:
    """One process per GPU of one node: allocate this rank's window, share it by
    CUDA IPC handle (torch.distributed all_gather_object, once), open the
    peers' windows (P2P over NVLink)."""
    import ctypes

    import torch.distributed as dist

    from . import _lib

    own, handle = _alloc_window(plan.n_recv, n_comp, dtype_bytes, True)
    infos = [None] * plan.world
    dist.all_gather_object(infos, (handle, list(plan.recv_counts)), group=group)
    L = _lib.lib()
    windows, opened = [], []
    for r, (h, _) in enumerate(infos):
        if r == plan.rank:
            windows.append(own)
            continue
        w = ctypes.c_void_p()
        _lib.check(L.txb_halo_window_open(ctypes.create_string_buffer(h, 64), ctypes.byref(w)), "txb_halo_window_open")
        windows.append(w.value)
        opened.append(w.value)

    def close():
        for w in opened:
            L.txb_halo_window_close(w)
        L.txb_halo_window_free(own)

    return PeerHalo(plan, n_comp, dtype_bytes, windows, [rc for _, rc in infos], on_close=close)
