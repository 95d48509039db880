"""Model-synthesised execution counters returned alongside results, as the
reference's fast lanes do (txfem/device.py:66-227, executor.py:153-157).

The CUDA lane does not count operations on the device; ncu's
dram__bytes_read/write is the measured counterpart (profiles/).  The
per-batch tallies below are the paper's closed-form model so that a caller
reading ``trace.totals()`` or ``write_csv`` sees the reference's numbers.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass, field, replace
from typing import IO, Optional

from .physics import CellAux, PhysicsForm
from .schedule import ExecutionGeometry

__all__ = ["BatchCounters", "ChunkTrace", "ExecutionTrace", "shared_image_entries",
           "shared_image_bytes", "batch_loaded_bytes", "aux_loaded_bytes", "model_batch_counters"]


@dataclass
class BatchCounters:
    flops_interp: int = 0
    flops_scale_f1: int = 0
    flops_scale_f0: int = 0
    flops_reduce_f1: int = 0
    flops_reduce_f0: int = 0
    flops_form: int = 0
    flops_aux: int = 0
    flops_redundant: int = 0
    bytes_loaded: int = 0
    bytes_aux: int = 0
    barriers: int = 0

    @property
    def model_flops(self) -> int:
        return self.flops_interp + self.flops_scale_f1 + self.flops_reduce_f1

    @property
    def total_flops(self) -> int:
        return (self.model_flops + self.flops_scale_f0 + self.flops_reduce_f0 + self.flops_form
                + self.flops_aux + self.flops_redundant)


@dataclass
class ChunkTrace:
    chunk_index: int
    batches: list = field(default_factory=list)
    task_log: Optional[list] = None

    @property
    def barrier_count(self) -> int:
        return sum(b.barriers for b in self.batches)


class ExecutionTrace:
    """Per-chunk counters of one integrate_transposed call (device.py:96-144).

    The CUDA lane's counters are the closed-form model, identical for every
    full batch, so a trace built with ``uniform`` stores one template and
    materialises ``chunks`` (n_chunks x n_cb BatchCounters) only when read;
    ``totals`` is closed-form.  (A 1 M-cell mesh has ~8,000 batches: building
    them eagerly cost more host time than the GPU work of the call.)"""

    def __init__(self, geom: ExecutionGeometry, scalar_width: int, chunks: Optional[list] = None,
                 remainder_cells: int = 0):
        self.geom = geom
        self.scalar_width = scalar_width
        self.remainder_cells = remainder_cells
        self._chunks = list(chunks) if chunks is not None else []
        self._uniform: Optional[BatchCounters] = None
        self._n_chunks = 0

    @classmethod
    def uniform(cls, geom: ExecutionGeometry, scalar_width: int, per_batch: BatchCounters,
                remainder_cells: int = 0) -> "ExecutionTrace":
        t = cls(geom, scalar_width, remainder_cells=remainder_cells)
        t._uniform, t._n_chunks = per_batch, geom.n_chunks
        t._chunks = None
        return t

    @property
    def chunks(self) -> list:
        if self._chunks is None:
            pb, n_cb = self._uniform, self.geom.n_cb
            self._chunks = [ChunkTrace(chunk_index=ci, batches=[replace(pb) for _ in range(n_cb)])
                            for ci in range(self._n_chunks)]
        return self._chunks

    def totals(self) -> BatchCounters:
        agg = BatchCounters()
        if self._chunks is None:  # closed form: every batch carries the template
            n = self._n_chunks * self.geom.n_cb
            for name in vars(agg):
                setattr(agg, name, n * getattr(self._uniform, name))
            return agg
        for chunk in self._chunks:
            for b in chunk.batches:
                for name in vars(agg):
                    setattr(agg, name, getattr(agg, name) + getattr(b, name))
        return agg

    def write_csv(self, stream: IO[str]) -> None:
        w = csv.writer(stream)
        w.writerow(["chunk", "batch", "flops", "bytes_loaded", "barriers"])
        for chunk in self.chunks:
            for i, b in enumerate(chunk.batches):
                w.writerow([chunk.chunk_index, i, b.model_flops, b.bytes_loaded, b.barriers])


def shared_image_entries(geom: ExecutionGeometry, needs_f0: bool) -> dict:
    """Reference smem image by area (device.py:147-161)."""
    d = geom.dim
    g = d + 1 if needs_f0 else d
    return {"tabulation": g * geom.n_bt * geom.n_q, "geometry": (d * d + 1) * geom.n_t,
            "coefficients": geom.n_t * geom.n_bt, "f_values": g * geom.n_t * geom.n_sqc}


def shared_image_bytes(geom: ExecutionGeometry, scalar_width: int, needs_f0: bool) -> int:
    return scalar_width * sum(shared_image_entries(geom, needs_f0).values())


def batch_loaded_bytes(geom: ExecutionGeometry, scalar_width: int) -> int:
    """Eq. 6 at the reference's layout granularity (device.py:168-180)."""
    d = geom.dim
    return scalar_width * ((d * d + 1) * geom.n_t + geom.n_t * geom.n_bt + (d + 1) * geom.n_t * geom.n_sqc)


def aux_loaded_bytes(geom: ExecutionGeometry, scalar_width: int, aux: Optional[CellAux]) -> int:
    if aux is None:
        return 0
    per_cell = aux.n_aux if aux.space == "p0" else aux.n_aux * geom.n_b
    return scalar_width * per_cell * geom.n_bc


def model_batch_counters(geom: ExecutionGeometry, form: PhysicsForm, scalar_width: int,
                         aux: Optional[CellAux] = None) -> BatchCounters:
    """Closed-form tallies for one full batch (device.py:188-227)."""
    d = geom.dim
    n_bc, n_q, n_bt, n_comp, n_b = geom.n_bc, geom.n_q, geom.n_bt, geom.n_comp, geom.n_b
    interp = n_bc * n_q * n_bt * (2 + (2 + 2 * d) * d)
    aux_flops = 0
    if aux is not None and aux.space == "p1":
        aux_flops = n_bc * n_q * 2 * n_b * aux.n_aux
        if form.uses_grad_a:
            aux_flops += n_bc * n_q * 2 * n_b * aux.n_aux * d
    return BatchCounters(
        flops_interp=interp,
        flops_scale_f1=n_bc * n_q * n_comp * 2 * d,
        flops_scale_f0=n_bc * n_q * n_comp * 2 if form.has_f0 else 0,
        flops_reduce_f1=n_bc * n_bt * n_q * (2 + 2 * d) * d,
        flops_reduce_f0=n_bc * n_bt * n_q * 2 if form.has_f0 else 0,
        flops_form=n_bc * n_q * n_comp * (form.flops_f1 + (form.flops_f0 if form.has_f0 else 0)),
        flops_aux=aux_flops,
        flops_redundant=(n_comp - 1) * (interp + aux_flops),
        bytes_loaded=batch_loaded_bytes(geom, scalar_width),
        bytes_aux=aux_loaded_bytes(geom, scalar_width, aux),
        barriers=1,
    )
