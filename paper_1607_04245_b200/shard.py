"""Contiguous cell-range partitioning across GPUs.

Cells are independent (txfem/_kernels_cy.pyx:69-123), so rank r of P owns the
contiguous range [lo, hi) of the global cell array, with range boundaries on
multiples of ``align`` cells so every rank's slices keep the 16-byte bulk-copy
alignment of the batch loader.  No collective touches the data path.
"""

from __future__ import annotations

__all__ = ["cell_range", "all_ranges"]


def cell_range(n_cells: int, rank: int, world: int, align: int = 64) -> tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if n_cells < 0 or align < 1:
        raise ValueError("n_cells must be >= 0 and align >= 1")
    units = -(-n_cells // align)  # ceil
    lo_u = units * rank // world
    hi_u = units * (rank + 1) // world
    return min(lo_u * align, n_cells), min(hi_u * align, n_cells)


def all_ranges(n_cells: int, world: int, align: int = 64):
    return [cell_range(n_cells, r, world, align) for r in range(world)]
