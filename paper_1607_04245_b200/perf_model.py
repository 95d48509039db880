"""The paper's closed-form traffic / flop model (§3.3, Eqs. 3-8;
txfem/perf_model.py:46-103) plus the compulsory-HBM-byte count the B200
roofline is reported against.

* ``traffic_and_flops`` — Eq. 6 bytes and Eq. 7 flops per batch.  Eq. 7 is the
  reference's reported-rate convention (cli.py:128-131): GF/s in
  bench.py is Eq.7 flops per cell x cells / time.
* ``compulsory_bytes_per_cell`` — what HBM must move at least once: read inv_j
  (d^2) + det_j (1) + coeffs (N_b N_comp) + aux (1 for P0, N_b for P1), write the
  element vector (N_b N_comp); times the scalar width.  For scalar P1 with
  N_q = 1 this equals Eq. 6 + the reference's aux bytes; for elasticity Eq. 6
  replicates geometry per component thread and over-counts.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Optional

from .schedule import ExecutionGeometry

__all__ = [
    "PerfEstimate", "shared_memory_bytes", "traffic_and_flops", "balance",
    "predict_bandwidth_bound", "occupancy_hint", "build_estimate", "flops_per_cell",
    "compulsory_bytes_per_cell",
]

DEFAULT_SHARED_MEM_CAP = 48 * 1024


@dataclass(frozen=True)
class PerfEstimate:
    geom: ExecutionGeometry
    scalar_width: int
    shared_bytes_block: int
    shared_bytes_per_cell: Fraction
    bytes_per_batch: int
    flops_per_batch: int
    balance: Fraction
    occupancy_hint: int


def shared_memory_bytes(geom: ExecutionGeometry, scalar_width: int, needs_f0: bool = True):
    """Eq. 3: per-block smem image M and M_c = M / N_bc (perf_model.py:46-65)."""
    d = geom.dim
    g = d + 1 if needs_f0 else d
    entries = ((d * d + 1) * geom.n_t + g * geom.n_bt * geom.n_q + geom.n_t * geom.n_bt
               + g * geom.n_t * geom.n_sqc)
    m = scalar_width * entries
    return m, Fraction(m, geom.n_bc)


def flops_per_cell(geom: ExecutionGeometry) -> int:
    """Eq. 7 per cell: interpolation + f1 scaling + basis-phase reduction."""
    d = geom.dim
    return ((2 + (2 + 2 * d) * d) * geom.n_bt * geom.n_q + 2 * d * geom.n_comp * geom.n_q
            + (2 + 2 * d) * d * geom.n_q * geom.n_bt)


def traffic_and_flops(geom: ExecutionGeometry, scalar_width: int) -> tuple[int, int]:
    """Eq. 6 bytes and Eq. 7 flops per batch (perf_model.py:68-85)."""
    d = geom.dim
    bytes_per_batch = scalar_width * geom.n_t * ((d * d + 1) + geom.n_bt + (d + 1) * geom.n_q)
    return bytes_per_batch, flops_per_cell(geom) * geom.n_bs * geom.n_bl


def balance(geom: ExecutionGeometry) -> Fraction:
    """beta at 4-byte scalars, flop/byte (perf_model.py:88-91); 41/22 for 2D Poisson."""
    b, f = traffic_and_flops(geom, 4)
    return Fraction(f, b)


def predict_bandwidth_bound(beta, achievable_bw_gbs: float) -> float:
    if beta <= 0 or achievable_bw_gbs < 0:
        raise ValueError("balance must be positive and bandwidth non-negative")
    return float(beta) * achievable_bw_gbs


def occupancy_hint(shared_bytes_block: int, cap: int = DEFAULT_SHARED_MEM_CAP) -> int:
    return cap // shared_bytes_block


def build_estimate(geom: ExecutionGeometry, scalar_width: int = 4, needs_f0: bool = False,
                   cap: int = DEFAULT_SHARED_MEM_CAP) -> PerfEstimate:
    m, m_c = shared_memory_bytes(geom, scalar_width, needs_f0)
    b, f = traffic_and_flops(geom, scalar_width)
    return PerfEstimate(geom, scalar_width, m, m_c, b, f, Fraction(f, b), occupancy_hint(m, cap))


def compulsory_bytes_per_cell(dim: int, n_comp: int, scalar_width: int,
                              aux_space: Optional[str] = None, n_aux: int = 1) -> int:
    """Minimum HBM bytes per cell of one integration pass (see module doc);
    ``n_aux`` auxiliary fields per point (run-time compiled forms)."""
    n_b = dim + 1
    aux = 0 if aux_space is None else (n_aux if aux_space == "p0" else n_b * n_aux)
    return scalar_width * (dim * dim + 1 + n_b * n_comp + aux + n_b * n_comp)
