"""Synthetic workloads of BASELINE.json's configs, generated on the device.

Conventions follow the reference CLI and tests (cli.py:71-117,
tests/conftest.py:18-34): a Kuhn mesh with the smallest refinement holding
``n_cells`` cells, sliced to exactly ``n_cells`` (cells are independent);
N(0,1) per-vertex coefficients from ``default_rng(seed)``; P0 kappa ~
U[0.5, 1.5) from ``default_rng(seed + 1)`` drawn for the full mesh.  Geometry
and the coefficient gather run on the GPU (csrc/txb_mesh.cu); the inputs are
bit-identical to the reference's (pinned by tests/golden/big_hashes.json).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .element import QuadratureRule, Tabulation, quadrature_rule, tabulate, two_point_rule
from .mesh import CellGeometry, FieldLayout, Mesh, compute_geometry, gather_coefficients, \
    generate_unit_simplex_mesh
from .physics import CellAux, PhysicsForm, elasticity_form, poisson_form, poisson_varcoef_form

__all__ = ["PHYSICS", "Workload", "refine_for", "make_workload", "kuhn_vertices", "kuhn_cells",
           "uniform_slice"]

# physics name -> (form factory, aux space)
PHYSICS = {
    "poisson": (poisson_form, None),
    "varcoef_p0": (poisson_varcoef_form, "p0"),
    "varcoef_p1": (poisson_varcoef_form, "p1"),
    "elasticity": (elasticity_form, None),
}


def refine_for(dim: int, n_cells: int) -> int:
    r = 1
    while (2 * r * r if dim == 2 else 6 * r ** 3) < n_cells:
        r += 1
    return r


def kuhn_vertices(dim: int, n: int) -> np.ndarray:
    """Vertex coordinates of generate_unit_simplex_mesh(dim, n) (mesh.py), which
    are cheap: (n+1)^dim rows against ~dim! n^dim cells."""
    ticks = np.linspace(0.0, 1.0, n + 1)
    m = n + 1
    if dim == 2:
        iy, ix = np.divmod(np.arange(m * m), m)
        return np.column_stack([ticks[ix], ticks[iy]])
    idx = np.arange(m ** 3)
    return np.column_stack([ticks[idx % m], ticks[(idx // m) % m], ticks[idx // (m * m)]])


def kuhn_cells(dim: int, n: int, lo: int, hi: int) -> np.ndarray:
    """Rows [lo, hi) of generate_unit_simplex_mesh(dim, n).cells without
    building the other rows: one rank's contiguous cell range (shard.cell_range)
    of an N-GPU job costs O(hi - lo) host memory, not O(N x cells)."""
    from .mesh import _CUBE_PERMS

    m = n + 1
    per = 2 if dim == 2 else 6
    c = np.arange(lo, hi, dtype=np.int64)
    sq, t = np.divmod(c, per)
    if dim == 2:
        sy, sx = np.divmod(sq, n)
        v00 = sy * m + sx
        v10, v01 = v00 + 1, v00 + m
        v11 = v01 + 1
        return np.ascontiguousarray(np.where((t == 0)[:, None], np.stack([v00, v10, v11], 1),
                                             np.stack([v00, v11, v01], 1)))
    corner = np.column_stack([sq // (n * n), (sq // n) % n, sq % n])
    out = np.empty((hi - lo, 4), dtype=np.int64)
    eye = np.eye(3, dtype=np.int64)
    for k_t, (perm, parity) in enumerate(_CUBE_PERMS):
        sel = t == k_t
        cn = corner[sel]
        p1 = cn + eye[perm[0]]
        p2 = p1 + eye[perm[1]]
        p3 = p2 + eye[perm[2]]
        path = (cn, p1, p2, p3) if parity > 0 else (cn, p1, p3, p2)
        for k, pt in enumerate(path):
            out[sel, k] = (pt[:, 2] * m + pt[:, 1]) * m + pt[:, 0]
    return out


def uniform_slice(seed: int, lo: int, hi: int, low: float = 0.5, high: float = 1.5) -> np.ndarray:
    """default_rng(seed).uniform(low, high, (N, 1))[lo:hi] without drawing the
    first lo values: PCG64 jumps ahead lo outputs (one 64-bit draw per double)."""
    bg = np.random.PCG64(seed)
    bg.advance(lo)
    return np.random.Generator(bg).uniform(low, high, (hi - lo, 1))


@dataclass
class Workload:
    dim: int
    physics: str
    n_cells: int
    form: PhysicsForm
    rule: QuadratureRule
    tab: Tabulation
    mesh: Mesh  # full Kuhn mesh (before slicing)
    cell_geom: CellGeometry  # float64 CUDA tensors
    coeffs: object  # (n, n_b, n_comp) float64 CUDA tensor
    aux: Optional[CellAux]  # float64 CUDA tensor values

    def cast(self, dtype: str):
        """(inv_j, det_j, coeffs, aux) cast once to the run precision (executor.py:77-90)."""
        import torch

        tdt = torch.float32 if dtype == "f32" else torch.float64
        c = lambda t: t.to(tdt).contiguous()  # noqa: E731
        aux = None if self.aux is None else CellAux(self.aux.space, c(self.aux.values))
        return c(self.cell_geom.inv_jacobians), c(self.cell_geom.determinants), c(self.coeffs), aux


def make_workload(dim: int, physics: str, n_cells: int, seed: int = 1234, n_q: int = 1) -> Workload:
    import torch

    factory, aux_space = PHYSICS[physics]
    form = factory(dim)
    rule = quadrature_rule(dim, 1) if n_q == 1 else two_point_rule(dim)
    tab = tabulate(dim, rule)
    full = generate_unit_simplex_mesh(dim, refine_for(dim, n_cells))
    cells = torch.from_numpy(np.ascontiguousarray(full.cells[:n_cells])).to("cuda")
    sliced = Mesh(dim, full.vertices, full.cells[:n_cells])
    geom = compute_geometry(sliced, cells=cells, device_out=True)
    layout = FieldLayout(form.n_comp)
    glob = np.random.default_rng(seed).standard_normal(layout.global_size(full))
    coeffs = gather_coefficients(sliced, layout, torch.from_numpy(glob).to("cuda"), cells=cells)
    aux = None
    if aux_space == "p0":
        vals = np.random.default_rng(seed + 1).uniform(0.5, 1.5, (full.n_cells, 1))[:n_cells]
        aux = CellAux("p0", torch.from_numpy(np.ascontiguousarray(vals)).to("cuda"))
    elif aux_space == "p1":
        nodal = np.random.default_rng(seed + 2).uniform(0.5, 1.5, (full.n_vertices, 1))
        aux = CellAux("p1", torch.from_numpy(np.ascontiguousarray(nodal[full.cells[:n_cells]])).to("cuda"))
    return Workload(dim, physics, n_cells, form, rule, tab, full, geom, coeffs, aux)
