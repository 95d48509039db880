#!/usr/bin/env python
"""Benchmark of the thread-transposed element-integration kernel on B200.

Contract (one JSON line from rank 0):
  metric   BASELINE.json's: element-integration GF/s (paper Eq. 7 flops), with
           HBM GB/s and the roofline fraction in ``roofline``.
  step     one integration pass over the workload's cells (one kernel launch).
  workload 3D P1 tetrahedra, variable-coefficient Laplacian (P0 kappa), f64,
           2^20 cells per GPU (BASELINE.json configs[1]); N GPUs own contiguous
           cell ranges of an N*2^20-cell Kuhn mesh (weak scaling, no collective
           on the data path).
  value    whole-job GF/s, inputs resident in HBM; 4+ rotating buffer sets so
           every step's inputs are out of L2 (set bytes x (sets-1) > 126 MB L2).
  e2e      the same metric through the reference-facing call with HOST numpy
           buffers (pinned): H2D + kernel + D2H inside the timed region.
  --impl reference   the reference's own CPU lane (oracle/_ref/_kernels_cy,
           built from /root/reference; else the C oracle port) on all host
           cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

L2_BYTES = 126 * 1024 * 1024
FALLBACK_HBM_GBS = 6650.0
METRIC = "element-integration GF/s (paper Eq.7 flops)"

CONFIGS = {
    # name: (dim, physics, dtype, cells per GPU)
    "3d_varcoef_f64": (3, "varcoef_p0", "f64", 1 << 20),
    "3d_varcoef_f32": (3, "varcoef_p0", "f32", 1 << 20),
    "2d_varcoef_f64": (2, "varcoef_p0", "f64", 1 << 20),
    "2d_varcoef_f32": (2, "varcoef_p0", "f32", 1 << 20),
    "2d_varcoef_f64_65536": (2, "varcoef_p0", "f64", 65536),
    "2d_elasticity_f64": (2, "elasticity", "f64", 1 << 20),
    "2d_elasticity_f32": (2, "elasticity", "f32", 1 << 20),
    "3d_elasticity_f64": (3, "elasticity", "f64", 1 << 20),
    "3d_elasticity_f32": (3, "elasticity", "f32", 1 << 20),
    "3d_varcoef_f32_2^24": (3, "varcoef_p0", "f32", 1 << 24),
    "3d_varcoef_f64_2^24": (3, "varcoef_p0", "f64", 1 << 24),
}
HEADLINE = "3d_varcoef_f64"
VARIANTS = ["3d_varcoef_f32", "2d_varcoef_f64", "2d_varcoef_f32", "2d_elasticity_f64", "2d_elasticity_f32",
            "3d_elasticity_f64", "3d_elasticity_f32", "2d_varcoef_f64_65536"]


def nccl_debug_env():
    """Communicator-init lines of NCCL (ranks, devices, NVLS / P2P transport) for
    the N > 1 runs, on STDERR: NCCL logs to stdout unless told otherwise, and
    stdout is the one JSON line.  A caller's own NCCL_DEBUG setting wins."""
    if "NCCL_DEBUG" not in os.environ:
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def config_model(name):
    from paper_1607_04245_b200.perf_model import compulsory_bytes_per_cell, flops_per_cell
    from paper_1607_04245_b200.schedule import derive_execution_geometry

    dim, physics, dtype, n = CONFIGS[name]
    n_comp = dim if physics == "elasticity" else 1
    width = 4 if dtype == "f32" else 8
    aux = "p0" if physics == "varcoef_p0" else None
    g = derive_execution_geometry(dim, dim + 1, n_comp, 1, 1, 1, n)
    return flops_per_cell(g), compulsory_bytes_per_cell(dim, n_comp, width, aux)


# ----------------------------------------------------------------------------
# clocks during the timed region (NVML, polled from a thread)
# ----------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._stop = threading.Event()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()
        if self.in_timed is None:
            self.in_timed = len(self.samples)

    in_timed = None  # samples taken inside the timed region (the first window)

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples),
                "samples_in_timed_region": self.in_timed,
                "window": "the timed region, then replays of the same timed graph (untimed) until "
                          ">= 0.25 s of load was sampled"}


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def rank_plan(name, rank, world):
    """(lo, hi, refinement) of rank r's contiguous cell range of the
    world x cells-per-GPU job (shard.cell_range, 256-cell aligned)."""
    from paper_1607_04245_b200.shard import cell_range
    from paper_1607_04245_b200.workload import refine_for

    dim, _, _, per_gpu = CONFIGS[name]
    total = per_gpu * world
    lo, hi = cell_range(total, rank, world, align=256)
    return lo, hi, refine_for(dim, total)


def rank_host_inputs(name, rank, world, seed=1234):
    """Host side of rank r's workload: its cells of the Kuhn mesh holding
    world x per-GPU cells (only rows [lo, hi) are generated), the mesh's vertex
    coordinates, the global N(0,1) coefficient vector and the rank's slice of
    the P0 kappa field (PCG64 jumped ahead to lo).  Identical to slicing the
    full single-process workload (tests/test_distributed.py)."""
    from paper_1607_04245_b200.workload import PHYSICS, kuhn_cells, kuhn_vertices, uniform_slice

    dim, physics, _, _ = CONFIGS[name]
    lo, hi, r = rank_plan(name, rank, world)
    factory, aux_space = PHYSICS[physics]
    form = factory(dim)
    verts = kuhn_vertices(dim, r)
    cells = kuhn_cells(dim, r, lo, hi)
    glob = np.random.default_rng(seed).standard_normal(verts.shape[0] * form.n_comp)
    kappa = uniform_slice(seed + 1, lo, hi) if aux_space == "p0" else None
    return dict(form=form, lo=lo, hi=hi, vertices=verts, cells=cells, glob=glob, kappa=kappa)


def rank_workload(name, rank, world, seed=1234):
    """Rank r's contiguous cell range of the N x cells-per-GPU Kuhn mesh: host
    generation of its rows only, geometry and gather on its GPU."""
    import torch

    from paper_1607_04245_b200.element import quadrature_rule, tabulate
    from paper_1607_04245_b200.mesh import FieldLayout, Mesh, compute_geometry, gather_coefficients
    from paper_1607_04245_b200.physics import CellAux

    dim, physics, dtype, per_gpu = CONFIGS[name]
    h = rank_host_inputs(name, rank, world, seed)
    form = h["form"]
    rule = quadrature_rule(dim, 1)
    tab = tabulate(dim, rule)
    cells = torch.from_numpy(h["cells"]).to("cuda")
    sliced = Mesh(dim, h["vertices"], h["cells"])
    geom = compute_geometry(sliced, cells=cells, device_out=True)
    layout = FieldLayout(form.n_comp)
    coeffs = gather_coefficients(sliced, layout, torch.from_numpy(h["glob"]).to("cuda"), cells=cells)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    aux = None
    if h["kappa"] is not None:
        aux = CellAux("p0", torch.from_numpy(np.ascontiguousarray(h["kappa"])).to("cuda", tdt))
    c = lambda t: t.to(tdt).contiguous()  # noqa: E731
    return dict(form=form, rule=rule, tab=tab, inv=c(geom.inv_jacobians), det=c(geom.determinants),
                coeffs=c(coeffs), aux=aux, n=h["hi"] - h["lo"], dtype=dtype, dim=dim)


def time_device(wl, steps, warmup, n_sets, barrier=None, sampler=None, jit=False):
    """Device-resident timing: K launches rotating over n_sets buffer sets,
    captured in one CUDA graph (so host launch overhead is not timed), bracketed
    by CUDA events on the launching stream.  Falls back to eager launches if
    capture is unavailable.  Returns (total_ms for the K steps, mode)."""
    import torch

    from paper_1607_04245_b200 import backend
    from paper_1607_04245_b200.physics import CellAux

    width = 4 if wl["dtype"] == "f32" else 8
    kernel = (backend.jit_kernel if jit else backend.cuda_kernel)(wl["form"], wl["rule"].n_q, wl["aux"], width)
    sets = []
    for _ in range(n_sets):
        aux = None if wl["aux"] is None else CellAux(wl["aux"].space, wl["aux"].values.clone())
        sets.append((wl["inv"].clone(), wl["det"].clone(), wl["coeffs"].clone(), aux,
                     torch.empty_like(wl["coeffs"])))
    tab, rule = wl["tab"], wl["rule"]
    npdt = np.float32 if wl["dtype"] == "f32" else np.float64
    B, D, W = (np.ascontiguousarray(x, dtype=npdt) for x in (tab.basis, tab.basis_der, rule.weights))

    def launch(i):
        inv, det, co, aux, out = sets[i % n_sets]
        backend.run_cuda(kernel, B, D, W, inv, det, co, aux, out)

    # warm-up writes EVERY set's output at least once (the determinism check
    # below compares all of them, whatever K and W are)
    for i in range(warmup_launches(warmup, n_sets)):
        launch(i)
    torch.cuda.synchronize()
    graph, mode = None, "graph"
    try:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, capture_error_mode="relaxed"):
            for i in range(steps):
                launch(warmup + i)
        graph.replay()  # untimed warm replay
        torch.cuda.synchronize()
    except Exception:  # pragma: no cover - capture unsupported
        graph, mode = None, "eager"
        torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if barrier:
        barrier()
    torch.cuda.synchronize()
    with (sampler if sampler else _null()):
        t0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(steps):
                launch(warmup + i)
        t1.record(stream)
        torch.cuda.synchronize()
    if sampler is not None and graph is not None:
        # a short timed region (small K) leaves few NVML samples: keep the same load
        # running (replays of the timed graph, untimed) while sampling for >= 0.25 s
        with sampler:
            t_end = time.perf_counter() + 0.25
            while time.perf_counter() < t_end:
                graph.replay()
                torch.cuda.synchronize()
    if barrier:
        barrier()
    total = t0.elapsed_time(t1)
    # every set holds identical inputs, so identical outputs: a cheap race/determinism check
    for k in range(1, n_sets):
        if not torch.equal(sets[0][4], sets[k][4]):
            raise RuntimeError(f"buffer set {k} differs from set 0 after identical launches")
    del graph
    return total, mode


def warmup_launches(warmup: int, n_sets: int) -> int:
    """Untimed launches before capture: at least W, and at least one per buffer set."""
    return max(warmup, n_sets)


def rotating_sets(set_bytes: int, min_sets: int = 4, cap: int = 64) -> int:
    """Buffer sets so that (sets - 1) x set bytes > 3 x L2: a step's inputs were
    evicted by the steps in between (L2 flushed by the rotation)."""
    return max(min_sets, min(cap, -(-3 * L2_BYTES // max(1, set_bytes)) + 1))


def time_mesh(name, steps, warmup, n_sets_min=4, given_geometry=False, tiled=True, n_cells=None):
    """Fused mesh kernel (geometry + gather + integrate, txb_integrate_mesh) on the
    config's Kuhn mesh: connectivity/aux/out rotate over buffer sets (> L2);
    vertex coordinates and the global coefficient vector are the mesh's own
    (small, L2-resident by nature).  Returns (ms per launch, compulsory bytes per cell)."""
    import torch

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200.workload import PHYSICS, refine_for

    dim, physics, dtype, n = CONFIGS[name]
    n = n_cells or n
    factory, aux_space = PHYSICS[physics]
    form = factory(dim)
    full = txb.generate_unit_simplex_mesh(dim, refine_for(dim, n))
    mesh = txb.Mesh(dim, full.vertices, np.ascontiguousarray(full.cells[:n]))
    npdt = np.float32 if dtype == "f32" else np.float64
    glob = torch.from_numpy(np.random.default_rng(1234).standard_normal(full.n_vertices * form.n_comp).astype(npdt)).cuda()
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    s = np.dtype(npdt).itemsize
    per_cell = (dim + 1) * 8 + {"p0": s, "p1": (dim + 1) * s}.get(aux_space, 0) + (dim + 1) * form.n_comp * s
    cells0 = torch.from_numpy(mesh.cells).cuda()
    os.environ["TXB_TILED"] = "1" if tiled else "0"
    tiles = None
    if tiled:
        from paper_1607_04245_b200 import executor

        tiles = executor.cell_tiles(cells0, dim, executor.default_tile_cells(dim, 1, given_geometry, s))
        # streamed per cell: local indices + the tile record instead of the int64 connectivity
        per_cell += 4 * tiles.local_bytes + tiles.vrec * 4 / tiles.tile_cells - (dim + 1) * 8
    n_sets = max(n_sets_min, -(-3 * L2_BYTES // int(per_cell * n)) + 1)
    verts = torch.from_numpy(np.ascontiguousarray(full.vertices)).cuda()
    geom = None
    if given_geometry:  # precomputed once (mesh setup); its bytes are streamed per launch
        g64 = txb.compute_geometry(mesh, cells=cells0, device_out=True)
        geom = txb.CellGeometry(g64.inv_jacobians.to(glob.dtype), g64.determinants.to(glob.dtype))
        per_cell += (dim * dim + 1) * s
    sets = []
    for _ in range(n_sets):
        aux = None
        if aux_space == "p0":
            aux = txb.CellAux("p0", torch.rand((n, 1), dtype=glob.dtype, device="cuda") + 0.5)
        elif aux_space == "p1":
            aux = txb.CellAux("p1", torch.rand((n, dim + 1, 1), dtype=glob.dtype, device="cuda") + 0.5)
        sets.append((cells0.clone(), aux, torch.empty((n, dim + 1, form.n_comp), dtype=glob.dtype, device="cuda")))
        if tiles is not None:  # each set's own tile tables, built before the timed graph
            executor.cell_tiles(sets[-1][0], dim, tiles.tile_cells)

    def launch(i):
        cells, aux, out = sets[i % n_sets]
        txb.integrate_mesh(mesh, txb.FieldLayout(form.n_comp), tab, rule, form, glob, aux, dtype=dtype,
                           cells=cells, vertices=verts, out=out, check_orientation=False, cell_geom=geom)

    for i in range(warmup):
        launch(i)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="relaxed"):
        for i in range(steps):
            launch(warmup + i)
    graph.replay()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    graph.replay()
    t1.record()
    torch.cuda.synchronize()
    os.environ.pop("TXB_TILED", None)
    return t0.elapsed_time(t1) / steps, per_cell


# A user physics form for the run-time compiled lane's bench rows: two P1
# auxiliary fields with their gradients and an f0 term (string-injection
# source, compiled by NVRTC).  Mirrors oracle/user_forms.py "advect".
_ADVECT_SIG = "(const real u[], const realv gradU[], const real a[], const realv gradA[], int comp)"
ADVECT_F1 = f"realv f1_advect{_ADVECT_SIG}\n{{\n  return a[0]*gradU[comp] + u[comp]*gradA[1];\n}}\n"
ADVECT_F0 = f"real f0_advect{_ADVECT_SIG}\n{{\n  return a[1]*u[comp] + dot(gradA[0], gradU[comp]);\n}}\n"


def strong_scaling_rows(world, rank, barrier, reduce_max, steps=10):
    """BASELINE.json configs[4] across the ranks: a FIXED total of 2^24 and 2^26
    cells (f32 and f64) split into contiguous per-rank ranges (strong scaling;
    the per-rank slice tiles the rank's 2^20-cell Kuhn workload, values do not
    affect timing).  Device time of `steps` launches per rank, max over ranks."""
    import torch

    from paper_1607_04245_b200.physics import CellAux

    rows = []
    for dtype in ("f32", "f64"):
        base = "3d_varcoef_" + dtype
        vf, vb = config_model(base)
        wl = rank_workload(base, rank, world)
        for lg in (24, 26):
            total = 1 << lg
            n = total // world
            reps = -(-n // wl["n"])
            cut = lambda t: t.repeat(reps, *([1] * (t.dim() - 1)))[:n].contiguous()  # noqa: E731
            big = dict(wl, n=n, inv=cut(wl["inv"]), det=cut(wl["det"]), coeffs=cut(wl["coeffs"]),
                       aux=CellAux("p0", cut(wl["aux"].values)))
            tot, _ = time_device(big, steps, 3, 1, barrier)
            tot = reduce_max(tot)
            ms = tot / steps
            rows.append({"config": f"3d_varcoef_{dtype}_2^{lg}_total", "dtype": dtype, "cells_total": total,
                         "cells_per_rank": n, "n_gpus": world, "ms_per_step": ms,
                         "gflops": vf * total / (ms * 1e-3) / 1e9, "gbs": vb * total / (ms * 1e-3) / 1e9,
                         "scaling": "strong"})
            del big
            torch.cuda.empty_cache()
        del wl
        torch.cuda.empty_cache()
    return rows


def api_rows(steps=20):
    """The reference's mesh-level call from the host (executor.integrate_transposed,
    executor.py:161-267): numpy global coefficients in, numpy residual out, every
    step (H2D of the coefficient vector, fused geometry-or-given + gather +
    integration kernel, deterministic scatter-add, D2H of the residual).  Wall
    time per call; the mesh's static device data is cached across calls."""
    import torch

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200.workload import PHYSICS, refine_for

    rows = []
    for name in ("3d_varcoef_f64", "3d_elasticity_f64"):
        dim, physics, dtype, n = CONFIGS[name]
        factory, aux_space = PHYSICS[physics]
        form = factory(dim)
        mesh = txb.generate_unit_simplex_mesh(dim, refine_for(dim, n))
        layout = txb.FieldLayout(form.n_comp)
        rule = txb.quadrature_rule(dim, 1)
        tab = txb.tabulate(dim, rule)
        glob = np.random.default_rng(3).standard_normal(layout.global_size(mesh))
        aux = None
        if aux_space == "p0":
            aux = txb.CellAux("p0", np.random.default_rng(4).uniform(0.5, 1.5, (mesh.n_cells, 1)))
        geom = txb.compute_geometry(mesh, device_out=True)  # mesh setup, once
        n_bl = 128 // (dim + 1)  # 128-cell batches (the tuned batch size); n_cb only feeds the trace model
        for label, cg in (("given_geometry", geom), ("geometry_in_kernel", None)):
            for _ in range(3):
                txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=n_bl, n_cb=8, dtype=dtype, shared_mem_limit=None,
                                         cell_geom=cg)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(steps):
                res, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=n_bl, n_cb=8,
                                                  dtype=dtype, cell_geom=cg, shared_mem_limit=None)
            dt = (time.perf_counter() - t0) / steps
            rows.append({"config": f"api_integrate_transposed_{label}_{name}", "cells": mesh.n_cells,
                         "vertices": mesh.n_vertices, "ms_per_call": dt * 1e3,
                         "gcells_per_s": mesh.n_cells / dt / 1e9,
                         "path": "host numpy in/out: H2D coefficients, fused mesh kernel, scatter-add, D2H residual"})
        # the same call with device-resident coefficients and kappa (CUDA tensors in, CUDA residual out):
        # what a GPU-resident solver loop pays per residual; wall time incl. the orientation-flag read
        glob_dev = torch.from_numpy(glob).cuda()
        aux_dev = None if aux is None else txb.CellAux("p0", torch.from_numpy(aux.values).cuda())
        for _ in range(3):
            txb.integrate_transposed(mesh, layout, tab, rule, form, glob_dev, aux_dev, n_bl=n_bl, n_cb=8,
                                     dtype=dtype, shared_mem_limit=None)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            res, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob_dev, aux_dev, n_bl=n_bl, n_cb=8,
                                              dtype=dtype, shared_mem_limit=None)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / steps
        rows.append({"config": f"api_integrate_transposed_device_{name}", "cells": mesh.n_cells,
                     "vertices": mesh.n_vertices, "ms_per_call": dt * 1e3, "gcells_per_s": mesh.n_cells / dt / 1e9,
                     "path": "CUDA tensors in/out: fused mesh kernel (in-kernel geometry) + scatter-add"})
        # the same residual captured once into a CUDA graph (ResidualGraph): copy-in + one replay per call
        rg = txb.ResidualGraph(mesh, layout, tab, rule, form, aux_dev, n_bl=n_bl, n_cb=8, dtype=dtype,
                               shared_mem_limit=None)
        for _ in range(3):
            rg(glob_dev)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            rg(glob_dev)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            rg(glob_dev)
        e1.record()
        torch.cuda.synchronize()
        rows.append({"config": f"api_residual_graph_device_{name}", "cells": mesh.n_cells,
                     "vertices": mesh.n_vertices, "ms_per_call": dt * 1e3, "gcells_per_s": mesh.n_cells / dt / 1e9,
                     "device_ms_per_call": e0.elapsed_time(e1) / steps,
                     "path": "ResidualGraph: copy of the global vector + one CUDA-graph replay (tiled mesh kernel + "
                             "scatter-add)"})
        del rg
        del glob_dev, aux_dev
        del geom
        torch.cuda.empty_cache()
    # a run-time compiled user form (f0, two P1 fields, grad a) at mesh level, device-resident:
    # the mesh entry point of the NVRTC lane (geometry + gather in-kernel) + scatter-add
    from paper_1607_04245_b200.physics import user_form

    dim, _, dtype, n = CONFIGS["3d_varcoef_f64"]
    mesh = txb.generate_unit_simplex_mesh(dim, refine_for(dim, n))
    form = user_form("advect", 3, 1, lambda s, c: None, 9, ADVECT_F1, n_aux=2, f0=lambda s, c: None,
                     flops_f0=7, source_f0=ADVECT_F0, uses_grad_a=True)
    layout = txb.FieldLayout(1)
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    glob_dev = torch.from_numpy(np.random.default_rng(5).standard_normal(mesh.n_vertices)).cuda()
    aux_dev = txb.CellAux("p1", torch.rand((mesh.n_cells, dim + 1, 2), dtype=torch.float64, device="cuda") + 0.5)
    call = lambda: txb.integrate_transposed(mesh, layout, tab, rule, form, glob_dev, aux_dev, n_bl=32,  # noqa: E731
                                            n_cb=8, dtype=dtype, shared_mem_limit=None)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    rows.append({"config": "api_integrate_transposed_device_user_advect_3d_f64", "cells": mesh.n_cells,
                 "vertices": mesh.n_vertices, "ms_per_call": dt * 1e3, "gcells_per_s": mesh.n_cells / dt / 1e9,
                 "path": "CUDA tensors in/out: run-time compiled form, tiled mesh entry point + scatter-add"})
    rg = txb.ResidualGraph(mesh, layout, tab, rule, form, aux_dev, n_bl=32, n_cb=8, dtype=dtype,
                           shared_mem_limit=None)
    for _ in range(3):
        rg(glob_dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        rg(glob_dev)
    e1.record()
    torch.cuda.synchronize()
    rows.append({"config": "api_residual_graph_device_user_advect_3d_f64", "cells": mesh.n_cells,
                 "vertices": mesh.n_vertices, "device_ms_per_call": e0.elapsed_time(e1) / steps,
                 "path": "ResidualGraph of the run-time compiled form (tiled mesh entry point + scatter-add)"})
    return rows


def residual_graph_rows(steps=50):
    """The mesh-level residual as a user's solver loop runs it: integrate_transposed
    (geometry + gather + integration + deterministic scatter-add) captured once as
    a ResidualGraph, replayed per residual; device time per residual, 2^20-cell
    3D Kuhn mesh (var-coef P0, f64), global vector device-resident."""
    import torch

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200.workload import refine_for

    mesh = txb.generate_unit_simplex_mesh(3, refine_for(3, 1 << 20))
    form = txb.poisson_varcoef_form(3)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    aux = txb.CellAux("p0", torch.rand((mesh.n_cells, 1), dtype=torch.float64, device="cuda") + 0.5)
    glob = torch.from_numpy(np.random.default_rng(5).standard_normal(mesh.n_vertices)).cuda()
    rg = txb.ResidualGraph(mesh, txb.FieldLayout(1), tab, rule, form, aux, n_bl=16, n_cb=8, dtype="f64",
                           shared_mem_limit=None)
    for _ in range(3):
        rg(glob)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        rg(glob)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    # a solver writing the graph's input buffer in place: one replay, no copy-in
    rg.glob.copy_(glob)
    e0.record()
    for _ in range(steps):
        rg()
    e1.record()
    torch.cuda.synchronize()
    ms_in_place = e0.elapsed_time(e1) / steps
    return [{"config": "residual_graph_3d_varcoef_f64", "cells": mesh.n_cells, "vertices": mesh.n_vertices,
             "ms_per_residual": ms, "ms_per_residual_in_place": ms_in_place,
             "gcells_per_s": mesh.n_cells / (ms * 1e-3) / 1e9,
             "path": "ResidualGraph: copy-in + one CUDA-graph replay (tiled mesh kernel, in-kernel float64 "
                     "geometry, + slot-ordered scatter-add); the reference's integrate_transposed ~290 ms"}]


def sweep_rows(peak):
    """BASELINE.json configs[4]: 3D P1 var-coef Laplacian at 2^24..2^27 cells on
    one GPU, f32 and f64.  The 2^20-cell Kuhn workload is tiled on the device
    (cells are independent; values do not affect timing).  Every size is larger
    than L2, so one buffer set; 10 graph-captured launches (5 at 2^27)."""
    import torch

    rows = []
    for dtype in ("f32", "f64"):
        base = "3d_varcoef_" + dtype
        vf, vb = config_model(base)
        wl = rank_workload(base, 0, 1)
        for lg in (24, 25, 26, 27):
            reps = 1 << (lg - 20)
            big = dict(wl, n=wl["n"] * reps, inv=wl["inv"].repeat(reps, 1, 1), det=wl["det"].repeat(reps),
                       coeffs=wl["coeffs"].repeat(reps, 1, 1))
            from paper_1607_04245_b200.physics import CellAux

            big["aux"] = CellAux("p0", wl["aux"].values.repeat(reps, 1))
            steps = 10 if lg < 27 else 5
            tot, _ = time_device(big, steps, 3, 1)
            ms = tot / steps
            rows.append({"config": f"3d_varcoef_{dtype}_2^{lg}", "dtype": dtype, "cells": big["n"],
                         "launch_ms": ms, "gflops": vf * big["n"] / (ms * 1e-3) / 1e9,
                         "gbs_launch": vb * big["n"] / (ms * 1e-3) / 1e9,
                         "frac": vb * big["n"] / (ms * 1e-3) / 1e9 / peak, "bytes_per_cell": vb,
                         "data": "2^20-cell Kuhn workload tiled on the device; one set (> L2)"})
            del big
            torch.cuda.empty_cache()
        del wl
        torch.cuda.empty_cache()
    return rows


def jit_rows(peak, steps):
    """Run-time compiled lane: the shipped var-coef and elasticity forms through
    NVRTC (same bytes as the ahead-of-time rows) and a user form with f0 + 2 P1
    fields + grad a."""
    import torch

    from paper_1607_04245_b200.perf_model import compulsory_bytes_per_cell
    from paper_1607_04245_b200.physics import CellAux, user_form

    rows = []
    for name in ("3d_varcoef_f64", "3d_varcoef_f32", "3d_elasticity_f64", "3d_elasticity_f32"):
        vf, vb = config_model(name)
        wl = rank_workload(name, 0, 1)
        ns = max(4, -(-3 * L2_BYTES // (vb * wl["n"])) + 1)
        tot, _ = time_device(wl, steps, 5, min(ns, 8), jit=True)
        ms = tot / steps
        rows.append({"config": "jit_" + name, "path": "txb_jit_integrate (shipped form's source, NVRTC)",
                     "dtype": wl["dtype"], "cells": wl["n"], "launch_ms": ms, "gflops": vf * wl["n"] / (ms * 1e-3) / 1e9,
                     "gbs_launch": vb * wl["n"] / (ms * 1e-3) / 1e9,
                     "frac": vb * wl["n"] / (ms * 1e-3) / 1e9 / peak, "bytes_per_cell": vb})
        del wl
        torch.cuda.empty_cache()
    for dtype in ("f64", "f32"):
        base = "3d_varcoef_" + dtype
        vf, _ = config_model(base)
        wl = rank_workload(base, 0, 1)
        n, tdt = wl["n"], wl["coeffs"].dtype
        wl["form"] = user_form("advect", 3, 1, lambda s, c: None, 9, ADVECT_F1, n_aux=2, f0=lambda s, c: None,
                               flops_f0=7, source_f0=ADVECT_F0, uses_grad_a=True)
        wl["aux"] = CellAux("p1", torch.rand((n, 4, 2), dtype=tdt, device="cuda") + 0.5)
        w = 4 if dtype == "f32" else 8
        vb = compulsory_bytes_per_cell(3, 1, w, "p1", n_aux=2)
        ns = max(4, -(-3 * L2_BYTES // (vb * n)) + 1)
        tot, _ = time_device(wl, steps, 5, min(ns, 8))
        ms = tot / steps
        rows.append({"config": "jit_3d_user_advect_" + dtype, "path": "txb_jit_integrate (user form: f0, 2 P1 aux, grad a)",
                     "dtype": dtype, "cells": n, "launch_ms": ms, "gcells_per_s": n / (ms * 1e-3) / 1e9,
                     "gbs_launch": vb * n / (ms * 1e-3) / 1e9, "frac": vb * n / (ms * 1e-3) / 1e9 / peak,
                     "bytes_per_cell": vb})
        del wl
        torch.cuda.empty_cache()
    return rows


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def time_e2e(wl, steps, warmup, pageable=False):
    """Through the reference-facing call with HOST buffers (pinned numpy; or
    plain pageable numpy arrays with ``pageable``): H2D + kernel + D2H per step
    inside the timed region (wall clock; the host call returns only after the
    result is in host memory)."""
    import torch

    from paper_1607_04245_b200 import backend
    from paper_1607_04245_b200.physics import CellAux

    def pinned(t):
        if pageable:
            return t.cpu().numpy().copy()
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h.numpy()

    inv, det, co = pinned(wl["inv"]), pinned(wl["det"]), pinned(wl["coeffs"])
    aux = None if wl["aux"] is None else CellAux("p0", pinned(wl["aux"].values))
    out = (np.empty(tuple(co.shape), dtype=co.dtype) if pageable else
           torch.empty(tuple(co.shape), dtype=wl["coeffs"].dtype, pin_memory=True).numpy())
    tab, rule = wl["tab"], wl["rule"]
    kernel = backend.cuda_kernel(wl["form"], rule.n_q, wl["aux"], co.dtype.itemsize)
    npdt = co.dtype
    B, D, W = (np.ascontiguousarray(x, dtype=npdt) for x in (tab.basis, tab.basis_der, rule.weights))
    for _ in range(warmup):
        backend.run_cuda(kernel, B, D, W, inv, det, co, aux, out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        backend.run_cuda(kernel, B, D, W, inv, det, co, aux, out)
    dt = time.perf_counter() - t0
    h2d = inv.nbytes + det.nbytes + co.nbytes + (aux.values.nbytes if aux is not None else 0)
    return dt, h2d, out.nbytes, out


def h2d_link_gbs(nbytes: int, reps: int = 5) -> float:
    """Pinned host -> device copy rate of this box's link (cudaMemcpy of nbytes,
    best of reps): the ceiling of the e2e path, whose inputs must cross it."""
    import torch

    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = float("inf")
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    del src, dst
    return nbytes / best / 1e9


def stream_probe(read_b, write_b, reps=20):
    """Measured achievable HBM GB/s of a STREAM-like kernel at the kernel's read:write ratio."""
    import ctypes

    import torch

    from paper_1607_04245_b200 import _lib

    scale = 8
    rb = (read_b * scale + 15) // 16 * 16
    wb = (write_b * scale + 15) // 16 * 16
    n_sets = 4
    src = [torch.empty(rb, dtype=torch.uint8, device="cuda").fill_(1) for _ in range(n_sets)]
    dst = [torch.empty(wb, dtype=torch.uint8, device="cuda") for _ in range(n_sets)]
    s = torch.cuda.current_stream()
    L = _lib.lib()
    for i in range(3):
        L.txb_stream_probe(src[i % n_sets].data_ptr(), rb, dst[i % n_sets].data_ptr(), wb,
                           ctypes.c_void_p(s.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for i in range(reps):
        _lib.check(L.txb_stream_probe(src[i % n_sets].data_ptr(), rb, dst[i % n_sets].data_ptr(), wb,
                                      ctypes.c_void_p(s.cuda_stream)))
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return (rb + wb) / (ms * 1e-3) / 1e9


# ----------------------------------------------------------------------------
# CPU arm: the reference's compiled lane over a fork pool
# ----------------------------------------------------------------------------
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


_CPU = {}


def _cpu_worker(idx, lo, hi, reps, bar, kind):
    from oracle import oracle

    a = _CPU
    sl = slice(lo, hi)
    out = np.empty(a["coeffs"][sl].shape, dtype=a["coeffs"].dtype)
    lane = oracle.ref_lane() if kind == "reference" else None
    aux = a["aux"][sl] if a["aux"] is not None else None
    for _ in range(reps):
        bar.wait()
        if lane is not None:
            oracle.ref_integrate(lane, a["fc"], a["am"], a["B"], a["D"], a["W"], a["inv"][sl], a["det"][sl],
                                 a["coeffs"][sl], aux, out)
        else:
            out[...] = oracle.integrate(a["fc"], a["am"], a["B"], a["D"], a["W"], a["inv"][sl], a["det"][sl],
                                        a["coeffs"][sl], aux, a["coeffs"].dtype)
        bar.wait()


def cpu_reference(name, reps, target_s=None, total_cells=None):
    """Time the reference CPU lane on all host cores (fork pool over contiguous
    ranges; threads do not scale: the Cython lane holds the GIL)."""
    import multiprocessing as mp

    from oracle import oracle

    dim, physics, dtype, n = CONFIGS[name]
    n = total_cells or n  # the reference arm integrates the same cells as our N-GPU arm
    npdt = np.float32 if dtype == "f32" else np.float64
    full, inv, det, coeffs, aux = oracle.workload(dim, physics, n)
    B, D, W = oracle.p1_tables(dim)
    c = lambda x: np.ascontiguousarray(x, dtype=npdt)  # noqa: E731
    kind = "reference" if oracle.ref_lane() is not None else "port"
    _CPU.update(fc=2 if physics == "elasticity" else 1, am=1 if aux is not None else 0, B=c(B), D=c(D), W=c(W),
                inv=c(inv), det=c(det), coeffs=c(coeffs), aux=None if aux is None else c(aux))
    P = host_cores()
    ctx = mp.get_context("fork")
    # one untimed calibration pass decides reps for the bounded sample
    if target_s is not None:
        t0 = time.perf_counter()
        _cpu_worker(0, 0, n // P, 1, _NoBarrier(), kind)
        one = max(time.perf_counter() - t0, 1e-4)
        reps = int(max(3, min(200, target_s / one)))
    bar = ctx.Barrier(P + 1)
    procs = []
    for i in range(P):
        lo, hi = n * i // P, n * (i + 1) // P
        p = ctx.Process(target=_cpu_worker, args=(i, lo, hi, reps + 1, bar, kind))
        p.start()
        procs.append(p)
    times = []
    for r in range(reps + 1):
        bar.wait()
        t0 = time.perf_counter()
        bar.wait()
        if r > 0:  # first rep is warm-up
            times.append(time.perf_counter() - t0)
    for p in procs:
        p.join()
    return dict(times=times, cores=P, kind=kind, n=n, dtype=dtype)


class _NoBarrier:
    def wait(self):
        pass


# ----------------------------------------------------------------------------
def _guarded(rows, label, fn, *args, **kw):
    """Run one extra row group; an exception becomes an {"error"} row instead of
    discarding the headline line (which is assembled before any extra)."""
    import traceback

    try:
        rows.extend(fn(*args, **kw))
    except Exception as e:  # noqa: BLE001 - recorded in the JSON line
        rows.append({"config": label, "error": f"{type(e).__name__}: {e}",
                     "where": traceback.format_exc(limit=3).splitlines()[-3:]})
    finally:
        try:
            import torch

            torch.cuda.synchronize()
            torch.cuda.empty_cache()
        except Exception:  # noqa: BLE001
            pass


def variant_rows(peak, steps):
    """The other BASELINE.json configurations on one GPU (parity configs timed
    like the headline: device-resident, rotating buffer sets > 3x L2)."""
    rows = []
    for v in VARIANTS:
        def one(v=v):
            vf, vb = config_model(v)
            vw = rank_workload(v, 0, 1)
            ns = rotating_sets(vb * vw["n"])
            k = variant_steps(vw["n"], steps)
            tot, _ = time_device(vw, k, 5, ns)
            vl = tot / k
            row = {"config": v, "dtype": vw["dtype"], "cells": vw["n"], "steps": k, "sets": ns,
                   "gflops": vf * vw["n"] / (vl * 1e-3) / 1e9,
                   "gbs_launch": vb * vw["n"] / (vl * 1e-3) / 1e9,
                   "frac": vb * vw["n"] / (vl * 1e-3) / 1e9 / peak, "launch_ms": vl,
                   "bytes_per_cell": vb}
            if vw["n"] <= (1 << 16):
                row["note"] = ("launch-latency bound (6 MB per launch): a plain copy kernel moving the same bytes "
                               "takes 3.5 us per chained launch, profiles/r1f_scan.md")
            return [row]
        _guarded(rows, v, one)
    return rows


def variant_steps(n_cells: int, steps: int) -> int:
    """Launches timed per variant: >= 200 (a short driver run still averages
    over many launches: one graph replay's fixed start costs ~1-2 % of a
    50-launch chain of 10 us launches), a quarter of K for long runs, capped at
    1000."""
    return min(1000, max(200, steps // 4)) if n_cells <= (1 << 20) else 40


def mesh_rows(peak, steps, configs=("3d_varcoef_f64", "3d_varcoef_f32", "3d_elasticity_f64", "3d_elasticity_f32",
                                     "2d_varcoef_f64", "2d_varcoef_f32"),
              modes=("given", "given_tiled", "tiled", "per_cell")):
    rows = []
    for v in configs:
        for mode in modes:
            def one(v=v, mode=mode):
                vf, _ = config_model(v)
                n = CONFIGS[v][3]
                ms, per_cell = time_mesh(v, variant_steps(n, steps), 5, given_geometry=mode.startswith("given"),
                                         tiled=mode in ("tiled", "given_tiled"))
                path = {"given": "txb_integrate_mesh: gather per cell fused into the integration, geometry streamed",
                        "given_tiled": "txb_integrate_mesh_tiled: geometry streamed, coefficients from per-tile "
                                       "vertex tables",
                        "per_cell": "txb_integrate_mesh: float64 geometry + gather per cell in-kernel",
                        "tiled": "txb_integrate_mesh_tiled: float64 geometry + gather from per-tile vertex "
                                 "tables in shared memory"}[mode]
                return [{
                    "config": {"given": "mesh_given_geometry_", "given_tiled": "mesh_tiled_given_geometry_",
                               "tiled": "mesh_tiled_geometry_in_kernel_",
                               "per_cell": "mesh_geometry_in_kernel_"}[mode] + v,
                    "path": path,
                    "cells": n, "launch_ms": ms, "gflops": vf * n / (ms * 1e-3) / 1e9,
                    "gcells_per_s": n / (ms * 1e-3) / 1e9, "bytes_per_cell": per_cell,
                    "gbs": per_cell * n / (ms * 1e-3) / 1e9, "frac": per_cell * n / (ms * 1e-3) / 1e9 / peak}]
            _guarded(rows, f"mesh_{v}_{mode}", one)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--no-variants", action="store_true", help="headline only (no BASELINE variant rows)")
    ap.add_argument("--extras", action="store_true",
                    help="also the mesh-fused rows, the 2^24..2^27 sweep, the mesh-level API rows and the "
                         "run-time compiled rows (minutes; not part of the default driver run)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=3.0)
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling runs)")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.warmup < 3:
        args.warmup = 3
    flops_cell, bytes_cell = config_model(args.config)
    dim, physics, dtype, per_gpu = CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        r = cpu_reference(args.config, args.steps + args.warmup, total_cells=per_gpu * max(world, args.gpus),
                          target_s=None if args.steps + args.warmup <= 200 else 60.0)
        ts = r["times"][args.warmup:] if len(r["times"]) > args.warmup else r["times"]
        t = sum(ts) / len(ts)
        gf = flops_cell * r["n"] / t / 1e9
        line = {
            "impl": "reference", "metric": METRIC, "value": gf,
            "unit": "GF/s", "n_gpus": args.gpus, "steps": len(ts), "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic (Kuhn mesh, seeded N(0,1) coefficients, P0 kappa)",
            "config": {"workload": f"{args.config}: {dim}D P1 {physics}, {r['n']} cells "
                                   f"({per_gpu} per GPU x {max(world, args.gpus)})"},
            "cpu_baseline": {"value": gf, "unit": "GF/s", "cores": r["cores"], "kind": r["kind"],
                             "sample": f"{r['n']} cells per step, fork pool of {r['cores']} processes over "
                                       f"contiguous ranges, reference _kernels_cy lane"},
            "e2e": {"value": gf, "unit": "GF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gbs": bytes_cell * r["n"] / t / 1e9,
        }
        print(json.dumps(line), flush=True)
        return

    import torch

    # one process per GPU; TXB_BENCH_BACKEND=gloo (+ device = local % count) lets the
    # multi-rank code path be exercised on a single-GPU box (timings then meaningless)
    dist_backend = os.environ.get("TXB_BENCH_BACKEND", "nccl")
    device = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    barrier = None
    dist = None
    if world > 1:
        import torch.distributed as dist

        if dist_backend == "nccl":
            # communicator init lines (ranks, devices, NVLS/P2P transport) on stderr; the
            # hot path itself runs no collective -- only the max-over-ranks time reduction
            nccl_debug_env()
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
            if rank == 0:
                print(f"[bench] nccl process group: world {world}, rank 0 on cuda:{device}", file=sys.stderr,
                      flush=True)
        else:
            dist.init_process_group(dist_backend)
        barrier = dist.barrier

    def reduce_max(x: float) -> float:
        """max over ranks (timing of a multi-GPU step is the slowest rank)."""
        return reduce_max_over_ranks(x, world, dist, "cuda" if dist_backend == "nccl" else "cpu")

    from paper_1607_04245_b200 import backend

    # ------------------------------------------------------------------ headline
    wl = rank_workload(args.config, rank, world)
    set_bytes = bytes_cell * wl["n"]
    n_sets = rotating_sets(set_bytes)
    sampler = ClockSampler(torch.cuda.current_device())
    total_ms, timing_mode = time_device(wl, args.steps, args.warmup, n_sets, barrier, sampler)
    total_ms = reduce_max(total_ms)
    cells_total = sum(cell_counts(per_gpu, world))
    ms_step = total_ms / args.steps  # one kernel launch per step
    gf = flops_cell * cells_total / (ms_step * 1e-3) / 1e9
    # the roofline's launch time is THIS rank's own (rank 0 prints it)
    launch_ms_local = ms_step

    # e2e through the host-buffer C ABI path
    e2e_steps = max(3, min(20, args.steps))
    if barrier:
        barrier()
    if args.no_e2e:
        e2e_s, h2d, d2h, e2e_gf = float("nan"), 0, 0, None
    else:
        e2e_s, h2d, d2h, _ = time_e2e(wl, e2e_steps, 2)
        e2e_s = reduce_max(e2e_s)
        e2e_gf = flops_cell * cells_total * e2e_steps / e2e_s / 1e9

    line = None
    if rank == 0:
        peak, peak_src = peaks()
        achieved = bytes_cell * wl["n"] / (launch_ms_local * 1e-3) / 1e9
        form = wl["form"]
        cfg = backend.launch_config(*backend.cuda_kernel(form, 1, wl["aux"], 4 if dtype == "f32" else 8),
                                    4 if dtype == "f32" else 8, dim, 1, form.n_comp, wl["n"])
        try:
            achievable = stream_probe(wl["inv"].nbytes + wl["det"].nbytes + wl["coeffs"].nbytes +
                                      (wl["aux"].values.nbytes if wl["aux"] is not None else 0),
                                      wl["coeffs"].nbytes)
        except Exception:  # noqa: BLE001 - optional context number
            achievable = None
        line = {
            "metric": METRIC,
            "value": gf, "unit": "GF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic (Kuhn mesh cells of the rank's range, seeded N(0,1) "
                                    "coefficients, P0 kappa U[0.5,1.5); generated per rank)",
            "config": {"workload": f"{args.config}: {dim}D P1 {physics}, {per_gpu} cells per GPU "
                                   f"(BASELINE.json configs[1])",
                       "cells_total": cells_total, "parallelism": f"cell-range x{world}",
                       "l2": f"inputs > L2: {n_sets} rotating buffer sets of {set_bytes / 1e6:.1f} MB "
                             f"(> 3 x 126 MB L2 between reuses)",
                       "launch": cfg},
            "gbs": bytes_cell * cells_total / (ms_step * 1e-3) / 1e9,
            "cells_per_s": cells_total / (ms_step * 1e-3),
            "roofline": roofline_entry(args.config, achieved, peak, peak_src, bytes_cell, flops_cell,
                                       achievable, launch_ms_local, timing_mode, args.steps, wl["n"]),
            "e2e": {"value": e2e_gf, "unit": "GF/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "path": "txb_integrate_cells_host (pinned numpy in/out)"},
            "gpu_launches": args.steps,
            "clocks": sampler.summary(),
        }
        if world == 1 and not args.no_cpu:
            try:
                r = cpu_reference(args.config, 3, target_s=args.cpu_seconds)
                t = statistics.median(r["times"])
                line["cpu_baseline"] = {
                    "value": flops_cell * r["n"] / t / 1e9, "unit": "GF/s", "cores": r["cores"],
                    "kind": r["kind"], "ms": t * 1e3,
                    "sample": f"{r['n']} cells ({args.config}) x {len(r['times'])} passes, fork pool of "
                              f"{r['cores']} processes, median pass"}
            except Exception as e:  # noqa: BLE001
                line["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"}
        if e2e_gf:
            # what bounds e2e: the step's inputs cross the host link (context, not a second metric)
            try:
                link = h2d_link_gbs(h2d)
                floor_ms = h2d / link / 1e6
                line["e2e"].update({"h2d_link_gbs": link, "h2d_floor_ms_per_step": floor_ms,
                                    "frac_of_h2d_floor": floor_ms / (e2e_s / e2e_steps * 1e3)})
            except Exception as e:  # noqa: BLE001
                line["e2e"]["h2d_link_error"] = f"{type(e).__name__}: {e}"
            # the same call with plain pageable numpy arrays (a reference user's buffers): context
            try:
                ps, _, _, _ = time_e2e(wl, 5, 1, pageable=True)
                line["e2e"]["pageable_value"] = flops_cell * wl["n"] * 5 / ps / 1e9
            except Exception as e:  # noqa: BLE001
                line["e2e"]["pageable_error"] = f"{type(e).__name__}: {e}"
    try:
        # -------------------------------------------------------------- extras
        # (each row group guarded: a failure is an error row, never a lost headline)
        if world == 1 and rank == 0:
            rows = []
            peak = line["roofline"]["peak"]
            if not args.no_variants:
                rows += variant_rows(peak, args.steps)
                # the mesh-level path (§8f rows 1 + 3): the tiled kernel, geometry in-kernel and given
                rows += mesh_rows(peak, args.steps, configs=("3d_varcoef_f64", "3d_varcoef_f32"),
                                  modes=("tiled", "given_tiled"))
                _guarded(rows, "residual_graph", residual_graph_rows)
            if args.extras:
                rows += mesh_rows(peak, args.steps)
                _guarded(rows, "sweep", sweep_rows, peak)
                _guarded(rows, "api", api_rows)
                _guarded(rows, "jit", jit_rows, peak, variant_steps(1 << 20, args.steps))
            if rows:
                line["variants"] = rows
        if world > 1:
            try:
                strong = strong_scaling_rows(world, rank, barrier, reduce_max)
            except Exception as e:  # noqa: BLE001
                strong = [{"error": f"{type(e).__name__}: {e}"}]
            if line is not None:
                line["strong_scaling"] = strong
    finally:
        if line is not None:
            print(json.dumps(line), flush=True)
        if world > 1:
            dist.destroy_process_group()


def cell_counts(per_gpu: int, world: int):
    """Cells of each rank's contiguous range of the world x per_gpu-cell job."""
    from paper_1607_04245_b200.shard import cell_range

    total = per_gpu * world
    return [hi - lo for lo, hi in (cell_range(total, r, world, align=256) for r in range(world))]


def reduce_max_over_ranks(x: float, world: int, dist, device: str) -> float:
    """max over ranks of a float (time of a multi-GPU step = the slowest rank)."""
    if world == 1:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def roofline_entry(config, achieved, peak, peak_src, bytes_cell, flops_cell, achievable, launch_ms, mode, steps,
                   n_cells):
    """The roofline object of the JSON line.  ``traffic`` is the ncu-measured
    DRAM read + write bytes of ONE launch (write-back included), per cell, from
    profiles/ncu_traffic.json (tools/traffic.py), scaled to this launch's cells."""
    prof = REPO / "profiles" / "ncu_traffic.json"
    traffic = traffic_split = None
    if prof.exists():
        ent = json.loads(prof.read_text()).get("configs", {}).get(config)
        if ent:
            rd = ent["read_bytes_per_cell"] * n_cells
            wr = ent["write_bytes_per_cell"] * n_cells
            traffic = rd + wr
            traffic_split = {"read": rd, "write": wr, "algorithmic": bytes_cell * n_cells,
                             "ratio": (rd + wr) / (bytes_cell * n_cells), "source": ent.get("source")}
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_split": traffic_split,
            "peak_source": peak_src, "bytes_per_cell": bytes_cell, "flops_per_cell_eq7": flops_cell,
            "achievable_stream_gbs": achievable,
            "frac_of_achievable": None if not achievable else achieved / achievable,
            "launch_ms": launch_ms,
            "timing": f"CUDA events on the launching stream around one {mode} replay of {steps} launches"}


if __name__ == "__main__":
    main()
