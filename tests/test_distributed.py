"""Multi-process (world_size 2, gloo, CPU) coverage of the cell-range sharding
used by bench.py under torchrun: ranges are disjoint, cover every cell, keep
16-byte alignment, and per-rank integration of the owned range (CPU oracle as
the stand-in device) reassembles to the single-process result bit for bit;
the timing reduction is the max over ranks."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1607_04245_b200.shard import all_ranges, cell_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("n,world,align", [(0, 2, 16), (1, 2, 16), (1000, 2, 16), (1 << 20, 8, 256),
                                           (12345, 3, 64), (5, 8, 16)])
def test_ranges_partition_the_cells(n, world, align):
    rs = all_ranges(n, world, align)
    assert rs[0][0] == 0 and rs[-1][1] == n
    for (a, b), (c, d) in zip(rs, rs[1:]):
        assert b == c and a <= b
    for lo, hi in rs[:-1]:
        assert lo % align == 0 and hi % align == 0 or hi == n
    sizes = [hi - lo for lo, hi in rs]
    assert max(sizes) - min(sizes) <= align


def _worker(rank, world, port, n, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle

        _, inv, det, coeffs, aux = oracle.workload(3, "varcoef_p0", n, seed=11)
        B, D, W = oracle.p1_tables(3)
        lo, hi = cell_range(n, rank, world, align=16)
        mine = oracle.integrate(1, 1, B, D, W, inv[lo:hi], det[lo:hi], coeffs[lo:hi], aux[lo:hi], np.float64)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, mine))
        # max-over-ranks timing reduction, as bench.py does with NCCL
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            full = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])])
            result_q.put((full.tobytes(), float(t[0])))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_reassembles_bitwise():
    from oracle import oracle

    n = 5003
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    ctxp = mp.start_processes(_worker, args=(2, _free_port(), n, q), nprocs=2, start_method="spawn", join=False)
    blob, tmax = q.get()  # drain before joining (the result is larger than a pipe buffer)
    while not ctxp.join(timeout=60):
        pass
    _, inv, det, coeffs, aux = oracle.workload(3, "varcoef_p0", n, seed=11)
    B, D, W = oracle.p1_tables(3)
    ref = oracle.integrate(1, 1, B, D, W, inv, det, coeffs, aux, np.float64)
    assert blob == ref.tobytes()
    assert tmax == 2.0


# ---------------------------------------------------------------------------
# bench.py's own rank logic (not a stand-in): input generation of a rank's
# range, the max-over-ranks reduction, the per-rank cell counts, and the
# buffer-set / launch arithmetic the driver's short runs depend on.
# ---------------------------------------------------------------------------
import bench  # noqa: E402


@pytest.mark.parametrize("steps", [1, 20, 4000])
@pytest.mark.parametrize("warmup", [3, 5, 10])
@pytest.mark.parametrize("name", sorted(bench.CONFIGS))
def test_bench_sets_are_all_written_before_the_check(name, steps, warmup):
    """Every buffer set gets written during warm-up (the determinism check
    compares all of them), and the rotation keeps reuse distance > 3 x L2."""
    _, bytes_cell = bench.config_model(name)
    n = bench.CONFIGS[name][3]
    for k in (steps, bench.variant_steps(n, steps)):
        ns = bench.rotating_sets(bytes_cell * n)
        assert 4 <= ns <= 64
        assert bench.warmup_launches(warmup, ns) >= max(warmup, ns)
        assert (ns - 1) * bytes_cell * n > 3 * bench.L2_BYTES or ns == 64
        assert k >= 1


def test_bench_variant_steps_bounded():
    assert bench.variant_steps(1 << 20, 20) == 200
    assert bench.variant_steps(1 << 20, 4000) == 1000
    assert bench.variant_steps(1 << 24, 20) == 40


def _bench_rank_worker(rank, world, port, name, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = bench.rank_host_inputs(name, rank, world)
        from oracle import oracle

        B, D, W = oracle.p1_tables(bench.CONFIGS[name][0])
        inv, det = oracle.geometry(h["vertices"], h["cells"])
        co = oracle.gather(h["cells"], h["glob"], h["form"].n_comp)
        am = 1 if h["kappa"] is not None else 0
        fc = {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}[h["form"].name]
        mine = oracle.integrate(fc, am, B, D, W, inv, det, co, h["kappa"], np.float64)
        parts = [None] * world
        dist.all_gather_object(parts, (h["lo"], h["hi"], mine.tobytes(), h["cells"].tobytes()))
        t = bench.reduce_max_over_ranks(float(10 * rank + 1), world, dist, "cpu")
        if rank == 0:
            parts.sort(key=lambda p: p[0])
            result_q.put((b"".join(p[2] for p in parts), b"".join(p[3] for p in parts),
                          [p[1] - p[0] for p in parts], t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["2d_varcoef_f64_65536"])
def test_bench_rank_logic_two_ranks_gloo(name):
    """bench.rank_host_inputs on 2 gloo ranks: each rank generates ONLY its
    cell range; concatenated, ranges and results equal the single-process
    workload of the 2 x per-GPU-cell job bit for bit; the timing reduction is
    the max over ranks; cell_counts matches the ranges."""
    from oracle import oracle

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    pc = mp.start_processes(_bench_rank_worker, args=(world, _free_port(), name, q), nprocs=world,
                            start_method="spawn", join=False)
    blob, cells_blob, counts, tmax = q.get()
    while not pc.join(timeout=120):
        pass
    h = bench.rank_host_inputs(name, 0, 1)  # world 1: rank 0 owns exactly the per-GPU cells
    dim, physics, _, per_gpu = bench.CONFIGS[name]
    from paper_1607_04245_b200.mesh import generate_unit_simplex_mesh
    from paper_1607_04245_b200.workload import refine_for

    full = generate_unit_simplex_mesh(dim, refine_for(dim, world * per_gpu))
    cells = full.cells[:world * per_gpu]
    assert cells_blob == np.ascontiguousarray(cells).tobytes()
    glob = np.random.default_rng(1234).standard_normal(full.n_vertices)
    kappa = np.random.default_rng(1235).uniform(0.5, 1.5, (full.n_cells, 1))[:world * per_gpu]
    B, D, W = oracle.p1_tables(dim)
    inv, det = oracle.geometry(full.vertices, cells)
    ref = oracle.integrate(1, 1, B, D, W, inv, det, oracle.gather(cells, glob, 1), kappa, np.float64)
    assert blob == ref.tobytes()
    assert counts == bench.cell_counts(per_gpu, world) and sum(counts) == world * per_gpu
    assert tmax == 11.0
    assert h["hi"] == per_gpu
