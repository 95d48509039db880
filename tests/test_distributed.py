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
