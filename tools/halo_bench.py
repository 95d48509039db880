"""Partitioned global residual across GPUs: integration + halo exchange
(NCCL all_to_all vs the peer-memory windows), device time max over ranks.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/halo_bench.py [cells_per_gpu]
  python tools/halo_bench.py --local W [cells_per_rank]   (W emulated ranks in one process on one GPU)

One process per GPU of one node.  Each rank owns a contiguous range of a
Kuhn mesh of N x cells_per_gpu tetrahedra (3D var-coef f64), integrates it
(fused mesh kernel) and assembles its owned vertices; the gathered residual is
checked against a single-GPU residual of the same mesh on rank 0 (bitwise).
Rank 0 prints one JSON line per exchange path.  (Tuning / evaluation aid; not
part of bench.py's contract.)
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.distributed as dist

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200 import halo
    from paper_1607_04245_b200.workload import refine_for

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    per_gpu = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    dim = 3
    full = txb.generate_unit_simplex_mesh(dim, refine_for(dim, per_gpu * world))
    mesh = txb.Mesh(dim, full.vertices, np.ascontiguousarray(full.cells[:per_gpu * world]))
    form = txb.poisson_varcoef_form(dim)
    layout = txb.FieldLayout(1)
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    glob = np.random.default_rng(1).standard_normal(mesh.n_vertices)
    aux = txb.CellAux("p0", np.random.default_rng(2).uniform(0.5, 1.5, (mesh.n_cells, 1)))
    plan = halo.build_halo_plan(mesh.cells, mesh.n_vertices, rank, world)
    peer = halo.distributed_peer_halo(plan, 1, 8)
    glob_dev = torch.from_numpy(glob).cuda()
    aux_dev = txb.CellAux("p0", torch.from_numpy(aux.values).cuda())

    def run(path):
        if path == "nccl":
            return txb.integrate_partitioned(mesh, layout, tab, rule, form, glob_dev, aux_dev, rank=rank,
                                             world=world, exchange=halo.all_to_all_exchange(), plan=plan)
        return txb.integrate_partitioned(mesh, layout, tab, rule, form, glob_dev, aux_dev, rank=rank, world=world,
                                         peer=peer)

    ref = None
    if rank == 0:
        ref, _ = txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=32, n_cb=8,
                                          shared_mem_limit=None)
    for path in ("nccl", "peer"):
        for _ in range(3):
            run(path)
        torch.cuda.synchronize()
        steps = 20
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            ids, res, _ = run(path)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if path == "peer":
            peer.check()
        parts = [None] * world
        dist.all_gather_object(parts, (ids, res.cpu().numpy()))
        if rank == 0:
            got = np.zeros(mesh.n_vertices)
            for i, v in parts:
                got[i] = v
            print(json.dumps({"path": path, "n_gpus": world, "cells": mesh.n_cells, "ms_per_residual": float(t[0]),
                              "halo_rows_per_rank": [int(plan.n_send)], "bitwise_equal": got.tobytes() == ref.tobytes()}),
                  flush=True)
    dist.barrier()
    peer.close()
    dist.destroy_process_group()


def local(world, per_rank):
    """All ranks in this process on one stream (highest rank first), peer
    windows in device memory: the summed device time of one residual over all
    ranks (integration + put + assembly per rank), the gathered residual
    checked bitwise across repeats."""
    import torch

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200 import halo
    from paper_1607_04245_b200.workload import refine_for

    dim = 3
    full = txb.generate_unit_simplex_mesh(dim, refine_for(dim, per_rank * world))
    mesh = txb.Mesh(dim, full.vertices, np.ascontiguousarray(full.cells[:per_rank * world]))
    form, layout = txb.poisson_varcoef_form(dim), txb.FieldLayout(1)
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    glob = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_vertices)).cuda()
    aux = txb.CellAux("p0", torch.from_numpy(np.random.default_rng(2).uniform(0.5, 1.5, (mesh.n_cells, 1))).cuda())
    plans = [halo.build_halo_plan(mesh.cells, mesh.n_vertices, r, world) for r in range(world)]
    group = halo.local_peer_group(plans, 1, 8)

    def residual():
        return [txb.integrate_partitioned(mesh, layout, tab, rule, form, glob, aux, rank=r, world=world,
                                          peer=group[r]) for r in reversed(range(world))]

    ref = None
    for _rep in range(2):
        for _ in range(3):
            residual()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            outs = residual()
        e1.record()
        torch.cuda.synchronize()
        for g in group:
            g.check()
        got = np.zeros(mesh.n_vertices)
        for ids, res, _ in outs:
            got[ids] = res.cpu().numpy()
        ref = got if ref is None else ref
        print(json.dumps({"mode": "local", "world": world, "cells_per_rank": per_rank,
                          "ms_per_residual_all_ranks": e0.elapsed_time(e1) / 10,
                          "rows_sent_per_rank": [int(p.n_send) for p in plans],
                          "same_bits": got.tobytes() == ref.tobytes()}), flush=True)
    group[0].close()


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--local":
        local(int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 20)
    else:
        main()
