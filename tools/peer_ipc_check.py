"""Cross-process check of the peer-memory halo exchange on ONE GPU: two (or
more) processes share their windows by CUDA IPC handle and run several
epochs; rank 0 compares the gathered residual with the oracle bit for bit.
(On one device the processes' kernels time-slice, so the spin-waits resolve
at context switches: a correctness check, not a timing.)

python tools/peer_ipc_check.py [world]
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1607_04245_b200 as txb
        from oracle import oracle
        from paper_1607_04245_b200 import halo

        dim = 3
        mesh = txb.generate_unit_simplex_mesh(dim, 8)
        form = txb.poisson_varcoef_form(dim)
        layout = txb.FieldLayout(1)
        rule = txb.quadrature_rule(dim, 1)
        tab = txb.tabulate(dim, rule)
        aux = txb.CellAux("p0", np.random.default_rng(2).uniform(0.5, 1.5, (mesh.n_cells, 1)))
        plan = halo.build_halo_plan(mesh.cells, mesh.n_vertices, rank, world, 64)
        peer = halo.distributed_peer_halo(plan, 1, 8)
        ok = True
        for epoch in range(3):
            glob = np.random.default_rng(30 + epoch).standard_normal(mesh.n_vertices)
            ids, res, _ = txb.integrate_partitioned(mesh, layout, tab, rule, form, glob, aux, rank=rank,
                                                    world=world, peer=peer)
            torch.cuda.synchronize()
            peer.check()
            parts = [None] * world
            dist.all_gather_object(parts, (ids, res.cpu().numpy()))
            if rank == 0:
                got = np.zeros(mesh.n_vertices)
                for i, v in parts:
                    got[i] = v
                inv, det = oracle.geometry(mesh.vertices, mesh.cells)
                elem = oracle.integrate(1, 1, tab.basis, tab.basis_der, rule.weights, inv, det,
                                        oracle.gather(mesh.cells, glob, 1), aux.values)
                ok &= got.tobytes() == oracle.scatter_add(mesh.cells, elem, mesh.n_vertices).tobytes()
        dist.barrier()
        peer.close()
        if rank == 0:
            q.put(ok)
    finally:
        dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = mp.start_processes(worker, args=(world, port, q), nprocs=world, start_method="spawn", join=False)
    ok = q.get()
    while not procs.join(timeout=120):
        pass
    print(f"peer_ipc_check world={world}: {'bit-identical to the oracle' if ok else 'MISMATCH'}")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
