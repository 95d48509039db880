"""Partitioned global assembly with a halo exchange (paper_1607_04245_b200/halo.py).

CPU: plan invariants; world_size 2 and 3 over gloo with the oracle standing
in for the device (element vectors, row gather, CSR chain) and the REAL
all_to_all_single exchange — the gathered owned residuals equal the
reference's np.add.at residual over the whole mesh bit for bit.
GPU: the device path (integration + pack kernel + scatter kernel) for several
emulated ranks in one process (a mailbox stands in for the collective; ranks
run from the highest down, since rank r only receives from ranks above it);
the peer-memory exchange (txb_halo_put / txb_halo_assemble) for a group of
ranks in one process and across processes through CUDA IPC windows."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import bitwise_equal
from oracle import oracle
from paper_1607_04245_b200 import halo
from paper_1607_04245_b200.mesh import generate_unit_simplex_mesh
from paper_1607_04245_b200.shard import all_ranges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def chain_assemble(plan, buf):
    """The CSR chain txb_scatter_add runs: per owned vertex, +0 then each row in order."""
    counts = np.diff(plan.offsets)
    out = np.zeros((plan.owned.size, buf.shape[1]), dtype=buf.dtype)
    for j in range(int(counts.max()) if counts.size else 0):
        live = np.nonzero(counts > j)[0]
        out[live] += buf[plan.incidence[plan.offsets[live] + j]]
    return out


@pytest.mark.parametrize("dim,refine,world,align", [(2, 12, 2, 16), (2, 12, 3, 16), (3, 4, 4, 16), (3, 4, 8, 1),
                                                    (3, 3, 5, 64), (2, 3, 4, 256)])
def test_plan_partitions_every_contribution(dim, refine, world, align):
    mesh = generate_unit_simplex_mesh(dim, refine)
    n, n_b = mesh.cells.shape
    owner = halo.vertex_owners(mesh.cells, mesh.n_vertices, world, align)
    plans = [halo.build_halo_plan(mesh.cells, mesh.n_vertices, r, world, align, owner) for r in range(world)]
    owned = np.concatenate([p.owned for p in plans])
    assert np.array_equal(np.sort(owned), np.unique(mesh.cells))  # each touched vertex owned exactly once
    assert sum(p.offsets[-1] for p in plans) == n * n_b          # every incidence contributes exactly once
    for r, p in enumerate(plans):
        assert (p.lo, p.hi) == all_ranges(n, world, align)[r]
        for s in range(world):  # what r sends to s is what s expects from r
            assert p.send_counts[s] == plans[s].recv_counts[r]
        assert all(p.send_counts[s] == 0 for s in range(r, world))
        assert all(p.recv_counts[s] == 0 for s in range(0, r + 1))
        assert p.incidence.dtype == np.int32 and p.incidence.max(initial=-1) < p.n_local_rows + p.n_recv


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("shuffle", [False, True])
def test_plan_slot_order(world, shuffle):
    """Owned vertices are listed in slot order (first chain row ascending);
    each chain is the vertex's contributions in (rank, cell, b) order — own
    rows first, then each higher rank's received rows — whatever the vertex
    numbering and cell order."""
    mesh = generate_unit_simplex_mesh(3, 4)
    cells = mesh.cells
    if shuffle:
        rng = np.random.default_rng(world)
        cells = rng.permutation(mesh.n_vertices)[cells][rng.permutation(len(cells))]
    n, n_b = cells.shape
    for r in range(world):
        p = halo.build_halo_plan(cells, mesh.n_vertices, r, world, 16)
        first = p.incidence[p.offsets[:-1]]
        assert np.all(np.diff(first) > 0)  # strictly ascending (distinct rows)
        assert np.all(first < p.n_local_rows)  # the owner's own row comes first
        # reference chain of every owned vertex: global incidence positions in ascending order
        flat = cells.ravel()
        for j in np.random.default_rng(r).choice(p.owned.size, min(60, p.owned.size), replace=False):
            v = p.owned[j]
            want = np.nonzero(flat == v)[0]  # (cell, b) positions, ascending = np.add.at order
            got = p.incidence[p.offsets[j]:p.offsets[j + 1]]
            own = want[(want >= p.lo * n_b) & (want < p.hi * n_b)] - p.lo * n_b
            assert np.array_equal(got[:own.size], own)
            assert got.size == want.size and np.all(got[own.size:] >= p.n_local_rows)


def _elem(mesh, lo, hi):
    inv, det = oracle.geometry(mesh.vertices, mesh.cells[lo:hi])
    glob = np.random.default_rng(5).standard_normal(mesh.n_vertices)
    co = oracle.gather(mesh.cells[lo:hi], glob, 1)
    kappa = np.random.default_rng(6).uniform(0.5, 1.5, (mesh.n_cells, 1))[lo:hi]
    B, D, W = oracle.p1_tables(mesh.dim)
    return oracle.integrate(1, 1, B, D, W, inv, det, co, kappa, np.float64)


def _worker(rank, world, port, dim, refine, align, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh = generate_unit_simplex_mesh(dim, refine)
        plan = halo.build_halo_plan(mesh.cells, mesh.n_vertices, rank, world, align)
        buf = np.zeros((plan.n_local_rows + plan.n_recv, 1))
        buf[:plan.n_local_rows] = _elem(mesh, plan.lo, plan.hi).reshape(-1, 1)
        send = torch.from_numpy(np.ascontiguousarray(buf[plan.send_rows]).reshape(-1))
        recv = torch.zeros(plan.n_recv, dtype=torch.float64)
        halo.all_to_all_exchange()(recv, send, plan.recv_counts, plan.send_counts)
        buf[plan.n_local_rows:, 0] = recv.numpy()
        parts = [None] * world
        dist.all_gather_object(parts, (plan.owned, chain_assemble(plan, buf)))
        if rank == 0:
            glob = np.zeros(mesh.n_vertices)
            for ids, vals in parts:
                glob[ids] = vals[:, 0]
            q.put(glob.tobytes())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dim,refine,world,align", [(2, 10, 2, 16), (3, 3, 3, 16)])
def test_gloo_halo_exchange_reproduces_reference_residual(dim, refine, world, align):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = mp.start_processes(_worker, args=(world, _free_port(), dim, refine, align, q), nprocs=world,
                               start_method="spawn", join=False)
    blob = q.get()
    while not procs.join(timeout=60):
        pass
    mesh = generate_unit_simplex_mesh(dim, refine)
    ref = oracle.scatter_add(mesh.cells, _elem(mesh, 0, mesh.n_cells), mesh.n_vertices)
    assert blob == ref.tobytes()


# ------------------------------------------------------------------ GPU ----

class Mailbox:
    def __init__(self):
        self.box = {}

    def exchange_for(self, rank, plan):
        def ex(recv, send, recv_splits, send_splits):
            o = 0
            for p, c in enumerate(send_splits):
                if c:
                    self.box[(rank, p)] = send[o:o + c].clone()
                o += c
            o = 0
            for s, c in enumerate(recv_splits):
                if c:
                    recv[o:o + c].copy_(self.box.pop((s, rank)))
                o += c
        return ex


@pytest.mark.gpu
@pytest.mark.parametrize("world,align", [(1, 256), (2, 256), (3, 64), (8, 16)])
@pytest.mark.parametrize("physics", ["varcoef_p0", "elasticity", "user_elastic_body"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_partitioned_integration_equals_reference_residual(world, align, physics, dtype):
    import paper_1607_04245_b200 as txb
    from oracle import user_forms

    dim = 3
    mesh = txb.generate_unit_simplex_mesh(dim, 9)
    if physics == "user_elastic_body":  # a run-time compiled form (f0, P0 field): its tiled mesh entry point
        form = user_forms.make_form(txb.user_form, "elastic_body", dim)
    else:
        form = txb.poisson_varcoef_form(dim) if physics == "varcoef_p0" else txb.elasticity_form(dim)
    layout = txb.FieldLayout(form.n_comp)
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    glob = np.random.default_rng(1).standard_normal(layout.global_size(mesh))
    aux = None
    if form.n_aux:
        aux = txb.CellAux("p0", np.random.default_rng(2).uniform(0.5, 1.5, (mesh.n_cells, 1)))
    npdt = np.float64 if dtype == "f64" else np.float32
    mb = Mailbox()
    got = np.zeros(layout.global_size(mesh), dtype=npdt)
    for r in reversed(range(world)):
        plan = halo.build_halo_plan(mesh.cells, mesh.n_vertices, r, world, align)
        ids, res, _ = txb.integrate_partitioned(mesh, layout, tab, rule, form, glob, aux, rank=r, world=world,
                                                exchange=mb.exchange_for(r, plan), dtype=dtype, plan=plan)
        torch.cuda.synchronize()
        got.reshape(-1, form.n_comp)[ids] = res.cpu().numpy().reshape(-1, form.n_comp)
    assert not mb.box
    # reference: every cell integrated, then np.add.at over the whole mesh (executor.py:266)
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    co = oracle.gather(mesh.cells, glob, form.n_comp)
    if physics == "user_elastic_body":
        s = user_forms.spec("elastic_body", dim)
        elem = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], tab.basis,
                                      tab.basis_der, rule.weights, inv, det, co, aux.values, npdt)
    else:
        fc = 1 if physics == "varcoef_p0" else 2
        elem = oracle.integrate(fc, 1 if aux is not None else 0, tab.basis, tab.basis_der, rule.weights, inv, det,
                                co, None if aux is None else aux.values, npdt)
    want = oracle.scatter_add(mesh.cells, elem, mesh.n_vertices)
    assert bitwise_equal(got, want)


# ---- peer-memory exchange (txb_halo_put / txb_halo_assemble) ------------------

@pytest.mark.parametrize("world,align", [(2, 16), (3, 16), (8, 1)])
def test_peer_layout_reproduces_reference_residual(world, align):
    """CPU emulation of the window protocol: every rank's owed rows stored at
    peer_send_layout's destinations, then the owner's CSR chain over
    [local rows | window rows] — bit-identical to np.add.at over the mesh."""
    mesh = generate_unit_simplex_mesh(3, 4)
    plans = [halo.build_halo_plan(mesh.cells, mesh.n_vertices, r, world, align) for r in range(world)]
    recv_counts_of = [p.recv_counts for p in plans]
    windows = [np.zeros((p.n_recv, 1)) for p in plans]
    rows = [_elem(mesh, p.lo, p.hi).reshape(-1, 1) for p in plans]
    for r, p in enumerate(plans):
        send_peer, send_dst, out_peers, in_peers = halo.peer_send_layout(p, recv_counts_of)
        assert list(out_peers) == [q for q in range(world) if p.send_counts[q]]
        assert list(in_peers) == [s for s in range(world) if p.recv_counts[s]]
        for i in range(p.n_send):
            windows[send_peer[i]][send_dst[i]] = rows[r][p.send_rows[i]]
    glob = np.zeros(mesh.n_vertices)
    for r, p in enumerate(plans):
        glob[p.owned] = chain_assemble(p, np.concatenate([rows[r], windows[r]]))[:, 0]
    ref = oracle.scatter_add(mesh.cells, _elem(mesh, 0, mesh.n_cells), mesh.n_vertices)
    assert glob.tobytes() == ref.tobytes()


def _residual_ref(mesh, form, tab, rule, glob, aux, npdt):
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    co = oracle.gather(mesh.cells, glob, form.n_comp)
    fc = 1 if form.n_aux else 2
    elem = oracle.integrate(fc, 1 if aux is not None else 0, tab.basis, tab.basis_der, rule.weights, inv, det,
                            co, None if aux is None else aux.values, npdt)
    return oracle.scatter_add(mesh.cells, elem, mesh.n_vertices)


@pytest.mark.gpu
@pytest.mark.parametrize("world,align", [(1, 256), (2, 256), (3, 64), (8, 16)])
@pytest.mark.parametrize("physics,dtype", [("varcoef_p0", "f64"), ("elasticity", "f32")])
def test_peer_exchange_single_process_group(world, align, physics, dtype):
    """All ranks in this process on one stream, highest rank first (rank r only
    waits for rows from ranks above it, and for acks two epochs old); four
    epochs with new coefficients each (slot reuse, acks)."""
    import paper_1607_04245_b200 as txb

    dim = 3
    mesh = txb.generate_unit_simplex_mesh(dim, 9)
    form = txb.poisson_varcoef_form(dim) if physics == "varcoef_p0" else txb.elasticity_form(dim)
    layout = txb.FieldLayout(form.n_comp)
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    npdt = np.float64 if dtype == "f64" else np.float32
    aux = None
    if form.n_aux:
        aux = txb.CellAux("p0", np.random.default_rng(2).uniform(0.5, 1.5, (mesh.n_cells, 1)))
    plans = [halo.build_halo_plan(mesh.cells, mesh.n_vertices, r, world, align) for r in range(world)]
    group = halo.local_peer_group(plans, form.n_comp, np.dtype(npdt).itemsize)
    try:
        for epoch in range(4):
            glob = np.random.default_rng(10 + epoch).standard_normal(layout.global_size(mesh))
            outs = [txb.integrate_partitioned(mesh, layout, tab, rule, form, glob, aux, rank=r, world=world,
                                              dtype=dtype, peer=group[r]) for r in reversed(range(world))]
            torch.cuda.synchronize()
            for g in group:
                g.check()
            got = np.zeros(layout.global_size(mesh), dtype=npdt)
            for ids, res, _ in outs:
                got.reshape(-1, form.n_comp)[ids] = res.cpu().numpy().reshape(-1, form.n_comp)
            assert bitwise_equal(got, _residual_ref(mesh, form, tab, rule, glob, aux, npdt)), epoch
    finally:
        group[0].close()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_across_processes_via_ipc(world):
    """Real CUDA IPC windows between processes (all on cuda:0 here; one per GPU
    in production): three epochs, gathered residual bit-identical to the oracle."""
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parents[1]
    env = dict(os.environ, TXB_HALO_TIMEOUT_MS="20000")
    r = subprocess.run([sys.executable, str(repo / "tools" / "peer_ipc_check.py"), str(world)], cwd=repo, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "bit-identical" in r.stdout, (r.stdout + r.stderr)[-3000:]


@pytest.mark.gpu
def test_peer_exchange_failed_sender_is_reported(monkeypatch):
    """A sender whose put times out waiting for an ack publishes a POISONED flag
    instead of a clean one: the owner reports error 3 and its owned residual is
    NaN -- never a stale slot assembled as if it were fresh."""
    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200.errors import CudaLaneError

    monkeypatch.setenv("TXB_HALO_TIMEOUT_MS", "200")
    dim, world = 3, 2
    mesh = txb.generate_unit_simplex_mesh(dim, 6)
    form = txb.poisson_form(dim)
    layout = txb.FieldLayout(1)
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    plans = [halo.build_halo_plan(mesh.cells, mesh.n_vertices, r, world, 16) for r in range(world)]
    assert plans[1].n_send > 0 and plans[0].n_recv > 0
    group = halo.local_peer_group(plans, 1, 8)
    glob = np.random.default_rng(3).standard_normal(layout.global_size(mesh))
    try:
        # rank 1 runs three epochs while rank 0 never assembles (never acks):
        # epoch 3's put times out on epoch 1's ack and poisons its flag
        for _ in range(3):
            txb.integrate_partitioned(mesh, layout, tab, rule, form, glob, None, rank=1, world=world,
                                      peer=group[1], check=False)
        torch.cuda.synchronize()
        with pytest.raises(CudaLaneError, match="ack"):
            group[1].check()
        with pytest.raises(CudaLaneError, match="poisoned"):
            txb.integrate_partitioned(mesh, layout, tab, rule, form, glob, None, rank=0, world=world,
                                      peer=group[0])
        ids, res, _ = txb.integrate_partitioned(mesh, layout, tab, rule, form, glob, None, rank=0, world=world,
                                                peer=group[0], check=False)
        torch.cuda.synchronize()
        assert torch.isnan(res).all()
    finally:
        group[0].close()
