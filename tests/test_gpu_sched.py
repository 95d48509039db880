"""Dynamic batch scheduling by cluster launch control (csrc/txb_pipeline.cuh).

Round 1 drew per-launch atomic counters from a rotating slot pool; a captured
CUDA graph baked its slots in, so a graph replayed next to eager launches that
wrapped onto the same slot could share a counter and silently skip batches.
The pipeline now schedules with `clusterlaunchcontrol.try_cancel`: no global
state, nothing to reset, nothing shared between launches.  These tests drive
exactly the hazardous pattern -- two captured graphs replayed concurrently on
two streams while more than 4096 eager launches run on a third -- and require
every result to stay bit-identical to the oracle.
"""

import numpy as np
import pytest

from conftest import bitwise_equal
from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1607_04245_b200 as txb  # noqa: E402
from paper_1607_04245_b200 import backend  # noqa: E402
from paper_1607_04245_b200.physics import CellAux  # noqa: E402


def _problem(n, seed, dim=3, physics="varcoef_p0"):
    B, D, W = oracle.p1_tables(dim)
    _, inv, det, coeffs, aux = oracle.workload(dim, physics, n, seed=seed)
    am = 1 if aux is not None else 0
    fc = 1 if physics == "varcoef_p0" else 2
    want = oracle.integrate(fc, am, B, D, W, inv, det, coeffs, aux, np.float64)
    dev = [None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (inv, det, coeffs, aux)]
    return (fc, am), (B, D, W), dev, want


def test_dynamic_mode_is_cluster_launch_control():
    """The tuned 3D var-coef f64 launch at 2^20 cells is dynamic: the grid has
    one CTA per scheduling unit (more CTAs than can be resident)."""
    cfg = backend.launch_config(1, 1, 8, 3, 1, 1, 1 << 20)
    assert cfg["grid"] > 148 * 8, cfg


def test_concurrent_graph_replays_and_4096_eager_launches():
    kernel, tabs, dev_a, want_a = _problem(200_000, seed=21)
    _, _, dev_b, want_b = _problem(120_000, seed=22)
    kernel_e, tabs_e, dev_e, want_e = _problem(3_000, seed=23, physics="elasticity")

    def launcher(dev, out, stream):
        inv, det, co, aux = dev
        ax = None if aux is None else CellAux("p0", aux)
        return lambda: backend.run_cuda(kernel, *tabs, inv, det, co, ax, out, stream=stream)

    graphs, outs = [], []
    for dev in (dev_a, dev_b):
        out = torch.full(tuple(dev[2].shape), float("nan"), dtype=torch.float64, device="cuda")
        outs.append(out)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            launcher(dev, out, s)()  # warm (module load) outside the capture
        s.synchronize()
        with torch.cuda.graph(g):
            run = launcher(dev, out, torch.cuda.current_stream())
            for _ in range(8):
                run()
        graphs.append(g)
    torch.cuda.synchronize()
    for o in outs:
        o.fill_(float("nan"))
    torch.cuda.synchronize()

    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    out_e = torch.full(tuple(dev_e[2].shape), float("nan"), dtype=torch.float64, device="cuda")
    eager = lambda: backend.run_cuda(kernel_e, *tabs_e, dev_e[0], dev_e[1], dev_e[2], None, out_e,  # noqa: E731
                                     stream=s3)
    mism = 0
    for rnd in range(3):
        with torch.cuda.stream(s1):
            graphs[0].replay()
        with torch.cuda.stream(s2):
            graphs[1].replay()
        with torch.cuda.stream(s3):
            for _ in range(1500):  # 4500 eager launches in all, interleaved with the replays
                eager()
        torch.cuda.synchronize()
        mism += not bitwise_equal(outs[0].cpu().numpy(), want_a)
        mism += not bitwise_equal(outs[1].cpu().numpy(), want_b)
        mism += not bitwise_equal(out_e.cpu().numpy(), want_e)
        for o in (*outs, out_e):
            o.fill_(float("nan"))
    assert mism == 0


def test_dynamic_grid_under_many_streams():
    """Sixteen concurrent dynamic launches on sixteen streams over disjoint
    slices of one output: each CTA cancels only CTAs of its own grid."""
    kernel, tabs, dev, want = _problem(400_000, seed=31)
    out = torch.full(tuple(dev[2].shape), float("nan"), dtype=torch.float64, device="cuda")
    b = np.linspace(0, 400_000, 17).astype(int) // 256 * 256
    b[-1] = 400_000
    streams = [torch.cuda.Stream() for _ in range(16)]
    torch.cuda.synchronize()
    for rep in range(4):
        for i, s in enumerate(streams):
            lo, hi = int(b[i]), int(b[i + 1])
            backend.run_cuda(kernel, *tabs, dev[0][lo:hi], dev[1][lo:hi], dev[2][lo:hi],
                             CellAux("p0", dev[3][lo:hi]), out[lo:hi], stream=s)
        torch.cuda.synchronize()
        assert bitwise_equal(out.cpu().numpy(), want)
        out.fill_(float("nan"))


@pytest.mark.parametrize("pct", ["0", "60", "100"])
def test_static_share_bounds(monkeypatch, pct):
    """TXB_STATIC_PCT 0 (every batch a cancellable unit), 60 (default), 100
    (round-robin only): same bits."""
    monkeypatch.setenv("TXB_STATIC_PCT", pct)
    kernel, tabs, dev, want = _problem(150_001, seed=41)
    out = torch.full(tuple(dev[2].shape), float("nan"), dtype=torch.float64, device="cuda")
    backend.run_cuda(kernel, *tabs, dev[0], dev[1], dev[2], CellAux("p0", dev[3]), out)
    torch.cuda.synchronize()
    assert bitwise_equal(out.cpu().numpy(), want)


def test_mesh_and_jit_kernels_schedule_dynamically():
    """The mesh-fused kernel and a run-time compiled form share the pipeline."""
    mesh = txb.generate_unit_simplex_mesh(3, 40)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    glob = np.random.default_rng(5).standard_normal(mesh.n_vertices)
    kappa = np.random.default_rng(6).uniform(0.5, 1.5, (mesh.n_cells, 1))
    form = txb.poisson_varcoef_form(3)
    elem = txb.integrate_mesh(mesh, txb.FieldLayout(1), tab, rule, form, torch.from_numpy(glob).cuda(),
                              txb.CellAux("p0", torch.from_numpy(kappa).cuda()), dtype="f64")
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    want = oracle.integrate(1, 1, tab.basis, tab.basis_der, rule.weights, inv, det,
                            oracle.gather(mesh.cells, glob, 1), kappa, np.float64)
    assert bitwise_equal(elem.cpu().numpy(), want)
    jit = backend.jit_kernel(form, 1, CellAux("p0", kappa))
    out = torch.empty((mesh.n_cells, 4, 1), dtype=torch.float64, device="cuda")
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    backend.run_cuda(jit, tab.basis, tab.basis_der, rule.weights, d(inv), d(det),
                     d(oracle.gather(mesh.cells, glob, 1)), CellAux("p0", d(kappa)), out)
    torch.cuda.synchronize()
    assert bitwise_equal(out.cpu().numpy(), want)
