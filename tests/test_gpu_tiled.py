"""The tiled mesh kernel (csrc/txb_integrate_tiled.cu): cell tiles with
batch-local vertex tables, the vertex rows gathered once per tile into shared
memory.  Bit-identical to the per-cell fused kernel and to the oracle's
geometry -> gather -> integrate (mesh.py:150-217, _kernels_cy.pyx:37-123)."""

import numpy as np
import pytest

from conftest import bitwise_equal
from oracle import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1607_04245_b200 as txb  # noqa: E402
from paper_1607_04245_b200 import executor  # noqa: E402

FORMS = [(txb.poisson_form, None), (txb.poisson_varcoef_form, "p0"), (txb.poisson_varcoef_form, "p1"),
         (txb.elasticity_form, None)]


def _problem(dim, n, factory, aux_space, seed, shuffle=False, n_cells=None):
    rng = np.random.default_rng(seed)
    mesh = txb.generate_unit_simplex_mesh(dim, n)
    verts = mesh.vertices + 0.15 / n * rng.uniform(-1, 1, mesh.vertices.shape)
    cells = mesh.cells
    if shuffle:  # random vertex numbering and cell order: up to 4 distinct vertices per cell in a tile
        perm = rng.permutation(mesh.n_vertices)
        verts = np.ascontiguousarray(verts[np.argsort(perm)])
        cells = np.ascontiguousarray(perm[cells][rng.permutation(mesh.n_cells)])
    if n_cells is not None:
        cells = np.ascontiguousarray(cells[:n_cells])
    mesh = txb.Mesh(dim, verts, cells)
    form = factory(dim)
    glob = rng.standard_normal(mesh.n_vertices * form.n_comp)
    aux = None
    if aux_space == "p0":
        aux = txb.CellAux("p0", rng.uniform(0.5, 1.5, (mesh.n_cells, 1)))
    elif aux_space == "p1":
        aux = txb.CellAux("p1", rng.uniform(0.5, 1.5, (mesh.n_vertices, 1))[mesh.cells])
    return mesh, form, glob, aux


def _oracle(mesh, form, glob, aux, rule, npdt):
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    tab = txb.tabulate(mesh.dim, rule)
    fc = {"poisson": 0, "poisson_varcoef": 1, "elasticity": 2}[form.name]
    am = {None: 0, "p0": 1, "p1": 2}[None if aux is None else aux.space]
    return oracle.integrate(fc, am, tab.basis, tab.basis_der, rule.weights, inv, det,
                            oracle.gather(mesh.cells, glob, form.n_comp), None if aux is None else aux.values, npdt)


@pytest.mark.parametrize("dim,n,shuffle", [(3, 5, False), (3, 6, True), (2, 30, False), (2, 13, True)])
@pytest.mark.parametrize("tile", [None, 64])
def test_tile_structure(dim, n, shuffle, tile):
    """records: each tile's distinct vertex ids ascending, count first; local:
    each cell's vertices are the listed ids at its local indices."""
    mesh, _, _, _ = _problem(dim, n, txb.poisson_form, None, seed=n, shuffle=shuffle)
    tile = tile or executor.default_tile_cells(dim, 1)
    cells = torch.from_numpy(mesh.cells).cuda()
    t = executor.CellTiles(cells, dim, tile)
    rec = t.records.view(t.n_tiles, t.vrec).cpu().numpy()
    dt = np.uint8 if t.local_bytes == 1 else np.uint16
    loc = t.local.cpu().numpy().view(dt).reshape(t.n_tiles * tile, 4)
    for k in range(t.n_tiles):
        cs = mesh.cells[k * tile:(k + 1) * tile]
        ids = np.unique(cs)
        assert rec[k, 0] == ids.size and not rec[k, 1:4].any()
        np.testing.assert_array_equal(rec[k, 4:4 + ids.size], ids)
        assert not rec[k, 4 + ids.size:].any()
        li = loc[k * tile:k * tile + len(cs), :dim + 1].astype(np.int64)
        np.testing.assert_array_equal(rec[k, 4 + li], cs)
    assert t.max_count == max(np.unique(mesh.cells[k * tile:(k + 1) * tile]).size for k in range(t.n_tiles))
    assert (t.local_bytes == 2) == (t.max_count > 256)


@pytest.mark.parametrize("dim,n,shuffle,n_cells", [(3, 6, False, None), (3, 7, True, 2000), (2, 26, False, 1297),
                                                   (2, 20, True, None)])
@pytest.mark.parametrize("factory,aux_space", FORMS)
def test_tiled_bitwise_vs_oracle_and_per_cell_kernel(dim, n, shuffle, n_cells, factory, aux_space, monkeypatch):
    mesh, form, glob, aux = _problem(dim, n, factory, aux_space, seed=3 * n + dim, shuffle=shuffle, n_cells=n_cells)
    layout = txb.FieldLayout(form.n_comp)
    for rule in (txb.quadrature_rule(dim, 1), txb.two_point_rule(dim)):
        tab = txb.tabulate(dim, rule)
        for dtype, npdt in (("f64", np.float64), ("f32", np.float32)):
            ref = _oracle(mesh, form, glob, aux, rule, npdt)
            g = torch.from_numpy(glob.astype(npdt)).cuda()
            inv, det = oracle.geometry(mesh.vertices, mesh.cells)
            geom = txb.CellGeometry(inv.astype(npdt), det.astype(npdt))
            for mode in ("tiled", "tiled_xpose", "per_cell"):
                monkeypatch.setenv("TXB_TILED", "0" if mode == "per_cell" else "1")
                monkeypatch.setenv("TXB_TILED_XPOSE", "1" if mode == "tiled_xpose" else "0")
                out = txb.integrate_mesh(mesh, layout, tab, rule, form, g, aux, dtype=dtype).cpu().numpy()
                assert bitwise_equal(out, ref), (mode, dtype, rule.n_q)
                # given geometry (cast once to the run precision, as executor.py:77-90): the same bits
                out = txb.integrate_mesh(mesh, layout, tab, rule, form, g, aux, dtype=dtype,
                                         cell_geom=geom).cpu().numpy()
                assert bitwise_equal(out, ref), (mode, dtype, rule.n_q, "given geometry")


@pytest.mark.parametrize("tile", ["64", "96", "192", "256"])
def test_tiled_tile_sizes(tile, monkeypatch):
    """Every legal tile size (a multiple of n_b*n_q and of the warp slice,
    at most 1024 vertex slots; > 6 slices loop over the consumer warps) gives the same bits; an illegal one is a ConfigurationError."""
    for dim in (2, 3):
        mesh, form, glob, aux = _problem(dim, 9 if dim == 3 else 40, txb.poisson_varcoef_form, "p0", seed=7)
        rule = txb.quadrature_rule(dim, 1)
        tab = txb.tabulate(dim, rule)
        ref = _oracle(mesh, form, glob, aux, rule, np.float64)
        monkeypatch.setenv("TXB_TILE_CELLS", tile)
        ok = int(tile) % (dim + 1) == 0 and int(tile) % 32 == 0 and int(tile) * (dim + 1) <= 1024
        g = torch.from_numpy(glob).cuda()
        if ok:
            out = txb.integrate_mesh(mesh, txb.FieldLayout(1), tab, rule, form, g, aux, dtype="f64")
            assert bitwise_equal(out.cpu().numpy(), ref)
        else:
            with pytest.raises(txb.ConfigurationError):
                txb.integrate_mesh(mesh, txb.FieldLayout(1), tab, rule, form, g, aux, dtype="f64")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_tiled_given_geometry_unaligned(dtype):
    """Given geometry whose bases are off 16 bytes (read from global memory,
    not bulk-copied): same bits as the oracle."""
    npdt = np.float64 if dtype == "f64" else np.float32
    tdt = torch.float64 if dtype == "f64" else torch.float32
    for dim in (2, 3):
        mesh, form, glob, aux = _problem(dim, 7 if dim == 3 else 25, txb.poisson_varcoef_form, "p0", seed=13)
        rule = txb.quadrature_rule(dim, 1)
        tab = txb.tabulate(dim, rule)
        ref = _oracle(mesh, form, glob, aux, rule, npdt)
        inv, det = oracle.geometry(mesh.vertices, mesh.cells)
        bi = torch.empty(inv.size + 1, dtype=tdt, device="cuda")
        bd = torch.empty(det.size + 1, dtype=tdt, device="cuda")
        gi, gd = bi[1:].view(inv.shape), bd[1:].view(det.shape)
        gi.copy_(torch.from_numpy(inv.astype(npdt)))
        gd.copy_(torch.from_numpy(det.astype(npdt)))
        out = txb.integrate_mesh(mesh, txb.FieldLayout(1), tab, rule, form, torch.from_numpy(glob.astype(npdt)).cuda(),
                                 aux, dtype=dtype, cell_geom=txb.CellGeometry(gi, gd))
        assert bitwise_equal(out.cpu().numpy(), ref), dim


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_tiled_unaligned_aux_and_out(dtype):
    """aux base off 16 bytes (read from global memory, not bulk-copied) and an
    out view off 16 bytes (scalar stores): same bits."""
    npdt = np.float64 if dtype == "f64" else np.float32
    tdt = torch.float64 if dtype == "f64" else torch.float32
    for dim in (2, 3):
        for factory, aux_space in ((txb.poisson_varcoef_form, "p0"), (txb.poisson_varcoef_form, "p1"),
                                   (txb.elasticity_form, None)):
            mesh, form, glob, aux = _problem(dim, 7 if dim == 3 else 25, factory, aux_space, seed=11)
            rule = txb.quadrature_rule(dim, 1)
            tab = txb.tabulate(dim, rule)
            ref = _oracle(mesh, form, glob, aux, rule, npdt)
            a = None
            if aux is not None:
                vals = aux.values.astype(npdt)
                buf = torch.empty(vals.size + 1, dtype=tdt, device="cuda")
                av = buf[1:].view(vals.shape)
                av.copy_(torch.from_numpy(vals))
                a = txb.CellAux(aux.space, av)
            obuf = torch.empty(ref.size + 1, dtype=tdt, device="cuda")
            out = obuf[1:].view(ref.shape)
            txb.integrate_mesh(mesh, txb.FieldLayout(form.n_comp), tab, rule, form,
                               torch.from_numpy(glob.astype(npdt)).cuda(), a, dtype=dtype, out=out)
            assert bitwise_equal(out.cpu().numpy(), ref), (dim, form.name, aux_space)


def test_tiled_orientation_error_names_first_bad_cell():
    mesh, form, glob, _ = _problem(3, 6, txb.poisson_form, None, seed=2)
    cells = mesh.cells.copy()
    for bad in (700, 1000):  # flip two cells' orientation (swap two vertices)
        cells[bad, [1, 2]] = cells[bad, [2, 1]]
    m = txb.Mesh(3, mesh.vertices, cells)
    rule = txb.quadrature_rule(3, 1)
    with pytest.raises(txb.OrientationError, match="cell 700"):
        txb.integrate_mesh(m, txb.FieldLayout(1), txb.tabulate(3, rule), rule, form, torch.from_numpy(glob).cuda(),
                           None)


def test_tiles_cached_per_connectivity_tensor():
    mesh, form, glob, aux = _problem(3, 5, txb.poisson_varcoef_form, "p0", seed=4)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    cells = torch.from_numpy(mesh.cells).cuda()
    a = executor.cell_tiles(cells, 3, 128)
    assert executor.cell_tiles(cells, 3, 128) is a
    assert executor.cell_tiles(cells[:], 3, 128) is a  # a view of the same memory
    assert executor.cell_tiles(cells.clone(), 3, 128) is not a
    assert executor.cell_tiles(cells[128:], 3, 128) is not a
    out1 = txb.integrate_mesh(mesh, txb.FieldLayout(1), tab, rule, form, torch.from_numpy(glob).cuda(), aux,
                              cells=cells)
    out2 = txb.integrate_mesh(mesh, txb.FieldLayout(1), tab, rule, form, torch.from_numpy(glob).cuda(), aux,
                              cells=cells)
    assert bitwise_equal(out1.cpu().numpy(), out2.cpu().numpy())


@pytest.mark.parametrize("exact_zero", [0, 1])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("seed", [0, 1])
def test_branch_free_geometry_is_correctly_rounded(dim, seed, exact_zero):
    """affine_inverse_fast (reciprocal pair + one Markstein correction, one
    range predicate per cell) against numpy's correctly rounded x / det on
    2^20 random simplices over 12 decades of scale: every cell it accepts is
    equal to numpy (zeros up to sign, which the fused kernels' +0-started
    output chains cannot see; with exact_zero -- the run-time compiled
    kernels' variant -- bit for bit, signed zeros included); cells it rejects
    are redone exactly."""
    import ctypes

    from paper_1607_04245_b200 import _lib

    rng = np.random.default_rng(100 + seed)
    n = 1 << 20
    scale = 10.0 ** rng.uniform(-6, 6, (n, 1, 1))
    x = rng.uniform(-1, 1, (n, dim + 1, dim)) * scale
    x[: n // 8] = np.round(x[: n // 8] * 64) / 64
    x[n // 8: n // 4] *= 2.0 ** rng.integers(-300, 300, (n // 8, 1, 1))  # many out of range: rejected
    verts = x.reshape(-1, dim)
    cells = np.arange(n * (dim + 1), dtype=np.int64).reshape(n, dim + 1)
    with np.errstate(all="ignore"):
        _, det = oracle.geometry(verts, cells)
        flip = det < 0  # orient every simplex positively (swap two vertices)
        cells[flip, 1], cells[flip, 2] = cells[flip, 2].copy(), cells[flip, 1].copy()
        inv, det = oracle.geometry(verts, cells)
    V = torch.from_numpy(verts).cuda()
    C = torch.from_numpy(cells).cuda()
    inv_d = torch.empty((n, dim, dim), dtype=torch.float64, device="cuda")
    det_d = torch.empty(n, dtype=torch.float64, device="cuda")
    ok = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().txb_debug_geometry_fast(dim, n, V.data_ptr(), C.data_ptr(), inv_d.data_ptr(),
                                                  det_d.data_ptr(), ok.data_ptr(), exact_zero, None))
    torch.cuda.synchronize()
    okh = ok.cpu().numpy().astype(bool)
    assert bitwise_equal(det_d.cpu().numpy(), det)
    a = inv_d.cpu().numpy()[okh]
    b = inv[okh]
    assert okh[: n // 8][det[: n // 8] > 0].all() and okh.mean() > 0.8
    assert ((det > 0) | ~okh).all()  # accepted cells are positively oriented and in range
    assert np.array_equal(a, b)  # == treats +0 and -0 as equal
    nz = b != 0
    assert np.array_equal(a[nz].view(np.int64), b[nz].view(np.int64))
    if exact_zero:
        assert np.array_equal(a.view(np.int64), b.view(np.int64))


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("seed", [0, 1])
def test_branch_free_float32_geometry(dim, seed):
    """affine_inverse_fast32 (float32 runs: one product by RN(1/det) per
    quotient, a midpoint-distance test instead of the correction) against
    float32(numpy's correctly rounded float64 x / det) on 2^20 random simplices:
    every accepted cell is bit-identical, signed zeros included; cells whose
    quotient is out of the float32-normal range are rejected."""
    from paper_1607_04245_b200 import _lib

    rng = np.random.default_rng(200 + seed)
    n = 1 << 20
    scale = 10.0 ** rng.uniform(-6, 6, (n, 1, 1))
    x = rng.uniform(-1, 1, (n, dim + 1, dim)) * scale
    x[: n // 8] = np.round(x[: n // 8] * 64) / 64
    x[n // 8: n // 4] *= 2.0 ** rng.integers(-300, 300, (n // 8, 1, 1))
    verts = x.reshape(-1, dim)
    cells = np.arange(n * (dim + 1), dtype=np.int64).reshape(n, dim + 1)
    with np.errstate(all="ignore"):
        _, det = oracle.geometry(verts, cells)
        flip = det < 0
        cells[flip, 1], cells[flip, 2] = cells[flip, 2].copy(), cells[flip, 1].copy()
        inv, det = oracle.geometry(verts, cells)
        inv32, det32 = inv.astype(np.float32), det.astype(np.float32)
    V = torch.from_numpy(verts).cuda()
    C = torch.from_numpy(cells).cuda()
    inv_d = torch.empty((n, dim, dim), dtype=torch.float32, device="cuda")
    det_d = torch.empty(n, dtype=torch.float32, device="cuda")
    ok = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().txb_debug_geometry_fast32(dim, n, V.data_ptr(), C.data_ptr(), inv_d.data_ptr(),
                                                    det_d.data_ptr(), ok.data_ptr(), None))
    torch.cuda.synchronize()
    okh = ok.cpu().numpy().astype(bool)
    assert bitwise_equal(det_d.cpu().numpy(), det32)
    assert okh[: n // 8][det[: n // 8] > 0].all() and okh.mean() > 0.8
    assert ((det > 0) | ~okh).all()
    a, b = inv_d.cpu().numpy()[okh], inv32[okh]
    assert np.array_equal(a.view(np.int32), b.view(np.int32))
    with np.errstate(all="ignore"):
        big = (np.abs(inv) >= 2.0 ** 127).any(axis=(1, 2)) | ((np.abs(inv) < 2.0 ** -125) & (inv != 0)).any(axis=(1, 2))
    assert not okh[big].any()


def test_float32_geometry_rejects_quotients_near_a_rounding_midpoint():
    """A quotient within a few double ulps of a float32 rounding midpoint
    (here 1/e with e = RN(1/(1 + 2^-24)), ~1 + 2^-24) is not decided by the
    one-product shortcut: the cell is rejected and the kernels redo it
    exactly; a neighbouring well-separated cell is accepted."""
    from paper_1607_04245_b200 import _lib

    e = 1.0 / (1.0 + 2.0 ** -24)
    verts = np.array([[0, 0], [1, 0], [0, e], [0, 0], [1, 0], [0, 0.75]], dtype=np.float64)
    cells = np.array([[0, 1, 2], [3, 4, 5]], dtype=np.int64)
    inv, det = oracle.geometry(verts, cells)
    V = torch.from_numpy(verts).cuda()
    C = torch.from_numpy(cells).cuda()
    inv_d = torch.empty((2, 2, 2), dtype=torch.float32, device="cuda")
    det_d = torch.empty(2, dtype=torch.float32, device="cuda")
    ok = torch.empty(2, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().txb_debug_geometry_fast32(2, 2, V.data_ptr(), C.data_ptr(), inv_d.data_ptr(),
                                                    det_d.data_ptr(), ok.data_ptr(), None))
    torch.cuda.synchronize()
    assert ok.cpu().tolist() == [0, 1]
    assert bitwise_equal(inv_d.cpu().numpy()[1], inv[1].astype(np.float32))


@pytest.mark.parametrize("dim", [2, 3])
def test_float32_mesh_near_midpoint_cells_bitwise(dim, monkeypatch):
    """The fused kernels redo a rejected cell exactly: on a structured mesh
    stretched by e = RN(1/(1 + 2^-24)) along one axis, invJ entries sit on
    float32 rounding midpoints (the shortcut rejects those cells), and the
    float32 mesh integration is still bit-identical to the oracle (float64
    geometry cast once) on every path that computes geometry in-kernel."""
    from paper_1607_04245_b200 import _lib

    n = 8 if dim == 2 else 4
    base = txb.generate_unit_simplex_mesh(dim, n)
    v = np.array(base.vertices, dtype=np.float64)
    v[:, 1] *= 1.0 / (1.0 + 2.0 ** -24)
    mesh = txb.Mesh(dim, v, base.cells)
    V = torch.from_numpy(v).cuda()
    C = torch.from_numpy(np.ascontiguousarray(mesh.cells)).cuda()
    nc = mesh.n_cells
    inv_d = torch.empty((nc, dim, dim), dtype=torch.float32, device="cuda")
    det_d = torch.empty(nc, dtype=torch.float32, device="cuda")
    ok = torch.empty(nc, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().txb_debug_geometry_fast32(dim, nc, V.data_ptr(), C.data_ptr(), inv_d.data_ptr(),
                                                    det_d.data_ptr(), ok.data_ptr(), None))
    torch.cuda.synchronize()
    assert (ok.cpu().numpy() == 0).any()  # the fallback is exercised
    rng = np.random.default_rng(dim)
    for factory, aux_space in FORMS:
        form = factory(dim)
        glob = rng.standard_normal(mesh.n_vertices * form.n_comp)
        aux = None
        if aux_space == "p0":
            aux = txb.CellAux("p0", rng.uniform(0.5, 1.5, (nc, 1)))
        elif aux_space == "p1":
            aux = txb.CellAux("p1", rng.uniform(0.5, 1.5, (mesh.n_vertices, 1))[mesh.cells])
        layout = txb.FieldLayout(form.n_comp)
        rule = txb.quadrature_rule(dim, 1)
        tab = txb.tabulate(dim, rule)
        ref = _oracle(mesh, form, glob, aux, rule, np.float32)
        g = torch.from_numpy(glob.astype(np.float32)).cuda()
        for tiled in ("1", "0"):
            monkeypatch.setenv("TXB_TILED", tiled)
            out = txb.integrate_mesh(mesh, layout, tab, rule, form, g, aux, dtype="f32").cpu().numpy()
            assert bitwise_equal(out, ref), (form.name, aux_space, tiled)


def test_tile_builder_rejects_out_of_range_ids():
    cells = torch.tensor([[0, 1, 2, 3], [1, 2, 3, (1 << 31) + 5]], dtype=torch.int64, device="cuda")
    with pytest.raises(IndexError):
        executor.CellTiles(cells, 3, 128)
    cells = torch.tensor([[0, 1, 2, -1]], dtype=torch.int64, device="cuda")
    with pytest.raises(IndexError):
        executor.CellTiles(cells, 3, 128)


def test_tiles_rebuilt_after_in_place_modification():
    """Tables are cached per connectivity tensor; an in-place change through
    torch (version counter) rebuilds them, so the result follows the new cells."""
    mesh, form, glob, aux = _problem(3, 5, txb.poisson_varcoef_form, "p0", seed=5)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    cells = torch.from_numpy(mesh.cells).cuda()
    g = torch.from_numpy(glob).cuda()
    txb.integrate_mesh(mesh, txb.FieldLayout(1), tab, rule, form, g, aux, cells=cells)
    flipped = mesh.cells.copy()
    flipped[:, [1, 2]] = flipped[:, [2, 1]]  # every cell negatively oriented now
    cells.copy_(torch.from_numpy(flipped))
    with pytest.raises(txb.OrientationError):
        txb.integrate_mesh(txb.Mesh(3, mesh.vertices, flipped), txb.FieldLayout(1), tab, rule, form, g, aux,
                           cells=cells)
