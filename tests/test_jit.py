"""Run-time compiled user physics (§8f row 4): the reference's string-injection
forms (txfem/physics.py:110-168, 260-304) compiled by NVRTC for sm_100a.

CPU tests: compilation (NVRTC needs no device), generated text, cubin
contents, the error surface (CodegenError / ValueError like the reference).
GPU tests: element vectors bit-identical to the reference's python lane
(tests/golden/user_cases.npz) and to the oracle's restatement of it on larger
seeded inputs; the shipped forms compiled at run time equal the ahead-of-time
kernel bit for bit; the mesh-level driver routes user forms through it."""

import os
import shutil
import subprocess

import numpy as np
import pytest

import paper_1607_04245_b200 as txb
from conftest import TOL, USER_CASES, bitwise_equal, rel_err
from oracle import oracle, user_forms
from paper_1607_04245_b200.physics import CellAux

SPECS = sorted(user_forms.SPECS)


def form_of(name, dim):
    return user_forms.make_form(txb.user_form, name, dim)


def aux_for(spec, n, rng, dtype=np.float64):
    if spec["aux"] is None:
        return None
    shape = (n, spec["n_aux"]) if spec["aux"] == "p0" else (n, spec["dim"] + 1, spec["n_aux"])
    return CellAux(spec["aux"], rng.uniform(0.5, 1.5, shape).astype(dtype))


# ------------------------------------------------------------------ CPU ----

@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("name", SPECS)
@pytest.mark.parametrize("width", [4, 8])
def test_user_forms_compile(name, dim, width):
    s = user_forms.spec(name, dim)
    f = form_of(name, dim)
    k = txb.jit_kernel(f, 1, aux_for(s, 2, np.random.default_rng(0)), width)
    assert f"f1_{name}" in k.source and "#include \"txb_jit_kernel.cuh\"" in k.source
    assert ("#define TXB_HAS_F0 1" in k.source) == f.has_f0
    assert len(k.cubin) > 1000
    # memoised on the generated text: same handle
    assert txb.jit_kernel(f, 1, aux_for(s, 2, np.random.default_rng(0)), width).handle == k.handle


@pytest.mark.skipif(shutil.which("cuobjdump") is None, reason="cuobjdump not on PATH")
def test_jit_cubin_is_sm100a_bulk_copy_pipeline(tmp_path):
    f = form_of("advect", 3)
    k = txb.jit_kernel(f, 2, aux_for(user_forms.spec("advect", 3), 2, np.random.default_rng(0)), 8)
    p = tmp_path / "k.cubin"
    p.write_bytes(k.cubin)
    sass = subprocess.run(["cuobjdump", "-sass", str(p)], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in sass
    assert "UBLKCP" in sass  # cp.async.bulk global -> shared (the batch loader)
    assert "SYNCS" in sass   # mbarrier ring
    funcs = {}
    for part in sass.split("Function : ")[1:]:
        funcs[part.split()[0]] = part
    assert {"txb_jit_integrate", "txb_jit_integrate_std"} <= set(funcs)  # mesh entry points: own program
    # -fmad=false: every product and sum rounds on its own
    assert "DFMA" not in funcs["txb_jit_integrate"] and "DFMA" not in funcs["txb_jit_integrate_std"]
    res = subprocess.run(["cuobjdump", "-res-usage", str(p)], capture_output=True, text=True, check=True).stdout
    assert "LOCAL:0" in res  # no spills


def test_shipped_forms_have_compilable_sources():
    for dim in (2, 3):
        for f in (txb.poisson_form(dim), txb.poisson_varcoef_form(dim), txb.elasticity_form(dim)):
            aux = CellAux("p0", np.ones((1, 1))) if f.n_aux else None
            txb.jit_kernel(f, 2, aux, 8)


def test_compile_errors_raise_codegen_error_with_log():
    bad = txb.user_form("bad", 2, 1, None, 0, "realv f1_bad(const real u[], const realv gradU[], const real a[], "
                        "const realv gradA[], int comp) { return gradU[comp] + undefined_symbol; }")
    with pytest.raises(txb.CodegenError, match="undefined_symbol"):
        txb.jit_kernel(bad, 1, None, 8)


def test_missing_sources_raise_codegen_error():
    f = txb.user_form("nosrc", 2, 1, lambda s, c: s.grad_u[c], 0, "")
    with pytest.raises(txb.CodegenError):
        txb.jit_kernel(f, 1, None, 8)
    g = txb.user_form("nof0src", 2, 1, lambda s, c: s.grad_u[c], 0, user_forms.spec("reaction", 2)["source_f1"],
                      f0=lambda s, c: s.u[c])
    with pytest.raises(txb.CodegenError):
        txb.jit_kernel(g, 1, None, 8)


def test_coverage_errors():
    f = form_of("reaction", 2)
    with pytest.raises(ValueError):
        txb.jit_kernel(f, 9, None, 8)  # n_q > 8
    with pytest.raises(ValueError):  # name is not a C identifier
        txb.jit_kernel(txb.user_form("not-an-id", 2, 1, None, 0, "x"), 1, None, 8)
    many = CellAux("p0", np.ones((1, 5)))
    g = txb.user_form("many_aux", 2, 1, None, 0, user_forms.spec("reaction", 2)["source_f1"].replace(
        "f1_reaction", "f1_many_aux"), n_aux=5)
    with pytest.raises(ValueError):
        txb.jit_kernel(g, 1, many, 8)  # n_aux > 4


def test_cuda_kernel_routes_user_forms_to_the_jit_lane():
    assert isinstance(txb.cuda_kernel(txb.poisson_form(3), 1, None, 8), tuple)  # ahead-of-time
    k = txb.cuda_kernel(form_of("reaction", 3), 1, None, 8)
    assert isinstance(k, txb.JitKernel) and k.has_f0
    aux2 = CellAux("p1", np.ones((1, 4, 1)))
    f = txb.poisson_varcoef_form(3)
    assert isinstance(txb.cuda_kernel(f, 1, aux2, 8), tuple)


# ------------------------------------------------------------------ GPU ----

def _dev(x, dt):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).cuda()


def _run(kernel, B, D, W, inv, det, co, aux, dt, n_bl=0, n_cb=0):
    import torch

    out = torch.empty(co.shape, dtype=torch.float64 if dt == np.float64 else torch.float32, device="cuda")
    ax = None if aux is None else CellAux(aux.space, _dev(aux.values, dt))
    txb.run_cuda(kernel, B, D, W, _dev(inv, dt), _dev(det, dt), _dev(co, dt), ax, out, n_bl=n_bl, n_cb=n_cb)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.gpu
@pytest.mark.parametrize("case", USER_CASES, ids=lambda c: c.name)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_jit_bitwise_matches_reference_python_lane(case, dtype):
    dt = np.float64 if dtype == "f64" else np.float32
    f = form_of(case.spec, case.dim)
    aux = None if case.aux is None else CellAux(case.aux_space, case.aux)
    k = txb.cuda_kernel(f, case.n_q, aux, np.dtype(dt).itemsize)
    assert isinstance(k, txb.JitKernel)
    got = _run(k, case.basis, case.basis_der, case.weights, case.inv_j, case.det_j, case.coeffs, aux, dt)
    want = case.py_f64 if dtype == "f64" else case.py_f32
    assert rel_err(got, want) <= TOL[dtype]
    assert bitwise_equal(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SPECS)
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("n", [0, 1, 33, 4099, 100_003])
def test_jit_matches_oracle_ragged_sizes(name, dim, n):
    rng = np.random.default_rng(n + dim)
    s = user_forms.spec(name, dim)
    f = form_of(name, dim)
    jac = np.eye(dim) + 0.2 * rng.uniform(-1, 1, (n, dim, dim))
    inv, det = np.linalg.inv(jac) if n else np.zeros((0, dim, dim)), np.linalg.det(jac) if n else np.zeros(0)
    co = rng.standard_normal((n, dim + 1, s["n_comp"]))
    aux = aux_for(s, n, rng)
    B, D, W = oracle.p1_tables(dim, 2)
    for dt in (np.float64, np.float32):
        k = txb.cuda_kernel(f, 2, aux, np.dtype(dt).itemsize)
        got = _run(k, B, D, W, inv, det, co, aux, dt)
        want = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], B, D, W, inv, det,
                                      co, None if aux is None else aux.values, dt)
        assert bitwise_equal(got, want), (name, dim, n, dt)


@pytest.mark.gpu
@pytest.mark.parametrize("n_q", [1, 3, 5, 8])
def test_jit_arbitrary_tabulation_and_decompositions(n_q):
    rng = np.random.default_rng(n_q)
    dim, n = 3, 5000
    s = user_forms.spec("advect", dim)
    f = form_of("advect", dim)
    B = rng.uniform(0, 1, (n_q, dim + 1))
    D = rng.uniform(-1, 1, (n_q, dim + 1, dim))
    W = rng.uniform(0.1, 0.5, n_q)
    jac = np.eye(dim) + 0.2 * rng.uniform(-1, 1, (n, dim, dim))
    inv, det = np.linalg.inv(jac), np.linalg.det(jac)
    co = rng.standard_normal((n, dim + 1, 1))
    aux = aux_for(s, n, rng)
    want = oracle.integrate_forms(s["f1_many"], s["f0_many"], True, "p1", B, D, W, inv, det, co, aux.values)
    k = txb.cuda_kernel(f, n_q, aux, 8)
    for n_bl, n_cb in ((0, 0), (1, 1), (2, 4), (8, 3)):
        got = _run(k, B, D, W, inv, det, co, aux, np.float64, n_bl=n_bl, n_cb=n_cb)
        assert bitwise_equal(got, want), (n_bl, n_cb)


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("physics", ["poisson", "varcoef_p0", "varcoef_p1", "elasticity"])
def test_shipped_forms_jit_equals_ahead_of_time_kernel(dim, physics):
    rng = np.random.default_rng(dim)
    n = 20_011
    factory = {"poisson": txb.poisson_form, "varcoef_p0": txb.poisson_varcoef_form,
               "varcoef_p1": txb.poisson_varcoef_form, "elasticity": txb.elasticity_form}[physics]
    f = factory(dim)
    jac = np.eye(dim) + 0.2 * rng.uniform(-1, 1, (n, dim, dim))
    inv, det = np.linalg.inv(jac), np.linalg.det(jac)
    co = rng.standard_normal((n, dim + 1, f.n_comp))
    aux = None
    if physics == "varcoef_p0":
        aux = CellAux("p0", rng.uniform(0.5, 1.5, (n, 1)))
    elif physics == "varcoef_p1":
        aux = CellAux("p1", rng.uniform(0.5, 1.5, (n, dim + 1, 1)))
    for n_q in (1, 2):
        B, D, W = oracle.p1_tables(dim, n_q)
        for dt in (np.float64, np.float32):
            w = np.dtype(dt).itemsize
            aot = txb.cuda_kernel(f, n_q, aux, w)
            assert isinstance(aot, tuple)
            jit = txb.jit_kernel(f, n_q, aux, w)
            a = _run(aot, B, D, W, inv, det, co, aux, dt)
            b = _run(jit, B, D, W, inv, det, co, aux, dt)
            assert bitwise_equal(a, b), (physics, n_q, dt)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SPECS)
@pytest.mark.parametrize("dim", [2, 3])
def test_jit_standard_table_entry_point_matches_generic(name, dim, monkeypatch):
    """The standard-P1-table entry point (txb_jit_integrate_std: T[0] = -sum of
    invJ rows, T[b] = invJ rows) and the generic one give the oracle's bits on
    a structured mesh, whose inverse Jacobians are full of exact +-0 (the sign
    of zero is where the two pull-backs may differ), midpoint and two-point
    rules, both precisions."""
    s = user_forms.spec(name, dim)
    f = form_of(name, dim)
    mesh = txb.generate_unit_simplex_mesh(dim, 14 if dim == 2 else 5)
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    assert (inv == 0).mean() > 0.2
    n = mesh.n_cells
    rng = np.random.default_rng(17)
    co = rng.standard_normal((n, dim + 1, f.n_comp))
    co[::7] = 0.0  # zero coefficient blocks: signed-zero products in grad u
    aux = aux_for(s, n, rng)
    for rule in (txb.quadrature_rule(dim, 1), txb.two_point_rule(dim)):
        tab = txb.tabulate(dim, rule)
        for dt in (np.float64, np.float32):
            k = txb.jit_kernel(f, rule.n_q, aux, np.dtype(dt).itemsize)
            want = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], tab.basis,
                                          tab.basis_der, rule.weights, inv, det, co,
                                          None if aux is None else aux.values, dt)
            monkeypatch.setenv("TXB_DISABLE_STD", "0")
            std = _run(k, tab.basis, tab.basis_der, rule.weights, inv, det, co, aux, dt)
            monkeypatch.setenv("TXB_DISABLE_STD", "1")
            gen = _run(k, tab.basis, tab.basis_der, rule.weights, inv, det, co, aux, dt)
            assert bitwise_equal(std, want), (rule.n_q, dt)
            assert bitwise_equal(gen, want), (rule.n_q, dt)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SPECS)
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("tiled", ["1", "0"])
@pytest.mark.parametrize("stretch", [False, True])
def test_integrate_transposed_user_forms_mesh_fused(name, dim, dtype, tiled, stretch, monkeypatch):
    """integrate_transposed with a run-time compiled form: the mesh entry point
    (float64 geometry + gather in-kernel, txb_jit_integrate_mesh) on a perturbed
    Kuhn mesh with a shuffled vertex numbering, midpoint and two-point rules,
    then the scatter-add — bit-identical to the oracle's geometry -> gather ->
    python-lane integration -> np.add.at, and to the unfused route (given
    geometry: gather + txb_jit_integrate).  tiled = 1: the tiled mesh entry
    point (txb_jit_integrate_mesh_tiled, per-tile vertex tables).  stretch:
    an unperturbed mesh stretched by RN(1/(1 + 2^-24)) along y, whose invJ
    entries sit on float32 rounding midpoints (the float32 geometry shortcut
    rejects those cells and the kernels redo them exactly)."""
    if stretch and dtype == "f64":
        pytest.skip("midpoint cells only matter for the float32 geometry path")
    monkeypatch.setenv("TXB_TILED", tiled)
    s = user_forms.spec(name, dim)
    f = form_of(name, dim)
    npdt = np.float64 if dtype == "f64" else np.float32
    base = txb.generate_unit_simplex_mesh(dim, (8 if stretch else 11) if dim == 2 else 4)
    rng = np.random.default_rng(dim * 7 + len(name))
    perm = rng.permutation(base.n_vertices)
    if stretch:
        verts = base.vertices[np.argsort(perm)] * np.array([1.0, 1.0 / (1.0 + 2.0 ** -24), 1.0][:dim])
    else:
        verts = base.vertices[np.argsort(perm)] + 0.02 * rng.uniform(-1, 1, base.vertices.shape)
    mesh = txb.Mesh(dim, np.ascontiguousarray(verts), np.ascontiguousarray(perm[base.cells]))
    layout = txb.FieldLayout(s["n_comp"])
    glob = rng.standard_normal(layout.global_size(mesh))
    aux = aux_for(s, mesh.n_cells, rng)
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    for rule in (txb.quadrature_rule(dim, 1), txb.two_point_rule(dim)):
        tab = txb.tabulate(dim, rule)
        res, _ = txb.integrate_transposed(mesh, layout, tab, rule, f, glob, aux, n_bl=8, n_cb=2, dtype=dtype,
                                          shared_mem_limit=None)
        elem = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], tab.basis,
                                      tab.basis_der, rule.weights, inv, det,
                                      oracle.gather(mesh.cells, glob, s["n_comp"]),
                                      None if aux is None else aux.values, npdt)
        g = txb.derive_execution_geometry(dim, tab.n_b, s["n_comp"], rule.n_q, 8, 2, mesh.n_cells)
        sp = g.n_chunks * g.n_chunk
        if sp < mesh.n_cells and npdt == np.float32:  # remainder: float64 then cast (executor.py:258-264)
            elem[sp:] = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], tab.basis,
                                               tab.basis_der, rule.weights, inv[sp:], det[sp:],
                                               oracle.gather(mesh.cells[sp:], glob, s["n_comp"]),
                                               None if aux is None else aux.values[sp:], np.float64).astype(npdt)
        want = oracle.scatter_add(mesh.cells, elem, mesh.n_vertices)
        assert bitwise_equal(res, want), (rule.n_q, dtype)
        res2, _ = txb.integrate_transposed(mesh, layout, tab, rule, f, glob, aux, n_bl=8, n_cb=2, dtype=dtype,
                                           shared_mem_limit=None, cell_geom=txb.CellGeometry(inv, det))
        assert bitwise_equal(res2, want)


@pytest.mark.gpu
def test_integrate_transposed_with_a_user_form():
    """Mesh-level driver: geometry -> gather -> run-time compiled integration ->
    deterministic scatter-add (executor.py:161-267) for the reaction form."""
    dim = 3
    mesh = txb.generate_unit_simplex_mesh(dim, 6)
    layout = txb.FieldLayout(1)
    rule = txb.quadrature_rule(dim, 1)
    tab = txb.tabulate(dim, rule)
    f = form_of("reaction", dim)
    glob = np.random.default_rng(3).standard_normal(mesh.n_vertices)
    res, _ = txb.integrate_transposed(mesh, layout, tab, rule, f, glob, None, n_bl=4, n_cb=2)
    inv, det = oracle.geometry(mesh.vertices, mesh.cells)
    co = oracle.gather(mesh.cells, glob, 1)
    s = user_forms.spec("reaction", dim)
    elem = oracle.integrate_forms(s["f1_many"], s["f0_many"], False, None, tab.basis, tab.basis_der, rule.weights,
                                  inv, det, co)
    want = oracle.scatter_add(mesh.cells, elem, mesh.n_vertices)
    assert bitwise_equal(res, want)


# ---- codegen.generate_kernel_source (txfem/codegen.py:50-256) --------------------

def test_generate_kernel_source_mirrors_reference_codegen():
    from paper_1607_04245_b200.codegen import generate_kernel_source

    geom = txb.derive_execution_geometry(3, 4, 1, 1, 8, 2, 1000)
    f = txb.poisson_varcoef_form(3)
    ks = generate_kernel_source(geom, f, "f64")
    assert "f1_poisson_varcoef" in ks.text and ks.entry_name == "txb_jit_integrate"
    assert ks.specialization == (3, 4, 1, 1, 8, "double")
    assert generate_kernel_source(geom, f, "f64").text == ks.text  # deterministic
    assert isinstance(ks.kernel, txb.JitKernel)
    with pytest.raises(txb.CodegenError):
        generate_kernel_source(geom, f, "f16")
    with pytest.raises(txb.CodegenError):  # form / geometry mismatch
        generate_kernel_source(txb.derive_execution_geometry(2, 3, 1, 1, 8, 2, 100), f, "f32")
    with pytest.raises(txb.CodegenError):
        generate_kernel_source(geom, txb.user_form("nosrc", 3, 1, None, 0, ""), "f32")
    two = txb.derive_execution_geometry(3, 4, 1, 2, 4, 2, 1000)
    ks2 = generate_kernel_source(two, form_of("advect", 3), "f32", aux_space="p1")
    assert "#define TXB_HAS_F0 1" in ks2.text and "#define TXB_GRAD_A 1" in ks2.text


from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402


@pytest.mark.gpu
@settings(max_examples=int(os.environ.get("TXB_HYPOTHESIS_EXAMPLES", 40)), deadline=None, suppress_health_check=list(HealthCheck))
@given(name=st.sampled_from(SPECS), dim=st.integers(2, 3), n_q=st.integers(1, 3), n=st.integers(0, 2500),
       dtype=st.sampled_from([np.float64, np.float32]), n_bl=st.sampled_from([0, 1, 5]), seed=st.integers(0, 999))
def test_jit_random_problems_bitwise(name, dim, n_q, n, dtype, n_bl, seed):
    rng = np.random.default_rng(seed)
    s = user_forms.spec(name, dim)
    f = form_of(name, dim)
    B = rng.uniform(0, 1, (n_q, dim + 1))
    D = rng.uniform(-1, 1, (n_q, dim + 1, dim))
    W = rng.uniform(0.1, 0.5, n_q)
    jac = np.eye(dim) + 0.3 * rng.uniform(-1, 1, (n, dim, dim))
    inv = np.linalg.inv(jac) if n else np.zeros((0, dim, dim))
    det = np.linalg.det(jac) if n else np.zeros(0)
    co = rng.standard_normal((n, dim + 1, s["n_comp"]))
    aux = aux_for(s, n, rng)
    k = txb.cuda_kernel(f, n_q, aux, np.dtype(dtype).itemsize)
    got = _run(k, B, D, W, inv, det, co, aux, dtype, n_bl=n_bl)
    want = oracle.integrate_forms(s["f1_many"], s["f0_many"], s["uses_grad_a"], s["aux"], B, D, W, inv, det, co,
                                  None if aux is None else aux.values, dtype)
    assert bitwise_equal(got, want)
