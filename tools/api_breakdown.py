"""Where the mesh-level call from numpy spends its time (1 M-tet 3D var-coef f64):
the whole integrate_transposed call, the H2D of kappa (pageable vs pinned staging),
the coefficient H2D, the residual D2H, the device-resident call, and a cProfile of
the Python side.  Run from the repo root: python tools/api_breakdown.py"""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1607_04245_b200 as txb
from paper_1607_04245_b200.workload import refine_for
mesh = txb.generate_unit_simplex_mesh(3, refine_for(3, 1 << 20))
form = txb.poisson_varcoef_form(3); layout = txb.FieldLayout(1)
rule = txb.quadrature_rule(3, 1); tab = txb.tabulate(3, rule)
glob = np.random.default_rng(3).standard_normal(layout.global_size(mesh))
aux = txb.CellAux("p0", np.random.default_rng(4).uniform(0.5, 1.5, (mesh.n_cells, 1)))
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
r = {}
r["call_ms"] = t(lambda: txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=32, n_cb=8, shared_mem_limit=None))
r["kappa_h2d_ms"] = t(lambda: torch.from_numpy(aux.values).cuda())
r["glob_h2d_ms"] = t(lambda: torch.from_numpy(glob).cuda())
res = torch.empty(mesh.n_vertices, dtype=torch.float64, device="cuda")
r["res_d2h_ms"] = t(lambda: res.cpu().numpy())
g = torch.from_numpy(glob).cuda(); a = txb.CellAux("p0", torch.from_numpy(aux.values).cuda())
r["device_call_ms"] = t(lambda: txb.integrate_transposed(mesh, layout, tab, rule, form, g, a, n_bl=32, n_cb=8, shared_mem_limit=None))
pk = torch.empty(aux.values.shape, dtype=torch.float64).pin_memory()
r["kappa_pin_copy_ms"] = t(lambda: pk.copy_(torch.from_numpy(aux.values)))
r["kappa_pinned_h2d_ms"] = t(lambda: pk.cuda(non_blocking=True))
import cProfile, pstats, io
pr = cProfile.Profile(); pr.enable()
for _ in range(10): txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=32, n_cb=8, shared_mem_limit=None)
torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(18); print(s.getvalue()[:4000])
print(json.dumps({k: round(v, 3) for k, v in r.items()}))
