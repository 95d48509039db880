"""ResidualGraph per form on the ~1 M-tet 3D Kuhn mesh (an NVRTC user form with f0,
two P1 fields and grad a; the ahead-of-time var-coef form): ms per residual.
Run from the repo root: python tools/residual_graph_forms.py"""
import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_1607_04245_b200 as txb
from paper_1607_04245_b200.physics import user_form
from paper_1607_04245_b200.workload import refine_for
mesh = txb.generate_unit_simplex_mesh(3, refine_for(3, 1 << 20))
rule = txb.quadrature_rule(3, 1); tab = txb.tabulate(3, rule)
glob = torch.from_numpy(np.random.default_rng(5).standard_normal(mesh.n_vertices)).cuda()
for name, form, aux in (
    ("user_advect", user_form("advect", 3, 1, lambda s, c: None, 9, bench.ADVECT_F1, n_aux=2, f0=lambda s, c: None,
                              flops_f0=7, source_f0=bench.ADVECT_F0, uses_grad_a=True),
     txb.CellAux("p1", torch.rand((mesh.n_cells, 4, 2), dtype=torch.float64, device="cuda") + 0.5)),
    ("varcoef_aot", txb.poisson_varcoef_form(3), txb.CellAux("p0", torch.rand((mesh.n_cells, 1), dtype=torch.float64, device="cuda") + 0.5)),
):
    g = txb.ResidualGraph(mesh, txb.FieldLayout(1), tab, rule, form, aux, n_bl=32, n_cb=8, shared_mem_limit=None)
    for _ in range(5): g(glob)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): g(glob)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"form": name, "residual_graph_ms": e0.elapsed_time(e1) / 50}))
