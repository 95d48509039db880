"""One ResidualGraph replay on the 2^20-cell 3D Kuhn mesh (var-coef P0, f64), for an ncu launch list:
ncu --metrics gpu__time_duration.sum python tools/residual_graph_profile.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_1607_04245_b200 as txb
    from paper_1607_04245_b200.workload import refine_for

    mesh = txb.generate_unit_simplex_mesh(3, refine_for(3, 1 << 20))
    form = txb.poisson_varcoef_form(3)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    aux = txb.CellAux("p0", torch.rand((mesh.n_cells, 1), dtype=torch.float64, device="cuda") + 0.5)
    glob = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_vertices)).cuda()
    g = txb.ResidualGraph(mesh, txb.FieldLayout(1), tab, rule, form, aux, n_bl=32, n_cb=8, shared_mem_limit=None)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(3):
        g(glob)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
