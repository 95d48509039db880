"""Host-side cost of one device-resident integrate_transposed call (small mesh: the
kernels are a few microseconds, the rest is Python + driver): cProfile top entries."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_1607_04245_b200 as txb

    mesh = txb.generate_unit_simplex_mesh(3, 4)
    form = txb.poisson_varcoef_form(3)
    rule = txb.quadrature_rule(3, 1)
    tab = txb.tabulate(3, rule)
    layout = txb.FieldLayout(1)
    glob = torch.from_numpy(np.random.default_rng(1).standard_normal(mesh.n_vertices)).cuda()
    aux = txb.CellAux("p0", torch.rand((mesh.n_cells, 1), dtype=torch.float64, device="cuda") + 0.5)
    call = lambda: txb.integrate_transposed(mesh, layout, tab, rule, form, glob, aux, n_bl=32, n_cb=8,  # noqa: E731
                                            shared_mem_limit=None)
    for _ in range(20):
        call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        call()
    torch.cuda.synchronize()
    print(f"integrate_transposed (384 cells, device-resident): {(time.perf_counter() - t0) / 200 * 1e6:.1f} us/call")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        call()
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
