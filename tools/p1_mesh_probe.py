"""Tiled mesh kernel with a P1 coefficient field (var-coef, kappa nodal per cell):
graph-timed us per launch, in-kernel and given geometry.  python tools/p1_mesh_probe.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

for dim in (3, 2):
    for dt in ("f64", "f32"):
        name = f"{dim}d_varcoef_p1_{dt}"
        bench.CONFIGS[name] = (dim, "varcoef_p1", dt, 1 << 20)
        for given in (False, True):
            ms, per_cell = bench.time_mesh(name, 200, 5, given_geometry=given)
            print(json.dumps({"config": name, "given_geometry": given, "us": round(ms * 1e3, 2),
                              "bytes_per_cell": round(per_cell, 1)}), flush=True)
