"""Run the fused mesh kernel a few times (for ncu): python tools/prof_mesh.py [config] [given|tiled|per_cell]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "3d_varcoef_f64"
mode = sys.argv[2] if len(sys.argv) > 2 else "tiled"
print(bench.time_mesh(name, 5, 3, given_geometry=mode == "given", tiled=mode == "tiled"))
