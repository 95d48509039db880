"""Mesh-fused kernel rows of bench.py (given geometry / tiled in-kernel geometry /
per-cell in-kernel geometry), one JSON row per line: python tools/mesh_rows.py [steps]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

peak, _ = bench.peaks()
for r in bench.mesh_rows(peak, int(sys.argv[1]) if len(sys.argv) > 1 else 200):
    print(json.dumps(r), flush=True)
