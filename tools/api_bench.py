"""Mesh-level API rows of bench.py on their own (integrate_transposed from the host)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

if __name__ == "__main__":
    for r in bench.api_rows():
        print(json.dumps(r), flush=True)
