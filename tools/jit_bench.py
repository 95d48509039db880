"""Run-time compiled lane rows of bench.py on their own (tuning aid)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

if __name__ == "__main__":
    peak, _ = bench.peaks()
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    for r in bench.jit_rows(peak, steps):
        print(json.dumps(r), flush=True)
