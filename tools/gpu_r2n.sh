#!/usr/bin/env bash
# Round-2 session N: full GPU suite + bench with extras (mesh rows incl. the tiled kernel, api rows).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2n}
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 1200 python bench.py --steps 20 --warmup 5 --extras > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
ls -la gpurun_out | grep ${T}
