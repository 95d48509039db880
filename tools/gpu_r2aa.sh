#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2aa}
timeout 1200 python -m pytest tests/test_jit.py tests/test_gpu_tiled.py tests/test_gpu_residual_graph.py tests/test_gpu_mesh.py -m gpu -q -x --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python tools/api_bench.py > gpurun_out/${T}_api.jsonl 2> gpurun_out/${T}_api.err
timeout 600 python tools/jit_bench.py > gpurun_out/${T}_jit.jsonl 2> gpurun_out/${T}_jit.err
