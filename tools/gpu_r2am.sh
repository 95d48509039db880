#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2am}
timeout 900 python -m pytest tests/test_gpu_mesh.py tests/test_halo.py tests/test_gpu_residual_graph.py tests/test_residual_golden.py -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for c in 3d_varcoef_f64 3d_elasticity_f64 3d_elasticity_f32 2d_varcoef_f64; do
  for w in 0 1; do TXB_SCATTER_VEC=$w timeout 300 python tools/pipeline_bench.py $c | sed "s/^/vec=$w /" >> gpurun_out/${T}_pipe.txt 2>&1; done
done
for w in 0 1; do TXB_SCATTER_VEC=$w timeout 300 python tools/pipeline_bench.py 3d_varcoef_f64 16777216 | sed "s/^/vec=$w /" >> gpurun_out/${T}_pipe.txt 2>&1; done
