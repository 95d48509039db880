#!/usr/bin/env bash
# Round-2 session X: the driver's exact commands + launch list + full captures (headline, tiled mesh kernel).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2x}
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
timeout 400 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo "rc=$?" >> gpurun_out/${T}_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 3 -c 1 \
  -o gpurun_out/${T}_prof_3dvar_f64 python bench.py --steps 5 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/${T}_ncu_full64.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_tiled_kernel -s 6 -c 1 \
  -o gpurun_out/${T}_prof_tiled_3dvar_f64 python tools/prof_mesh.py 3d_varcoef_f64 > gpurun_out/${T}_ncu_tiled.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
ls -la gpurun_out | grep ${T}
