#!/usr/bin/env bash
# One GPU session: parity tests, bench (default + quick variants), ncu launch list and
# one full capture of the headline kernel.  Outputs land in gpurun_out/ (scratch).
set -u
TAG=${1:-r1}
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 --maxfail 20 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_3dvar_f64 python bench.py --steps 5 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_full64.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 3 -c 1 \
  -o gpurun_out/${TAG}_prof_3dvar_f32 python bench.py --config 3d_varcoef_f32 --steps 5 --warmup 3 --no-variants --no-cpu --no-e2e > gpurun_out/${TAG}_ncu_full32.log 2>&1
ls -la gpurun_out | tail -20
