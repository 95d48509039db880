#!/usr/bin/env bash
# Round-2 session C: reference-seam and residual-golden GPU tests, traffic with an evicting sweep.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2c}
timeout 1500 python -m pytest tests/test_reference_seam.py tests/test_residual_golden.py -m gpu -q --timeout 1400 > gpurun_out/${T}_seam.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_seam.log
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --replay-mode range --metrics $M --csv --log-file gpurun_out/${T}_traffic_range.csv python tools/traffic.py run > gpurun_out/${T}_traffic_range.log 2>&1
timeout 600 ncu --profile-from-start off --cache-control all --clock-control none -k regex:integrate --metrics $M --csv --log-file gpurun_out/${T}_traffic_kernel.csv python tools/traffic.py run > gpurun_out/${T}_traffic_kernel.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 20 --warmup 5 --no-variants --no-cpu --no-e2e > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 6 -c 1 -o gpurun_out/${T}_prof_3dvar_f64 python bench.py --steps 5 --warmup 5 --no-variants --no-cpu --no-e2e > gpurun_out/${T}_ncu_full64.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:integrate_kernel -s 6 -c 1 -o gpurun_out/${T}_prof_3dvar_f32 python bench.py --config 3d_varcoef_f32 --steps 5 --warmup 5 --no-variants --no-cpu --no-e2e > gpurun_out/${T}_ncu_full32.log 2>&1
ls -la gpurun_out | grep ${T}
