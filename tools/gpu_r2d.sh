#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2d}
timeout 1500 python -m pytest tests/test_reference_seam.py tests/test_residual_golden.py tests/test_api_surface.py tests/test_halo.py -m gpu -q --timeout 1400 > gpurun_out/${T}_seam.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_seam.log
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --replay-mode range --metrics $M --csv --log-file gpurun_out/${T}_traffic_range.csv python tools/traffic.py run > gpurun_out/${T}_traffic_range.log 2>&1
timeout 600 ncu --profile-from-start off --cache-control all --clock-control none -k regex:integrate --metrics $M --csv --log-file gpurun_out/${T}_traffic_kernel.csv python tools/traffic.py run > gpurun_out/${T}_traffic_kernel.log 2>&1
ls -la gpurun_out | grep ${T}
