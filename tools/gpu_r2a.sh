#!/usr/bin/env bash
# Round-2 session A: the driver's exact bench command, the reference arm, the
# write-back-inclusive traffic capture, and the GPU tests.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2a}
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --replay-mode range --profile-from-start off --metrics $M --csv --log-file gpurun_out/${T}_traffic_range.csv python tools/traffic.py run > gpurun_out/${T}_traffic_range.log 2>&1
timeout 600 ncu --profile-from-start off --cache-control all --clock-control none -k regex:integrate --metrics $M --csv --log-file gpurun_out/${T}_traffic_kernel.csv python tools/traffic.py run > gpurun_out/${T}_traffic_kernel.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
ls -la gpurun_out | grep ${T}
