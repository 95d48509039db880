#!/usr/bin/env bash
# Round-2 session B: cluster-launch-control scheduling -- new scheduling tests,
# the full GPU suite, the driver's bench command, traffic capture.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2b}
timeout 300 python -m pytest tests/test_gpu_sched.py -q -x --timeout 240 > gpurun_out/${T}_sched.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_sched.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$?" >> gpurun_out/${T}_bench.err
TXB_DYNAMIC=0 timeout 600 python bench.py --gpus 1 --steps 2000 --warmup 5 --no-cpu > gpurun_out/${T}_bench_static.json 2> gpurun_out/${T}_bench_static.err
timeout 600 python bench.py --gpus 1 --steps 2000 --warmup 5 --no-cpu > gpurun_out/${T}_bench_2000.json 2> gpurun_out/${T}_bench_2000.err
timeout 300 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --replay-mode range --metrics $M --csv --log-file gpurun_out/${T}_traffic_range.csv python tools/traffic.py run > gpurun_out/${T}_traffic_range.log 2>&1
timeout 600 ncu --profile-from-start off --cache-control all --clock-control none -k regex:integrate --metrics $M --csv --log-file gpurun_out/${T}_traffic_kernel.csv python tools/traffic.py run > gpurun_out/${T}_traffic_kernel.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --maxfail 20 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
ls -la gpurun_out | grep ${T}
