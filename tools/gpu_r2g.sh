#!/usr/bin/env bash
# Round-2 session G: gather micro-benchmark (+ L1 wavefront counts) and the 2-rank torchrun test.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2g}
[ -x tools/probes/gather_probe ] || nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/probes/gather_probe tools/probes/gather_probe.cu
timeout 120 tools/probes/gather_probe > gpurun_out/${T}_gather.txt 2>&1
timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_lg.sum,l1tex__data_pipe_lsu_wavefronts_mem_lg_cmd_read.sum -k regex:probe -c 6 --csv tools/probes/gather_probe > gpurun_out/${T}_gather_ncu.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x > gpurun_out/${T}_multirank.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_multirank.log
ls -la gpurun_out | grep ${T}
