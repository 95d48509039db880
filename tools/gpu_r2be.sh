#!/usr/bin/env bash
# Tiled mesh kernel register budget variants (tune_libs/, built with -D'TXB_TILED_MIN_BLOCKS(NCOMP)=...'): mesh rows.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
cp paper_1607_04245_b200/libtxb.so /tmp/libtxb_orig.so
for lib in ${LIBS:-default 2_2 4_2 3_1 default}; do
  cp tune_libs/libtxb_$lib.so paper_1607_04245_b200/libtxb.so
  timeout 600 python tools/mesh_rows.py 200 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if 'tiled' in d['config']: print('$lib', d['config'], round(d['launch_ms']*1000,2))"
done | tee gpurun_out/r2be.txt
cp /tmp/libtxb_orig.so paper_1607_04245_b200/libtxb.so
