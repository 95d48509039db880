#!/usr/bin/env bash
# Elasticity launch-bound variants (tune_libs/, built with -DTXB_ELAST_THREADS/-DTXB_ELAST_MINB): us per launch.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
cp paper_1607_04245_b200/libtxb.so /tmp/libtxb_orig.so
for lib in ${LIBS:-default 128_4 192_3 256_2 default}; do
  cp tune_libs/libtxb_$lib.so paper_1607_04245_b200/libtxb.so
  for cfg in 3d_elasticity_f32 3d_elasticity_f64 2d_elasticity_f32 2d_elasticity_f64; do
    timeout 300 python bench.py --config $cfg --steps 400 --warmup 10 --no-variants --no-cpu --no-e2e 2>/dev/null | \
      python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', '$cfg', round(d['ms_per_step']*1000,2), round(d['roofline']['frac'],4), d['config'].get('launch'))"
  done
done | tee gpurun_out/r2bd.txt
cp /tmp/libtxb_orig.so paper_1607_04245_b200/libtxb.so
