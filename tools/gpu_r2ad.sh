#!/usr/bin/env bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${1:-r2ad}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py tests/test_jit.py tests/test_gpu_mesh.py -m gpu -q -x --timeout 600 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
cat > /tmp/tail_scan.py <<'PY'
import json, os, sys
sys.path.insert(0, '.')
import bench
peak, _ = bench.peaks()
for name in ["3d_varcoef_f64", "3d_varcoef_f32", "2d_varcoef_f64", "2d_varcoef_f32", "2d_elasticity_f64", "2d_elasticity_f32", "3d_elasticity_f64", "3d_elasticity_f32"]:
    _, bpc = bench.config_model(name)
    wl = bench.rank_workload(name, 0, 1)
    ns = bench.rotating_sets(bpc * wl["n"])
    for rep in range(2):
        for env in ({"TXB_TAIL_SPLIT": "0"}, {"TXB_TAIL_SPLIT": "1"}):
            os.environ.update(env)
            tot, _ = bench.time_device(wl, 200, 5, ns)
            us = tot / 200 * 1e3
            print(json.dumps({"config": name, "env": env, "us": round(us, 3), "frac": round(bpc * wl["n"] / (us * 1e-6) / 1e9 / peak, 4)}), flush=True)
    del wl
PY
timeout 900 python /tmp/tail_scan.py > gpurun_out/${T}_tail.jsonl 2>&1
