"""The driver's scaling command, run for real: ``torch.distributed.run
--nproc-per-node 2 bench.py --gpus 2 --steps 20 --warmup 5``.  The GPU box has
one B200, so both ranks share it and talk over gloo (TXB_BENCH_BACKEND=gloo;
NCCL refuses two ranks on one device); every rank still launches the CUDA
kernels on its own cell range, reduces its device time as the max over ranks,
and rank 0 prints the one JSON line (weak headline + strong-scaling rows of
BASELINE.json configs[4]).  Timings are meaningless here (two ranks share one
GPU); the test checks that the N>1 script runs unchanged and what it prints."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.gpu
@pytest.mark.timeout(900)
def test_torchrun_two_ranks_bench_line():
    env = dict(os.environ, TXB_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "20", "--warmup", "5"]
    p = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=850)
    assert p.returncode == 0, p.stderr[-4000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-4000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 20 and d["warmup"] == 5
    assert d["scaling"] == "weak"
    assert d["config"]["cells_total"] == 2 * (1 << 20)
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["e2e"]["value"] and d["e2e"]["value"] > 0
    assert d["roofline"]["frac"] > 0
    strong = d["strong_scaling"]
    assert all("error" not in r for r in strong), strong
    assert {r["config"] for r in strong} == {f"3d_varcoef_{t}_2^{lg}_total" for t in ("f32", "f64")
                                             for lg in (24, 26)}
    for r in strong:
        assert r["n_gpus"] == 2 and r["cells_per_rank"] * 2 == r["cells_total"] and r["gflops"] > 0


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_torchrun_two_ranks_reference_arm():
    """--impl reference under torchrun: rank 0 alone runs and prints; rank 1 exits 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl",
           "reference", "--gpus", "2", "--steps", "3", "--warmup", "3"]
    p = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=550)
    assert p.returncode == 0, p.stderr[-4000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_nccl_init_logs_stay_off_stdout():
    """bench.py's N > 1 runs turn on NCCL's init log (NCCL_DEBUG=INFO) for the
    communicator evidence; NCCL writes it to stdout by default, and the driver
    reads stdout as the one JSON line.  A one-rank NCCL group (the only NCCL
    group one B200 allows) with bench.nccl_debug_env(): the INIT lines land on
    stderr, stdout holds only what the process prints itself."""
    code = ("import os, sys, torch, torch.distributed as dist; sys.path.insert(0, '.'); import bench; "
            "bench.nccl_debug_env(); torch.cuda.set_device(0); "
            "dist.init_process_group('nccl', rank=0, world_size=1, device_id=torch.device('cuda', 0)); "
            "t = torch.ones(1, device='cuda'); dist.all_reduce(t); torch.cuda.synchronize(); "
            "dist.destroy_process_group(); print('{\"ok\": 1}')")
    env = {k: v for k, v in os.environ.items() if not k.startswith("NCCL_DEBUG")}
    env.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    p = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True, text=True, timeout=280)
    assert p.returncode == 0, p.stderr[-4000:]
    assert p.stdout.strip() == '{"ok": 1}', p.stdout[-2000:]
    assert "NCCL INFO" in p.stderr
