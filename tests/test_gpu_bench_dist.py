"""bench.py --gpus 2 end to end on the one GPU of the box (EBS_BENCH_GLOO=1: gloo with
host-staged halos, both ranks on cuda:0, no kernel waits on another process): every N > 1
branch of bench_dist.py runs -- weak-scaled C2, strong C2, C4 / C5 solvers, the JSON line --
and the distributed C5 solve ends on the single-GPU residual norm."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_gloo(gpu):
    env = dict(os.environ, EBS_BENCH_GLOO="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--steps", "8", "--warmup", "3", "--size", "9"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["value"] > 0
    assert line["config"]["n_nodes"] == 513 * (512 * 2 + 1)
    assert line["strong_c2"]["value"] > 0 and line["e2e"]["value"] > 0
    assert line["gpu_launches"] > 0
    c5 = line["solvers"]["C5"]
    assert "error" not in c5 and c5["ranks"] == 2 and c5["iterations"] == 500
    assert abs(c5["final_norm"] - 1.279564e-08) <= 1e-6 * 1.279564e-08 * 10
    assert "error" not in line["solvers"]["C4"]
