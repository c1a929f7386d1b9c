"""bench.py --gpus 2 end to end on the one GPU of the box (EBS_BENCH_GLOO=1: both ranks on
cuda:0, gloo for the host plumbing, no kernel waits on another process -- the peer-memory
transport with a host barrier after every put phase (CUDA-IPC windows between the two
processes), or NCCL's stand-in with host-staged halos): every N > 1
branch of bench_dist.py runs -- `value` = the fixed C2 mesh strong-scaled (the N=1
workload), the weak-scaled C2 extra, C4 / C5 solver strong scaling with E(N) against the
in-job single-GPU run and the C5 norm history checked against it, the JSON line."""

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


@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_bench_two_ranks_gloo(gpu, transport):
    env = dict(os.environ, EBS_BENCH_GLOO="1", EBS_TRANSPORT=transport, EBS_PEER_TIMEOUT="120")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--steps", "8", "--warmup", "3", "--size", "9", "--c4-size", "9",
           "--c5-size", "48"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0
    assert line["config"]["n_nodes"] == 513 * 513          # the N=1 C2 workload (level 9)
    assert line["config"]["parallelism"].startswith("element slabs x2")
    assert line["weak_c2"]["value"] > 0 and line["weak_c2"]["n_nodes"] == 513 * (512 * 2 + 1)
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert line["transport"].startswith("peer memory" if transport == "peer" else "NCCL")
    assert line["roofline"]["frac"] > 0
    ss = line["strong_scaling"]
    for cfg, its in (("C4", 200), ("C5", 500)):
        row = ss[cfg]
        assert "error" not in row, row
        assert row["ranks"] == 2 and row["iterations"] == its and row["efficiency"] > 0
        assert row["t1_it_per_s"] > 0 and not row["diverged"] and row["transport"] == transport
    assert ss["C5"]["history_vs_1gpu"]["ok_1e-8"], ss["C5"]["history_vs_1gpu"]
    assert ss["C4"]["history_vs_1gpu"]["ok_1e-8"], ss["C4"]["history_vs_1gpu"]
