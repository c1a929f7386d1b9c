"""bench.py on one GPU at a reduced C2 level: the JSON line keeps the driver's contract
(metric / value / unit / steps / roofline / cpu_baseline / e2e / clocks / gpu_launches), the
headline goes through ebs_residual_many with the one-at-a-time figure beside it, and every
in-bench consistency assert (pipelined == C-ABI == public API rows, bitwise) holds."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_single_gpu_bench_line(gpu):
    steps = 6
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--size", "8", "--steps",
                        str(steps), "--warmup", "3", "--no-extra", "--cpu-budget", "0.5"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["unit"] == "GDoF/s" and d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert d["value"] > 0 and abs(d["value"] - d["config"]["n_nodes"] / d["ms_per_step"] / 1e6) \
        <= 1e-9 * d["value"]
    assert "workload" in d["config"] and "ebs_residual_many" in d["config"]["mode"]
    assert d["sequential"]["value"] > 0 and d["sequential"]["ms_per_step"] > 0
    assert d["gpu_launches"] == 3 * steps           # x permutation, -0.0 fill, SELL pass per step
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-12
    assert r["bytes_per_launch"] > 0 and r["kernel_ms"] > 0 and "step_frac" in r
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 8 * d["config"]["n_nodes"]
    assert e["value"] < d["value"]                   # the copies are inside its timed region
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["exact_mode"]["value"] > 0 and d["exact_mode"]["sequential_value"] > 0
