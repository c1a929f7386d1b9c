"""bench.py --impl reference on CPU: the reference's own residual (baseline/_ref, the
unmodified ebsolve package) or, without that install, the oracle port -- one JSON line
with the contract's keys, on the same workload recipe (here at level 6)."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--size", "6"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "GDoF/s"
    assert line["config"]["n_nodes"] == 65 * 65
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "ebsolve")):
        assert cb["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
