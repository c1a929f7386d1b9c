"""The two-pass coalesced caller <-> internal permutation (csrc/perm.cu), used automatically
for vectors beyond the L2-resident crossover (>= 8M nodes), forced here on small meshes
(EBS_PERM2_MIN_NODES=0 in a subprocess): residual, matvec and solver outputs bit-identical
to the direct path / the oracle."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as o
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
for cfg, size in ((2, 8), (4, 7), (5, 8)):
    p = config_problem(cfg, seed=2, size=size)
    b, d, m = p["batch"], p["dirichlet"], p["mesh"]
    inp = o.config_inputs(cfg, seed=2, size=size)
    _, _, A, b_e = o.element_matrices(inp["nodes"], inp["elements"], nu=p["nu"],
                                      f_vals=inp.get("f_vals"))
    indt = np.ascontiguousarray(inp["elements"].T)
    x = np.random.default_rng(3).uniform(-1, 1, m.n_nodes)
    assert np.array_equal(eb.residual(b, x).cpu().numpy(), o.residual(A, b_e, indt, x))
    assert np.array_equal(eb.matvec(b, x, d).cpu().numpy(),
                          o.matvec_masked(A, indt, x, inp["dirichlet"]))
    xs, hs = eb.richardson(b, d, np.ones(m.n_nodes), eb.SpectralBounds(0.1, 8.0), 7) \
        if cfg != 5 else eb.jacobi(b, d, np.zeros(m.n_nodes), 7)
    print("ok", cfg, float(xs.abs().sum()), hs.residual_norms[-1])
'''


def _run(env_value):
    env = dict(os.environ, EBS_PERM2_MIN_NODES=str(env_value))
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


def test_two_pass_permutation_bitwise(gpu):
    forced = _run(0)                # every plan uses the two-pass schedule
    direct = _run(1 << 40)          # never
    assert forced == direct         # solver outputs identical to the last bit printed
