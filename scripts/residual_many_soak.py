"""Soak of ebs_residual_many (two residuals in flight): 15k rows over 2D permuted, 2D jittered +
permuted and 3D structured meshes, both modes, each compared bit for bit with ebs_residual on
the same vector.  python scripts/residual_many_soak.py  ->  soak ok 0"""
import sys; sys.path.insert(0, '.')
import torch, numpy as np
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
bad = 0
for cfg, size in ((2, 9), (4, 8), (3, 24)):
    p = config_problem(cfg, seed=cfg, size=size)
    b, n = p["batch"], p["mesh"].n_nodes
    g = torch.Generator(device="cuda").manual_seed(cfg)
    for rep in range(10):
        K = 257
        xs = torch.rand((K, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        for det in (True, False):
            out = eb.residual_many(b, xs, deterministic=det)
            for k in range(K):
                if not torch.equal(out[k], eb.residual(b, xs[k], deterministic=det, check_finite=False)):
                    bad += 1
    print(f"config {cfg} size {size}: n={n}, mismatching rows so far {bad}", flush=True)
print("soak", "ok" if bad == 0 else "FAILED", bad)
