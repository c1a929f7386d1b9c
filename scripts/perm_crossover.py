"""Fast residual in caller numbering on n x n grids between levels 11 and 12: direct
gather / red output vs the two-pass coalesced permutation (run once per library)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200 import _device as D  # noqa: E402
from paper_1911_03973_b200._lib import EBS_RES_FAST, load  # noqa: E402

lib = load()
for side in [int(a) for a in sys.argv[1:]] or [2049, 2500, 2897, 3300, 3700, 4097]:
    m = eb.build_grid_mesh(side)
    m = eb.permute_nodes(m, np.random.default_rng(0).permutation(m.n_nodes))
    b = eb.build_element_batch(m, nu=1.0)
    n = m.n_nodes
    pl = b.operator(n)
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
    r = D.empty(n)
    s = D.stream()
    for _ in range(5):
        lib.ebs_residual(pl.handle, D.ptr(x), D.ptr(r), EBS_RES_FAST, 0, None, s)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(20):
        lib.ebs_residual(pl.handle, D.ptr(x), D.ptr(r), EBS_RES_FAST, 0, None, s)
    e[1].record()
    torch.cuda.synchronize()
    t = e[0].elapsed_time(e[1]) / 1e3 / 20
    print(f"side {side}: {n} nodes ({n * 8 / 1e6:.0f} MB/vector): {t * 1e6:.0f} us, "
          f"{n / t / 1e9:.2f} GDoF/s", flush=True)
    del b, pl, m
    torch.cuda.empty_cache()
