"""Throughput vs mesh size: the fast residual (caller numbering, ebs_residual) on 2D levels
6..12 and the Jacobi-PCG iteration on 3D N = 16..256 -- where the GPU leaves the
latency-bound regime and saturates HBM.  Device time, CUDA events, after warm-up."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200 import _device as D  # noqa: E402
from paper_1911_03973_b200._lib import EBS_RES_FAST, load  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
lib = load()
print("2D residual r = b - A x (x, r in caller numbering, random permutation)")
for L in range(6, 13):
    m = eb.permute_nodes(eb.build_unit_square_mesh(L),
                         np.random.default_rng(0).permutation((2**L + 1) ** 2))
    b = eb.build_element_batch(m, nu=1.0)
    n, ne = m.n_nodes, m.n_elements
    pl = b.operator(n)
    x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).cuda()
    r = D.empty(n)
    s = D.stream()
    K = max(20, int(2e8 // (ne * 100)))
    for _ in range(5):
        lib.ebs_residual(pl.handle, D.ptr(x), D.ptr(r), EBS_RES_FAST, 0, None, s)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(K):
        lib.ebs_residual(pl.handle, D.ptr(x), D.ptr(r), EBS_RES_FAST, 0, None, s)
    e[1].record()
    torch.cuda.synchronize()
    t = e[0].elapsed_time(e[1]) / 1e3 / K
    byt = ne * (8 * 9 + 12) + 24 * n
    print(f"  level {L:2d}: {n:9d} nodes  {t * 1e6:9.1f} us  {n / t / 1e9:6.2f} GDoF/s  "
          f"{byt / t / 1e9:7.0f} GB/s = {byt / t / 1e9 / peak:.2f} of peak", flush=True)
    del b, pl, m
    torch.cuda.empty_cache()
print("3D Jacobi-PCG iteration (ν = 1, 200 iterations)")
for N in (16, 32, 64, 128, 256):
    m = eb.build_unit_cube_mesh(N)
    b = eb.build_element_batch(m, nu=1.0)
    d = eb.DirichletData(eb.face_z0_nodes(m), torch.zeros(eb.face_z0_nodes(m).numel(),
                                                         dtype=torch.float64, device="cuda"))
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    eb.pcg(b, d, x0, 200)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    _, h = eb.pcg(b, d, x0, 200)
    e[1].record()
    torch.cuda.synchronize()
    t = e[0].elapsed_time(e[1]) / 1e3 / 200
    byt = m.n_elements * (8 * 16 + 16) + 104 * m.n_nodes
    print(f"  N {N:3d}: {m.n_elements:10d} tets  {t * 1e6:8.1f} us/it  {1 / t:8.1f} it/s  "
          f"{byt / t / 1e9:7.0f} GB/s = {byt / t / 1e9 / peak:.2f} of peak", flush=True)
    del b, m
    torch.cuda.empty_cache()
