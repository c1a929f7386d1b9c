"""Fused element assembly (ebs_assemble_p1: K_e, M_e, A_e, b_e) timed alone with CUDA
events on the BASELINE meshes; algorithmic bytes n_e(4 nb + 24 nb^2 + 8 nb) + 8 dim n_n
 against the measured HBM peak."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200 import _device as D  # noqa: E402
from paper_1911_03973_b200._lib import load  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
lib = load()
for name, m in (("C2 level 11", eb.build_unit_square_mesh(11)),
                ("C4 level 12", eb.build_unit_square_mesh(12)),
                ("C3 N=128", eb.build_unit_cube_mesh(128)),
                ("C5 N=256", eb.build_unit_cube_mesh(256))):
    nb, n_e, n_n, dim = m.conn.shape[0], m.n_elements, m.n_nodes, m.dim
    K, M, A = (D.empty((n_e, nb, nb)) for _ in range(3))
    b = D.empty((nb, n_e))
    bad = D.zeros(1, torch.int64)
    s = D.stream()

    def run():
        lib.ebs_assemble_p1(dim, n_e, D.ptr(m.nodes), D.ptr(m.conn), ctypes.c_double(1.0), None,
                            ctypes.c_double(1.0), D.ptr(K), D.ptr(M), D.ptr(A), D.ptr(b),
                            D.ptr(bad), s)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        run()
    ev[1].record()
    torch.cuda.synchronize()
    t = ev[0].elapsed_time(ev[1]) / 10 / 1e3
    byt = n_e * (4 * nb + 24 * nb * nb + 8 * nb) + 8 * dim * n_n
    print(f"{name}: {n_e} elements, {t * 1e3:.3f} ms, {byt / 1e9:.2f} GB -> "
          f"{byt / t / 1e9:.0f} GB/s = {byt / t / 1e9 / peak:.3f} of peak", flush=True)
    del K, M, A, b
    torch.cuda.empty_cache()
