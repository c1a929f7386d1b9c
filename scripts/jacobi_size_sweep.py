"""Per-iteration time of the 1-GPU damped Jacobi (C4 recipe) vs mesh level: the fixed cost per
sweep (intercept) that dominates small slabs.  python scripts/jacobi_size_sweep.py"""
import sys
sys.path.insert(0, '.')
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
for size in (9, 10, 11, 12):
    p = config_problem(4, seed=0, size=size)
    b, d, m = p["batch"], p["dirichlet"], p["mesh"]
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    eb.jacobi(b, d, x0, 200, omega=0.8); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); eb.jacobi(b, d, x0, 200, omega=0.8); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / 200
    by = m.n_elements * 84 + 32 * m.n_nodes
    print(f"level {size}: {m.n_elements} tri, {t*1e6:.1f} us/it, {by/t/1e9:.0f} GB/s, chunks {(m.n_nodes+31)//32}", flush=True)
    del p, b
    torch.cuda.empty_cache()
