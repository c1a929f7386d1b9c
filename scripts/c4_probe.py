"""C4 damped Jacobi x200 (level 12 jittered + permuted, nu=10) and C2 internal matvec:
device time per iteration -- quick A/B of kernel variants (EBS_LIB_PATH)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 12
p = config_problem(4, seed=0, size=size)
batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
eb.jacobi(batch, d, x0, 200, omega=0.8)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, h = eb.jacobi(batch, d, x0, 200, omega=0.8)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 200)
print(f"C4 jacobi: {best * 1e3:.1f} us/it  {1e3 / best:.0f} it/s  final {h.residual_norms[-1]:.12e}")
