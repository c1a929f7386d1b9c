"""ncu target: BASELINE C4 (level 12, jittered + permuted, nu = 10) damped Jacobi, two short
solves of 6 iterations: `ncu --set full -k regex:k_jacobi_step -s 6 -c 1 python
scripts/jacobi_ncu_target.py`."""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem

torch.cuda.set_device(0)
p = config_problem(4, seed=0)
x0 = torch.zeros(p["mesh"].n_nodes, dtype=torch.float64, device="cuda")
for _ in range(2):
    eb.jacobi(p["batch"], p["dirichlet"], x0, 6, omega=0.8)
torch.cuda.synchronize()
