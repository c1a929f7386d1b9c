"""ncu target: builds a BASELINE config (argv[1], default 5) and runs two short PCG solves
(6 iterations each), e.g. `ncu --set full -k regex:k_pcg_ -s 6 -c 3 python
scripts/pcg_ncu_target.py 5`."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
torch.cuda.set_device(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = config_problem(cfg, seed=0)
x0 = torch.zeros(p["mesh"].n_nodes, dtype=torch.float64, device="cuda")
for _ in range(2):
    eb.pcg(p["batch"], p["dirichlet"], x0, 6)
torch.cuda.synchronize()
