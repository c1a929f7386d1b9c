"""ncu target: BASELINE C3 with a seeded random node permutation (the unstructured-numbering
3D path: first-appearance ids, 8 B delta words) -- two short PCG solves of 6 iterations,
e.g. `ncu --set full -k regex:k_pcg_matvec -s 6 -c 1 python scripts/c3p_ncu_target.py`."""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

torch.cuda.set_device(0)
p = config_problem(3, seed=0, assemble=False)
m = eb.permute_nodes(p["mesh"], np.random.default_rng(1).permutation(p["mesh"].n_nodes))
nd = eb.face_z0_nodes(m)
d = eb.DirichletData(nd, torch.zeros(nd.numel(), dtype=torch.float64, device="cuda"))
batch = eb.build_element_batch(m, nu=p["nu"])
print("plan flags", batch.operator(m.n_nodes).info())
x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
for _ in range(2):
    eb.pcg(batch, d, x0, 6)
torch.cuda.synchronize()
