"""ncu target: the peer-memory slab loops emulated on one GPU (dist.emulate(..., peer=True):
P ranks' windows in this process, every put before any get) -- BASELINE C5 Jacobi-PCG
(single reduction, fused all-reduce) or C4 damped Jacobi on P = 8 slabs, a few iterations
twice:
  ncu --set full -k regex:"k_peer_matvec_sweep|k_peer_combine_q|k_vec_cg1_update" -s 24 -c 3 \
      python scripts/peer_ncu_target.py 5
  ncu --set full -k regex:"k_peer_jacobi_sweep|k_peer_combine_jacobi" -s 24 -c 2 \
      python scripts/peer_ncu_target.py 4"""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1911_03973_b200 import dist  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

torch.cuda.set_device(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
p = config_problem(cfg)
m = p["mesh"]
prob, _ = dist.emulate(p["batch"], m.n_nodes, p["dirichlet"], P, peer=True)
del p
x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
xin = [op.to_internal(x0) for op in prob.ops]
for _ in range(2):
    if cfg == 4:
        dist.jacobi(prob, xin, 6, 0.8)
    else:
        dist.pcg(prob, xin, 6)
torch.cuda.synchronize()
prob.comm.status()
