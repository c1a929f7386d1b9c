"""ncu target: the slab PCG of BASELINE C5 on ONE rank through the distributed loop
(dist.pcg, single-reduction recurrence, LocalTransport), 6 iterations twice:
`ncu --set full -k regex:"k_vec_cg1_update|k_dist_matvec_sweep" -s 4 -c 3 python
scripts/dist_ncu_target.py`."""
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1911_03973_b200 import dist  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

torch.cuda.set_device(0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
p = config_problem(cfg, assemble=False)
op, _ = dist.rank_operator(p["mesh"], p["nu"], p["f"], p["dirichlet"], 1, 0)
prob = dist.setup([op], dist.LocalTransport())
x0 = op.zeros()
for _ in range(2):
    dist.pcg(prob, [x0], 6)
torch.cuda.synchronize()
