"""Slab PCG at one rank (dist.pcg, LocalTransport) vs the 1-GPU PCG on BASELINE C5 (or
argv[1]): it/s of both -- A/B of the vector kernels through EBS_LIB_PATH."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200 import dist  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
iters = 100
p = config_problem(cfg)
batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")


def tm(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return iters / (e0.elapsed_time(e1) / 1e3)


from bench import ClockSampler  # noqa: E402
samp = ClockSampler().start()
samp.on()
one = tm(lambda: eb.pcg(batch, d, x0, iters))
del batch
torch.cuda.empty_cache()
op, _ = dist.rank_operator(m, p["nu"], p["f"], d, 1, 0)
prob = dist.setup([op], dist.LocalTransport())
xz = op.zeros()
r1 = tm(lambda: dist.pcg(prob, [xz], iters, graph=True))
r2 = tm(lambda: dist.pcg(prob, [xz], iters, graph=True, reductions=2))
rs = [tm(lambda: dist.pcg(prob, [xz], iters, graph=True)) for _ in range(4)]
samp.off()
samp.stop()
print(f"C{cfg}: 1-GPU pcg {one:.0f} it/s; slab pcg (1 rank) single-reduction {r1:.0f}, "
      f"two-reduction {r2:.0f} it/s; repeats {[round(v) for v in rs]}; graphs {dist.GRAPH_STATS}; "
      f"clocks {samp.summary()}")
