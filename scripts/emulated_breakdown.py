"""Per-kernel device time per iteration of the emulated P-slab loop (one GPU, CUPTI via
torch.profiler): where the partitioning overhead of scripts/emulated_scaling.py goes.
Usage: python scripts/emulated_breakdown.py CFG P [peer]"""
import sys
from collections import defaultdict

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1911_03973_b200 import dist  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
iters = 64
p = config_problem(cfg)
batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
peer = len(sys.argv) > 3 and sys.argv[3] == "peer"
prob, _ = dist.emulate(batch, m.n_nodes, d, P, peer=peer)
x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
xin = [op.to_internal(x0) for op in prob.ops]
if cfg == 2:  # the caller-order slab residual (bench value), graph of `iters` residuals
    x = torch.from_numpy(p["x"]).cuda()
    xl = [x[op.global_ids].contiguous() for op in prob.ops]
    rl, xi, sr = ([op.zeros() for op in prob.ops] for _ in range(3))

    def body():
        for _ in range(iters):
            dist.residual_local(prob, xl, rl, xi, sr)
    body()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        body()
    run = g.replay
elif cfg == 4:
    run = lambda: dist.jacobi(prob, xin, iters, 0.8, graph=True)  # noqa: E731
else:
    run = lambda: dist.pcg(prob, xin, iters, graph=True)  # noqa: E731
run()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
tot, cnt = defaultdict(float), defaultdict(int)
gap, prev = 0.0, None
for e in evs:
    tot[e.name[:60]] += e.time_range.elapsed_us()
    cnt[e.name[:60]] += 1
    if prev is not None and e.time_range.start > prev:
        gap += e.time_range.start - prev
    prev = max(prev or 0, e.time_range.end)
span = (evs[-1].time_range.end - evs[0].time_range.start) if evs else 0
print(f"C{cfg} P={P}: {span / iters:.1f} us/it span, idle {gap / iters:.1f} us/it; per rank-iteration:")
for k in sorted(tot, key=tot.get, reverse=True)[:12]:
    print(f"  {tot[k] / iters / P:8.2f} us  x{cnt[k] / iters / P:4.1f}  {k}")
# the two SELL sweeps of a rank-iteration: interface chunks first, then the interior
sw = [e.time_range.elapsed_us() for e in evs if "_sweep" in e.name]
if sw:
    # per iteration: the P ranks' interface sweeps, then the P interior sweeps (P = 1 and
    # no interface: interior only)
    has_if = any(op.if_chunks.numel() for op in prob.ops)
    a = [t for k, t in enumerate(sw) if has_if and (k % (2 * P)) < P]
    b = [t for k, t in enumerate(sw) if not has_if or (k % (2 * P)) >= P]
    a = a or [0.0]
    print(f"  interface sweep {sum(a) / len(a):.2f} us, interior sweep {sum(b) / len(b):.2f} us "
          f"(mean per launch); chunks per rank: interface "
          f"{sum(op.if_chunks.numel() for op in prob.ops) / P:.0f}, interior "
          f"{sum(op.in_chunks.numel() for op in prob.ops) / P:.0f}")
