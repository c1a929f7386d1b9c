"""Timeline of the host-buffer residual pipeline (the ebs_residual_many_host schedule
replayed from Python with timing events around every copy and residual): where the
steps lose time against the both-directions PCIe rate.  python scripts/e2e_timeline_probe.py"""
import sys
sys.path.insert(0, '.')
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200 import _device as D
from paper_1911_03973_b200._lib import EBS_RES_FAST, call
from paper_1911_03973_b200.inputs import config_problem

p = config_problem(2, seed=0)
b, n = p["batch"], p["mesh"].n_nodes
NB, k = 3, 24
h_x = torch.empty(n, dtype=torch.float64).uniform_(-1, 1).pin_memory()
out = torch.empty((k, n), dtype=torch.float64).pin_memory()
xb = [D.empty(n) for _ in range(NB)]
rb = [D.empty(n) for _ in range(NB)]
comp = torch.cuda.current_stream()
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(2):
    t = {key: [E() for _ in range(k)] for key in ("h0", "h1", "c0", "c1", "d0", "d1")}
    x_in = [torch.cuda.Event() for _ in range(k)]
    used = [torch.cuda.Event() for _ in range(k)]
    rread = [torch.cuda.Event() for _ in range(k)]
    start = E()
    torch.cuda.synchronize()
    start.record(comp)
    h2d.wait_stream(comp); d2h.wait_stream(comp)
    with b.using(n) as pl:
        for i in range(k):
            j = i % NB
            if i >= NB:
                h2d.wait_event(used[i - NB])
            t["h0"][i].record(h2d)
            with torch.cuda.stream(h2d):
                xb[j].copy_(h_x, non_blocking=True)
            t["h1"][i].record(h2d)
            x_in[i].record(h2d)
            comp.wait_event(x_in[i])
            if i >= NB:
                comp.wait_event(rread[i - NB])
            t["c0"][i].record(comp)
            call("ebs_residual", pl.handle, D.ptr(xb[j]), D.ptr(rb[j]), EBS_RES_FAST, 0, None, D.stream())
            t["c1"][i].record(comp)
            used[i].record(comp)
            d2h.wait_event(used[i])
            t["d0"][i].record(d2h)
            with torch.cuda.stream(d2h):
                out[i].copy_(rb[j], non_blocking=True)
            t["d1"][i].record(d2h)
            rread[i].record(d2h)
    comp.wait_stream(d2h)
    end = E(); end.record(comp)
    torch.cuda.synchronize()
    print(f"rep {rep}: {start.elapsed_time(end) / k:.3f} ms/step", flush=True)
    if rep:
        for i in range(k):
            f = lambda key: start.elapsed_time(t[key][i])
            print(f"  {i:2d}  H2D {f('h0'):7.3f}-{f('h1'):7.3f} ({f('h1') - f('h0'):.3f})  "
                  f"res {f('c0'):7.3f}-{f('c1'):7.3f}  D2H {f('d0'):7.3f}-{f('d1'):7.3f} ({f('d1') - f('d0'):.3f})")
