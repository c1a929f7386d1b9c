"""C2 caller-numbering residual: the fused red.add output (ebs_residual, fast mode) against
the split form -- x permutation, SELL pass with INTERNAL-order output (coalesced), then a
gather of r back into the caller's numbering (ebs_to_user, random reads of an L2-resident
r_int).  Both give bit-identical r (checked).  Prints us per residual for each, with a
per-kernel breakdown of the split form."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_03973_b200 import _device as D  # noqa: E402
from paper_1911_03973_b200._lib import EBS_RES_FAST, load  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

p = config_problem(2, seed=0)
batch, m = p["batch"], p["mesh"]
pl = batch.operator(m.n_nodes)
lib = load()
n = m.n_nodes
x = torch.from_numpy(p["x"]).cuda()
r = D.empty(n)
r2 = D.empty(n)
xi = D.empty(n)
ri = D.empty(n)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 50


def fused():
    lib.ebs_residual(pl.handle, D.ptr(x), D.ptr(r), EBS_RES_FAST, 0, None, s)


def split(ev=None):
    lib.ebs_to_internal(pl.handle, D.ptr(x), D.ptr(xi), None, s)
    if ev: ev[0].record()
    lib.ebs_plan_apply(pl.handle, 1, D.ptr(xi), D.ptr(ri), 0, 0, s)
    if ev: ev[1].record()
    lib.ebs_to_user(pl.handle, D.ptr(ri), D.ptr(r2), s)


def timeit(f, k=K):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


fused()
split()
torch.cuda.synchronize()
print("bitwise equal:", bool(torch.equal(r.view(torch.int64), r2.view(torch.int64))))
for rep in range(3):
    print(f"rep {rep}: fused {timeit(fused):.1f} us   split {timeit(split):.1f} us")
# breakdown of the split form
ts = []
for _ in range(20):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[2].record()
    split(ev[:2])
    ev[3].record()
    torch.cuda.synchronize()
    ts.append((ev[2].elapsed_time(ev[0]) * 1e3, ev[0].elapsed_time(ev[1]) * 1e3,
               ev[1].elapsed_time(ev[3]) * 1e3))
ts.sort(key=lambda t: sum(t))
g, a, u = ts[len(ts) // 2]
print(f"split breakdown (median): to_internal {g:.1f}  sell internal {a:.1f}  to_user {u:.1f} us")
