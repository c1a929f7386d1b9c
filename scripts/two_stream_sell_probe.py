"""Where does the two-stream gain of scripts/two_stream_probe.py come from?  The SELL pass
alone (ebs_plan_apply on internal-order vectors: no x permutation, no fill, no scattered
output) back to back on one stream vs alternating between two streams (two plans).  If the
persistent sweep had a long tail, the second stream's sweep would fill it."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200 import _device as D  # noqa: E402
from paper_1911_03973_b200._lib import load  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

p = config_problem(2, seed=0)
m = p["mesh"]
batches = [p["batch"], eb.build_element_batch(eb.Mesh(m.nodes, None, m.boundary_nodes, conn=m.conn.clone()), nu=1.0)]
plans = [b.operator(m.n_nodes) for b in batches]
lib = load()
n = m.n_nodes
xi = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(2)]
ri = [D.empty(n) for _ in range(2)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
K = 100


def run(two):
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for k in range(K):
        i = k % 2 if two else 0
        st = streams[i]
        lib.ebs_plan_apply(plans[i].handle, 1, D.ptr(xi[i]), D.ptr(ri[i]), 0, 0,
                           ctypes.c_void_p(st.cuda_stream))
    for s in streams:
        cur.wait_stream(s)


for name, two in (("one stream", False), ("two streams", True)) * 3:
    run(two); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); run(two); e1.record(); torch.cuda.synchronize()
    print(f"SELL pass, internal order, {name:12s} {e0.elapsed_time(e1) / K * 1e3:7.1f} us per pass", flush=True)
