"""Do independent C2 residuals overlap usefully on two streams?  Two plans of the same mesh
(each with its own workspace), residual k on stream k % 2: the gather / fill of one step can
fill the tail of the other's SELL pass.  python scripts/two_stream_probe.py"""
import sys
sys.path.insert(0, '.')
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem

p = config_problem(2, seed=0)
m = p["mesh"]
batches = [p["batch"], eb.build_element_batch(eb.Mesh(m.nodes, None, m.boundary_nodes, conn=m.conn.clone()), nu=1.0)]
x = torch.as_tensor(p["x"], device="cuda")
outs = [torch.empty_like(x) for _ in range(2)]
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
K = 100


def one_stream():
    for k in range(K):
        eb.residual(batches[0], x, deterministic=False, out=outs[0], check_finite=False)


def two_streams():
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for k in range(K):
        with torch.cuda.stream(streams[k % 2]):
            eb.residual(batches[k % 2], x, deterministic=False, out=outs[k % 2], check_finite=False)
    for s in streams:
        cur.wait_stream(s)


for name, fn in (("one stream", one_stream), ("two streams", two_streams)) * 3:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / K
    print(f"{name:12s} {t * 1e3:7.1f} us per residual, {m.n_nodes / t / 1e6:.2f} GDoF/s", flush=True)
assert torch.equal(outs[0], outs[1])
