"""ebs_residual_many (two residuals in flight inside ONE plan) vs k x ebs_residual, C2, with
bitwise comparison; eager and CUDA-graph replay.  python scripts/two_stream_probe2.py"""
import sys
sys.path.insert(0, '.')
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem

p = config_problem(2, seed=0)
m, batch = p["mesh"], p["batch"]
n = m.n_nodes
K = 100
x = torch.as_tensor(p["x"], device="cuda")
xs = x.unsqueeze(0).expand(K, n)
out = torch.empty((K, n), dtype=torch.float64, device="cuda")
ref = eb.residual(batch, x, deterministic=False)


def loop():
    for k in range(K):
        eb.residual(batch, x, deterministic=False, out=out[k], check_finite=False)


def many():
    eb.residual_many(batch, xs, out=out, deterministic=False, check_finite=False)


def timed(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


for rep in range(3):
    out.zero_()
    tl = timed(loop)
    out.zero_()
    tm = timed(many)
    ok = all(torch.equal(out[k], ref) for k in (0, 1, K // 2, K - 1))
    print(f"k x residual {tl:6.1f} us ({n / tl / 1e3:.2f} GDoF/s) | residual_many {tm:6.1f} us "
          f"({n / tm / 1e3:.2f} GDoF/s) bitwise {ok}", flush=True)
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    many(); torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        many()
    for rep in range(3):
        out.zero_()
        t = timed(g.replay)
        ok = all(torch.equal(out[k], ref) for k in (0, 1, K - 1))
        print(f"residual_many graph replay {t:6.1f} us ({n / t / 1e3:.2f} GDoF/s) bitwise {ok}", flush=True)
# exact mode + non-finite flags
xs2 = torch.stack([x, x * 2, x * 3])
xs2[1, 5] = float("nan")
try:
    eb.residual_many(batch, xs2)
    print("ERROR: no ValueError")
except ValueError as e:
    print("non-finite:", e)
xs2[1, 5] = 0.5
o = eb.residual_many(batch, xs2)
print("exact bitwise:", all(torch.equal(o[i], eb.residual(batch, xs2[i])) for i in range(3)))
