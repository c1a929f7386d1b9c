"""PCIe ceiling for the e2e leg: pinned host <-> HBM copy bandwidth of a C2-sized vector
(33.6 MB), H2D alone, D2H alone and both directions at once on two copy streams, then
the pipelined residual_many call for comparison.  python scripts/pcie_probe.py"""
import sys
sys.path.insert(0, '.')
import torch

n = 4198401
nb = 8 * n
reps = 32
h_x = torch.empty(n, dtype=torch.float64).pin_memory()
h_r = torch.empty(n, dtype=torch.float64).pin_memory()
d_x = torch.empty(n, dtype=torch.float64, device="cuda")
d_r = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    s1.wait_stream(cur); s2.wait_stream(cur)
    fn()
    cur.wait_stream(s1); cur.wait_stream(s2)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def h2d():
    with torch.cuda.stream(s1):
        for _ in range(reps):
            d_x.copy_(h_x, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        for _ in range(reps):
            h_r.copy_(d_r, non_blocking=True)


def both():
    h2d(); d2h()


for name, fn, dirs in (("H2D", h2d, 1), ("D2H", d2h, 1), ("both", both, 2)):
    t = timed(fn)
    print(f"{name:5s}: {reps * nb / t / 1e9:6.1f} GB/s per direction, {t / reps * 1e3:.3f} ms per 33.6 MB step"
          f" (e2e ceiling {n / (t / reps) / 1e9:.2f} GDoF/s)", flush=True)

import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
p = config_problem(2, seed=0)
b = p["batch"]
xs = h_x.unsqueeze(0).expand(reps, n)
out = torch.empty((reps, n), dtype=torch.float64).pin_memory()
h_x.uniform_(-1, 1)
t = timed(lambda: eb.residual_many(b, xs, out=out, deterministic=False))
print(f"residual_many: {t / reps * 1e3:.3f} ms per step, {n / (t / reps) / 1e9:.2f} GDoF/s", flush=True)

# both directions, each copy split over two streams (two copy engines per direction)
s3, s4 = torch.cuda.Stream(), torch.cuda.Stream()
half = n // 2


def both_split():
    cur = torch.cuda.current_stream()
    s3.wait_stream(cur); s4.wait_stream(cur)
    with torch.cuda.stream(s1):
        for _ in range(reps):
            d_x[:half].copy_(h_x[:half], non_blocking=True)
    with torch.cuda.stream(s3):
        for _ in range(reps):
            d_x[half:].copy_(h_x[half:], non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(reps):
            h_r[:half].copy_(d_r[:half], non_blocking=True)
    with torch.cuda.stream(s4):
        for _ in range(reps):
            h_r[half:].copy_(d_r[half:], non_blocking=True)
    cur.wait_stream(s3); cur.wait_stream(s4)


t = timed(both_split)
print(f"both, 2 streams/dir: {reps * nb / t / 1e9:6.1f} GB/s per direction", flush=True)

import time
for k in (32, 100):
    xs = h_x.unsqueeze(0).expand(k, n)
    out = torch.empty((k, n), dtype=torch.float64).pin_memory()
    eb.residual_many(b, xs, out=out, deterministic=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eb.residual_many(b, xs, out=out, deterministic=False, check_finite=False)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"residual_many k={k}: host issue {(t1 - t0) / k * 1e3:.3f} ms/step, wall {(t2 - t0) / k * 1e3:.3f} ms/step "
          f"({n / ((t2 - t0) / k) / 1e9:.2f} GDoF/s)", flush=True)
    del out
