"""bench.py's e2e leg replayed with variations: as in the bench (2-row warm call, then one
k = 100 call timed by events), with a full-size warm call first, and without the NVML
clock sampler.  python scripts/e2e_bench_replica.py"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import bench
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem

p = config_problem(2, seed=0)
b, n = p["batch"], p["mesh"].n_nodes
x_np = np.random.default_rng(0).uniform(-1, 1, n)
k = 100


def leg(full_warm, sampler):
    x_host = torch.from_numpy(x_np).pin_memory()
    r_many = torch.empty((k, n), dtype=torch.float64).pin_memory()
    xs = x_host.unsqueeze(0).expand(k, n)
    eb.residual_many(b, xs[:k if full_warm else 2], out=r_many[:k if full_warm else 2], deterministic=False)
    torch.cuda.synchronize()
    smp = bench.ClockSampler().start() if sampler else None
    if smp:
        smp.on()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eb.residual_many(b, xs, out=r_many, deterministic=False)
    e1.record()
    torch.cuda.synchronize()
    if smp:
        smp.stop()
    t = e0.elapsed_time(e1) / k
    print(f"full_warm={full_warm} sampler={sampler}: {t:.3f} ms/step ({n / t / 1e6:.2f} GDoF/s)", flush=True)


for fw, sm in ((False, True), (False, False), (True, True), (True, False), (False, True)):
    leg(fw, sm)
