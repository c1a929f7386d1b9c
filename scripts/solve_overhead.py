"""Per-solve fixed cost and per-iteration cost of the 1-GPU solvers (C3 PCG, C4 Jacobi):
device time of solves with 0..400 iterations, plus the SM clock (NVML) during each."""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__))))
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402

try:
    import pynvml
    pynvml.nvmlInit()
    H = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:  # noqa: BLE001
    H = None


def clocks():
    if H is None:
        return (0, 0)
    return (pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM),
            pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_MEM))


cfgs = [int(a) for a in sys.argv[1:]] or [4, 3]
for cfg in cfgs:
    p = config_problem(cfg)
    b, d, m = p["batch"], p["dirichlet"], p["mesh"]
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    run = ((lambda it: eb.jacobi(b, d, x0, it, omega=0.8)) if cfg == 4
           else (lambda it: eb.pcg(b, d, x0, it)))
    run(200)
    torch.cuda.synchronize()
    for it in (0, 32, 96, 200, 400):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(it)
        e1.record()
        c = clocks()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"C{cfg} iters={it:4d}: {ms:8.2f} ms  per-it {ms / max(it, 1) * 1e3:7.1f} us"
              f"  sm/mem MHz {c}", flush=True)
