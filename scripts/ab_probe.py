"""Quick A/B of libebs builds (EBS_LIB_PATH): C2 caller-order residual, C2 internal matvec,
C4 Jacobi x200, C3 / C5 PCG -- device time."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_1911_03973_b200 as eb  # noqa: E402
from paper_1911_03973_b200 import _device as D  # noqa: E402
from paper_1911_03973_b200._lib import EBS_RES_FAST, load  # noqa: E402
from paper_1911_03973_b200.inputs import config_problem  # noqa: E402


def t_events(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


which = sys.argv[1:] or ["c2", "c4", "c3", "c5"]
lib = load()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
if "c2" in which:
    p = config_problem(2, seed=0)
    batch, m = p["batch"], p["mesh"]
    pl = batch.operator(m.n_nodes)
    x = torch.from_numpy(p["x"]).cuda()
    r = D.empty(m.n_nodes)
    xi = D.empty(m.n_nodes)
    y = D.empty(m.n_nodes)
    lib.ebs_to_internal(pl.handle, D.ptr(x), D.ptr(xi), None, s)
    res = lambda: [lib.ebs_residual(pl.handle, D.ptr(x), D.ptr(r), EBS_RES_FAST, 0, None, s) for _ in range(100)]  # noqa: E731
    mv = lambda: [lib.ebs_plan_apply(pl.handle, 0, D.ptr(xi), D.ptr(y), 0, 0, s) for _ in range(100)]  # noqa: E731
    res(); mv()
    print(f"C2 residual {t_events(res) * 10:.1f} us   internal matvec {t_events(mv) * 10:.1f} us")
    del p, batch, pl
for cfg, iters in (("c4", 200), ("c3", 200), ("c5", 100)):
    if cfg not in which:
        continue
    p = config_problem(int(cfg[1]), seed=0)
    batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
    x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
    run = (lambda: eb.jacobi(batch, d, x0, iters, omega=0.8)) if cfg == "c4" else \
        (lambda: eb.pcg(batch, d, x0, iters))
    run()
    ms = t_events(run)
    print(f"{cfg.upper()} {iters / ms * 1e3:.0f} it/s ({ms / iters * 1e3:.1f} us/it)")
    del p, batch
    torch.cuda.empty_cache()
