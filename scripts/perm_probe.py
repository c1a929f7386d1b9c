"""Time the caller -> internal x permutation and the full caller-order residual at C2
(or another level) for the libebs build selected by EBS_LIB_PATH.

    EBS_LIB_PATH=... python scripts/perm_probe.py [--size 11] [--steps 200]

Prints one JSON line: µs per ebs_to_internal, per SELL pass (ebs_plan_apply into a
-0.0-filled caller-order r), per ebs_residual (back to back, and replayed as a graph)."""

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=11)
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    import torch

    from paper_1911_03973_b200 import _device as D
    from paper_1911_03973_b200._lib import EBS_RES_FAST, load
    from paper_1911_03973_b200.inputs import config_problem

    torch.cuda.set_device(0)
    p = config_problem(2, seed=0, size=a.size)
    batch, m = p["batch"], p["mesh"]
    n = m.n_nodes
    pl = batch.operator(n)
    lib = load()
    h = pl.handle
    st = torch.cuda.current_stream()
    s = ctypes.c_void_p(st.cuda_stream)
    x = torch.from_numpy(p["x"]).cuda()
    xi, r = D.empty(n), D.empty(n)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    K = a.steps

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / K)
        return best

    def perm():
        for _ in range(K):
            lib.ebs_to_internal(h, P(x), P(xi), None, s)

    def sell():
        for _ in range(K):
            lib.ebs_plan_apply(h, 1, P(xi), P(r), 1, 0, s)

    def res():
        for _ in range(K):
            lib.ebs_residual(h, P(x), P(r), EBS_RES_FAST, 0, None, s)

    out = {"lib": os.path.basename(os.environ.get("EBS_LIB_PATH", "libebs.so")), "n": n,
           "perm_us": timeit(perm), "sell_us": timeit(sell), "residual_us": timeit(res)}
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cs = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(K):
            lib.ebs_residual(h, P(x), P(r), EBS_RES_FAST, 0, None, cs)
    out["residual_graph_us"] = timeit(lambda: g.replay())
    out["gdofs_graph"] = n / out["residual_graph_us"] / 1e3
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
