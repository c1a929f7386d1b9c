"""Time the C2 caller-numbering residual (ebs_residual, fast mode) per call; with the debug
build (EBS_LIB_PATH=.../variants/libebs_dbg.so) the fused pass prints its fallback count."""
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
x = torch.from_numpy(p["x"]).cuda()
r = D.empty(m.n_nodes)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for _ in range(3):
    lib.ebs_residual(pl.handle, D.ptr(x), D.ptr(r), EBS_RES_FAST, 0, None, s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    lib.ebs_residual(pl.handle, D.ptr(x), D.ptr(r), EBS_RES_FAST, 0, None, s)
e1.record()
torch.cuda.synchronize()
print(f"us per residual: {e0.elapsed_time(e1) / K * 1e3:.1f}")
