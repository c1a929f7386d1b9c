"""Does write-combined pinned memory (cudaHostAllocWriteCombined) as the SOURCE of the
host->device copies raise the e2e ceiling?  A C2-sized vector (33.6 MB), 32 copies back to
back: H2D alone and H2D while the D2H of the step before runs (the pipeline's steady
state), from ordinary pinned memory and from write-combined pinned memory, plus NUMA-agnostic
cudaHostAllocPortable and cudaHostRegister'ed malloc memory for reference.
python scripts/pcie_wc_probe.py"""
import ctypes
import sys

sys.path.insert(0, '.')
import torch

n = 4198401
nb = 8 * n
reps = 32
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaHostAlloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                               ctypes.c_void_p]
H2D, D2H = 1, 2


def host_alloc(flags):
    p = ctypes.c_void_p()
    rc = rt.cudaHostAlloc(ctypes.byref(p), nb, flags)
    assert rc == 0, rc
    return p


torch.cuda.init()
d_x = torch.empty(n, dtype=torch.float64, device="cuda")
d_r = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h_r = host_alloc(0)
srcs = {"pinned (default)": host_alloc(0), "pinned portable": host_alloc(1),
        "pinned write-combined": host_alloc(4)}
for p in srcs.values():  # touch every page once from the host (streaming writes)
    ctypes.memset(p, 1, nb)
ctypes.memset(h_r, 0, nb)


def run(src, with_d2h):
    def go():
        for _ in range(reps):
            rt.cudaMemcpyAsync(d_x.data_ptr(), src, nb, H2D, ctypes.c_void_p(s1.cuda_stream))
            if with_d2h:
                rt.cudaMemcpyAsync(h_r, d_r.data_ptr(), nb, D2H, ctypes.c_void_p(s2.cuda_stream))
    go()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(s1); b0.record(s2)
    go()
    a1.record(s1); b1.record(s2)
    torch.cuda.synchronize()
    return a0.elapsed_time(a1) / reps, b0.elapsed_time(b1) / reps


for rep in range(2):
    for name, src in srcs.items():
        h, _ = run(src, False)
        hb, db = run(src, True)
        print(f"{name:24s} H2D alone {h:.3f} ms ({nb / h / 1e6:5.1f} GB/s) | with D2H: H2D {hb:.3f} ms "
              f"({nb / hb / 1e6:5.1f} GB/s), D2H {db:.3f} ms ({nb / db / 1e6:5.1f} GB/s) -> e2e ceiling "
              f"{n / max(hb, db) / 1e6:.2f} GDoF/s", flush=True)
