"""Host<->device copy throughput on this box: 33.6 MB vectors (C2's x and r) from/to pinned
memory, one direction alone and both at once, split over 1, 2 or 4 streams per direction."""
import torch

n = 4198401
x_h = torch.empty(n, dtype=torch.float64).pin_memory()
r_h = torch.empty(n, dtype=torch.float64).pin_memory()
x_d = torch.empty(n, dtype=torch.float64, device="cuda")
r_d = torch.empty(n, dtype=torch.float64, device="cuda")
K = 20


def run(split, h2d=True, d2h=True):
    ss_in = [torch.cuda.Stream() for _ in range(split)]
    ss_out = [torch.cuda.Stream() for _ in range(split)]
    bounds = [n * i // split for i in range(split + 1)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss_in + ss_out:
        s.wait_stream(torch.cuda.current_stream())
    for _ in range(K):
        for i in range(split):
            lo, hi = bounds[i], bounds[i + 1]
            if h2d:
                with torch.cuda.stream(ss_in[i]):
                    x_d[lo:hi].copy_(x_h[lo:hi], non_blocking=True)
            if d2h:
                with torch.cuda.stream(ss_out[i]):
                    r_h[lo:hi].copy_(r_d[lo:hi], non_blocking=True)
    for s in ss_in + ss_out:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    moved = K * 8 * n * (int(h2d) + int(d2h))
    return moved / t / 1e9


for split in (1, 2, 4):
    print(f"split {split}: H2D {run(split, True, False):6.1f} GB/s  D2H {run(split, False, True):6.1f}"
          f" GB/s  both {run(split):6.1f} GB/s aggregate", flush=True)
