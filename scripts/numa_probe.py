"""Pinned-copy bandwidth vs the NUMA node of the host buffer: the process is bound to the
cores of each node in turn (first touch puts the pinned pages there), then H2D / D2H /
both-direction rates of a 33.6 MB vector.  python scripts/numa_probe.py"""
import glob
import os
import sys
sys.path.insert(0, '.')
import torch

n = 4198401
nb = 8 * n
reps = 16


def cpus_of(node):
    s = open(f"/sys/devices/system/node/node{node}/cpulist").read().strip()
    out = []
    for part in s.split(","):
        a, _, b = part.partition("-")
        out += list(range(int(a), int(b or a) + 1))
    return out


nodes = sorted(int(p.rsplit("node", 1)[1]) for p in glob.glob("/sys/devices/system/node/node[0-9]*"))
print("nodes", nodes, {nd: len(cpus_of(nd)) for nd in nodes}, "cpus", os.cpu_count(), flush=True)
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("gpu0 numa node (nvml):", pynvml.nvmlDeviceGetNumaNodeId(h) if hasattr(pynvml, "nvmlDeviceGetNumaNodeId") else "?",
          "pci", pynvml.nvmlDeviceGetPciInfo(h).busId, flush=True)
except Exception as e:
    print("nvml:", e)
try:
    bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
except Exception:
    bus = None
for p in glob.glob("/sys/bus/pci/devices/*/numa_node"):
    pass
d_x = torch.empty(n, dtype=torch.float64, device="cuda")
d_r = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for nd in nodes:
    os.sched_setaffinity(0, cpus_of(nd))
    h_x = torch.empty(n, dtype=torch.float64).pin_memory()
    h_r = torch.empty(n, dtype=torch.float64).pin_memory()
    h_x.fill_(1.0); h_r.fill_(0.0)
    res = {}
    for name in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        e0.record(cur); s1.wait_stream(cur); s2.wait_stream(cur)
        for _ in range(reps):
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d_x.copy_(h_x, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h_r.copy_(d_r, non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2); e1.record(cur)
        torch.cuda.synchronize()
        res[name] = reps * nb / (e0.elapsed_time(e1) / 1e3) / 1e9
    print(f"node {nd}: H2D {res['h2d']:.1f} GB/s  D2H {res['d2h']:.1f} GB/s  both {res['both']:.1f} GB/s per direction", flush=True)
    del h_x, h_r
