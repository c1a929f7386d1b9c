import subprocess, threading, time, sys
sys.path.insert(0, '.')
import torch
import paper_1911_03973_b200 as eb
from paper_1911_03973_b200.inputs import config_problem
p = config_problem(4)
batch, d, m = p["batch"], p["dirichlet"], p["mesh"]
x0 = torch.zeros(m.n_nodes, dtype=torch.float64, device="cuda")
eb.jacobi(batch, d, x0, 200, omega=0.8); torch.cuda.synchronize()
samples = []
stop = False
def sampler():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append(out)
        time.sleep(0.05)
th = threading.Thread(target=sampler); th.start()
t0 = time.time(); n = 0
while time.time() - t0 < 6:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); eb.jacobi(batch, d, x0, 200, omega=0.8); e1.record(); torch.cuda.synchronize()
    n += 1
    print(f"run {n}: {200 / (e0.elapsed_time(e1) / 1e3):.0f} it/s", flush=True)
stop = True; th.join()
for s in samples[::4]: print(s)
