import time, torch, sys
sys.path.insert(0, '.')
from paper_1911_03973_b200.inputs import stacked_c2_problem
from paper_1911_03973_b200 import dist
t0 = time.perf_counter()
p = stacked_c2_problem(8)
torch.cuda.synchronize(); t1 = time.perf_counter()
m = p["mesh"]
for rank in (0, 3, 7):
    op, maps = dist.rank_operator(m, p["nu"], p["f"], None, 8, rank)
    torch.cuda.synchronize()
    print("rank", rank, "local nodes", op.n, "if", {q: int(v.numel()) for q, v in op.if_idx.items()},
          "if_chunks", op.if_chunks.numel(), "in_chunks", op.in_chunks.numel())
    del op
t2 = time.perf_counter()
print(f"stacked mesh {m.n_nodes} nodes {m.n_elements} elems: build {t1-t0:.2f}s, 3 rank ops {t2-t1:.2f}s, peak mem {torch.cuda.max_memory_allocated()/1e9:.1f} GB")
