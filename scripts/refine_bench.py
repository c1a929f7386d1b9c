"""uniform_refine at level 11 -> 12 (8.4M -> 33.5M triangles): device (ebs_refine_tri)
vs the reference algorithm on the host (oracle restatement of mesh.py:157-208, NumPy,
one thread) -- and the level-12 generator for comparison.  Checks the device result
against build_unit_square_mesh(12) bit for bit."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle as o  # noqa: E402
import paper_1911_03973_b200 as eb  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 11
m = eb.build_unit_square_mesh(level)
eb.uniform_refine(eb.build_unit_square_mesh(4))  # warm
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    fine = eb.uniform_refine(m)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
direct = eb.build_unit_square_mesh(level + 1)
ok = torch.equal(fine.nodes, direct.nodes) and torch.equal(fine.conn, direct.conn)
print(f"device uniform_refine level {level}->{level + 1}: best {min(ts):.3f} s "
      f"({fine.n_elements} triangles), equals build_unit_square_mesh({level + 1}): {ok}")
nodes, elements, _ = o.unit_square_mesh(level)
t0 = time.perf_counter()
fn, fe = o.uniform_refine(nodes, elements)
th = time.perf_counter() - t0
print(f"host reference algorithm (oracle restatement, NumPy 1 thread): {th:.1f} s; "
      f"device result identical: {np.array_equal(fine.nodes.cpu().numpy(), fn) and np.array_equal(fine.elements.cpu().numpy(), fe)}")
