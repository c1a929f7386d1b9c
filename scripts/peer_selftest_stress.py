"""Long run of the concurrent peer-protocol self-test (ebs_peer_selftest) over meshes and
rank counts 2..8, 2000 rounds each: python scripts/peer_selftest_stress.py"""
import sys, os
sys.path.insert(0, '.')
from paper_1911_03973_b200 import dist
from paper_1911_03973_b200.inputs import config_problem
for cfg, size in ((4, 7), (5, 8), (4, 9)):
    pr = config_problem(cfg, seed=3, size=size)
    m = pr["mesh"]
    for P in (2, 3, 4, 5, 6, 7, 8):
        prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], P, peer=True)
        n = prob.comm.selftest(2000)
        prob.comm.status()
        print(f"C{cfg} size {size} P={P}: 2000 rounds, {n} wrong values", flush=True)
        prob.comm.close()
