import sys, torch
sys.path.insert(0, '.')
from paper_1911_03973_b200 import dist
from paper_1911_03973_b200._lib import load
from paper_1911_03973_b200.inputs import config_problem
pr = config_problem(4, seed=1, size=8)
m = pr["mesh"]
prob, _ = dist.emulate(pr["batch"], m.n_nodes, pr["dirichlet"], 4)
x0 = [op.zeros() for op in prob.ops]
lib = load()
for run, name in ((lambda it: dist.jacobi(prob, x0, it), "jacobi"), (lambda it: dist.pcg(prob, x0, it), "pcg")):
    run(2); torch.cuda.synchronize()
    a = lib.ebs_launch_count(); run(10); torch.cuda.synchronize(); b = lib.ebs_launch_count()
    a2 = lib.ebs_launch_count(); run(20); torch.cuda.synchronize(); b2 = lib.ebs_launch_count()
    print(name, "libebs launches per iteration per rank:", ((b2 - a2) - (b - a)) / 10 / 4)
