import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2203_15340_b200 import ils
from workloads import make_problem
pr = make_problem("c2")
A = torch.from_numpy(pr.A).cuda(); b = torch.from_numpy(pr.b).cuda()
h = ils.ils_create(A, b, pr.p, pr.q, pr.n)
for rep in range(2):
    x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
    ils.ils_sp_solve(h, None, x, 0.0, 16, ils.ils_default_opts(stop=ils.ILS_STOP_NONE))
torch.cuda.synchronize()
