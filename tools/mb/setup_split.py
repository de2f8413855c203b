"""Development aid: split SP setup time on a config into Gram (SP-SCD setup) and Cholesky +
inverse + P (the rest of SP setup), fresh handle each, CUDA-event times from the report."""
import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2203_15340_b200 import ils
from workloads import make_problem
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
pr = make_problem(cfg)
A = torch.from_numpy(pr.A).cuda(); b = torch.from_numpy(pr.b).cuda()
for rep in range(3):
    h = ils.ils_create(A, b, pr.p, pr.q, pr.n)
    x = np.zeros(pr.n)
    st, r1 = ils.ils_rgs_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=1, check_every=1))
    st, r2 = ils.ils_sp_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE))
    ils.ils_destroy(h)
    h = ils.ils_create(A, b, pr.p, pr.q, pr.n)
    st, r3 = ils.ils_sp_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE))
    ils.ils_destroy(h)
    print(f"{cfg}: gram {r1.setup_ms:.2f} ms, chol+inv+P {r2.setup_ms:.2f} ms, SP setup fresh {r3.setup_ms:.2f} ms", flush=True)
