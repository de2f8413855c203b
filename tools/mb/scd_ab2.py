import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2203_15340_b200 import ils
from workloads import make_dense
for n in (384, 512, 768, 1000):
    pr = make_dense(4 * n, n // 2, n, 0.3, seed=1)
    A = torch.from_numpy(pr.A).cuda(); b = torch.from_numpy(pr.b).cuda()
    out = []
    for env, nt in (("1", "256"), ("1", "128")):
        os.environ["ILS_SCD_CTA"] = env
        os.environ["ILS_SCD_NT"] = nt
        h = ils.ils_create(A, b, pr.p, pr.q, n)
        x = np.zeros(n)
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=20000, check_every=20000, inner_tol=0.0)
        ils.ils_rgs_solve(h, None, x, 0.0, 1, o)
        st, rep = ils.ils_rgs_solve(h, None, x, 0.0, 2, o)
        out.append(f"nt={nt}: {rep.solve_ms / 40000 * 1e3:.3f}")
        ils.ils_destroy(h)
    print(f"n={n}: " + ", ".join(out), flush=True)
