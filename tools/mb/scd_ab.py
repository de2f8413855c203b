import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2203_15340_b200 import ils
from workloads import make_dense
for n in (64, 128, 200, 256):
    pr = make_dense(4 * n, n // 2, n, 0.3, seed=1)
    A = torch.from_numpy(pr.A).cuda(); b = torch.from_numpy(pr.b).cuda()
    res = []
    for env in ("0", "1"):
        os.environ["ILS_SCD_CTA"] = env
        h = ils.ils_create(A, b, pr.p, pr.q, n)
        x = np.zeros(n)
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=20000, check_every=20000, inner_tol=0.0)
        ils.ils_rgs_solve(h, None, x, 0.0, 1, o)
        st, rep = ils.ils_rgs_solve(h, None, x, 0.0, 2, o)
        res.append(rep.solve_ms / 40000 * 1e3)
        ils.ils_destroy(h)
    print(f"n={n}: warp {res[0]:.3f} us/step, cta {res[1]:.3f} us/step", flush=True)
