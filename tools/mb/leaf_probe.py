"""Development aid: SP setup time (Gram excluded: Cholesky + inverse + P) against n, to size the
64x64 leaf cost of the recursive factorisation. Prints ms per setup for n = 64 .. 2048."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2203_15340_b200 import ils
from workloads import make_dense
for n in (64, 128, 256, 512, 1024, 2048):
    pr = make_dense(2 * n + 64, 32, n, 0.3, seed=1)
    A = torch.from_numpy(pr.A).cuda(); b = torch.from_numpy(pr.b).cuda()
    best_g, best_c = 1e9, 1e9
    for rep in range(4):
        h = ils.ils_create(A, b, pr.p, pr.q, pr.n)
        x = np.zeros(pr.n)
        st, r1 = ils.ils_rgs_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=1, check_every=1))
        st, r2 = ils.ils_sp_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE))
        ils.ils_destroy(h)
        best_g, best_c = min(best_g, r1.setup_ms), min(best_c, r2.setup_ms)
    print(f"n={n}: leaves {n // 64}, gram {best_g:.3f} ms, chol+inv+P {best_c:.3f} ms", flush=True)
