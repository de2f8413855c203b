"""Development aid: SP-SCD inner steps at the paper's size (Table 2, 43000 x 13000) through the
C ABI, fixed horizon (1 outer step, T inner steps, one chunk), for timing and ncu captures."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2203_15340_b200 import ils
from workloads import make_paper
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
pr = make_paper(30000, 13000, 13000, seed=0)
A = torch.from_numpy(pr.A).cuda(); b = torch.from_numpy(pr.b).cuda()
del pr
h = ils.ils_create(A, b, 30000, 13000, 13000)
x = torch.zeros(13000, dtype=torch.float64, device="cuda")
for rep in range(2):
    o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=T, check_every=T, inner_tol=0.0, seed=rep)
    st, r = ils.ils_rgs_solve(h, None, x, 0.0, 1, o)
    print(f"rep {rep}: setup {r.setup_ms:.1f} ms solve {r.solve_ms:.2f} ms = {1e3 * r.solve_ms / T:.2f} us/step "
          f"(hot {r.hot_ms[2]:.2f} ms)", flush=True)
ils.ils_destroy(h)
