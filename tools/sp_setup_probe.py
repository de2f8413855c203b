"""Development probe: one SP solve on a config (first call: Gram + Cholesky + inverse + P, then the
iterations); for launch lists of the setup under ncu (--metrics gpu__time_duration.sum)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2203_15340_b200 import ils  # noqa: E402
from workloads import make_problem  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    pr = make_problem(cfg)
    if cfg == "c3":
        t = {k: torch.from_numpy(getattr(pr, k)).cuda() for k in ("vals", "b", "row_ptr", "col_idx")}
        mk = lambda: ils.ils_create(t["vals"], t["b"], pr.p, pr.q, pr.n, row_ptr=t["row_ptr"], col_idx=t["col_idx"])
    else:
        A = torch.from_numpy(pr.A).cuda()
        b = torch.from_numpy(pr.b).cuda()
        mk = lambda: ils.ils_create(A, b, pr.p, pr.q, pr.n)
    for r in range(reps):
        h = mk()
        x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
        st, rep = ils.ils_sp_solve(h, None, x, 0.0, 16, ils.ils_default_opts(stop=ils.ILS_STOP_NONE))
        d = rep.as_dict()
        print(f"{cfg} rep {r}: setup {d['setup_ms']:.3f} ms solve {d['solve_ms']:.3f} ms", flush=True)
        ils.ils_destroy(h)


if __name__ == "__main__":
    main()
