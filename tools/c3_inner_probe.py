"""Development probe: one capped SP-RK-RGS / SP-SCD inner solve on configs[3] (CSR), for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_15340_b200 import ils  # noqa: E402
from workloads import make_problem  # noqa: E402


def main():
    methods = sys.argv[1].split(",") if len(sys.argv) > 1 else ["rk", "rgs"]
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
    pr = make_problem("c3")
    t = {k: torch.from_numpy(getattr(pr, k)).cuda() for k in ("vals", "b", "row_ptr", "col_idx")}
    h = ils.ils_create(t["vals"], t["b"], pr.p, pr.q, pr.n, row_ptr=t["row_ptr"], col_idx=t["col_idx"])
    for m in [mm for mm in methods for _ in range(2)]:   # second call: setup (Gram) already built
        x = np.zeros(pr.n)
        fn = ils.ils_rk_solve if m == "rk" else ils.ils_rgs_solve
        st, rep = fn(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=T, inner_tol=0.0,
                                                               check_every=T, weighted=1 if m == "rcd" else 0))
        d = rep.as_dict()
        print(m, T, "solve_ms %.2f" % d["solve_ms"], "us/step %.3f" % (1e3 * d["solve_ms"] / T), flush=True)
    ils.ils_destroy(h)


if __name__ == "__main__":
    main()
