"""Quick GPU probe: time each method through the C ABI on a config and print the reports.
Development aid (not the bench). x_ref: x* for consistent configs, else ils_direct_solve."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_15340_b200 import ils  # noqa: E402
from workloads import make_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--methods", default="sp,rk,rgs,rcd")
    ap.add_argument("--max-inner", type=int, default=1_000_000)
    ap.add_argument("--max-iter", type=int, default=200)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--fixed", type=int, default=0, help="fixed horizon: 1 outer x FIXED inner steps, no stopping")
    ap.add_argument("--check-every", type=int, default=0)
    ap.add_argument("--sp-form", type=int, default=0)
    a = ap.parse_args()
    t0 = time.time()
    pr = make_problem(a.config)
    print(f"gen {a.config}: {time.time() - t0:.1f}s", flush=True)
    dev = "cuda:0"
    if a.config == "c3":
        t = {k: torch.from_numpy(getattr(pr, k)).to(dev) for k in ("vals", "b", "row_ptr", "col_idx")}
        h = ils.ils_create(t["vals"], t["b"], pr.p, pr.q, pr.n, row_ptr=t["row_ptr"], col_idx=t["col_idx"])
        n, B = pr.n, 1
        xr = torch.from_numpy(np.load(os.path.join(ROOT, "workloads", "xref", "c3_seed0.npy"))).to(dev)
    elif a.config == "c4":
        A = torch.from_numpy(pr.A).to(dev)
        b = torch.from_numpy(pr.b).to(dev)
        xr = torch.from_numpy(pr.xstar).to(dev)
        h = ils.ils_create(A, b, pr.p, pr.q, pr.n, batch=pr.batch)
        n, B = pr.n, pr.batch
    else:
        A = torch.from_numpy(pr.A).to(dev)
        b = torch.from_numpy(pr.b).to(dev)
        h = ils.ils_create(A, b, pr.p, pr.q, pr.n)
        n, B = pr.n, 1
        if pr.consistent:
            xr = torch.from_numpy(pr.xstar).to(dev)
        else:
            xr = torch.zeros(n, dtype=torch.float64, device=dev)
            ils.ils_direct_solve(h, xr)
    itol = 1e-12 if pr.tol <= 1e-10 else 1e-10
    for m in a.methods.split(","):
        for rep in range(a.reps):
            x = torch.zeros(B * n, dtype=torch.float64, device=dev)
            o = ils.ils_default_opts(x_ref=xr.data_ptr(), inner_tol=itol, max_inner=a.max_inner,
                                     check_every=a.check_every)
            o.sp_form = a.sp_form
            max_iter = a.max_iter
            if a.fixed:
                o.stop, o.inner_tol, o.max_inner, max_iter = ils.ILS_STOP_NONE, 0.0, a.fixed, 1
            fn = {"sp": ils.ils_sp_solve, "rk": ils.ils_rk_solve, "rgs": ils.ils_rgs_solve,
                  "rcd": ils.ils_rgs_solve}[m]
            if m == "rcd":
                o.weighted = 1
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            st, r = fn(h, None, x, pr.tol, max_iter, o)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t1) * 1e3
            d = r.as_dict()
            d.update(method=m, rep=rep, status=st, wall_ms=wall, check_every=a.check_every, fixed=a.fixed)
            if B == 1:
                d["err"] = float(torch.linalg.norm(x - xr) / torch.linalg.norm(xr))
            print(json.dumps(d), flush=True)
    ils.ils_destroy(h)


if __name__ == "__main__":
    main()
