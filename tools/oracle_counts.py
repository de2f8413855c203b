"""Run the ORACLE's full solves on a workload and record iteration counts and CPU times
(calls only oracle/ and workloads/). Output: profiles/oracle_<cfg>_counts.json.
Used by bench.py's reference arm to extrapolate bounded oracle samples to a full solve."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import ils_oracle as O  # noqa: E402
from workloads import make_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--inner-tol", type=float, default=None)
    ap.add_argument("--max-inner", type=int, default=1_000_000)
    ap.add_argument("--methods", default="sp,rk,rgs")
    a = ap.parse_args()
    pr = make_problem(a.config)
    itol = a.inner_tol if a.inner_tol is not None else (1e-12 if pr.tol <= 1e-10 else 1e-10)
    t0 = time.perf_counter()
    xref = pr.xstar if pr.consistent else O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2)
    out = {"config": a.config, "tol": pr.tol, "inner_tol": itol, "max_inner": a.max_inner,
           "xref_s": time.perf_counter() - t0, "rho": O.spectral_radius_sp(pr.A1, pr.A2)}
    args = (pr.A1, pr.A2, pr.b1, pr.b2)
    for m in a.methods.split(","):
        t0 = time.perf_counter()
        if m == "sp":
            r = O.sp_solve(*args, tol=pr.tol, x_ref=xref, max_iter=1000)
        elif m == "rk":
            r = O.sp_rk_rgs_solve(*args, tol=pr.tol, x_ref=xref, max_iter=1000, inner_tol=itol,
                                  max_inner=a.max_inner)
        else:
            r = O.sp_scd_solve(*args, tol=pr.tol, x_ref=xref, max_iter=1000, inner_tol=itol,
                               max_inner=a.max_inner)
        out[m] = {"outer": r.outer_iters, "inner_total": r.inner_iters_total, "inner_hist": r.inner_hist,
                  "converged": r.converged, "final_err": r.final_metric, "cpu_s": time.perf_counter() - t0}
        print(m, out[m], flush=True)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"oracle_{a.config}_counts.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
