"""SP-SCD alpha-policy study (Remark 4.1) on B200 through the
C ABI: alpha_t uniform on {1..n} (the paper's Alg. 5 step 7), fixed alpha in
{1, sqrt(n), n/2, n} (alpha = n is the Motzkin / greedy coordinate case, run on the mask-free fast
path), and the column-norm-weighted alpha = 1 case (SP-RCD). For each policy:
outer and inner counts to the config tolerance, time, inner steps per second, error vs x_ref, over
several seeds (the paper averages 10 trials).

    python tools/alpha_study.py --config c1 --seeds 3 --out profiles/r01_alpha_study
"""
import argparse
import json
import math
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
    ap.add_argument("--seeds", type=int, default=3)
    ap.add_argument("--max-inner", type=int, default=2_000_000)
    ap.add_argument("--out", default="")
    ap.add_argument("--subsets", action="store_true",
                    help="Q9 study: Feistel-prefix subsets (reading R9) against exact uniform subsets "
                         "(ILS_SUBSET_EXACT) under the same alpha policies")
    a = ap.parse_args()
    pr = make_problem(a.config)
    n = pr.n
    dev = "cuda:0"
    A = torch.from_numpy(pr.A).to(dev)
    b = torch.from_numpy(pr.b).to(dev)
    h = ils.ils_create(A, b, pr.p, pr.q, n)
    if pr.consistent:
        xr = torch.from_numpy(pr.xstar).to(dev)
    else:
        xr = torch.zeros(n, dtype=torch.float64, device=dev)
        ils.ils_direct_solve(h, xr)
    itol = 1e-12 if pr.tol <= 1e-10 else 1e-10
    policies = [("uniform (paper)", dict(alpha_mode=ils.ILS_ALPHA_UNIFORM)),
                ("alpha = 1", dict(alpha_mode=ils.ILS_ALPHA_FIXED, alpha_k=1)),
                (f"alpha = sqrt(n) = {int(math.isqrt(n))}", dict(alpha_mode=ils.ILS_ALPHA_FIXED, alpha_k=int(math.isqrt(n)))),
                (f"alpha = n/2 = {n // 2}", dict(alpha_mode=ils.ILS_ALPHA_FIXED, alpha_k=n // 2)),
                (f"alpha = n (Motzkin)", dict(alpha_mode=ils.ILS_ALPHA_FIXED, alpha_k=n)),
                ("weighted alpha = 1 (SP-RCD)", dict(alpha_mode=ils.ILS_ALPHA_FIXED, alpha_k=1, weighted=1))]
    if a.subsets:   # quantify the deviation of the pseudo-uniform subsets (Q9)
        E = ils.ILS_SUBSET_EXACT
        sq = int(math.isqrt(n))
        policies = []
        for nm, am, ak in (("uniform alpha_t (paper)", ils.ILS_ALPHA_UNIFORM, 1),
                           (f"alpha = sqrt(n) = {sq}", ils.ILS_ALPHA_FIXED, sq),
                           (f"alpha = n/2 = {n // 2}", ils.ILS_ALPHA_FIXED, n // 2)):
            policies.append((f"{nm}, Feistel prefix (R9)", dict(alpha_mode=am, alpha_k=ak)))
            policies.append((f"{nm}, exact uniform subset", dict(alpha_mode=am | E, alpha_k=ak)))
    rows = []
    for name, kw in policies:
        runs = []
        for seed in range(a.seeds):
            x = torch.zeros(n, dtype=torch.float64, device=dev)
            o = ils.ils_default_opts(x_ref=xr.data_ptr(), inner_tol=itol, max_inner=a.max_inner, seed=seed, **kw)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st, rep = ils.ils_rgs_solve(h, None, x, pr.tol, 500, o)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) * 1e3
            err = float(torch.linalg.norm(x - xr) / torch.linalg.norm(xr))
            runs.append(dict(seed=seed, outer=rep.outer_iters, inner=rep.inner_iters_total, converged=bool(rep.converged),
                             ms=wall, solve_ms=rep.solve_ms, err=err))
            print(name, json.dumps(runs[-1]), flush=True)
        inner = np.array([r["inner"] for r in runs], dtype=float)
        ms = np.array([r["solve_ms"] for r in runs])
        rows.append(dict(policy=name, outer=float(np.mean([r["outer"] for r in runs])), inner_mean=float(inner.mean()),
                         inner_median=float(np.median(inner)), solve_ms_mean=float(ms.mean()),
                         us_per_step=float(1e3 * ms.sum() / max(inner.sum(), 1)), err_max=max(r["err"] for r in runs),
                         all_converged=all(r["converged"] for r in runs), runs=runs))
    ils.ils_destroy(h)
    md = [f"SP-SCD alpha policies on {a.config} (p={pr.p}, q={pr.q}, n={n}), tol {pr.tol:g}, inner_tol {itol:g}, "
          f"{a.seeds} seeds, one B200.", "",
          "| policy | outer | inner steps (mean / median) | solve ms (mean) | us / inner step | max error | converged |",
          "|---|---:|---:|---:|---:|---:|---|"]
    for r in rows:
        md.append(f"| {r['policy']} | {r['outer']:.1f} | {r['inner_mean']:.0f} / {r['inner_median']:.0f} | "
                  f"{r['solve_ms_mean']:.1f} | {r['us_per_step']:.3f} | {r['err_max']:.2e} | {r['all_converged']} |")
    text = "\n".join(md) + "\n"
    print(text)
    if a.out:
        with open(a.out + ".json", "w") as f:
            json.dump(dict(config=a.config, rows=rows), f, indent=1)
        with open(a.out + ".md", "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
