"""Per-seed statistics of the randomized methods ("for randomized methods: seed 0
(the parity run) plus mean / median over 10 seeds"; the paper averages 10 trials):
SP-RK-RGS and SP-SCD on a config to its tolerance through the C ABI, one fresh handle per run
(setup included), for seeds 0..N-1.

    python tools/seed_study.py --config c1 --seeds 10 --out profiles/r01_seeds_c1
"""
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
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    pr = make_problem(a.config)
    dev = "cuda:0"
    A = torch.from_numpy(pr.A).to(dev)
    b = torch.from_numpy(pr.b).to(dev)
    if pr.consistent:
        xr = torch.from_numpy(pr.xstar).to(dev)
    else:
        xr = torch.from_numpy(np.load(os.path.join(ROOT, "workloads", "xref", f"{a.config}_seed0.npy"))).to(dev)
    itol = 1e-12 if pr.tol <= 1e-10 else 1e-10
    rows = {}
    for name, fn in (("SP-RK-RGS", ils.ils_rk_solve), ("SP-SCD", ils.ils_rgs_solve)):
        runs = []
        for seed in range(a.seeds):
            h = ils.ils_create(A, b, pr.p, pr.q, pr.n)
            x = torch.zeros(pr.n, dtype=torch.float64, device=dev)
            o = ils.ils_default_opts(x_ref=xr.data_ptr(), inner_tol=itol, max_inner=1_000_000, seed=seed)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st, rep = fn(h, None, x, pr.tol, 1000, o)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) * 1e3
            ils.ils_destroy(h)
            err = float(torch.linalg.norm(x - xr) / torch.linalg.norm(xr))
            runs.append(dict(seed=seed, outer=rep.outer_iters, inner=rep.inner_iters_total, ms=wall,
                             setup_ms=rep.setup_ms, solve_ms=rep.solve_ms, err=err, converged=bool(rep.converged)))
            print(name, json.dumps(runs[-1]), flush=True)
        rows[name] = runs
    md = [f"Randomized methods over {a.seeds} seeds on {a.config} (p={pr.p}, q={pr.q}, n={pr.n}), tol {pr.tol:g}, "
          f"inner_tol {itol:g}, fresh handle per run (setup included), one B200.", "",
          "| method | seed 0: outer / inner / ms | mean outer | mean inner | median inner | mean ms | median ms | min / max ms | max error | all converged |",
          "|---|---|---:|---:|---:|---:|---:|---|---:|---|"]
    for name, runs in rows.items():
        inner = np.array([r["inner"] for r in runs], float)
        ms = np.array([r["ms"] for r in runs])
        r0 = runs[0]
        md.append(f"| {name} | {r0['outer']} / {r0['inner']} / {r0['ms']:.1f} | {np.mean([r['outer'] for r in runs]):.1f} | "
                  f"{inner.mean():.0f} | {np.median(inner):.0f} | {ms.mean():.1f} | {np.median(ms):.1f} | "
                  f"{ms.min():.1f} / {ms.max():.1f} | {max(r['err'] for r in runs):.2e} | {all(r['converged'] for r in runs)} |")
    text = "\n".join(md) + "\n"
    print(text)
    if a.out:
        with open(a.out + ".json", "w") as f:
            json.dump(dict(config=a.config, runs=rows), f, indent=1)
        with open(a.out + ".md", "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
