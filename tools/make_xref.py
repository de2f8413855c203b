"""Write the reference solutions x_ref of the inconsistent workloads (c1) with the ORACLE.

x_ref solves A^T J A x = A^T J b (Eq. Sec12) by the oracle's fp64 Cholesky of
M = A1^T A1 - A2^T A2 (BASELINE.json configs[1]: "reference solution from the oracle's fp64
Cholesky of A^T J A"). Calls only oracle/ and workloads/. Output: workloads/xref/<cfg>_seed<s>.npy
plus a .json with the data fingerprint, so bench.py (GPU leg) can use x_ref without running the
oracle itself.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import ils_oracle as O  # noqa: E402
from workloads import fingerprint, make_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    seed = a.seed
    while True:   # configs[3]: "regenerate with seed+1 if the oracle's Cholesky of A^T J A fails"
        pr = make_problem(a.config, seed=seed)
        if hasattr(pr, "scipy"):
            S = pr.scipy()
            A1, A2, b1, b2 = S[:pr.p], S[pr.p:], pr.b[:pr.p], pr.b[pr.p:]
        else:
            A1, A2, b1, b2 = pr.A1, pr.A2, pr.b1, pr.b2
        try:
            x = O.direct_solve(A1, A2, b1, b2)
            break
        except np.linalg.LinAlgError:
            seed += 1
    out = os.path.join(ROOT, "workloads", "xref")
    os.makedirs(out, exist_ok=True)
    base = os.path.join(out, f"{a.config}_seed{a.seed}")
    np.save(base + ".npy", x)
    meta = {"config": a.config, "seed": a.seed, "data_seed": seed, "n": int(pr.n),
            "fingerprint": fingerprint(pr if hasattr(pr, "scipy") else pr.A, pr.b),
            "rho": O.spectral_radius_sp(A1, A2) if not hasattr(pr, "scipy") else None,
            "err_xstar": float(np.linalg.norm(x - pr.xstar) / np.linalg.norm(pr.xstar)),
            "writer": "tools/make_xref.py (oracle.ils_oracle.direct_solve)"}
    with open(base + ".json", "w") as f:
        json.dump(meta, f, indent=1)
    print(meta)


if __name__ == "__main__":
    main()
