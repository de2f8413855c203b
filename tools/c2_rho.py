"""Write profiles/c2_rho.json: the SP iteration-matrix spectral radius of configs[2] measured by the
ORACLE (oracle.ils_oracle.spectral_radius_sp, Theorem 2.1) -- reading R16 / SURVEY
Q16: the literal construction's lambda_max(A2^T A2) = 0.9 lambda_min(A1^T A1) is only an upper bound
on rho. Calls oracle/ only (a stored value, never from the CUDA path)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import ils_oracle as O  # noqa: E402
from workloads import make_problem  # noqa: E402


def main():
    pr = make_problem("c2")
    t0 = time.perf_counter()
    rho = O.spectral_radius_sp(pr.A1, pr.A2)
    G = pr.A1.T @ pr.A1
    lam1 = float(np.linalg.eigvalsh(G)[0])
    lam2 = float(np.linalg.eigvalsh(pr.A2.T @ pr.A2)[-1])
    out = {"config": "c2", "rho": rho, "bound_lmax_A2bar_over_lmin_A1bar": lam2 / lam1,
           "lambda_min_A1bar": lam1, "lambda_max_A2bar": lam2, "seconds": round(time.perf_counter() - t0, 1),
           "source": "oracle.ils_oracle.spectral_radius_sp (Theorem 2.1, PAPER.md:157-174), tools/c2_rho.py",
           "reading": "R16: the config text's 'rho about 0.9' is the bound lambda_max(A2^T A2)/lambda_min(A1^T A1)"}
    with open(os.path.join(ROOT, "profiles", "c2_rho.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
