"""Development probe: the SP K1 + P stream on configs[2] (fixed 16 outer steps, no stopping) under
ring-geometry overrides (ILS_SP_STAGE bytes, ILS_SP_NS stages); prints kernel ms and GB/s against the
algorithmic 8q(n+1) + 8n^2 bytes per outer step."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2203_15340_b200 import ils  # noqa: E402
from workloads import make_problem  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    variants = sys.argv[2:] or ["default"]
    pr = make_problem(cfg)
    A = torch.from_numpy(pr.A).cuda()
    b = torch.from_numpy(pr.b).cuda()
    h = ils.ils_create(A, b, pr.p, pr.q, pr.n)
    K = 16
    byt = K * (8.0 * pr.q * (pr.n + 1) + 8.0 * pr.n * pr.n)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for v in variants:
        for k in ("ILS_SP_STAGE", "ILS_SP_NS"):
            os.environ.pop(k, None)
        if v != "default":
            for kv in v.split(","):
                k, val = kv.split("=")
                os.environ[k] = val
        ts = []
        for rep in range(6):
            x = torch.zeros(pr.n, dtype=torch.float64, device="cuda")
            flush.add_(1)
            torch.cuda.synchronize()
            o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE)
            st, rep_ = ils.ils_sp_solve(h, None, x, 0.0, K, o)
            d = rep_.as_dict()
            if rep >= 1:
                ts.append(d["solve_ms"])
        ms = sorted(ts)[len(ts) // 2]
        print(f"{cfg} {v:40s} solve {ms:.4f} ms  {byt / ms / 1e6:.0f} GB/s", flush=True)
    ils.ils_destroy(h)


if __name__ == "__main__":
    main()
