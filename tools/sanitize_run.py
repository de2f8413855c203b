"""Short runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
SP row stream (c1 rows, 3 outer steps, and the RK check mode), the look-ahead SP-RK-RGS kernel with
its in-kernel checks (c1, one outer step of 2200 inner steps, a check every 500), the one-CTA small
kernel (c0), SP-SCD one-CTA and one-warp kernels, forced-large cluster SCD and gmode RK, CSR kernels,
and the batched kernels (64 instances). Horizons are short: the sanitizers run every kernel ~100x
slower. Exits non-zero on any library error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_15340_b200 import ils  # noqa: E402
from workloads import make_batched, make_dense, make_problem, make_sparse  # noqa: E402


def run(h, n, fn, batch=1, **kw):
    x = np.zeros(batch * n)
    o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, **kw)
    st, rep = fn(h, None, x, 0.0, kw.pop("K", 1) if "K" in kw else 1, o)
    return rep


def dense(pr):
    A = torch.from_numpy(pr.A).cuda()
    b = torch.from_numpy(pr.b).cuda()
    return ils.ils_create(A, b, pr.p, pr.q, pr.n), (A, b)


def main():
    which = sys.argv[1:] or ["c1", "c0", "large", "csr", "batched"]
    if "c1" in which:
        pr = make_problem("c1")
        h, keep = dense(pr)
        x = np.zeros(pr.n)
        ils.ils_sp_solve(h, None, x, 0.0, 3, ils.ils_default_opts(stop=ils.ILS_STOP_NONE))
        ils.ils_rk_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=2200,
                                                                  check_every=500, inner_tol=1e-30))
        os.environ["ILS_RK_LA"] = "0"   # the chunked blocked kernel + row-stream check
        ils.ils_rk_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=1200,
                                                                  check_every=400, inner_tol=1e-30))
        del os.environ["ILS_RK_LA"]
        ils.ils_rgs_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=1500,
                                                                   check_every=500, inner_tol=0.0))
        ils.ils_destroy(h)
        print("c1 done", flush=True)
    if "c0" in which:
        pr = make_problem("c0")
        h, keep = dense(pr)
        x = np.zeros(pr.n)
        for fn in (ils.ils_sp_solve, ils.ils_rk_solve, ils.ils_rgs_solve):
            fn(h, None, x, 0.0, 2, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=600, check_every=50,
                                                        inner_tol=0.0))
        ils.ils_destroy(h)
        print("c0 done", flush=True)
    if "large" in which:
        os.environ["ILS_FORCE_LARGE"] = "1"
        pr = make_dense(2000, 300, 200, 0.4, noise=0.05, seed=5)
        h, keep = dense(pr)
        x = np.zeros(pr.n)
        for fn in (ils.ils_sp_solve, ils.ils_rk_solve, ils.ils_rgs_solve):
            fn(h, None, x, 0.0, 2, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=300, check_every=100,
                                                        inner_tol=0.0))
        ils.ils_destroy(h)
        del os.environ["ILS_FORCE_LARGE"]
        print("large done", flush=True)
    if "csr" in which:
        pr = make_sparse(3000, 600, 200, 6, seed=7)
        t = {k: torch.from_numpy(getattr(pr, k)).cuda() for k in ("vals", "b", "row_ptr", "col_idx")}
        h = ils.ils_create(t["vals"], t["b"], pr.p, pr.q, pr.n, row_ptr=t["row_ptr"], col_idx=t["col_idx"])
        x = np.zeros(pr.n)
        for fn, kw in ((ils.ils_sp_solve, {}), (ils.ils_rk_solve, {}), (ils.ils_rgs_solve, {}),
                       (ils.ils_rgs_solve, {"weighted": 1})):
            fn(h, None, x, 0.0, 2, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=300, check_every=100,
                                                        inner_tol=0.0, **kw))
        ils.ils_destroy(h)
        print("csr done", flush=True)
    if "batched" in which:
        bt = make_batched(batch=64, base_seed=3)
        h = ils.ils_create(bt.A, bt.b, bt.p, bt.q, bt.n, batch=bt.batch)
        x = np.zeros(bt.batch * bt.n)
        for fn, kw in ((ils.ils_sp_solve, {}), (ils.ils_rk_solve, {}), (ils.ils_rgs_solve, {}),
                       (ils.ils_rgs_solve, {"weighted": 1})):
            fn(h, None, x, 0.0, 2, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=256, check_every=32,
                                                        inner_tol=0.0, **kw))
        ils.ils_destroy(h)
        print("batched done", flush=True)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
