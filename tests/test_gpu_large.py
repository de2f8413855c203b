"""GPU parity for the dense n > 8192 paths (the paper's own Tables 2-5
use n = 13000-15000): two-pass SP right-hand side and inner check (large.cu), global-z RK-RGS
(rk_rgs.cu gmode), shared-memory-residual SCD with dense A1bar rows (sparse.cu kernel).

ILS_FORCE_LARGE=1 (read by ils_create) routes a small problem through the same kernels, so the
element-by-element parity runs at sizes the oracle finishes in seconds; one test runs a real
n > 8192 problem. Bars as in test_gpu_parity.py (iterates within 1e-9 relative at fixed horizons,
inner step counts exact).
"""
import numpy as np
import pytest

from oracle import ils_oracle as O
from workloads import make_dense

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2203_15340_b200 import ils  # noqa: E402

DEV = "cuda:0"


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _par(a, b):
    """Parity distance of two iterates: the larger of the norm-wise relative difference (the
    north_star bar) and the element-wise max |a_i - b_i| / max |b_i|, so that a wrong small
    coordinate cannot hide inside the norm."""
    a, b = np.asarray(a), np.asarray(b)
    d = np.abs(a - b)
    return max(_rel(a, b), float(d.max() / max(np.abs(b).max(), 1e-300)) if d.size else 0.0)


class Big:
    def __init__(self, pr, monkeypatch=None, force=True):
        if monkeypatch is not None:
            monkeypatch.setenv("ILS_FORCE_LARGE", "1" if force else "0")
        A = torch.from_numpy(pr.A).to(DEV)
        b = torch.from_numpy(pr.b).to(DEV)
        self.h = ils.ils_create(A, b, pr.p, pr.q, pr.n)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        ils.ils_destroy(self.h)


SHAPES = [(200, 100, 50, 0.3), (257, 33, 31, 0.3), (90, 0, 17, 0.3), (1000, 300, 130, 0.4)]


@pytest.mark.parametrize("cols", ["0", "2"])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("form", [0, 1])
def test_large_sp_fixed_horizon(shape, form, cols, monkeypatch):
    p, q, n, s = shape
    # c = base + alpha X^T y of the two-pass right-hand side and of the P apply: the 32-column kernel
    # ("0") and the tiled kernel forced at these sizes ("2": odd n takes its single-column tail, q = 0
    # its empty row range, in-place base == c on the correction form)
    monkeypatch.setenv("ILS_COLS_TILED", cols)
    pr = make_dense(p, q, n, s, seed=31)
    K = 6
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, sp_form=form)
    hist = np.zeros((K, n))
    x = np.zeros(n)
    with Big(pr, monkeypatch) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, sp_form=form, x_hist=hist.ctypes.data)
        st, rep = ils.ils_sp_solve(hh.h, None, x, 0.0, K, o)
    assert rep.outer_iters == K
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


def test_large_sp_rr_stop_and_relative_residual(monkeypatch):
    pr = make_dense(300, 60, 40, 0.3, seed=32)
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, tol=1e-12, stop=O.STOP_RR, max_iter=200)
    x = np.zeros(pr.n)
    with Big(pr, monkeypatch) as hh:
        st, rep = ils.ils_sp_solve(hh.h, None, x, 1e-12, 200, ils.ils_default_opts(stop=ils.ILS_STOP_RR))
        assert rep.converged and rep.final_metric < 1e-12
        assert abs(rep.outer_iters - ref.outer_iters) <= 1
        xt = np.linspace(-1.0, 1.0, pr.n)
        rr = ils.ils_relative_residual(hh.h, xt)
    assert abs(rr - O.relative_residual(pr.A1, pr.A2, pr.b1, pr.b2, xt)) <= 1e-12 * max(rr, 1.0)


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("T,ce,itol", [(1, 50, 0.0), (7, 3, 0.0), (333, 50, 0.0), (5000, 64, 1e-6)])
def test_large_rk_fixed_horizon(shape, T, ce, itol, monkeypatch):
    p, q, n, s = shape
    pr = make_dense(p, q, n, s, seed=33)
    K = 3
    ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=5, max_inner=T,
                            check_every=ce, inner_tol=itol)
    hist = np.zeros((K, n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(n)
    with Big(pr, monkeypatch) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=5, max_inner=T, check_every=ce, inner_tol=itol,
                                 x_hist=hist.ctypes.data, inner_hist=inner.ctypes.data)
        ils.ils_rk_solve(hh.h, None, x, 0.0, K, o)
    assert list(inner) == list(ref.inner_hist)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("mode", [(0, 1, 0), (1, 1, 0), (1, 5, 0), (1, 10 ** 6, 0), (1, 1, 1)])
def test_large_scd_fixed_horizon(shape, mode, monkeypatch):
    """(alpha_mode, alpha_k, weighted): weighted = 1 is SP-RCD."""
    p, q, n, s = shape
    pr = make_dense(p, q, n, s, seed=34)
    amode, ak, wt = mode
    K, T, ce = 3, 300, 40
    ref = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=9, max_inner=T,
                         check_every=ce, inner_tol=1e-9, alpha_mode=amode, alpha_fixed=ak, weighted=bool(wt))
    hist = np.zeros((K, n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(n)
    with Big(pr, monkeypatch) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=9, max_inner=T, check_every=ce, inner_tol=1e-9,
                                 alpha_mode=amode, alpha_k=min(ak, 2 ** 31 - 1), weighted=wt, x_hist=hist.ctypes.data,
                                 inner_hist=inner.ctypes.data)
        ils.ils_rgs_solve(hh.h, None, x, 0.0, K, o)
    assert list(inner) == list(ref.inner_hist)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


def test_large_methods_converge(monkeypatch):
    pr = make_dense(400, 80, 60, 0.3, seed=35)
    xs = O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2)
    for fn in (ils.ils_sp_solve, ils.ils_rk_solve, ils.ils_rgs_solve):
        x = np.zeros(pr.n)
        with Big(pr, monkeypatch) as hh:
            o = ils.ils_default_opts(x_ref=xs.ctypes.data, inner_tol=1e-12, max_inner=400000)
            st, rep = fn(hh.h, None, x, 1e-10, 300, o)
        assert st == ils.ILS_OK and _rel(x, xs) <= 1e-10, fn


def test_large_real_n_above_8192(monkeypatch):
    """A dense problem with n = 8300 (> 8192, npad 8320) on the default routing: SP (both forms),
    SP-RK-RGS, SP-SCD and SP-RCD at short fixed horizons against the oracle."""
    p, q, n = 8700, 300, 8300
    pr = make_dense(p, q, n, 0.3, seed=36)
    monkeypatch.delenv("ILS_FORCE_LARGE", raising=False)
    K = 2
    ref_sp = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE)
    ref_rk = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=2, max_inner=400,
                               check_every=100, inner_tol=0.0)
    ref_scd = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=2, max_inner=400,
                             check_every=100, inner_tol=0.0, alpha_mode=1, alpha_fixed=64)
    ref_rcd = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=2, max_inner=400,
                             check_every=100, inner_tol=0.0, weighted=True)
    with Big(pr) as hh:
        for fn, ref, kw in ((ils.ils_sp_solve, ref_sp, {}), (ils.ils_sp_solve, ref_sp, {"sp_form": 1}),
                            (ils.ils_rk_solve, ref_rk, {"max_inner": 400, "check_every": 100}),
                            (ils.ils_rgs_solve, ref_scd, {"max_inner": 400, "check_every": 100, "alpha_mode": 1,
                                                          "alpha_k": 64}),
                            (ils.ils_rgs_solve, ref_rcd, {"max_inner": 400, "check_every": 100, "weighted": 1})):
            hist = np.zeros((K, n))
            x = np.zeros(n)
            o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=2, inner_tol=0.0, x_hist=hist.ctypes.data, **kw)
            fn(hh.h, None, x, 0.0, K, o)
            for k in range(K):
                assert _par(hist[k], ref.x_hist[k]) <= 1e-9, (fn, kw, k)
        # the explicit B = P A2bar of sp_form 2 is not formed at n >= 8192 (P is applied implicitly)
        with pytest.raises(ils.IlsError) as e:
            ils.ils_sp_solve(hh.h, None, np.zeros(n), 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, sp_form=2))
        assert e.value.status == ils.ILS_ERR_UNSUPPORTED


@pytest.mark.parametrize("shape", [(3000, 200, 200), (2500, 1, 300), (1500, 1, 70)])
def test_paper_family_parity(shape):
    """The paper's own families (§5.2, q = n; §5.3 Minkowski, q = 1)
    at reduced sizes on the default routing: all three methods at fixed horizons against the oracle."""
    from workloads import make_paper
    p, q, n = shape
    pr = make_paper(p, q, n, seed=37)
    K = 3
    refs = [
        (ils.ils_sp_solve, O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE), {}),
        (ils.ils_rk_solve, O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=4,
                                             max_inner=500, check_every=100, inner_tol=1e-6),
         dict(max_inner=500, check_every=100, inner_tol=1e-6)),
        (ils.ils_rgs_solve, O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=4,
                                           max_inner=300, check_every=60, inner_tol=1e-6, alpha_mode=0),
         dict(max_inner=300, check_every=60, inner_tol=1e-6, alpha_mode=0)),
    ]
    with Big(pr, force=False) as hh:
        for fn, ref, kw in refs:
            hist = np.zeros((K, n))
            inner = np.zeros(K, dtype=np.int64)
            x = np.zeros(n)
            o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=4, x_hist=hist.ctypes.data,
                                     inner_hist=inner.ctypes.data, **kw)
            fn(hh.h, None, x, 0.0, K, o)
            if fn is not ils.ils_sp_solve:
                assert list(inner) == list(ref.inner_hist), fn
            for k in range(K):
                assert _par(hist[k], ref.x_hist[k]) <= 1e-9, (fn, k)
