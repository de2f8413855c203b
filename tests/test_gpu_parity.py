"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars: integer/index work bit-exact; iterates within 1e-9 relative
(BASELINE.json north_star) at fixed horizons; converged solutions within the config tolerance.
"""
import numpy as np
import pytest

from oracle import ils_oracle as O
from oracle import index_stream as ix
from workloads import make_dense, make_problem

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


class H:
    """Handle on a problem; A, b passed as device tensors (or host arrays if host=True)."""

    def __init__(self, pr, host=False):
        self.pr = pr
        if host:
            self.h = ils.ils_create(pr.A, pr.b, pr.p, pr.q, pr.n)
        else:
            A = torch.from_numpy(pr.A).to(DEV)
            b = torch.from_numpy(pr.b).to(DEV)
            self.h = ils.ils_create(A, b, pr.p, pr.q, pr.n)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        ils.ils_destroy(self.h)


SHAPES = [(200, 100, 50, 0.3), (130, 37, 67, 0.3), (64, 1, 64, 0.2), (257, 40, 3, 0.3), (90, 0, 17, 0.3)]


# ------------------------------------------------------------------ index stream: bit-exact
@pytest.mark.parametrize("shape", SHAPES + [(8000, 2000, 1000, 0.5)])
def test_sampling_tables_bitwise(shape):
    p, q, n, s = shape
    pr = make_dense(p, q, n, s, seed=1)
    with H(pr) as hh:
        N, S = ils.ils_get_sampling_tables(hh.h, n)
    No = ix.column_norms_sq(pr.A1)
    _, So = ix.weights_prefix(No)
    assert np.array_equal(N.view(np.uint64), No.view(np.uint64))
    assert [int(v) for v in S] == So


@pytest.mark.parametrize("n", [1, 2, 3, 50, 1000])
def test_rk_index_replay(n):
    pr = make_dense(max(n, 8) + 5, 3, n, 0.3, seed=2)
    _, So = ix.weights_prefix(ix.column_norms_sq(pr.A1))
    with H(pr) as hh:
        for seed, k, t0 in [(0, 0, 0), (7, 3, 12345), (2 ** 40 + 5, 17, 2 ** 33 - 7)]:
            j1, j2 = ils.ils_rk_indices(hh.h, seed, k, t0, 3000)
            o1, o2 = ix.rk_rgs_indices(seed, k, t0, 3000, So)
            assert np.array_equal(j1, o1) and np.array_equal(j2, o2)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 50, 1000, 4000])
def test_scd_subset_replay(n):
    for (seed, k, t) in [(0, 0, 0), (3, 2, 99), (11, 9, 123456)]:
        for mode, ak in [(0, 1), (1, 1), (1, max(1, n // 3)), (1, n)]:
            alpha, mask = ils.ils_scd_subset(n, seed, k, t, mode, ak)
            a_o, tau = ix.scd_subset(seed, k, t, n, mode, ak)
            assert alpha == a_o
            assert np.array_equal(np.flatnonzero(mask), tau)


# ------------------------------------------------------------------ reference solution
@pytest.mark.parametrize("shape", SHAPES)
def test_direct_solve(shape):
    p, q, n, s = shape
    pr = make_dense(p, q, n, s, noise=0.1, seed=3)
    xo = O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2)
    x = np.zeros(n)
    with H(pr, host=True) as hh:
        ils.ils_direct_solve(hh.h, x)
        rr = ils.ils_relative_residual(hh.h, x)
    assert _par(x, xo) <= 1e-10
    assert rr <= 1e-20 and abs(rr - O.relative_residual(pr.A1, pr.A2, pr.b1, pr.b2, x)) <= 1e-18


def test_not_spd_and_argument_errors():
    A1 = np.eye(4)
    A = np.vstack([A1, 1.2 * np.eye(4)])
    b = np.ones(8)
    h = ils.ils_create(A, b, 4, 4, 4)
    with pytest.raises(ils.IlsError) as e:
        ils.ils_direct_solve(h, np.zeros(4))
    assert e.value.status == ils.ILS_ERR_NOT_SPD
    ils.ils_destroy(h)
    Az = np.vstack([np.diag([1.0, 0.0, 2.0]), np.ones((1, 3))])
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(np.ascontiguousarray(Az), np.ones(4), 3, 1, 3)
    assert e.value.status == ils.ILS_ERR_ZERO_COLUMN
    An = np.ones((5, 3))
    An[2, 1] = np.nan
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(An, np.ones(5), 4, 1, 3)
    assert e.value.status == ils.ILS_ERR_ARG
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(np.ones((5, 3)), np.ones(5), 2, 3, 3)
    assert e.value.status == ils.ILS_ERR_SHAPE


@pytest.mark.parametrize("where", ["A1", "A2", "lastcol", "b1", "b2"])
@pytest.mark.parametrize("dev", [False, True])
def test_nonfinite_input_rejected(where, dev):
    """The fused ingest pass (ingest_dense_kernel) flags NaN / Inf anywhere in A or b, host or
    device input."""
    pr = make_dense(70, 20, 33, 0.3, seed=21)
    A, b = pr.A.copy(), pr.b.copy()
    if where == "A1":
        A[3, 5] = np.inf
    elif where == "A2":
        A[75, 0] = np.nan
    elif where == "lastcol":
        A[89, 32] = -np.inf
    elif where == "b1":
        b[0] = np.nan
    else:
        b[89] = np.inf
    if dev:
        A, b = torch.from_numpy(A).to(DEV), torch.from_numpy(b).to(DEV)
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(A, b, 70, 20, 33)
    assert e.value.status == ils.ILS_ERR_ARG


@pytest.mark.parametrize("dev", [False, True])
def test_strided_input_matches_contiguous(dev):
    """lda > n (row stride) through the fused ingest: identical tables and SP iterates."""
    pr = make_dense(130, 37, 67, 0.3, seed=22)
    lda = 80
    As = np.zeros((pr.m, lda))
    As[:, :pr.n] = pr.A
    As[:, pr.n:] = np.nan   # never read
    Ain, bin_ = (torch.from_numpy(As).to(DEV), torch.from_numpy(pr.b).to(DEV)) if dev else (As, pr.b)
    h1 = ils.ils_create(Ain, bin_, pr.p, pr.q, pr.n, lda=lda)
    h2 = ils.ils_create(pr.A, pr.b, pr.p, pr.q, pr.n)
    try:
        N1, S1 = ils.ils_get_sampling_tables(h1, pr.n)
        N2, S2 = ils.ils_get_sampling_tables(h2, pr.n)
        assert np.array_equal(N1, N2) and np.array_equal(S1, S2)
        x1, x2 = np.zeros(pr.n), np.zeros(pr.n)
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE)
        ils.ils_sp_solve(h1, None, x1, 0.0, 5, o)
        ils.ils_sp_solve(h2, None, x2, 0.0, 5, o)
        assert np.array_equal(x1, x2)
    finally:
        ils.ils_destroy(h1)
        ils.ils_destroy(h2)


# ------------------------------------------------------------------ SP (Alg. 1)
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("form", [0, 1])
def test_sp_fixed_horizon(shape, form):
    p, q, n, s = shape
    pr = make_dense(p, q, n, s, noise=0.05, seed=4)
    K = 6
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, sp_form=form)
    hist = np.zeros((K, n))
    x = np.zeros(n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, sp_form=form, x_hist=hist.ctypes.data)
        st, rep = ils.ils_sp_solve(hh.h, None, x, 0.0, K, o)
    assert rep.outer_iters == K
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k
    assert _par(x, ref.x) <= 1e-9


@pytest.mark.parametrize("cfg", ["c0", "c1"])
def test_sp_converges(cfg):
    pr = make_problem(cfg)
    xref = pr.xstar if pr.consistent else O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2)
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, tol=pr.tol, x_ref=xref, max_iter=500)
    x = torch.zeros(pr.n, dtype=torch.float64, device=DEV)
    xr_t = torch.from_numpy(xref).to(DEV)
    with H(pr) as hh:
        o = ils.ils_default_opts(x_ref=xr_t.data_ptr())
        st, rep = ils.ils_sp_solve(hh.h, None, x, pr.tol, 500, o)
    assert st == ils.ILS_OK and rep.converged
    assert _rel(x.cpu().numpy(), xref) <= pr.tol
    assert abs(rep.outer_iters - ref.outer_iters) <= 1


def test_sp_q0_one_step():
    pr = make_dense(90, 0, 17, 0.3, noise=0.5, seed=5)
    xls = np.linalg.lstsq(pr.A1, pr.b1, rcond=None)[0]
    x = np.zeros(17)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE)
        ils.ils_sp_solve(hh.h, None, x, 0.0, 1, o)
    assert _par(x, xls) <= 1e-11


def test_sp_rr_stop():
    pr = make_dense(120, 40, 30, 0.3, noise=0.2, seed=6)
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, tol=1e-12, stop=O.STOP_RR, max_iter=100)
    x = np.zeros(30)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_RR)
        st, rep = ils.ils_sp_solve(hh.h, None, x, 1e-12, 100, o)
    assert rep.converged and rep.final_metric < 1e-12
    assert abs(rep.outer_iters - ref.outer_iters) <= 1


# ------------------------------------------------------------------ SP-RK-RGS (Alg. 2)
@pytest.mark.parametrize("shape", [(200, 100, 50, 0.3), (130, 37, 67, 0.3), (257, 40, 3, 0.3), (64, 1, 64, 0.2)])
@pytest.mark.parametrize("T", [1, 2, 7, 333])
def test_rk_fixed_horizon(shape, T):
    p, q, n, s = shape
    pr = make_dense(p, q, n, s, noise=0.05, seed=7)
    K = 3
    ce = 50
    ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=5,
                            max_inner=T, check_every=ce, inner_tol=0.0)
    hist = np.zeros((K, n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=5, max_inner=T, check_every=ce, inner_tol=0.0,
                                 x_hist=hist.ctypes.data, inner_hist=inner.ctypes.data)
        st, rep = ils.ils_rk_solve(hh.h, None, x, 0.0, K, o)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k
    # inner_tol = 0 stops only on an exactly zero gradient; with tiny n the iteration can reach
    # that at a check on one side and not the other (a stop decision at a threshold, R25)
    for g, o_ in zip(inner, ref.inner_hist):
        assert g == o_ or (n <= 3 and g % ce == 0 and g < o_)


def test_rk_cluster_path_c1_horizon(monkeypatch):
    """c1 rows (p = 8000) exercise the 16-CTA cluster/DSMEM blocked kernel without look-ahead
    (ILS_RK_LA=0; the look-ahead default is covered by test_rk_lookahead_kernel_c1_horizon)."""
    monkeypatch.setenv("ILS_RK_LA", "0")
    pr = make_problem("c1")
    K, T, ce = 2, 3000, 1000
    ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=0,
                            max_inner=T, check_every=ce, inner_tol=0.0)
    hist = np.zeros((K, pr.n))
    x = np.zeros(pr.n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=0, max_inner=T, check_every=ce, inner_tol=0.0,
                                 x_hist=hist.ctypes.data)
        ils.ils_rk_solve(hh.h, None, x, 0.0, K, o)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


def test_rk_lookahead_kernel_c1_horizon(monkeypatch):
    """The look-ahead SP-RK-RGS kernel (opt-in, ILS_RK_LA=1: block i+1's exchange in flight during
    block i, stale-state products corrected through A1bar) against the oracle at c1 size."""
    monkeypatch.setenv("ILS_RK_LA", "1")
    pr = make_problem("c1")
    K, T, ce = 2, 3000, 1000
    ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=1,
                            max_inner=T, check_every=ce, inner_tol=0.0)
    hist = np.zeros((K, pr.n))
    x = np.zeros(pr.n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=1, max_inner=T, check_every=ce, inner_tol=0.0,
                                 x_hist=hist.ctypes.data)
        ils.ils_rk_solve(hh.h, None, x, 0.0, K, o)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


@pytest.mark.parametrize("T,ce", [(1, 1000), (5, 3), (7, 4), (130, 64)])
def test_rk_cluster_short_horizons(T, ce):
    """16-CTA cluster path (p = 8000) at short / ragged horizons and check intervals: partial last
    blocks, a horizon shorter than the TMA ring, checks inside a block of 4 steps."""
    pr = make_dense(8000, 400, 300, 0.5, seed=47)
    K = 2
    ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=2, max_inner=T,
                            check_every=ce, inner_tol=0.0)
    hist = np.zeros((K, pr.n))
    x = np.zeros(pr.n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=2, max_inner=T, check_every=ce, inner_tol=0.0,
                                 x_hist=hist.ctypes.data)
        ils.ils_rk_solve(hh.h, None, x, 0.0, K, o)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


@pytest.mark.parametrize("shape", [(10000, 500, 700), (7900, 300, 1500)])
@pytest.mark.parametrize("T,ce", [(6, 5), (2003, 250)])
@pytest.mark.parametrize("la", ["1", "0"])
def test_rk_cluster_geometries(shape, T, ce, la, monkeypatch):
    """Other 16-CTA geometries: 5 compute warps (p = 10000) and n = 1500 (four column slots next to
    the Gram ring), with the look-ahead kernel (default) and without (ILS_RK_LA=0); iterates and
    inner counts against the oracle."""
    monkeypatch.setenv("ILS_RK_LA", la)
    p, q, n = shape
    pr = make_dense(p, q, n, 0.5, seed=48)
    K = 2
    ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=6, max_inner=T,
                            check_every=ce, inner_tol=1e-6)
    hist = np.zeros((K, pr.n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(pr.n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=6, max_inner=T, check_every=ce, inner_tol=1e-6,
                                 x_hist=hist.ctypes.data, inner_hist=inner.ctypes.data)
        ils.ils_rk_solve(hh.h, None, x, 0.0, K, o)
    assert list(inner) == list(ref.inner_hist)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


def test_rk_converges_c0():
    pr = make_problem("c0")
    ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, tol=1e-10, x_ref=pr.xstar, inner_tol=1e-12,
                            max_inner=100000)
    x = np.zeros(pr.n)
    with H(pr) as hh:
        o = ils.ils_default_opts(x_ref=pr.xstar.ctypes.data, inner_tol=1e-12, max_inner=100000)
        st, rep = ils.ils_rk_solve(hh.h, None, x, 1e-10, 100, o)
    assert st == ils.ILS_OK and _rel(x, pr.xstar) <= 1e-10
    assert rep.outer_iters == ref.outer_iters
    assert abs(rep.inner_iters_total - ref.inner_iters_total) <= 50 * rep.outer_iters


# ------------------------------------------------------------------ SP-SCD / SP-RCD (Alg. 5)
@pytest.mark.parametrize("n,force_large", [(40, False), (1000, False), (1000, True)])
@pytest.mark.parametrize("mode", [(0, 1), (1, 10 ** 6)])
def test_scd_argmax_ties(n, force_large, mode, monkeypatch):
    """Exact ties in the Alg. 5 step 8 argmax: A1 = 2 I, A2 = I / 2 (q = n),
    b = (+-1, ...): r_j^2 is the same for every coordinate until it is zeroed, so every step is a
    tie that must go to the smallest index of tau_t (reading of argmax). Covers the
    one-warp (n = 40), one-CTA (n = 1000) and 16-CTA cluster (forced large) kernels; inner counts
    and iterates against the oracle."""
    from workloads.configs import IlsProblem
    monkeypatch.setenv("ILS_FORCE_LARGE", "1" if force_large else "0")
    A = np.vstack([2.0 * np.eye(n), 0.5 * np.eye(n)])
    b = np.where(np.arange(2 * n) % 3 == 0, -1.0, 1.0)
    pr = IlsProblem(name="ties", A=np.ascontiguousarray(A), b=b, p=n, q=n, xstar=np.zeros(n), consistent=False,
                    tol=1e-8)
    amode, ak = mode
    K, T, ce = 2, 3 * n // 2, n // 4
    ref = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=12, max_inner=T,
                         check_every=ce, inner_tol=0.0, alpha_mode=amode, alpha_fixed=ak)
    hist = np.zeros((K, n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=12, max_inner=T, check_every=ce, inner_tol=0.0,
                                 alpha_mode=amode, alpha_k=min(ak, 2 ** 31 - 1), x_hist=hist.ctypes.data,
                                 inner_hist=inner.ctypes.data)
        ils.ils_rgs_solve(hh.h, None, x, 0.0, K, o)
    assert list(inner) == list(ref.inner_hist)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-12, k


@pytest.mark.parametrize("shape", [(200, 100, 50, 0.3), (130, 37, 67, 0.3), (257, 40, 3, 0.3)])
@pytest.mark.parametrize("mode", [(0, 1, 0), (1, 1, 0), (1, 5, 0), (1, 10 ** 6, 0), (0, 1, 1)])
def test_scd_fixed_horizon(shape, mode):
    p, q, n, s = shape
    amode, ak, weighted = mode
    pr = make_dense(p, q, n, s, noise=0.05, seed=8)
    K, T, ce = 3, 300, 40
    ref = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=9, max_inner=T,
                         check_every=ce, inner_tol=0.0, alpha_mode=amode, alpha_fixed=ak,
                         weighted=bool(weighted))
    hist = np.zeros((K, n))
    x = np.zeros(n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=9, max_inner=T, check_every=ce, inner_tol=0.0,
                                 alpha_mode=amode, alpha_k=min(ak, 2 ** 31 - 1), weighted=weighted,
                                 x_hist=hist.ctypes.data)
        ils.ils_rgs_solve(hh.h, None, x, 0.0, K, o)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


def test_scd_converges_c0():
    pr = make_problem("c0")
    x = np.zeros(pr.n)
    with H(pr) as hh:
        o = ils.ils_default_opts(x_ref=pr.xstar.ctypes.data, inner_tol=1e-12, max_inner=100000)
        st, rep = ils.ils_rgs_solve(hh.h, None, x, 1e-10, 100, o)
    assert st == ils.ILS_OK and _rel(x, pr.xstar) <= 1e-10


# ------------------------------------------------------------------ batched (K4)
@pytest.mark.parametrize("method", ["sp", "rk", "rgs", "rcd", "motzkin"])
def test_batched_vs_oracle(method):
    from workloads import make_batched
    bt = make_batched(batch=24, p=96, q=32, n=32, base_seed=100)
    K = 3
    T, ce = 200, 32
    x = np.zeros((bt.batch, bt.n))
    h = ils.ils_create(bt.A, bt.b, bt.p, bt.q, bt.n, batch=bt.batch)
    try:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=T, check_every=ce, inner_tol=0.0, seed=100,
                                 weighted=1 if method == "rcd" else 0)
        if method == "motzkin":   # alpha = n: tau_t = [n], global argmax (Remark 4.1)
            o.alpha_mode, o.alpha_k = ils.ILS_ALPHA_FIXED, bt.n
        fn = {"sp": ils.ils_sp_solve, "rk": ils.ils_rk_solve, "rgs": ils.ils_rgs_solve,
              "rcd": ils.ils_rgs_solve, "motzkin": ils.ils_rgs_solve}[method]
        fn(h, None, x, 0.0, K, o)
    finally:
        ils.ils_destroy(h)
    for i in range(bt.batch):
        A1, A2 = bt.A[i, :bt.p], bt.A[i, bt.p:]
        b1, b2 = bt.b[i, :bt.p], bt.b[i, bt.p:]
        kw = dict(max_iter=K, stop=O.STOP_NONE)
        if method == "sp":
            ref = O.sp_solve(A1, A2, b1, b2, **kw)
        elif method == "rk":
            ref = O.sp_rk_rgs_solve(A1, A2, b1, b2, seed=100 + i, max_inner=T, check_every=ce, inner_tol=0.0, **kw)
        elif method == "motzkin":
            ref = O.sp_scd_solve(A1, A2, b1, b2, seed=100 + i, max_inner=T, check_every=ce, inner_tol=0.0,
                                 alpha_mode=1, alpha_fixed=bt.n, **kw)
        else:
            ref = O.sp_scd_solve(A1, A2, b1, b2, seed=100 + i, max_inner=T, check_every=ce, inner_tol=0.0,
                                 weighted=(method == "rcd"), **kw)
        assert _par(x[i], ref.x) <= 1e-9, (method, i)


def test_batched_converges_c4_subset():
    from workloads import make_batched
    bt = make_batched(batch=256, base_seed=0)
    for fn in (ils.ils_sp_solve, ils.ils_rk_solve, ils.ils_rgs_solve):
        x = np.zeros((bt.batch, bt.n))
        its = np.zeros(bt.batch, dtype=np.int64)
        sts = np.zeros(bt.batch, dtype=np.int32)
        h = ils.ils_create(bt.A, bt.b, bt.p, bt.q, bt.n, batch=bt.batch)
        try:
            o = ils.ils_default_opts(x_ref=bt.xstar.ctypes.data, inner_tol=1e-12, max_inner=100000)
            st, rep = fn(h, None, x, 1e-10, 200, o, inst_iters=its, inst_status=sts)
        finally:
            ils.ils_destroy(h)
        assert st == ils.ILS_OK and sts.all()
        err = np.linalg.norm(x - bt.xstar, axis=1) / np.linalg.norm(bt.xstar, axis=1)
        assert err.max() <= 1e-10


# ------------------------------------------------------------------ paper-literal precompute (sp_form 2)
@pytest.mark.parametrize("method", ["sp", "rk", "rgs"])
def test_literal_precompute_forms(method):
    """Alg. 1 literal (B = P A2bar, c = P A^T J b) and the precomputed-A2bar right-hand side of
    Alg. 2 / Alg. 5 (sp_form = 2) against the oracle's literal forms at a fixed horizon."""
    pr = make_dense(180, 60, 40, 0.3, noise=0.05, seed=21)
    K = 4
    kw = dict(max_iter=K, stop=O.STOP_NONE)
    if method == "sp":
        ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, sp_form=2, **kw)
    elif method == "rk":
        ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, seed=4, max_inner=200, check_every=40, inner_tol=0.0,
                                rhs_literal=True, **kw)
    else:
        ref = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, seed=4, max_inner=200, check_every=40, inner_tol=0.0,
                             rhs_literal=True, **kw)
    hist = np.zeros((K, pr.n))
    x = np.zeros(pr.n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, sp_form=2, seed=4, max_inner=200, check_every=40,
                                 inner_tol=0.0, x_hist=hist.ctypes.data)
        fn = {"sp": ils.ils_sp_solve, "rk": ils.ils_rk_solve, "rgs": ils.ils_rgs_solve}[method]
        fn(hh.h, None, x, 0.0, K, o)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


# ------------------------------------------------------------------ full-size bench configurations
def test_c1_full_size_inner_counts_match_oracle():
    """BASELINE.json configs[1] in the bench's configuration (x_ref stop at 1e-8, inner_tol 1e-10,
    max_inner 1e6, seed 0): every outer step's inner-step count of SP-RK-RGS and SP-SCD equals the
    oracle's (profiles/oracle_c1_counts.json, written by tools/oracle_counts.py from oracle/ only),
    which pins the whole index stream and every inner stop decision at full size."""
    import json
    import os
    ref = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "profiles", "oracle_c1_counts.json")))
    pr = make_problem("c1")
    xref = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "workloads", "xref", "c1_seed0.npy"))
    xr_t = torch.from_numpy(xref).to(DEV)
    with H(pr) as hh:
        for name, fn in (("rk", ils.ils_rk_solve), ("rgs", ils.ils_rgs_solve)):
            x = torch.zeros(pr.n, dtype=torch.float64, device=DEV)
            inner = np.zeros(200, dtype=np.int64)
            o = ils.ils_default_opts(x_ref=xr_t.data_ptr(), inner_tol=ref["inner_tol"], max_inner=ref["max_inner"],
                                     inner_hist=inner.ctypes.data)
            st, rep = fn(hh.h, None, x, pr.tol, 200, o)
            assert st == ils.ILS_OK and rep.converged, name
            assert rep.outer_iters == ref[name]["outer"], name
            assert list(inner[:rep.outer_iters]) == ref[name]["inner_hist"], name
            err = _rel(x.cpu().numpy(), xref)
            assert err <= pr.tol and abs(err - ref[name]["final_err"]) <= 1e-9 * ref[name]["final_err"] + 1e-12, name


def test_scd_c1_fixed_horizon():
    """c1 size through the CTA SP-SCD kernel (n = 1000, V = 4) against the oracle, 3000 steps."""
    pr = make_problem("c1")
    K, T, ce = 1, 3000, 1000
    ref = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=0, max_inner=T,
                         check_every=ce, inner_tol=0.0)
    hist = np.zeros((K, pr.n))
    x = np.zeros(pr.n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=0, max_inner=T, check_every=ce, inner_tol=0.0,
                                 x_hist=hist.ctypes.data)
        ils.ils_rgs_solve(hh.h, None, x, 0.0, K, o)
    assert _par(hist[0], ref.x_hist[0]) <= 1e-9


def test_c4_full_size_all_instances_converge():
    """BASELINE.json configs[4]: all 4096 instances, every method, each within 1e-10 of its x*."""
    pr = make_problem("c4")
    for fn in (ils.ils_sp_solve, ils.ils_rk_solve, ils.ils_rgs_solve):
        x = torch.zeros((pr.batch, pr.n), dtype=torch.float64, device=DEV)
        A = torch.from_numpy(pr.A).to(DEV)
        b = torch.from_numpy(pr.b).to(DEV)
        xs = torch.from_numpy(pr.xstar).to(DEV)
        sts = np.zeros(pr.batch, dtype=np.int32)
        h = ils.ils_create(A, b, pr.p, pr.q, pr.n, batch=pr.batch)
        try:
            o = ils.ils_default_opts(x_ref=xs.data_ptr(), inner_tol=1e-12, max_inner=1_000_000)
            st, rep = fn(h, None, x, pr.tol, 1000, o, inst_status=sts)
        finally:
            ils.ils_destroy(h)
        assert st == ils.ILS_OK and sts.all(), fn
        err = (torch.linalg.norm(x - xs, dim=1) / torch.linalg.norm(xs, dim=1)).max().item()
        assert err <= pr.tol, (fn, err)


# ------------------------------------------------------------------ determinism (include/ils.h)
@pytest.mark.parametrize("cfg", ["c0", "c1"])
def test_bitwise_deterministic_runs(cfg):
    """Same inputs and seed give bitwise-identical iterates and counts (fixed-order reductions, no
    floating-point atomics on the dense paths): two fresh handles, every method, a short horizon."""
    pr = make_problem(cfg)
    outs = []
    for _ in range(2):
        res = []
        with H(pr) as hh:
            for fn in (ils.ils_sp_solve, ils.ils_rk_solve, ils.ils_rgs_solve):
                x = np.zeros(pr.n)
                inner = np.zeros(3, dtype=np.int64)
                o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=7, max_inner=2500, inner_tol=1e-6,
                                         inner_hist=inner.ctypes.data)
                fn(hh.h, None, x, 0.0, 3, o)
                res.append((x.copy(), inner.copy()))
        outs.append(res)
    for (xa, ia), (xb, ib) in zip(outs[0], outs[1]):
        assert np.array_equal(xa, xb) and np.array_equal(ia, ib)


@pytest.mark.parametrize("method", ["sp", "rk"])
def test_auto_form_choice_and_iterates(method):
    """sp_form = ILS_SP_FORM_AUTO (include/ils.h "Automatic form"): a short expected
    horizon keeps the streaming form 0, a long one takes the literal precompute (form 2); either way the
    iterates equal the oracle's for the form the report names."""
    pr = make_dense(180, 400, 40, 0.2, noise=0.05, seed=23)   # q >> n: the literal form's saving is large
    K = 3
    fn = {"sp": ils.ils_sp_solve, "rk": ils.ils_rk_solve}[method]
    for exp_outer, want in ((1, 0), (10 ** 6, 2)):
        hist = np.zeros((K, pr.n))
        x = np.zeros(pr.n)
        with H(pr) as hh:
            o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, sp_form=ils.ILS_SP_FORM_AUTO, expected_outer=exp_outer,
                                     seed=4, max_inner=200, check_every=40, inner_tol=0.0, x_hist=hist.ctypes.data)
            st, rep = fn(hh.h, None, x, 0.0, K, o)
        assert rep.sp_form_used == want, (exp_outer, rep.sp_form_used)
        kw = dict(max_iter=K, stop=O.STOP_NONE)
        if method == "sp":
            ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, sp_form=want, **kw)
        else:
            ref = O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, seed=4, max_inner=200, check_every=40, inner_tol=0.0,
                                    rhs_literal=(want == 2), **kw)
        for k in range(K):
            assert _par(hist[k], ref.x_hist[k]) <= 1e-9, (exp_outer, k)


def test_batched_zero_column_and_not_spd_errors():
    """Batched handles report the errors include/ils.h promises: an instance with a
    zero A1 column fails ils_create with ILS_ERR_ZERO_COLUMN; an instance whose A1^T A1 is singular
    (two equal columns 2 e_0: the second Cholesky pivot is exactly 4 - 2 * 2 = 0) makes SP return
    ILS_ERR_NOT_SPD with inst_status -1 for that instance."""
    from workloads import make_batched
    bt = make_batched(batch=8, p=96, q=32, n=32, base_seed=500)
    A = bt.A.copy()
    A[5, :96, 7] = 0.0
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(A, bt.b, bt.p, bt.q, bt.n, batch=bt.batch)
    assert e.value.status == ils.ILS_ERR_ZERO_COLUMN
    A = bt.A.copy()
    A[3, :96, 0] = 0.0
    A[3, :96, 1] = 0.0
    A[3, 0, 0] = 2.0
    A[3, 0, 1] = 2.0
    h = ils.ils_create(A, bt.b, bt.p, bt.q, bt.n, batch=bt.batch)
    try:
        x = np.zeros((bt.batch, bt.n))
        sts = np.zeros(bt.batch, dtype=np.int32)
        with pytest.raises(ils.IlsError) as e:
            ils.ils_sp_solve(h, None, x, 0.0, 3, ils.ils_default_opts(stop=ils.ILS_STOP_NONE), inst_status=sts)
        assert e.value.status == ils.ILS_ERR_NOT_SPD
        assert sts[3] == -1
    finally:
        ils.ils_destroy(h)


@pytest.mark.parametrize("n", [1, 2, 5, 17, 50, 1000, 4000])
def test_exact_subset_replay(n):
    """ILS_SUBSET_EXACT: alpha_t and the membership of the key-selection subset are
    bit-exact against the oracle's independent implementation of the include/ils.h text."""
    for (seed, k, t) in [(0, 0, 0), (3, 2, 99), (11, 9, 123456)]:
        for mode, ak in [(0, 1), (1, 1), (1, max(1, n // 3)), (1, n)]:
            alpha, mask = ils.ils_scd_subset(n, seed, k, t, mode | ils.ILS_SUBSET_EXACT, ak)
            a_o, tau = ix.scd_subset(seed, k, t, n, mode | ix.SUBSET_EXACT, ak)
            assert alpha == a_o
            assert np.array_equal(np.flatnonzero(mask), tau)


@pytest.mark.parametrize("shape,force_large", [((200, 100, 50), False), ((1400, 300, 1000), False),
                                               ((260, 60, 130), True)])
def test_scd_exact_subsets_fixed_horizon(shape, force_large, monkeypatch):
    """SP-SCD with exact uniform subsets through the one-warp (n = 50), one-CTA (n = 1000) and
    forced-large cluster kernels: inner counts and iterates against the oracle."""
    monkeypatch.setenv("ILS_FORCE_LARGE", "1" if force_large else "0")
    p, q, n = shape
    pr = make_dense(p, q, n, 0.3, noise=0.05, seed=24)
    K, T, ce = 2, 400, 100
    mode = ils.ILS_ALPHA_UNIFORM | ils.ILS_SUBSET_EXACT
    ref = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=8, max_inner=T,
                         check_every=ce, inner_tol=0.0, alpha_mode=mode)
    hist = np.zeros((K, n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(n)
    with H(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=8, max_inner=T, check_every=ce, inner_tol=0.0,
                                 alpha_mode=mode, x_hist=hist.ctypes.data, inner_hist=inner.ctypes.data)
        ils.ils_rgs_solve(hh.h, None, x, 0.0, K, o)
    assert list(inner) == list(ref.inner_hist)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


@pytest.mark.parametrize("shape,force_large", [((40, 5, 1), False), ((60, 10, 3), False), ((200, 100, 50), False),
                                               ((1400, 300, 1000), False), ((2000, 200, 1500), False),
                                               ((260, 60, 130), True), ((6000, 300, 5000), True)])
@pytest.mark.parametrize("mode", [(0, 1), (1, 7), (1, 10 ** 6)])
def test_scd_masks_forward_kernel_matches_decrypt_kernel(shape, force_large, mode, monkeypatch):
    """The membership masks of Alg. 5 step 8 built forward (tau_t = {pi(i) : i <
    alpha_t}, tabulated rounds, scd_masks_fwd_kernel) and by decrypting every coordinate
    (pi^{-1}(s) < alpha_t, scd_masks_kernel) give bit-identical SP-SCD iterates and inner counts
    through the one-warp, one-CTA (V = 4, 8) and cluster kernels; one of them against the oracle."""
    monkeypatch.setenv("ILS_FORCE_LARGE", "1" if force_large else "0")
    p, q, n = shape
    pr = make_dense(p, q, n, 0.3, noise=0.05, seed=31)
    amode, ak = mode
    K, T, ce = 2, 300, 100
    runs = []
    for fwd in ("0", "1"):
        monkeypatch.setenv("ILS_MASKS_FWD", fwd)
        hist = np.zeros((K, n))
        inner = np.zeros(K, dtype=np.int64)
        x = np.zeros(n)
        with H(pr) as hh:
            o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=5, max_inner=T, check_every=ce, inner_tol=0.0,
                                     alpha_mode=amode, alpha_k=min(ak, 2 ** 31 - 1), x_hist=hist.ctypes.data,
                                     inner_hist=inner.ctypes.data)
            ils.ils_rgs_solve(hh.h, None, x, 0.0, K, o)
        runs.append((hist, inner))
    assert np.array_equal(runs[0][0], runs[1][0]) and list(runs[0][1]) == list(runs[1][1])
    if n <= 1000:
        ref = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=5, max_inner=T,
                             check_every=ce, inner_tol=0.0, alpha_mode=amode, alpha_fixed=ak)
        for k in range(K):
            assert _par(runs[1][0][k], ref.x_hist[k]) <= 1e-9, k


@pytest.mark.parametrize("shape", [(2600, 300, 2100), (1400, 200, 700)])
def test_sp_leaf_variants_match_oracle(shape, monkeypatch):
    """SP (Alg. 1; its setup Gram -> Cholesky -> inverse -> P, step 2) with the blocked
    64x64 leaf (default) and with the column-at-a-time leaf (ILS_LEAF_OLD=1): both within 1e-9 of the
    oracle's iterates."""
    p, q, n = shape
    pr = make_dense(p, q, n, 0.3, noise=0.05, seed=41)
    K = 3
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE)
    for old in ("0", "1"):
        monkeypatch.setenv("ILS_LEAF_OLD", old)
        hist = np.zeros((K, n))
        x = np.zeros(n)
        with H(pr) as hh:
            ils.ils_sp_solve(hh.h, None, x, 0.0, K, ils.ils_default_opts(stop=ils.ILS_STOP_NONE, x_hist=hist.ctypes.data))
        for k in range(K):
            assert _par(hist[k], ref.x_hist[k]) <= 1e-9, (old, k)


@pytest.mark.parametrize("n", [1, 5, 17, 24, 31])
@pytest.mark.parametrize("method", ["rgs", "rcd"])
def test_batched_scd_generic_n_vs_oracle(n, method):
    """Batched SP-SCD / SP-RCD (Alg. 5) at n != 32: the generic kernel (Feistel
    domains 4^h of 4, 16 and 64 with cycle walking through values >= n) against the oracle per
    instance; n = 32 (c4) takes the specialised kernel (test_batched_vs_oracle)."""
    from workloads import make_batched
    bt = make_batched(batch=12, p=3 * n + 8, q=max(n // 2, 1), n=n, base_seed=300)
    K, T, ce = 3, 150, 25
    x = np.zeros((bt.batch, bt.n))
    h = ils.ils_create(bt.A, bt.b, bt.p, bt.q, bt.n, batch=bt.batch)
    try:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, max_inner=T, check_every=ce, inner_tol=0.0, seed=300,
                                 weighted=1 if method == "rcd" else 0)
        ils.ils_rgs_solve(h, None, x, 0.0, K, o)
    finally:
        ils.ils_destroy(h)
    for i in range(bt.batch):
        A1, A2 = bt.A[i, :bt.p], bt.A[i, bt.p:]
        b1, b2 = bt.b[i, :bt.p], bt.b[i, bt.p:]
        ref = O.sp_scd_solve(A1, A2, b1, b2, max_iter=K, stop=O.STOP_NONE, seed=300 + i, max_inner=T,
                             check_every=ce, inner_tol=0.0, weighted=(method == "rcd"))
        assert _par(x[i], ref.x) <= 1e-9, (method, n, i)
