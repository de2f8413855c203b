"""GPU parity for the CSR input path (BASELINE.json configs[3]) through the C ABI, against the CPU
oracle run on the same matrix (densified at test sizes; scipy.sparse at full size).

Bars as in test_gpu_parity.py: sampling tables bit-exact, iterates within 1e-9 relative at fixed
horizons, converged solutions within the config tolerance.
"""
import json
import os

import numpy as np
import pytest

from oracle import ils_oracle as O
from oracle import index_stream as ix
from workloads import make_problem, make_sparse

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2203_15340_b200 import ils  # noqa: E402

DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _par(a, b):
    """Parity distance of two iterates: the larger of the norm-wise relative difference (the
    north_star bar) and the element-wise max |a_i - b_i| / max |b_i|, so that a wrong small
    coordinate cannot hide inside the norm."""
    a, b = np.asarray(a), np.asarray(b)
    d = np.abs(a - b)
    return max(_rel(a, b), float(d.max() / max(np.abs(b).max(), 1e-300)) if d.size else 0.0)


class HS:
    """Handle on a sparse problem; CSR arrays passed as device tensors (or host arrays)."""

    def __init__(self, pr, host=False):
        if host:
            self.h = ils.ils_create(pr.vals, pr.b, pr.p, pr.q, pr.n, row_ptr=pr.row_ptr, col_idx=pr.col_idx)
        else:
            t = {k: torch.from_numpy(getattr(pr, k)).to(DEV) for k in ("vals", "b", "row_ptr", "col_idx")}
            self._keep = t
            self.h = ils.ils_create(t["vals"], t["b"], pr.p, pr.q, pr.n, row_ptr=t["row_ptr"], col_idx=t["col_idx"])

    def __enter__(self):
        return self

    def __exit__(self, *a):
        ils.ils_destroy(self.h)


def _dense(pr):
    A = pr.dense()
    return A[:pr.p], A[pr.p:], pr.b[:pr.p], pr.b[pr.p:]


SHAPES = [(600, 120, 80, 6), (300, 0, 45, 4), (257, 33, 31, 5), (1000, 300, 130, 3)]


@pytest.mark.parametrize("shape", SHAPES)
def test_sparse_sampling_tables_bitwise(shape):
    p, q, n, k = shape
    pr = make_sparse(p, q, n, k, seed=11)
    A1, _, _, _ = _dense(pr)
    with HS(pr) as hh:
        N, S = ils.ils_get_sampling_tables(hh.h, n)
    No = ix.column_norms_sq(A1)
    _, So = ix.weights_prefix(No)
    assert np.array_equal(N.view(np.uint64), No.view(np.uint64))
    assert [int(v) for v in S] == So


@pytest.mark.parametrize("shape", SHAPES)
def test_sparse_direct_solve_and_rr(shape):
    p, q, n, k = shape
    pr = make_sparse(p, q, n, k, seed=12)
    A1, A2, b1, b2 = _dense(pr)
    xo = O.direct_solve(A1, A2, b1, b2)
    x = np.zeros(n)
    with HS(pr, host=True) as hh:
        ils.ils_direct_solve(hh.h, x)
        rr0 = ils.ils_relative_residual(hh.h, np.zeros(n))
    assert _par(x, xo) <= 1e-10
    assert abs(rr0 - 1.0) <= 1e-14


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("form", [0, 1])
def test_sparse_sp_fixed_horizon(shape, form):
    """form 0: the paper's x_{k+1} = P (A1^T b1 + A2^T (A2 x_k - b2)); form 1: the correction form
    x_{k+1} = x_k + P A^T J (b - A x_k) (DESIGN.md readings)."""
    p, q, n, k = shape
    pr = make_sparse(p, q, n, k, seed=13)
    A1, A2, b1, b2 = _dense(pr)
    K = 6
    ref = O.sp_solve(A1, A2, b1, b2, max_iter=K, stop=O.STOP_NONE, sp_form=form)
    hist = np.zeros((K, n))
    x = np.zeros(n)
    with HS(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, sp_form=form, x_hist=hist.ctypes.data)
        st, rep = ils.ils_sp_solve(hh.h, None, x, 0.0, K, o)
    assert rep.outer_iters == K
    for kk in range(K):
        assert _par(hist[kk], ref.x_hist[kk]) <= 1e-9, kk


def test_sparse_sp_rr_stop():
    pr = make_sparse(500, 100, 60, 5, seed=14)
    A1, A2, b1, b2 = _dense(pr)
    ref = O.sp_solve(A1, A2, b1, b2, tol=1e-12, stop=O.STOP_RR, max_iter=100)
    x = np.zeros(pr.n)
    with HS(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_RR)
        st, rep = ils.ils_sp_solve(hh.h, None, x, 1e-12, 100, o)
        assert rep.converged and rep.final_metric < 1e-12
        assert abs(rep.outer_iters - ref.outer_iters) <= 1


@pytest.mark.parametrize("T", [1, 7, 333])
def test_sparse_rk_fixed_horizon(T):
    pr = make_sparse(600, 120, 80, 6, seed=15)
    A1, A2, b1, b2 = _dense(pr)
    K, ce = 3, 50
    ref = O.sp_rk_rgs_solve(A1, A2, b1, b2, max_iter=K, stop=O.STOP_NONE, seed=3, max_inner=T, check_every=ce,
                            inner_tol=0.0)
    hist = np.zeros((K, pr.n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(pr.n)
    with HS(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=3, max_inner=T, check_every=ce, inner_tol=0.0,
                                 x_hist=hist.ctypes.data, inner_hist=inner.ctypes.data)
        ils.ils_rk_solve(hh.h, None, x, 0.0, K, o)
    for kk in range(K):
        assert _par(hist[kk], ref.x_hist[kk]) <= 1e-9, kk
    assert list(inner) == list(ref.inner_hist)


@pytest.mark.parametrize("mode", [(0, 1, 0), (1, 1, 0), (1, 5, 0), (1, 10 ** 6, 0), (1, 1, 1)])
def test_sparse_scd_fixed_horizon(mode):
    """(alpha_mode, alpha_k, weighted): weighted = 1 is SP-RCD."""
    pr = make_sparse(600, 120, 80, 6, seed=16)
    A1, A2, b1, b2 = _dense(pr)
    amode, ak, wt = mode
    K, T, ce = 3, 300, 40
    ref = O.sp_scd_solve(A1, A2, b1, b2, max_iter=K, stop=O.STOP_NONE, seed=9, max_inner=T, check_every=ce,
                         inner_tol=0.0, alpha_mode=amode, alpha_fixed=ak, weighted=bool(wt))
    hist = np.zeros((K, pr.n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(pr.n)
    with HS(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=9, max_inner=T, check_every=ce, inner_tol=0.0,
                                 alpha_mode=amode, alpha_k=min(ak, 2 ** 31 - 1), weighted=wt,
                                 x_hist=hist.ctypes.data, inner_hist=inner.ctypes.data)
        ils.ils_rgs_solve(hh.h, None, x, 0.0, K, o)
    assert list(inner) == list(ref.inner_hist)
    for kk in range(K):
        assert _par(hist[kk], ref.x_hist[kk]) <= 1e-9, kk


def test_sparse_rcd_converges():
    """Weighted SP-RCD on CSR input reaches the planted solution (consistent system)."""
    pr = make_sparse(800, 160, 60, 6, seed=19, noise=0.0)
    x = np.zeros(pr.n)
    with HS(pr) as hh:
        o = ils.ils_default_opts(x_ref=pr.xstar.ctypes.data, inner_tol=1e-12, max_inner=400000, weighted=1)
        st, rep = ils.ils_rgs_solve(hh.h, None, x, 1e-10, 200, o)
    assert st == ils.ILS_OK and _rel(x, pr.xstar) <= 1e-10


def test_sparse_methods_converge():
    pr = make_sparse(800, 160, 60, 6, seed=17, noise=0.0)
    tol = 1e-10
    for fn in (ils.ils_sp_solve, ils.ils_rk_solve, ils.ils_rgs_solve):
        x = np.zeros(pr.n)
        with HS(pr) as hh:
            o = ils.ils_default_opts(x_ref=pr.xstar.ctypes.data, inner_tol=1e-12, max_inner=200000)
            st, rep = fn(hh.h, None, x, tol, 200, o)
        assert st == ils.ILS_OK and _rel(x, pr.xstar) <= tol, fn


def test_sparse_csr_validation():
    pr = make_sparse(40, 10, 8, 3, seed=18)
    bad = pr.col_idx.copy()
    bad[1], bad[2] = bad[2], bad[1]   # unsorted within row 0
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(pr.vals, pr.b, pr.p, pr.q, pr.n, row_ptr=pr.row_ptr, col_idx=bad)
    assert e.value.status == ils.ILS_ERR_ARG
    bad = pr.col_idx.copy()
    bad[5] = pr.n   # out of range
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(pr.vals, pr.b, pr.p, pr.q, pr.n, row_ptr=pr.row_ptr, col_idx=bad)
    assert e.value.status == ils.ILS_ERR_ARG
    rp = pr.row_ptr.copy()
    rp[-1] -= 1
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(pr.vals, pr.b, pr.p, pr.q, pr.n, row_ptr=rp, col_idx=pr.col_idx)
    assert e.value.status == ils.ILS_ERR_ARG
    v = pr.vals.copy()
    v[3] = np.inf
    with pytest.raises(ils.IlsError) as e:
        ils.ils_create(v, pr.b, pr.p, pr.q, pr.n, row_ptr=pr.row_ptr, col_idx=pr.col_idx)
    assert e.value.status == ils.ILS_ERR_ARG


def test_sparse_c3_full_size_sp():
    """configs[3] at full size in the bench's launch configuration: SP reaches 1e-8 against the
    oracle-written x_ref (tools/make_xref.py, oracle Cholesky of A^T J A)."""
    base = os.path.join(ROOT, "workloads", "xref", "c3_seed0")
    meta = json.load(open(base + ".json"))
    pr = make_problem("c3", seed=meta["data_seed"])
    xref = np.load(base + ".npy")
    xr_t = torch.from_numpy(xref).to(DEV)
    x = torch.zeros(pr.n, dtype=torch.float64, device=DEV)
    with HS(pr) as hh:
        o = ils.ils_default_opts(x_ref=xr_t.data_ptr())
        st, rep = ils.ils_sp_solve(hh.h, None, x, pr.tol, 100, o)
    assert st == ils.ILS_OK and rep.converged
    assert _rel(x.cpu().numpy(), xref) <= pr.tol


@pytest.mark.parametrize("method", ["sp", "rk", "rgs"])
@pytest.mark.parametrize("shape", [(500, 100, 60, 5), (2000, 400, 300, 8)])
def test_sparse_literal_precompute_forms(method, shape):
    """CSR input with the paper-literal precompute (sp_form = 2; Alg. 1 steps 2-3, PAPER.md:134-135:
    B = P A2bar, c = P A^T J b; Alg. 2 / Alg. 5 step 5: b_hat = A2bar x_k + A^T J b with A2bar =
    A2^T A2 formed from the CSC of A2) against the oracle's literal forms at a fixed horizon."""
    p, q, n, k = shape
    pr = make_sparse(p, q, n, k, seed=23)
    A1, A2, b1, b2 = _dense(pr)
    K = 4
    kw = dict(max_iter=K, stop=O.STOP_NONE)
    if method == "sp":
        ref = O.sp_solve(A1, A2, b1, b2, sp_form=2, **kw)
    elif method == "rk":
        ref = O.sp_rk_rgs_solve(A1, A2, b1, b2, seed=6, max_inner=300, check_every=50, inner_tol=0.0,
                                rhs_literal=True, **kw)
    else:
        ref = O.sp_scd_solve(A1, A2, b1, b2, seed=6, max_inner=300, check_every=50, inner_tol=0.0,
                             rhs_literal=True, **kw)
    hist = np.zeros((K, n))
    x = np.zeros(n)
    with HS(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, sp_form=2, seed=6, max_inner=300, check_every=50,
                                 inner_tol=0.0, x_hist=hist.ctypes.data)
        fn = {"sp": ils.ils_sp_solve, "rk": ils.ils_rk_solve, "rgs": ils.ils_rgs_solve}[method]
        st, rep = fn(hh.h, None, x, 0.0, K, o)
        assert rep.sp_form_used == 2
    for kk in range(K):
        assert _par(hist[kk], ref.x_hist[kk]) <= 1e-9, kk


@pytest.mark.parametrize("shape", [(3000, 200, 20, 5), (600, 120, 80, 6), (257, 33, 31, 5)])
def test_sparse_gram_staged_bitwise(shape, monkeypatch):
    """The staged Gram-row kernel (default) against the one-warp kernel (ILS_SPGRAM_OLD=1): same
    per-address fma order, so the SP iterates (through P built from A1bar) are bitwise equal, also
    with a 7-contribution window (rows straddling windows, ILS_SPGRAM_CCAP=7) and columns longer than
    one 256-entry chunk (3000 rows x 5 nnz over 20 columns: ~750 entries per column); and within
    1e-9 of the oracle."""
    p, q, n, k = shape
    pr = make_sparse(p, q, n, k, seed=21)
    A1, A2, b1, b2 = _dense(pr)
    K = 3
    ref = O.sp_solve(A1, A2, b1, b2, max_iter=K, stop=O.STOP_NONE)
    hists = []
    for env in ({"ILS_SPGRAM_OLD": "1"}, {}, {"ILS_SPGRAM_CCAP": "7"}):
        monkeypatch.delenv("ILS_SPGRAM_OLD", raising=False)
        monkeypatch.delenv("ILS_SPGRAM_CCAP", raising=False)
        for kk, v in env.items():
            monkeypatch.setenv(kk, v)
        hist = np.zeros((K, n))
        x = np.zeros(n)
        with HS(pr) as hh:
            o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, x_hist=hist.ctypes.data)
            ils.ils_sp_solve(hh.h, None, x, 0.0, K, o)
        hists.append(hist)
    assert np.array_equal(hists[0], hists[1])
    assert np.array_equal(hists[0], hists[2])
    for kk in range(K):
        assert _par(hists[1][kk], ref.x_hist[kk]) <= 1e-9, kk


@pytest.mark.parametrize("cols", ["0", "2"])
@pytest.mark.parametrize("th", [1, 2, 3, 64])
@pytest.mark.parametrize("shape", [(4000, 900, 700, 6), (3000, 0, 333, 5)])
def test_sparse_sp_tree_inverse(monkeypatch, shape, th, cols):
    """The n >= 8192 form of P (x = Z^T (Z c) on the Cholesky recursion's tree, whole inverses only of
    the diagonal blocks of <= ILS_ZT_TH 64-blocks, L21 by the recursive triangular solve), forced at
    small n (ILS_ZT_MIN_NPAD): SP iterates against the oracle for trees of depth 0 .. 4."""
    p, q, n, k = shape
    monkeypatch.setenv("ILS_ZT_MIN_NPAD", "64")
    monkeypatch.setenv("ILS_ZT_TH", str(th))
    # x = Z^T t passes (c = base + alpha X^T y, also lower-triangular X): the 32-column kernel ("0") and
    # the tiled two-columns-per-thread kernel with its chunk reduction forced at these small panels ("2")
    monkeypatch.setenv("ILS_COLS_TILED", cols)
    pr = make_sparse(p, q, n, k, seed=21)
    A1, A2, b1, b2 = _dense(pr)
    K = 5
    ref = O.sp_solve(A1, A2, b1, b2, max_iter=K, stop=O.STOP_NONE)
    hist = np.zeros((K, n))
    x = np.zeros(n)
    with HS(pr) as hh:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, x_hist=hist.ctypes.data)
        st, rep = ils.ils_sp_solve(hh.h, None, x, 0.0, K, o)
        xd = np.zeros(n)
        ils.ils_direct_solve(hh.h, xd)
    assert rep.outer_iters == K
    for kk in range(K):
        assert _par(hist[kk], ref.x_hist[kk]) <= 1e-9, kk
    assert _par(xd, O.direct_solve(A1, A2, b1, b2)) <= 1e-9
