"""Row-sharded handles (include/ils.h "Row sharding") on the one GPU this
run has: a world-size-1 NCCL communicator drives the sharded code path (local partials, NCCL
all-reduce, replicated P apply / SP-SCD inner solve) through the C ABI; results are compared with
the CPU oracle at the usual bars. The N > 1 reduction algebra is covered on CPU with gloo
(tests/test_multiprocess.py::test_sharded_oracle_algebra_gloo)."""
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


@pytest.fixture(scope="module")
def comm():
    c = ils.ils_comm_create(ils.ils_comm_unique_id(), 1, 0)
    yield c
    ils.ils_comm_destroy(c)


def _handle(pr, comm):
    A = torch.from_numpy(pr.A).to(DEV)
    b = torch.from_numpy(pr.b).to(DEV)
    return ils.ils_create(A, b, pr.p, pr.q, pr.n, comm=comm), (A, b)


@pytest.mark.parametrize("shape", [(200, 100, 50, 0.3), (257, 33, 31, 0.3), (1000, 300, 130, 0.4)])
@pytest.mark.parametrize("form", [0, 1])
def test_sharded_sp_fixed_horizon(comm, shape, form):
    p, q, n, s = shape
    pr = make_dense(p, q, n, s, seed=41)
    K = 6
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, sp_form=form)
    hist = np.zeros((K, n))
    x = np.zeros(n)
    h, keep = _handle(pr, comm)
    try:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, sp_form=form, x_hist=hist.ctypes.data)
        st, rep = ils.ils_sp_solve(h, None, x, 0.0, K, o)
    finally:
        ils.ils_destroy(h)
    assert rep.outer_iters == K
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


def test_sharded_sp_stops_and_residual(comm):
    pr = make_dense(300, 60, 40, 0.3, seed=42)
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, tol=1e-12, stop=O.STOP_RR, max_iter=200)
    xs = O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2)
    h, keep = _handle(pr, comm)
    try:
        x = np.zeros(pr.n)
        st, rep = ils.ils_sp_solve(h, None, x, 1e-12, 200, ils.ils_default_opts(stop=ils.ILS_STOP_RR))
        assert rep.converged and abs(rep.outer_iters - ref.outer_iters) <= 1
        x = np.zeros(pr.n)
        st, rep = ils.ils_sp_solve(h, None, x, 1e-10, 200, ils.ils_default_opts(x_ref=xs.ctypes.data))
        assert rep.converged and _rel(x, xs) <= 1e-10
        xt = np.linspace(-1.0, 1.0, pr.n)
        rr = ils.ils_relative_residual(h, xt)
        assert abs(rr - O.relative_residual(pr.A1, pr.A2, pr.b1, pr.b2, xt)) <= 1e-12 * max(rr, 1.0)
    finally:
        ils.ils_destroy(h)


@pytest.mark.parametrize("mode", [(0, 1, 0), (1, 5, 0), (1, 10 ** 6, 0), (1, 1, 1)])
def test_sharded_scd_fixed_horizon(comm, mode):
    amode, ak, weighted = mode
    pr = make_dense(600, 120, 80, 0.3, seed=43)
    K, T, ce = 3, 300, 40
    ref = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=9, max_inner=T,
                         check_every=ce, inner_tol=1e-9, alpha_mode=amode, alpha_fixed=ak, weighted=bool(weighted))
    hist = np.zeros((K, pr.n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(pr.n)
    h, keep = _handle(pr, comm)
    try:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=9, max_inner=T, check_every=ce, inner_tol=1e-9,
                                 alpha_mode=amode, alpha_k=min(ak, 2 ** 31 - 1), weighted=weighted,
                                 x_hist=hist.ctypes.data, inner_hist=inner.ctypes.data)
        ils.ils_rgs_solve(h, None, x, 0.0, K, o)
    finally:
        ils.ils_destroy(h)
    assert list(inner) == list(ref.inner_hist)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k


def test_sharded_unsupported_modes_and_shapes(comm):
    pr = make_dense(200, 100, 50, 0.3, seed=44)
    h, keep = _handle(pr, comm)
    try:
        x = np.zeros(pr.n)
        for call in (lambda: ils.ils_rk_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE)),
                     lambda: ils.ils_sp_solve(h, None, x, 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE,
                                                                                        sp_form=2)),
                     lambda: ils.ils_direct_solve(h, x)):
            with pytest.raises(ils.IlsError) as e:
                call()
            assert e.value.status == ils.ILS_ERR_UNSUPPORTED
    finally:
        ils.ils_destroy(h)
    # a shard may hold fewer than n rows of A1 (the global p >= n is the caller's contract); with
    # one rank that leaves A1^T A1 singular, which the Cholesky reports
    A = torch.from_numpy(np.ascontiguousarray(pr.A[pr.p - 30:])).to(DEV)
    b = torch.from_numpy(np.ascontiguousarray(pr.b[pr.p - 30:])).to(DEV)
    h = ils.ils_create(A, b, 30, pr.q, pr.n, comm=comm)
    try:
        with pytest.raises(ils.IlsError) as e:
            ils.ils_sp_solve(h, None, np.zeros(pr.n), 0.0, 1, ils.ils_default_opts(stop=ils.ILS_STOP_NONE))
        assert e.value.status == ils.ILS_ERR_NOT_SPD
    finally:
        ils.ils_destroy(h)
    with pytest.raises(ils.IlsError) as e:   # without a communicator p < n is a shape error
        ils.ils_create(A, b, 30, pr.q, pr.n)
    assert e.value.status == ils.ILS_ERR_SHAPE


def test_sharded_with_large_n_routing(comm, monkeypatch):
    """Sharded handle on the n > 8192 routing (forced at small n): two-pass right-hand side and the
    cluster SP-SCD kernel, each followed by the NCCL all-reduce."""
    monkeypatch.setenv("ILS_FORCE_LARGE", "1")
    pr = make_dense(600, 120, 80, 0.3, seed=46)
    K = 3
    ref_sp = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, sp_form=1)
    ref_scd = O.sp_scd_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=K, stop=O.STOP_NONE, seed=3, max_inner=200,
                             check_every=40, inner_tol=1e-9, alpha_mode=0)
    h, keep = _handle(pr, comm)
    try:
        for fn, ref, kw in ((ils.ils_sp_solve, ref_sp, dict(sp_form=1)),
                            (ils.ils_rgs_solve, ref_scd, dict(seed=3, max_inner=200, check_every=40, inner_tol=1e-9))):
            hist = np.zeros((K, pr.n))
            x = np.zeros(pr.n)
            o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, x_hist=hist.ctypes.data, **kw)
            fn(h, None, x, 0.0, K, o)
            for k in range(K):
                assert _par(hist[k], ref.x_hist[k]) <= 1e-9, (fn, k)
    finally:
        ils.ils_destroy(h)
