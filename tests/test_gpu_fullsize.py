"""GPU parity at the large configs' own sizes and for the kernel instantiations they select.

SURVEY.md §8(c) Mode F (fixed horizon, stopping disabled): both sides run exactly K outer x T inner
steps from x0 = 0 with the same seed; the iterates after every outer step must agree within 1e-9
relative (north_star), norm-wise and element-wise (`_par`), and the inner step counts must be
equal. Horizons: c2 K = 2, T = 1e4 (Alg. 2 steps 7-12 PAPER.md:296-301; Alg. 5 steps 6-11
PAPER.md:692-699); c3 K = 2, T = 1e4.

Besides c2 (p = 40000: `rk_rgs_kernel<16,8>` single-step cluster kernel; n = 4000:
`scd_chunk_kernel<16>`) and c3 (CSR: single-CTA sparse kernels, 160 KB shared residual), the file
covers the instantiations no other test reaches: forced-large routing at p > 32768 (the U = 8 gmode
kernel), the single-step kernel on a 16-CTA geometry (ILS_RK_SINGLE_STEP=1), dense SP-SCD at
n = 1500 (V = 8) and n = 8000 (V = 32), the one-warp kernel with V = 8 (n = 200), and CSR input
with > 512 stored entries per column.
"""
import os

import numpy as np
import pytest

from oracle import ils_oracle as O
from workloads import make_dense, make_problem, make_sparse

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
from paper_2203_15340_b200 import ils  # noqa: E402

DEV = "cuda:0"


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _par(a, b):
    """Parity distance of two iterates: the larger of the norm-wise relative difference (the
    north_star bar) and the element-wise max |a_i - b_i| / max |b_i|."""
    a, b = np.asarray(a), np.asarray(b)
    d = np.abs(a - b)
    return max(_rel(a, b), float(d.max() / max(np.abs(b).max(), 1e-300)) if d.size else 0.0)


def _handle(pr):
    if hasattr(pr, "row_ptr"):
        t = {k: torch.from_numpy(getattr(pr, k)).to(DEV) for k in ("vals", "b", "row_ptr", "col_idx")}
        h = ils.ils_create(t["vals"], t["b"], pr.p, pr.q, pr.n, row_ptr=t["row_ptr"], col_idx=t["col_idx"])
        return h, t
    t = (torch.from_numpy(pr.A).to(DEV), torch.from_numpy(pr.b).to(DEV))
    return ils.ils_create(t[0], t[1], pr.p, pr.q, pr.n), t


def _mode_f(pr, args, method, K, T, ce, seed, h=None, **kw):
    """Run the GPU and the oracle for K outer x T inner steps (no stopping); compare per outer step."""
    ofn = O.sp_rk_rgs_solve if method == "rk" else O.sp_scd_solve
    ref = ofn(*args, max_iter=K, stop=O.STOP_NONE, seed=seed, max_inner=T, check_every=ce, inner_tol=0.0, **kw)
    hist = np.zeros((K, pr.n))
    inner = np.zeros(K, dtype=np.int64)
    x = np.zeros(pr.n)
    own = h is None
    if own:
        h, keep = _handle(pr)
    try:
        o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, seed=seed, max_inner=T, check_every=ce, inner_tol=0.0,
                                 x_hist=hist.ctypes.data, inner_hist=inner.ctypes.data,
                                 alpha_mode=kw.get("alpha_mode", 0), alpha_k=min(kw.get("alpha_fixed", 1), 2 ** 31 - 1),
                                 weighted=int(kw.get("weighted", False)))
        fn = ils.ils_rk_solve if method == "rk" else ils.ils_rgs_solve
        st, rep = fn(h, None, x, 0.0, K, o)
    finally:
        if own:
            ils.ils_destroy(h)
    assert rep.outer_iters == K
    assert list(inner) == list(ref.inner_hist) == [T] * K
    errs = [_par(hist[k], ref.x_hist[k]) for k in range(K)]
    print(f"[mode F] {pr.__class__.__name__} p={pr.p} q={pr.q} n={pr.n} {method} {kw} K={K} T={T} ce={ce}: "
          f"inner {list(inner)} parity {['%.2e' % e for e in errs]}")
    for k in range(K):
        assert errs[k] <= 1e-9, (k, errs)
    return errs


# ------------------------------------------------------------------ configs[2] at full size
@pytest.fixture(scope="module")
def c2():
    pr = make_problem("c2")
    return pr, (pr.A1, pr.A2, pr.b1, pr.b2)


@pytest.fixture(scope="module")
def c2_handle(c2):
    pr, _ = c2
    h, keep = _handle(pr)
    yield h
    ils.ils_destroy(h)


def test_c2_full_size_sp_iterates_and_convergence(c2, c2_handle):
    """configs[2] at full size (p=40000, q=10000, n=4000, ill-conditioned) in the bench's launch
    configuration: the first two SP iterates match the oracle's (1e-9, the paper-form floor is
    ~1e-10, SURVEY Appendix A probe 3) and SP reaches 1e-8 against x* (consistent b = A x*)."""
    pr, args = c2
    K = 2
    ref = O.sp_solve(*args, max_iter=K, stop=O.STOP_NONE)
    hist = np.zeros((K, pr.n))
    x = torch.zeros(pr.n, dtype=torch.float64, device=DEV)
    xs = torch.from_numpy(pr.xstar).to(DEV)
    o = ils.ils_default_opts(stop=ils.ILS_STOP_NONE, x_hist=hist.ctypes.data)
    ils.ils_sp_solve(c2_handle, None, x, 0.0, K, o)
    for k in range(K):
        assert _par(hist[k], ref.x_hist[k]) <= 1e-9, k
    o = ils.ils_default_opts(x_ref=xs.data_ptr())
    st, rep = ils.ils_sp_solve(c2_handle, None, x, pr.tol, 100, o)
    assert st == ils.ILS_OK and rep.converged
    assert _rel(x.cpu().numpy(), pr.xstar) <= pr.tol


def test_c2_full_size_rk_rgs_mode_f(c2, c2_handle):
    """SP-RK-RGS on configs[2]: K = 2, T = 1e4 (check_every = n = 4000, so two inner checks with
    the r = w - A1 z reset per outer step) through `rk_rgs_kernel<16,8>`."""
    pr, args = c2
    _mode_f(pr, args, "rk", K=2, T=10000, ce=pr.n, seed=0, h=c2_handle)


@pytest.mark.parametrize("kw", [{}, {"weighted": True}], ids=["scd", "rcd"])
def test_c2_full_size_scd_mode_f(c2, c2_handle, kw):
    """SP-SCD (uniform alpha_t, `scd_chunk_kernel<16>`) and weighted SP-RCD on configs[2]:
    K = 2, T = 1e4, check_every = n."""
    pr, args = c2
    _mode_f(pr, args, "rgs", K=2, T=10000, ce=pr.n, seed=0, h=c2_handle, **kw)


# ------------------------------------------------------------------ configs[3] at full size
@pytest.fixture(scope="module")
def c3():
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    meta = json.load(open(os.path.join(root, "workloads", "xref", "c3_seed0.json")))
    pr = make_problem("c3", seed=meta["data_seed"])
    S = pr.scipy()
    return pr, (S[:pr.p], S[pr.p:], pr.b[:pr.p], pr.b[pr.p:])


@pytest.fixture(scope="module")
def c3_handle(c3):
    pr, _ = c3
    h, keep = _handle(pr)
    yield h
    ils.ils_destroy(h)


def test_c3_full_size_rk_rgs_mode_f(c3, c3_handle):
    """SP-RK-RGS on configs[3] (CSR, p = 500000, n = 20000) against the oracle's column-wise CSC
    path (pinned to the dense oracle by test_sparse_column_path_matches_the_pinned_dense_oracle):
    K = 2, T = 1e4, an inner check (r reset) every 2500 steps."""
    pr, args = c3
    _mode_f(pr, args, "rk", K=2, T=10000, ce=2500, seed=0, h=c3_handle)


@pytest.mark.parametrize("kw", [{}, {"weighted": True}], ids=["scd", "rcd"])
def test_c3_full_size_scd_mode_f(c3, c3_handle, kw):
    """SP-SCD (uniform alpha_t; the shared-residual kernel with r = 160 KB in shared memory) and
    weighted SP-RCD on configs[3]: K = 2, T = 1e4, a check every 2500 steps."""
    pr, args = c3
    _mode_f(pr, args, "rgs", K=2, T=10000, ce=2500, seed=0, h=c3_handle, **kw)


# ------------------------------------------------------------------ kernel instantiations
@pytest.mark.parametrize("single,T,ce", [("0", 3000, 1000), ("0", 2999, 997), ("1", 3000, 1000)])
def test_rk_forced_large_u8_gmode(single, T, ce, monkeypatch):
    """p > 32768 with forced-large routing: the slice exceeds 2048 rows, so U = 8 rows per thread
    with z and the prefix sums in global memory (gmode) -- the geometry the paper's Tables 3-5 sizes
    and c2 run (p = 40000-60000): the blocked kernel with B steps per cluster reduction
    (`rk_rgs_block_kernel<16,8,B>` gmode; T, ce not multiples of B mask the tail steps) and, with
    ILS_RK_SINGLE_STEP=1, the one-step kernel (`rk_rgs_kernel<16,8>` gmode)."""
    monkeypatch.setenv("ILS_FORCE_LARGE", "1")
    monkeypatch.setenv("ILS_RK_SINGLE_STEP", single)
    pr = make_dense(40000, 500, 300, 0.4, noise=0.05, seed=61)
    _mode_f(pr, (pr.A1, pr.A2, pr.b1, pr.b2), "rk", K=2, T=T, ce=ce, seed=3)


def test_rk_single_step_kernel_16cta(monkeypatch):
    """ILS_RK_SINGLE_STEP=1 (read at create) forces the one-step-per-exchange kernel on a 16-CTA
    geometry (p = 10000, U = 4) that would otherwise take the blocked look-ahead kernel."""
    monkeypatch.setenv("ILS_RK_SINGLE_STEP", "1")
    pr = make_dense(10000, 500, 700, 0.5, noise=0.05, seed=62)
    _mode_f(pr, (pr.A1, pr.A2, pr.b1, pr.b2), "rk", K=2, T=2003, ce=250, seed=4)


@pytest.mark.parametrize("shape,tag", [((200, 60, 200), "warp V=8"), ((1700, 200, 1500), "CTA V=8"),
                                       ((8100, 200, 8000), "CTA V=32")])
def test_scd_dense_vector_widths(shape, tag):
    """Dense SP-SCD kernels by coordinates per lane / thread: the one-warp kernel with V = 8
    (n = 200), the 256-thread CTA kernel with V = 8 (n = 1500) and V = 32 (n = 8000)."""
    p, q, n = shape
    pr = make_dense(p, q, n, 0.3, noise=0.05, seed=63)
    T = 3000 if n < 8000 else 2000
    _mode_f(pr, (pr.A1, pr.A2, pr.b1, pr.b2), "rgs", K=2, T=T, ce=max(n // 2, 100), seed=5)


@pytest.mark.parametrize("method,kw", [("rk", {}), ("rgs", {}), ("rgs", {"weighted": True})],
                         ids=["rk", "scd", "rcd"])
def test_csr_long_columns(method, kw):
    """CSR input with ~1333 stored entries per A1 column (> 512: the global-column path of the
    sparse kernels), against the dense oracle on the densified matrix."""
    pr = make_sparse(20000, 2000, 30, 2, seed=64)
    A = pr.dense()
    args = (A[:pr.p], A[pr.p:], pr.b[:pr.p], pr.b[pr.p:])
    _mode_f(pr, args, method, K=2, T=600, ce=100, seed=6, **kw)
