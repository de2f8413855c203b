"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: values the paper
(or the SPEC worked examples derived from it) fixes, closed forms, invariants from
the paper's proofs, library routines for special cases, or brute force.
See DESIGN.md "Oracle pins" for the P-numbering.
"""
import json
import os
import subprocess
import shutil

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import ils_oracle as O
from oracle import index_stream as ix
from workloads import PAPER_TABLES, make_dense, make_paper, make_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _np(d, k):
    return np.array(d[k], dtype=np.float64)


# ---------------------------------------------------------------- P1: 2x2 example
def test_p1_two_by_two_closed_form():
    g = _load("sp_2x2.json")
    A1, A2, b1, b2 = _np(g, "A1"), _np(g, "A2"), _np(g, "b1"), _np(g, "b2")
    assert np.array_equal(O.normal_matrix(A1, A2), _np(g, "M"))
    assert np.array_equal(O.ajb(A1, A2, b1, b2), _np(g, "AJb"))
    assert np.allclose(O.direct_solve(A1, A2, b1, b2), _np(g, "x_star"), atol=1e-15)
    A = np.vstack([A1, A2])
    b = np.concatenate([b1, b2])
    assert np.allclose(O.qr_cholesky_solve(A, b, 2), _np(g, "x_star"), atol=1e-14)
    for form in (0, 1):
        rep = O.sp_solve(A1, A2, b1, b2, max_iter=4, stop=O.STOP_NONE, sp_form=form)
        for k, xk in enumerate(_np(g, "sp_iterates")):
            assert np.allclose(rep.x_hist[k], xk, atol=1e-15), (form, k)
    assert abs(O.spectral_radius_sp(A1, A2) - g["rho"]) < 1e-15
    assert O.relative_residual(A1, A2, b1, b2, np.zeros(2)) == g["rr_at_zero"]
    assert O.relative_residual(A1, A2, b1, b2, _np(g, "x_star")) == g["rr_at_xstar"]
    # the squared reading of RR (R15): 9/160 at x_1, where the unsquared ratio would be 0.237
    assert O.relative_residual(A1, A2, b1, b2, _np(g, "sp_iterates")[0]) == g["rr_at_x1"]


# ---------------------------------------------------------------- P2: single steps
def test_p2_single_steps():
    g = _load("steps.json")
    for c in g["rk"]:
        A1 = np.array(c["A1"], float)
        w, _ = O.rk_step(A1.T.copy(), ix.column_norms_sq(A1), np.array(c["bhat"], float),
                         np.array(c["w"], float), c["j1"])
        assert np.allclose(w, c["w_next"], atol=1e-15), c["_cite"]
    for c in g["rgs"]:
        A1 = np.array(c["A1"], float)
        z0 = np.array(c["z"], float)
        z, az, _ = O.rgs_step(A1.T.copy(), ix.column_norms_sq(A1), np.array(c["w"], float),
                              z0, A1 @ z0, c["j2"])
        assert np.allclose(z, c["z_next"], atol=1e-15), c["_cite"]
        assert np.allclose(az, A1 @ z, atol=1e-15)
    for c in g["rcd"]:
        G = np.array(c["G"], float)
        beta0 = np.array(c["beta"], float)
        r0 = np.array(c["bhat"], float) - G @ beta0
        beta, r, _ = O.rcd_step(G, np.diag(G).copy(), beta0, r0, c["j"])
        assert np.allclose(beta, c["beta_next"]) and np.allclose(r, c["r_next"]), c["_cite"]
    for c in g["select"]:
        assert O.scd_select(np.array(c["r"], float), c["tau"]) == c["j"], c["_cite"]


# ---------------------------------------------------------------- P3/P4/P5 direct solves
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_p5_direct_vs_qr_cholesky_vs_library(seed):
    pr = make_dense(40, 15, 20, 0.3, noise=0.1, seed=seed)
    x1 = O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2)
    x2 = O.qr_cholesky_solve(pr.A, pr.b, pr.p)
    M = pr.A.T @ np.diag(np.r_[np.ones(pr.p), -np.ones(pr.q)]) @ pr.A
    x3 = np.linalg.solve(M, pr.A.T @ np.r_[pr.b1, -pr.b2])
    for xa in (x2, x3):
        assert np.linalg.norm(x1 - xa) <= 1e-10 * np.linalg.norm(xa)


def test_p3_q0_is_ordinary_least_squares():
    pr = make_dense(60, 0, 12, 0.3, noise=0.5, seed=3)
    xls = np.linalg.lstsq(pr.A1, pr.b1, rcond=None)[0]          # SVD-based library LS
    assert np.linalg.norm(O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2) - xls) <= 1e-12 * np.linalg.norm(xls)
    rep = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=1, stop=O.STOP_NONE)
    assert np.linalg.norm(rep.x - xls) <= 1e-12 * np.linalg.norm(xls)   # B = 0: exact in one step
    assert O.spectral_radius_sp(pr.A1, pr.A2) == 0.0


def test_p4_consistent_fixed_point_and_convergence():
    pr = make_problem("c0")
    xs = pr.xstar
    assert np.linalg.norm(O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2) - xs) <= 1e-13 * np.linalg.norm(xs)
    c = O.sp_rhs(pr.A1, pr.A2, pr.b1, pr.b2, xs)
    assert np.linalg.norm(np.linalg.solve(pr.A1.T @ pr.A1, c) - xs) <= 1e-13 * np.linalg.norm(xs)
    rep = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, tol=1e-12, x_ref=xs, max_iter=200)
    assert rep.converged and rep.final_metric <= 1e-12


# ---------------------------------------------------------------- P6/P7 SP invariants
def test_p6_spectral_radius_library_and_energy_contraction():
    pr = make_dense(60, 30, 20, 0.3, noise=0.2, seed=5)
    A1, A2 = pr.A1, pr.A2
    rho = O.spectral_radius_sp(A1, A2)
    ev = sla.eigh(A2.T @ A2, A1.T @ A1, eigvals_only=True)   # generalized symmetric eigensolver
    assert abs(rho - ev.max()) <= 1e-12 and rho < 1.0
    xr = O.direct_solve(A1, A2, pr.b1, pr.b2)
    rep = O.sp_solve(A1, A2, pr.b1, pr.b2, max_iter=12, stop=O.STOP_NONE)
    G = A1.T @ A1
    en = [np.sqrt((e @ G @ e)) for e in [np.zeros(20) - xr] + [x - xr for x in rep.x_hist]]
    for k in range(len(en) - 1):
        assert en[k + 1] <= rho * en[k] * (1 + 1e-9) + 1e-14
    # sp_form 1 (correction form) is the same iteration in exact arithmetic (R14)
    rep1 = O.sp_solve(A1, A2, pr.b1, pr.b2, max_iter=12, stop=O.STOP_NONE, sp_form=1)
    assert np.linalg.norm(rep1.x - rep.x) <= 1e-12 * np.linalg.norm(rep.x)


def test_p6_non_spd_gives_rho_ge_one():
    # A1 = I, A2 = 1.2 I: M = -0.44 I is not SPD (condition 1.3 fails), rho = 1.44
    A1 = np.eye(4)
    A2 = 1.2 * np.eye(4)
    assert not O.is_spd(O.normal_matrix(A1, A2))
    assert O.spectral_radius_sp(A1, A2) >= 1.0


def test_p7_gradient_identity():
    pr = make_dense(50, 20, 15, 0.3, noise=0.3, seed=7)
    A1, A2, b1, b2 = pr.A1, pr.A2, pr.b1, pr.b2
    x = np.random.default_rng(0).standard_normal(15)
    c0 = O.sp_rhs(A1, A2, b1, b2, x)
    x1 = np.linalg.solve(A1.T @ A1, c0)
    c1 = O.sp_rhs(A1, A2, b1, b2, x1)
    grad = A1.T @ (A1 @ x1 - b1) - A2.T @ (A2 @ x1 - b2)       # A^T J (A x_{k+1} - b)
    assert np.linalg.norm(grad - (c0 - c1)) <= 1e-11 * np.linalg.norm(c0)


# ---------------------------------------------------------------- RK-RGS (Alg. 2)
def test_p1b_orthogonal_columns_finite_termination():
    """Disjoint column supports: <a_j, w> = bhat_j exactly after the first RK step at j,
    and z_j = <a_j, w>/N_j after each RGS step at j; so z_j = bhat_j/N_j once an RGS
    step at j follows (or shares a step with) the first RK step at j."""
    p, n = 12, 4
    A1 = np.zeros((p, n))
    rng = np.random.default_rng(1)
    for j in range(n):
        A1[3 * j:3 * j + 3, j] = rng.uniform(0.5, 2.0, 3) * (j + 1)
    N = ix.column_norms_sq(A1)
    _, S = ix.weights_prefix(N)
    bhat = rng.standard_normal(n)
    T = 40
    z, steps = O.rk_rgs_inner(A1.T.copy(), N, S, bhat, seed=11, k=0, max_inner=T,
                              check_every=10 ** 9, inner_tol=0.0)
    J1, J2 = ix.rk_rgs_indices(11, 0, 0, T, S)
    for j in range(n):
        rk_first = next((t for t in range(T) if J1[t] == j), None)
        rgs_after = rk_first is not None and any(J2[t] == j for t in range(rk_first, T))
        if rgs_after:
            assert abs(z[j] - bhat[j] / N[j]) <= 1e-14 * abs(bhat[j] / N[j])
        elif not any(J2[t] == j for t in range(T)):
            assert z[j] == 0.0


def test_p8_theorem31_inner_limit_is_sp_iterate():
    pr = make_dense(40, 10, 12, 0.3, seed=9)
    A1 = pr.A1
    N = ix.column_norms_sq(A1)
    _, S = ix.weights_prefix(N)
    bhat = np.random.default_rng(2).standard_normal(12)
    z, steps = O.rk_rgs_inner(A1.T.copy(), N, S, bhat, seed=0, k=0, max_inner=200000,
                              check_every=12, inner_tol=1e-13)
    zstar = sla.solve(A1.T @ A1, bhat, assume_a="pos")
    assert np.linalg.norm(z - zstar) <= 1e-11 * np.linalg.norm(zstar)
    assert steps < 200000


def test_p9_p11_p12_step_identities():
    pr = make_dense(30, 5, 8, 0.3, seed=4)
    A1 = pr.A1
    A1T = A1.T.copy()
    N = ix.column_norms_sq(A1)
    rng = np.random.default_rng(3)
    bhat = rng.standard_normal(8)
    w = A1 @ rng.standard_normal(8)     # w in range(A1)
    z = rng.standard_normal(8)
    for j1, j2 in [(0, 3), (5, 5), (7, 1), (2, 2)]:
        w1, _ = O.rk_step(A1T, N, bhat, w, j1)
        assert abs(A1T[j1] @ w1 - bhat[j1]) <= 1e-12 * (1 + abs(bhat[j1]))        # P11
        z1, az1, _ = O.rgs_step(A1T, N, w1, z, A1 @ z, j2)
        assert abs(A1T[j2] @ (w1 - A1 @ z1)) <= 1e-11 * np.linalg.norm(w1)        # P12
        if j1 == j2:                                                               # P9
            G = A1.T @ A1
            beta, _, _ = O.rcd_step(G, N, z, bhat - G @ z, j1)
            assert np.allclose(z1, beta, rtol=0, atol=1e-12 * (1 + np.abs(beta).max()))
        # range invariant (Thm 3.1 context): w stays in range(A1)
        Q, _ = np.linalg.qr(A1)
        assert np.linalg.norm(w1 - Q @ (Q.T @ w1)) <= 1e-12 * np.linalg.norm(w1)


def test_p14_rk_rgs_expected_rate_median():
    """Thm 3.2 bound: E||z_t - z*||^2_{A1bar} <= q^t ||z*||^2 + t s q^t ||w*||^2,
    q = 1 - smin^2/||A1||_F^2, s = smax^2/||A1||_F^2. Median over seeds, slack 3."""
    pr = make_dense(30, 5, 6, 0.3, seed=12)
    A1 = pr.A1
    N = ix.column_norms_sq(A1)
    _, S = ix.weights_prefix(N)
    bhat = np.random.default_rng(5).standard_normal(6)
    G = A1.T @ A1
    zs = np.linalg.solve(G, bhat)
    wstar = A1 @ zs
    sv = np.linalg.svd(A1, compute_uv=False)
    fro2 = float(np.sum(sv ** 2))
    qf = 1 - sv[-1] ** 2 / fro2
    T = 150
    bound = qf ** T * (zs @ G @ zs) + T * (sv[0] ** 2 / fro2) * qf ** T * (wstar @ wstar)
    errs = []
    for seed in range(40):
        z, _ = O.rk_rgs_inner(A1.T.copy(), N, S, bhat, seed=seed, k=0, max_inner=T,
                              check_every=10 ** 9, inner_tol=0.0)
        e = z - zs
        errs.append(e @ G @ e)
    assert np.median(errs) <= 3 * bound


# ---------------------------------------------------------------- SCD (Alg. 5 / Alg. 3)
def test_p10_scd_energy_identity_and_monotone():
    pr = make_dense(40, 10, 10, 0.3, seed=6)
    A1 = pr.A1
    G = A1.T @ A1
    N = ix.column_norms_sq(A1)
    _, S = ix.weights_prefix(N)
    bhat = np.random.default_rng(4).standard_normal(10)
    bs = np.linalg.solve(G, bhat)
    prev = {"e": bs @ G @ bs}
    seen = []

    def hook(t, j, beta, r):
        e = (beta - bs) @ G @ (beta - bs)
        seen.append((prev["e"], e, j))
        prev["e"] = e

    # record r before the step: identity uses r_t^(j)^2 / A1bar_jj
    rs = []

    def hook2(t, j, beta, r):
        hook(t, j, beta, r)
        rs.append(r.copy())

    O.scd_inner(G, N, S, bhat, seed=3, k=0, max_inner=60, check_every=10 ** 9, inner_tol=0.0,
                step_hook=hook2)
    r_prev = bhat.copy()
    for (e0, e1, j), r_after in zip(seen, rs):
        drop = r_prev[j] ** 2 / G[j, j]
        assert abs((e0 - e1) - drop) <= 1e-9 * max(e0, 1e-300)
        assert e1 <= e0 * (1 + 1e-12)
        r_prev = r_after


def test_p13_alpha_n_is_global_argmax():
    n = 9
    r = np.random.default_rng(8).standard_normal(n)
    for t in range(20):
        alpha, tau = ix.scd_subset(0, 0, t, n, alpha_mode=1, alpha_fixed=n)
        assert alpha == n and list(tau) == list(range(n))
        assert O.scd_select(r, tau) == int(np.argmax(r * r))


def test_p13_p17_exact_sampler_special_cases():
    rng = np.random.default_rng(9)
    n = 6
    B = rng.standard_normal((10, n))
    G = B.T @ B
    r = rng.standard_normal(n)
    d1 = O.scd_exact_select_distribution(G, r, 1)       # alpha=1: A1bar_jj / trace
    for j in range(n):
        assert abs(d1.get(j, 0.0) - G[j, j] / np.trace(G)) <= 1e-14
    dn = O.scd_exact_select_distribution(G, r, n)       # alpha=n: global argmax w.p. 1
    assert dn == {int(np.argmax(r * r)): 1.0}


def test_p17_feistel_subset_matches_exact_uniform_selection():
    """Equal diagonal A1bar: Alg. 3's subset law is uniform (Remark 4.1);
    the selected-index law of Alg. 5 with the Feistel subsets must match it (chi-square)."""
    from scipy.stats import chisquare
    n, alpha = 6, 3
    G = np.eye(n) * 2.0
    r = np.array([0.3, -1.2, 0.7, 2.0, -0.1, 1.5])
    exact = O.scd_exact_select_distribution(G, r, alpha)
    counts = np.zeros(n)
    T = 6000
    for t in range(T):
        _, tau = ix.scd_subset(17, 0, t, n, alpha_mode=1, alpha_fixed=alpha)
        counts[O.scd_select(r, tau)] += 1
    support = [j for j in range(n) if exact.get(j, 0) > 0]
    assert all(counts[j] == 0 for j in range(n) if j not in support)
    f_exp = np.array([exact[j] * T for j in support])
    assert chisquare(counts[support], f_exp).pvalue > 1e-3


# ---------------------------------------------------------------- index stream (P15/P16)
def test_p15_philox_known_answers():
    g = _load("philox_kat.json")
    for v in g["vectors"]:
        out = ix.philox4x32_10(np.array([int(h, 16) for h in v["ctr"]]),
                               [int(h, 16) for h in v["key"]])
        assert [int(o) for o in out] == [int(h, 16) for h in v["out"]]


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_p15_philox_matches_curand_host(tmp_path):
    """The CUDA toolkit's curand_Philox4x32_10 (library routine) compiled for the host."""
    src = tmp_path / "ph.cu"
    src.write_text(r'''
#include <cstdio>
#include <vector_types.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
int main(){ unsigned s=1u;
  for(int i=0;i<64;i++){ uint4 c; uint2 k;
    s=s*1664525u+1013904223u; c.x=s; s=s*1664525u+1013904223u; c.y=s;
    s=s*1664525u+1013904223u; c.z=s; s=s*1664525u+1013904223u; c.w=s;
    s=s*1664525u+1013904223u; k.x=s; s=s*1664525u+1013904223u; k.y=s;
    uint4 r=curand_Philox4x32_10(c,k);
    printf("%u %u %u %u %u %u %u %u %u %u\n",c.x,c.y,c.z,c.w,k.x,k.y,r.x,r.y,r.z,r.w);} }
''')
    exe = tmp_path / "ph"
    subprocess.run(["nvcc", "-Wno-deprecated-gpu-targets", "-o", str(exe), str(src)], check=True,
                   capture_output=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    for line in out.strip().splitlines():
        v = [int(s) for s in line.split()]
        got = ix.philox4x32_10(np.array(v[:4]), v[4:6])
        assert [int(o) for o in got] == v[6:]


def test_p16_weighted_sampler_definition_and_chisquare():
    from scipy.stats import chisquare
    N = np.array([1.0, 2.0, 3.0, 4.0])
    W, S = ix.weights_prefix(N)
    assert W[-1] == 2 ** 32 and W[0] == 2 ** 30
    rng = np.random.default_rng(0)
    for _ in range(2000):                                  # brute-force definition check
        U = int(rng.integers(0, 2 ** 63)) * 2 + int(rng.integers(0, 2))
        j = ix.sample_weighted(U, S)
        v = (U * S[-1]) >> 64
        assert S[j] > v and (j == 0 or S[j - 1] <= v)
    J1, J2 = ix.rk_rgs_indices(0, 0, 0, 20000, S)
    exp = np.array(W, float) / S[-1]
    for J in (J1, J2):
        assert chisquare(np.bincount(J, minlength=4), exp * len(J)).pvalue > 1e-3


def test_p16_column_norms_and_weights():
    A = np.random.default_rng(1).standard_normal((300, 7))
    N = ix.column_norms_sq(A)
    assert np.allclose(N, np.sum(A * A, axis=0), rtol=1e-13, atol=0)
    with pytest.raises(ValueError):
        ix.weights_prefix(np.array([1.0, 0.0]))


@pytest.mark.parametrize("n", [1, 2, 3, 5, 50, 1000, 1024, 4000, 20000])
def test_p16_feistel_is_a_permutation(n):
    _, keys = ix.scd_alpha_keys(5, 3, 7, max(n, 1))
    perm = ix.feistel_forward(np.arange(n, dtype=np.uint64), keys, n)
    assert sorted(perm.tolist()) == list(range(n))


def test_p16_alpha_uniform_and_subset_uniform():
    from scipy.stats import chisquare
    n = 5
    alphas = [ix.scd_alpha_keys(1, 0, t, n)[0] for t in range(5000)]
    assert chisquare(np.bincount(alphas, minlength=n + 1)[1:]).pvalue > 1e-3
    from itertools import combinations
    pairs = {c: i for i, c in enumerate(combinations(range(n), 2))}
    cnt = np.zeros(len(pairs))
    for t in range(20000):
        _, tau = ix.scd_subset(2, 1, t, n, alpha_mode=1, alpha_fixed=2)
        cnt[pairs[tuple(int(v) for v in tau)]] += 1
    assert chisquare(cnt).pvalue > 1e-3


# ---------------------------------------------------------------- whole-method convergence
def test_methods_converge_on_c0():
    pr = make_problem("c0")
    args = (pr.A1, pr.A2, pr.b1, pr.b2)
    for solve in (O.sp_solve, O.sp_rk_rgs_solve):
        kw = {} if solve is O.sp_solve else dict(inner_tol=1e-12, max_inner=100000)
        rep = solve(*args, tol=1e-10, x_ref=pr.xstar, **kw)
        assert rep.converged and rep.final_metric <= 1e-10
    rep = O.sp_scd_solve(*args, tol=1e-10, x_ref=pr.xstar, inner_tol=1e-12, max_inner=100000,
                         max_iter=3, stop=O.STOP_NONE)
    # three outer steps of SCD equal three exact SP steps up to the inner tolerance
    sp = O.sp_solve(*args, max_iter=3, stop=O.STOP_NONE)
    assert np.linalg.norm(rep.x - sp.x) <= 1e-9 * np.linalg.norm(sp.x)
    assert O.spectral_radius_sp(pr.A1, pr.A2) < 1.0 and O.is_spd(O.normal_matrix(pr.A1, pr.A2))


def test_paper_literal_forms_match_the_pinned_forms():
    """Alg. 1 literal (explicit B = P A2bar, c = P A^T J b; sp_form 2) and the precomputed-A2bar
    right-hand side of Alg. 2 / Alg. 5 equal the pinned streaming forms (the same iteration in
    exact arithmetic, PAPER.md:126 vs :134-139; P1 closed form on the 2x2 example)."""
    g = _load("sp_2x2.json")
    A1, A2, b1, b2 = _np(g, "A1"), _np(g, "A2"), _np(g, "b1"), _np(g, "b2")
    rep = O.sp_solve(A1, A2, b1, b2, max_iter=4, stop=O.STOP_NONE, sp_form=2)
    for k, xk in enumerate(_np(g, "sp_iterates")):
        assert np.allclose(rep.x_hist[k], xk, atol=1e-15), k
    pr = make_dense(150, 40, 30, 0.3, noise=0.1, seed=2)
    args = (pr.A1, pr.A2, pr.b1, pr.b2)
    r0 = O.sp_solve(*args, max_iter=5, stop=O.STOP_NONE)
    r2 = O.sp_solve(*args, max_iter=5, stop=O.STOP_NONE, sp_form=2)
    for a, b in zip(r2.x_hist, r0.x_hist):
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
    for fn, kw in ((O.sp_rk_rgs_solve, dict(max_inner=300)), (O.sp_scd_solve, dict(max_inner=300))):
        ra = fn(*args, max_iter=3, stop=O.STOP_NONE, inner_tol=0.0, check_every=50, **kw)
        rb = fn(*args, max_iter=3, stop=O.STOP_NONE, inner_tol=0.0, check_every=50, rhs_literal=True, **kw)
        assert np.linalg.norm(ra.x - rb.x) <= 1e-10 * np.linalg.norm(ra.x)


def test_sparse_inputs_match_the_pinned_dense_oracle():
    """The oracle on scipy.sparse CSR inputs (configs[3]) equals the pinned dense oracle on the
    same matrix: only the storage differs (PAPER.md:43-46 direct solve, Alg. 1 SP iterates)."""
    from workloads import make_sparse
    pr = make_sparse(400, 80, 30, 5, seed=3)
    S = pr.scipy()
    A = pr.dense()
    sp_args = (S[:pr.p], S[pr.p:], pr.b[:pr.p], pr.b[pr.p:])
    de_args = (A[:pr.p], A[pr.p:], pr.b[:pr.p], pr.b[pr.p:])
    xs, xd = O.direct_solve(*sp_args), O.direct_solve(*de_args)
    assert np.linalg.norm(xs - xd) <= 1e-12 * np.linalg.norm(xd)
    rs = O.sp_solve(*sp_args, max_iter=4, stop=O.STOP_NONE)
    rd = O.sp_solve(*de_args, max_iter=4, stop=O.STOP_NONE)
    for a, b in zip(rs.x_hist, rd.x_hist):
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
    assert abs(O.relative_residual(*sp_args, xs) - O.relative_residual(*de_args, xd)) <= 1e-20
    # the generator's CSR layout: sorted distinct columns, row_ptr consistent
    assert np.all(np.diff(pr.row_ptr) == 5)
    assert all(np.all(np.diff(pr.col_idx[pr.row_ptr[i]:pr.row_ptr[i + 1]]) > 0) for i in range(pr.m))


@pytest.mark.parametrize("shape", [(400, 80, 30, 5), (3000, 200, 12, 2), (150, 40, 60, 7)])
def test_sparse_column_path_matches_the_pinned_dense_oracle(shape):
    """P18b: the oracle's column-wise CSC path (rk_rgs_inner_sparse, scd_inner_sparse,
    column_norms_sq_csc -- what it runs on configs[3] at full size) equals the pinned dense path on
    the densified matrix: column norms bit for bit, identical inner counts (stop decisions) and
    iterates to rounding, for SP-RK-RGS, SP-SCD (uniform alpha, Motzkin) and weighted SP-RCD.
    Shape (3000, 200, 12, 2) gives ~500 stored entries per column."""
    from workloads import make_sparse
    p, q, n, k = shape
    pr = make_sparse(p, q, n, k, seed=31)
    S = pr.scipy()
    A = pr.dense()
    A1c = S[:p].tocsc()
    A1c.sort_indices()
    Nd = ix.column_norms_sq(A[:p])
    Ns = ix.column_norms_sq_csc(A1c.indptr, A1c.data, n)
    assert np.array_equal(Nd.view(np.uint64), Ns.view(np.uint64))
    sp_args = (S[:p], S[p:], pr.b[:p], pr.b[p:])
    de_args = (A[:p], A[p:], pr.b[:p], pr.b[p:])
    kw = dict(max_iter=3, stop=O.STOP_NONE, seed=4, max_inner=700, check_every=50, inner_tol=1e-7)
    cases = [(O.sp_rk_rgs_solve, {}), (O.sp_scd_solve, {}), (O.sp_scd_solve, dict(alpha_mode=1, alpha_fixed=n)),
             (O.sp_scd_solve, dict(weighted=True))]
    for fn, extra in cases:
        rs = fn(*sp_args, **kw, **extra)
        rd = fn(*de_args, **kw, **extra)
        assert rs.inner_hist == rd.inner_hist, (fn.__name__, extra)
        for a, b in zip(rs.x_hist, rd.x_hist):
            assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b), (fn.__name__, extra)


# ---------------------------------------------------------------- P19 the paper's own families
def test_p19_paper_family_structure():
    """§5.2 / §5.3 generator: A1, b in [0,1), A2 = 7*eye(q,n)."""
    pr = make_paper(400, 30, 30, seed=3)
    assert np.array_equal(pr.A2, 7.0 * np.eye(30))
    assert pr.A1.min() >= 0.0 and pr.A1.max() < 1.0 and pr.b.min() >= 0.0 and pr.b.max() < 1.0
    assert abs(pr.A1.mean() - 0.5) < 0.01 and abs(pr.A1.var() - 1.0 / 12.0) < 0.005
    mk = make_paper(300, 1, 40, seed=4)
    assert mk.q == 1 and np.array_equal(mk.A2[0], 7.0 * np.eye(1, 40)[0])
    with pytest.raises(ValueError):
        make_paper(10, 5, 4)
    assert [len(v) for v in PAPER_TABLES.values()] == [3, 3, 3, 3]
    assert PAPER_TABLES["t2"][0] == (30000, 13000, 13000) and PAPER_TABLES["t5"][2] == (60000, 1, 15000)


def test_p19_song_family_spectral_radius_closed_form():
    """q = n, A2 = 7I: B = (A1^T A1)^{-1} A2^T A2 = 49 (A1^T A1)^{-1}, so rho(B) = 49 / lambda_min(A1^T A1)
    (Theorem 2.1); SP converges iff lambda_min > 49 (condition Sec13)."""
    pr = make_paper(2500, 60, 60, seed=5)
    lam = np.linalg.eigvalsh(pr.A1.T @ pr.A1).min()
    rho = O.spectral_radius_sp(pr.A1, pr.A2)
    assert abs(rho - 49.0 / lam) <= 1e-12 * max(rho, 1.0)
    assert rho < 1.0 and O.is_spd(O.normal_matrix(pr.A1, pr.A2))
    rep = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=200, stop=O.STOP_NONE)
    xs = O.direct_solve(pr.A1, pr.A2, pr.b1, pr.b2)
    G = pr.A1.T @ pr.A1
    errs = [np.sqrt((x - xs) @ G @ (x - xs)) for x in rep.x_hist[:6]]
    for k in range(5):   # energy-norm contraction by rho per outer step (Theorem 2.1)
        assert errs[k + 1] <= rho * errs[k] * (1 + 1e-9) + 1e-13


def test_p19_minkowski_sherman_morrison():
    """Minkowski space q = 1: A^T J A = A1^T A1 - 49 e1 e1^T, a rank-one
    downdate. rho(B) = 49 [(A1^T A1)^{-1}]_11 and the SP / SP-RK-RGS limit equals the
    Sherman-Morrison solution built from solves with A1^T A1 only."""
    pr = make_paper(2000, 1, 30, seed=6)
    G = pr.A1.T @ pr.A1
    e = np.zeros(30)
    e[0] = 1.0
    Gi_e = np.linalg.solve(G, e)
    assert abs(O.spectral_radius_sp(pr.A1, pr.A2) - 49.0 * Gi_e[0]) <= 1e-12
    rhs = pr.A1.T @ pr.b1 - 7.0 * pr.b2[0] * e
    y = np.linalg.solve(G, rhs)
    x_sm = y + 49.0 * Gi_e * y[0] / (1.0 - 49.0 * Gi_e[0])
    for rep in (O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, tol=1e-14, stop=O.STOP_RR, max_iter=500),
                O.sp_rk_rgs_solve(pr.A1, pr.A2, pr.b1, pr.b2, tol=1e-14, stop=O.STOP_RR, max_iter=500, seed=1,
                                  max_inner=200000, inner_tol=1e-10)):
        assert rep.converged
        # ||x - x*|| <= ||M^{-1}||_2 ||A^T J (b - A x)||_2 with M = A^T J A = G - 49 e1 e1^T
        g = pr.A1.T @ (pr.b1 - pr.A1 @ rep.x) - pr.A2.T @ (pr.b2 - pr.A2 @ rep.x)
        bound = np.linalg.norm(g) / np.linalg.eigvalsh(G - 49.0 * np.outer(e, e)).min()
        assert np.linalg.norm(rep.x - x_sm) <= bound * (1 + 1e-6) + 1e-14
        assert np.linalg.norm(rep.x - x_sm) <= 1e-4 * np.linalg.norm(x_sm)


def test_oracle_not_imported_by_product():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2203_15340_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_p16b_exact_subsets_are_uniform_and_match_alg3():
    """SURVEY.md §8 f3 (include/ils.h ILS_SUBSET_EXACT): the key-selection subsets are exactly uniform
    -- every size-alpha subset equally likely (chi-square over all C(5,2) pairs) -- and the selected
    index of Alg. 5 step 9 then follows the exact Alg. 3 step-10 law (Eq. Sec4.111)
    reweighted to uniform subsets; key ties are broken by index (u, s) lexicographically."""
    from itertools import combinations
    from scipy.stats import chisquare
    n = 5
    pairs = {c: i for i, c in enumerate(combinations(range(n), 2))}
    cnt = np.zeros(len(pairs))
    for t in range(12000):
        _, tau = ix.scd_subset(2, 1, t, n, alpha_mode=1 | ix.SUBSET_EXACT, alpha_fixed=2)
        cnt[pairs[tuple(int(v) for v in tau)]] += 1
    assert chisquare(cnt).pvalue > 1e-3
    # alpha_t policy unchanged by the flag
    a0 = [ix.scd_subset(1, 0, t, 9, alpha_mode=0)[0] for t in range(50)]
    a1 = [ix.scd_subset(1, 0, t, 9, alpha_mode=ix.SUBSET_EXACT)[0] for t in range(50)]
    assert a0 == a1
    # the selected index: argmax of r^2 over a uniform 3-subset of 6 -> P(j = the i-th largest) =
    # C(6-1-i, 2) / C(6, 3) (the subset contains j and two of the smaller ones)
    r = np.array([0.3, -2.0, 1.1, 0.7, -1.5, 0.1])
    order = np.argsort(-r * r)
    exp = np.array([sum(1 for c in combinations(range(6), 3) if order[min(order.tolist().index(s) for s in c)] == j)
                    for j in range(6)], dtype=float)
    got = np.zeros(6)
    for t in range(6000):
        _, tau = ix.scd_subset(5, 2, t, 6, alpha_mode=1 | ix.SUBSET_EXACT, alpha_fixed=3)
        got[O.scd_select(r, tau)] += 1
    sup = exp > 0
    assert np.all(got[~sup] == 0)
    assert chisquare(got[sup], exp[sup] / exp.sum() * got.sum()).pvalue > 1e-3
