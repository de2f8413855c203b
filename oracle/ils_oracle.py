"""ORACLE -- test infrastructure, NOT the product.

A plain, slow, fp64 CPU implementation of what the hot path computes, written
from PAPER.md (arXiv 2203.15340, Zhang & Li) in the paper's order and notation.
Each function cites the passage it follows ("PAPER.md:L" = line L of the LaTeX).
Library primitives (matmul, Cholesky, triangular solve, eigvalsh, QR) serve as
single steps; there is no blocking, fusion or reordering beyond the algorithm.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module. It shares no code with the CUDA path
(paper_2203_15340_b200/); the only shared module is workloads/ (input data).

Parity pins: see tests/test_oracle_pins.py and DESIGN.md "Oracle pins".
Functions with no independent pin are marked "parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

from . import index_stream as ix

# ----------------------------------------------------------------------------
# Problem-level definitions (§1)
# ----------------------------------------------------------------------------


def _dense(M) -> np.ndarray:
    """A scipy.sparse result (sparse CSR inputs, config c3) as a dense ndarray; identity otherwise.
    Densifying changes no value: it only lets a dense library routine (Cholesky) take the step."""
    return M.toarray() if hasattr(M, "toarray") else np.asarray(M)


def apply_J(p: int, v: np.ndarray) -> np.ndarray:
    """J v with J = diag(I_p, -I_q)."""
    w = np.array(v, dtype=np.float64, copy=True)
    w[p:] = -w[p:]
    return w


def normal_matrix(A1: np.ndarray, A2: np.ndarray) -> np.ndarray:
    """M = A^T J A = A1^T A1 - A2^T A2, symmetrised (M + M^T)/2."""
    M = _dense(A1.T @ A1 - A2.T @ A2)
    return 0.5 * (M + M.T)


def ajb(A1, A2, b1, b2) -> np.ndarray:
    """A^T J b = A1^T b1 - A2^T b2 (right side of the normal equation Sec12)."""
    return A1.T @ b1 - A2.T @ b2


def is_spd(M: np.ndarray) -> bool:
    """Condition (1.3): Cholesky succeeds with positive pivots."""
    try:
        np.linalg.cholesky(M)
        return True
    except np.linalg.LinAlgError:
        return False


def direct_solve(A1, A2, b1, b2) -> np.ndarray:
    """x_ref: solve the normal equation A^T J A x = A^T J b (Eq. Sec12)
    by Cholesky of M = A1^T A1 - A2^T A2 and two triangular solves."""
    M = normal_matrix(A1, A2)
    L = np.linalg.cholesky(M)
    y = sla.solve_triangular(L, ajb(A1, A2, b1, b2), lower=True)
    return sla.solve_triangular(L.T, y, lower=False)


def qr_cholesky_solve(A: np.ndarray, b: np.ndarray, p: int) -> np.ndarray:
    """QR-Cholesky method: A = QR, solve (Q^T J Q) y = Q^T J b by
    Cholesky, x = R^{-1} y."""
    Q, R = np.linalg.qr(A, mode="reduced")
    JQ = apply_J(p, Q)
    K = Q.T @ JQ
    K = 0.5 * (K + K.T)
    L = np.linalg.cholesky(K)
    rhs = Q.T @ apply_J(p, b)
    y = sla.solve_triangular(L.T, sla.solve_triangular(L, rhs, lower=True), lower=False)
    return sla.solve_triangular(R, y, lower=False)


def relative_residual(A1, A2, b1, b2, x) -> float:
    """RR = ||A^T J (A x - b)||_2^2 / ||A^T J b||_2^2 (§5; squared ratio)."""
    num = A1.T @ (A1 @ x - b1) - A2.T @ (A2 @ x - b2)
    den = ajb(A1, A2, b1, b2)
    dd = float(den @ den)
    if dd == 0.0:
        raise ValueError("A^T J b = 0: RR undefined")
    return float(num @ num) / dd


def sp_rhs(A1, A2, b1, b2, x) -> np.ndarray:
    """b_hat = A2^T A2 x_k + A^T J b (Alg. 2 step 5; Eq. Sec3.41), evaluated as
    c_k = A1^T b1 + A2^T (A2 x_k - b2) -- the same vector, one pass over A2."""
    return A1.T @ b1 + A2.T @ (A2 @ x - b2)


def sp_rhs_literal(A2bar, AJb, x) -> np.ndarray:
    """b_hat = A2bar x_k + A^T J b with the precomputed A2bar = A2^T A2 (Alg. 2 steps 2, 3, 5,
    PAPER.md:291-294; Alg. 5 steps 2, 4) -- the paper's literal layout."""
    return A2bar @ x + AJb


def spectral_radius_sp(A1, A2) -> float:
    """rho((A1^T A1)^{-1} A2^T A2) (Theorem 2.1) as
    lambda_max(L^{-1} A2bar L^{-T}) with A1bar = L L^T (a similarity transform)."""
    L = np.linalg.cholesky(A1.T @ A1)
    Li_A2 = sla.solve_triangular(L, A2.T, lower=True)        # L^{-1} A2^T
    K = Li_A2 @ Li_A2.T
    ev = np.linalg.eigvalsh(0.5 * (K + K.T))
    return float(np.max(np.abs(ev))) if ev.size else 0.0


# ----------------------------------------------------------------------------
# Reports and stopping (§5 protocol; BASELINE.json XREF rule)
# ----------------------------------------------------------------------------

STOP_XREF, STOP_RR, STOP_NONE = 0, 1, 2


@dataclass
class Report:
    x: np.ndarray
    outer_iters: int = 0
    inner_iters_total: int = 0
    converged: bool = False
    final_metric: float = float("nan")
    inner_hist: list = field(default_factory=list)
    x_hist: list = field(default_factory=list)


def _outer_stop(stop, x, x_ref, tol, A1, A2, b1, b2):
    """Returns (stop?, metric). XREF: ||x - x_ref|| <= tol ||x_ref|| (BASELINE.json);
    RR: RR(x) < tol; NONE: never (fixed-horizon parity)."""
    if stop == STOP_XREF:
        m = float(np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
        return m <= tol, m
    if stop == STOP_RR:
        m = relative_residual(A1, A2, b1, b2, x)
        return m < tol, m
    return False, float("nan")


# ----------------------------------------------------------------------------
# Alg. 1 -- SP
# ----------------------------------------------------------------------------


def sp_solve(A1, A2, b1, b2, x0=None, tol=1e-8, max_iter=20000, stop=STOP_XREF,
             x_ref=None, sp_form=0) -> Report:
    """SP method, Alg. 1: x_{k+1} = (A1^T A1)^{-1} A2^T A2 x_k + (A1^T A1)^{-1} A^T J b
    (Eq. Sec23). P = (A1^T A1)^{-1} is applied by Cholesky solves
    (SPEC reading, R12). sp_form 0: x_{k+1} = P c_k with c_k = sp_rhs(x_k);
    sp_form 1 (correction form, identical in exact arithmetic): x_{k+1} = x_k + P A^T J (b - A x_k);
    sp_form 2 (Alg. 1 literal): B = P A2bar and c = P A^T J b formed explicitly
    (P applied to the columns of A2bar by Cholesky solves), x_{k+1} = B x_k + c."""
    n = A1.shape[1]
    L = np.linalg.cholesky(_dense(A1.T @ A1))

    def apply_P(v):
        return sla.solve_triangular(L.T, sla.solve_triangular(L, v, lower=True), lower=False)

    if sp_form == 2:
        B = apply_P(_dense(A2.T @ A2))          # Alg. 1 step 3: B = (A1^T A1)^{-1} A2^T A2
        c = apply_P(ajb(A1, A2, b1, b2))        # Alg. 1 step 4: c = (A1^T A1)^{-1} A^T J b

    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    rep = Report(x=x)
    for k in range(max_iter):
        if sp_form == 0:
            x = apply_P(sp_rhs(A1, A2, b1, b2, x))
        elif sp_form == 2:
            x = B @ x + c                        # Alg. 1 step 6
        else:
            g = A1.T @ (b1 - A1 @ x) - A2.T @ (b2 - A2 @ x)
            x = x + apply_P(g)
        rep.outer_iters = k + 1
        rep.x_hist.append(x.copy())
        done, rep.final_metric = _outer_stop(stop, x, x_ref, tol, A1, A2, b1, b2)
        if done:
            rep.converged = True
            break
    rep.x = x
    return rep


# ----------------------------------------------------------------------------
# Alg. 2 -- SP-RK-RGS
# ----------------------------------------------------------------------------


def rk_step(A1T, N, bhat, w, j1):
    """Alg. 2 step 9: w_{t+1} = w_t + (bhat_j1 - A1_(j1)^T w_t)/||A1_(j1)||^2 A1_(j1).
    A1T[j] is column j of A1. Returns (w_{t+1}, s1)."""
    s1 = (bhat[j1] - A1T[j1] @ w) / N[j1]
    return w + s1 * A1T[j1], s1


def rgs_step(A1T, N, w, z, az, j2):
    """Alg. 2 step 11: z_{t+1} = z_t + A1_(j2)^T (w_{t+1} - A1 z_t)/||A1_(j2)||^2 e_j2.
    az = A1 z_t is maintained incrementally (SPEC reading R21). Returns (z, az, s2)."""
    s2 = (A1T[j2] @ (w - az)) / N[j2]
    z = z.copy()
    z[j2] += s2
    return z, az + s2 * A1T[j2], s2


def rk_rgs_inner(A1T, N, S, bhat, seed, k, max_inner, check_every, inner_tol,
                 step_hook=None):
    """Inner loop of Alg. 2 for outer iteration k.

    z_0 = w_0 = 0 (step 6). For t = 0,1,...: (j1, j2) from the index stream
    (steps 8, 10); RK step on A1^T w = bhat (step 9); RGS step on A1 z = w (step 11).
    "until convergence" (step 7, silent -- reading R2): after every check_every steps
    g = A1^T (A1 z) - bhat, stop if ||g|| <= inner_tol ||bhat||. The check reads z only: the
    incrementally maintained A1 z (reading R21) is never recomputed, as in Alg. 2 itself.
    Stops at max_inner steps. Returns (z, steps)."""
    p, n = A1T.shape[1], A1T.shape[0]
    w = np.zeros(p)
    z = np.zeros(n)
    az = np.zeros(p)
    nb = float(np.linalg.norm(bhat))
    if nb == 0.0:
        return z, 0
    t = 0
    CH = 4096
    while t < max_inner:
        cnt = min(CH, max_inner - t)
        J1, J2 = ix.rk_rgs_indices(seed, k, t, cnt, S)
        for c in range(cnt):
            j1, j2 = int(J1[c]), int(J2[c])
            w, s1 = rk_step(A1T, N, bhat, w, j1)
            z, az, s2 = rgs_step(A1T, N, w, z, az, j2)
            t += 1
            if step_hook is not None:
                step_hook(t, j1, j2, w, z, az)
            if t % check_every == 0:
                g = A1T @ (A1T.T @ z) - bhat
                if float(np.linalg.norm(g)) <= inner_tol * nb:
                    return z, t
    return z, t


def _issparse(M) -> bool:
    return hasattr(M, "tocsc")


def _csc_sorted(M):
    """A scipy.sparse matrix in CSC with ascending row indices in every column (canonical)."""
    C = M.tocsc(copy=True)
    C.sort_indices()
    return C


def rk_rgs_inner_sparse(A1c, N, S, bhat, seed, k, max_inner, check_every, inner_tol):
    """rk_rgs_inner (Alg. 2 steps 6-12) for A1 stored by columns (scipy CSC,
    configs[3]): the same steps in the same order, each column A1_(j) touched only on its stored
    rows. The dense step's remaining entries are exact zeros, which add nothing to the dots and
    leave w_i and (A1 z)_i unchanged, so this is the dense loop with the zero terms skipped
    (pinned against rk_rgs_inner in tests/test_oracle_pins.py). Returns (z, steps)."""
    p, n = A1c.shape
    ip, ri, va = A1c.indptr, A1c.indices, A1c.data
    w = np.zeros(p)
    z = np.zeros(n)
    az = np.zeros(p)
    nb = float(np.linalg.norm(bhat))
    if nb == 0.0:
        return z, 0
    t = 0
    CH = 4096
    while t < max_inner:
        cnt = min(CH, max_inner - t)
        J1, J2 = ix.rk_rgs_indices(seed, k, t, cnt, S)
        for c in range(cnt):
            j1, j2 = int(J1[c]), int(J2[c])
            r1, v1 = ri[ip[j1]:ip[j1 + 1]], va[ip[j1]:ip[j1 + 1]]
            s1 = (bhat[j1] - v1 @ w[r1]) / N[j1]           # step 9 (RK on A1^T w = b_hat)
            w[r1] += s1 * v1
            r2, v2 = ri[ip[j2]:ip[j2 + 1]], va[ip[j2]:ip[j2 + 1]]
            s2 = (v2 @ (w[r2] - az[r2])) / N[j2]          # step 11 (RGS on A1 z = w)
            z[j2] += s2
            az[r2] += s2 * v2
            t += 1
            if t % check_every == 0:                      # reading R2 (no recomputation of A1 z)
                g = A1c.T @ (A1c @ z) - bhat
                if float(np.linalg.norm(g)) <= inner_tol * nb:
                    return z, t
    return z, t


def sp_rk_rgs_solve(A1, A2, b1, b2, x0=None, tol=1e-8, max_iter=20000, stop=STOP_XREF,
                    x_ref=None, seed=0, max_inner=100000, check_every=None,
                    inner_tol=1e-12, rhs_literal=False) -> Report:
    """SP-RK-RGS, Alg. 2: outer b_hat = A2bar x_k + A^T J b (step 5),
    inner RK-RGS (steps 6-12), x_{k+1} = z (step 13)."""
    n = A1.shape[1]
    if _issparse(A1):   # CSR/CSC input (configs[3]): the column-wise path, same steps
        A1c = _csc_sorted(A1)
        N = ix.column_norms_sq_csc(A1c.indptr, A1c.data, n)
    else:
        A1T = np.ascontiguousarray(A1.T)
        N = ix.column_norms_sq(A1)
    _, S = ix.weights_prefix(N)
    ce = n if check_every is None else check_every
    if rhs_literal:   # Alg. 2 steps 2-3
        A2bar, AJb = _dense(A2.T @ A2), ajb(A1, A2, b1, b2)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    rep = Report(x=x)
    for k in range(max_iter):
        bhat = sp_rhs_literal(A2bar, AJb, x) if rhs_literal else sp_rhs(A1, A2, b1, b2, x)
        if _issparse(A1):
            x, steps = rk_rgs_inner_sparse(A1c, N, S, bhat, seed, k, max_inner, ce, inner_tol)
        else:
            x, steps = rk_rgs_inner(A1T, N, S, bhat, seed, k, max_inner, ce, inner_tol)
        rep.inner_iters_total += steps
        rep.inner_hist.append(steps)
        rep.outer_iters = k + 1
        rep.x_hist.append(x.copy())
        done, rep.final_metric = _outer_stop(stop, x, x_ref, tol, A1, A2, b1, b2)
        if done:
            rep.converged = True
            break
    rep.x = x
    return rep


# ----------------------------------------------------------------------------
# Alg. 5 -- practical SP-SCD and SP-RCD
# ----------------------------------------------------------------------------


def rcd_step(G, N, beta, r, j):
    """Alg. 5 steps 10-11 (garble r_k read as r_t, reading R11):
    s = r_j / A1bar_jj; beta_j += s; r -= s A1bar_(j). A1bar_jj = ||A1_(j)||^2 = N_j
    (reading R13). Returns (beta, r, s)."""
    s = r[j] / N[j]
    beta = beta.copy()
    beta[j] += s
    return beta, r - s * G[j], s


def scd_select(r, tau) -> int:
    """Alg. 5 step 9: j_t = argmax_{s in tau} |r^(s)|^2, ties to the smallest s
    (reading R10). tau must be sorted ascending."""
    tau = np.asarray(tau)
    vals = r[tau] * r[tau]
    return int(tau[int(np.argmax(vals))])


def scd_inner(G, N, S, bhat, seed, k, max_inner, check_every, inner_tol,
              alpha_mode=0, alpha_fixed=1, weighted=False, step_hook=None):
    """Inner loop of Alg. 5: beta_0 = 0, r_0 = bhat (step 5);
    per step alpha_t (step 7), tau_t (step 8), j_t = argmax (step 9), RCD update (10-11).
    weighted=True: SP-RCD, j from the column-norm distribution (alpha = 1, Remark 4.1).
    Stop rule (reading R2): every check_every steps r = bhat - G beta recomputed,
    stop if ||r|| <= inner_tol ||bhat||. Returns (beta, steps)."""
    n = G.shape[0]
    beta = np.zeros(n)
    r = bhat.copy()
    nb = float(np.linalg.norm(bhat))
    if nb == 0.0:
        return beta, 0
    t = 0
    while t < max_inner:
        if weighted:
            j = int(ix.rcd_indices(seed, k, t, 1, S)[0])
        else:
            _, tau = ix.scd_subset(seed, k, t, n, alpha_mode, alpha_fixed)
            j = scd_select(r, tau)
        beta, r, s = rcd_step(G, N, beta, r, j)
        t += 1
        if step_hook is not None:
            step_hook(t, j, beta, r)
        if t % check_every == 0:
            r = bhat - G @ beta
            if float(np.linalg.norm(r)) <= inner_tol * nb:
                return beta, t
    return beta, t


def scd_inner_sparse(Gc, N, S, bhat, seed, k, max_inner, check_every, inner_tol,
                     alpha_mode=0, alpha_fixed=1, weighted=False):
    """scd_inner (Alg. 5 steps 5-11) with A1bar = A1^T A1 stored sparse (scipy
    CSR, configs[3]): step 11's update r -= s A1bar_(j) touches only the stored entries of row j;
    the skipped entries are exact zeros (r_i - s*0 = r_i). Pinned against scd_inner in
    tests/test_oracle_pins.py. Returns (beta, steps)."""
    n = Gc.shape[0]
    ip, ci, va = Gc.indptr, Gc.indices, Gc.data
    beta = np.zeros(n)
    r = bhat.copy()
    nb = float(np.linalg.norm(bhat))
    if nb == 0.0:
        return beta, 0
    t = 0
    while t < max_inner:
        if weighted:
            j = int(ix.rcd_indices(seed, k, t, 1, S)[0])
        else:
            _, tau = ix.scd_subset(seed, k, t, n, alpha_mode, alpha_fixed)
            j = scd_select(r, tau)
        s = r[j] / N[j]                                   # step 10 (A1bar_jj = N_j, R13)
        beta[j] += s
        cols = ci[ip[j]:ip[j + 1]]
        r[cols] -= s * va[ip[j]:ip[j + 1]]                # step 11
        t += 1
        if t % check_every == 0:
            r = bhat - Gc @ beta
            if float(np.linalg.norm(r)) <= inner_tol * nb:
                return beta, t
    return beta, t


def sp_scd_solve(A1, A2, b1, b2, x0=None, tol=1e-8, max_iter=20000, stop=STOP_XREF,
                 x_ref=None, seed=0, max_inner=100000, check_every=None, inner_tol=1e-12,
                 alpha_mode=0, alpha_fixed=1, weighted=False, rhs_literal=False) -> Report:
    """SP-SCD, Alg. 5. A1bar = A1^T A1 formed once (step 2); the outer
    right side b_hat = A2bar x_k + A^T J b (step 4) is formed as sp_rhs(x_k)."""
    n = A1.shape[1]
    sparse = _issparse(A1)
    if sparse:   # CSR/CSC input (configs[3]): A1bar kept sparse, same steps
        A1c = _csc_sorted(A1)
        G = (A1c.T @ A1c).tocsr()
        G.sort_indices()
        N = ix.column_norms_sq_csc(A1c.indptr, A1c.data, n)
    else:
        G = A1.T @ A1
        N = ix.column_norms_sq(A1)
    _, S = ix.weights_prefix(N)
    ce = n if check_every is None else check_every
    if rhs_literal:   # Alg. 5 step 2
        A2bar, AJb = _dense(A2.T @ A2), ajb(A1, A2, b1, b2)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    rep = Report(x=x)
    for k in range(max_iter):
        bhat = sp_rhs_literal(A2bar, AJb, x) if rhs_literal else sp_rhs(A1, A2, b1, b2, x)
        inner = scd_inner_sparse if sparse else scd_inner
        x, steps = inner(G, N, S, bhat, seed, k, max_inner, ce, inner_tol, alpha_mode, alpha_fixed, weighted)
        rep.inner_iters_total += steps
        rep.inner_hist.append(steps)
        rep.outer_iters = k + 1
        rep.x_hist.append(x.copy())
        done, rep.final_metric = _outer_stop(stop, x, x_ref, tol, A1, A2, b1, b2)
        if done:
            rep.converged = True
            break
    rep.x = x
    return rep


def scd_exact_select_distribution(G, r, alpha: int) -> dict:
    """Alg. 3 step 10 (Eq. Sec4.111) for tiny n: enumerate all size-alpha
    subsets tau, s(tau) = argmax_{s in tau} r_s^2 (ties smallest), P(tau) proportional to
    A1bar_{s(tau), s(tau)}. Returns the induced distribution of the selected index."""
    from itertools import combinations
    n = G.shape[0]
    probs = {}
    tot = 0.0
    for tau in combinations(range(n), alpha):
        s = scd_select(r, list(tau))
        wgt = G[s, s]
        probs[s] = probs.get(s, 0.0) + wgt
        tot += wgt
    return {k: v / tot for k, v in probs.items()}
