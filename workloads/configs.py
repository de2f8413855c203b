"""Seeded generators for the five BASELINE.json workloads.

Recipe: numpy ``Generator(Philox(seed))`` with a fixed draw
order A1, A2, x*, noise. The paper measures only on its own synthetic families
(§5.2, §5.3); BASELINE.json names five
synthetic configs which are generated here. No dataset is involved.

Nothing in this module implements the paper's method: it produces (A, b, x*)
and the problem dimensions only.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np


@dataclass
class IlsProblem:
    """ILS data min (b-Ax)^T J (b-Ax), J = diag(I_p, -I_q) (Eq. Sec11).

    A is stored row-major as [A1; A2] (partition Sec121).
    """

    name: str
    A: np.ndarray          # (m, n) float64, rows 0..p-1 = A1, p..m-1 = A2
    b: np.ndarray          # (m,) float64
    p: int
    q: int
    xstar: np.ndarray      # generating solution x* (n,)
    consistent: bool       # b == A x* exactly (then x_ref = x*)
    tol: float             # target relative error (BASELINE.json)
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.A.shape[1]

    @property
    def m(self) -> int:
        return self.A.shape[0]

    @property
    def A1(self) -> np.ndarray:
        return self.A[: self.p]

    @property
    def A2(self) -> np.ndarray:
        return self.A[self.p:]

    @property
    def b1(self) -> np.ndarray:
        return self.b[: self.p]

    @property
    def b2(self) -> np.ndarray:
        return self.b[self.p:]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def make_dense(p: int, q: int, n: int, a2_scale: float, noise: float = 0.0,
               seed: int = 0, tol: float = 1e-8, name: str = "dense") -> IlsProblem:
    """A1 ~ N(0,1) (p x n), A2 ~ a2_scale*N(0,1) (q x n), x* ~ N(0,1), b = A x* + noise*N(0,1).

    BASELINE.json configs[0] (p,q,n)=(200,100,50), scale 0.3, consistent;
    configs[1] (8000,2000,1000), scale 0.5, noise 0.01 on all m entries.
    """
    rng = _rng(seed)
    A1 = rng.standard_normal((p, n))
    A2 = a2_scale * rng.standard_normal((q, n))
    xstar = rng.standard_normal(n)
    A = np.ascontiguousarray(np.vstack([A1, A2]))
    b = A @ xstar
    if noise > 0.0:
        b = b + noise * rng.standard_normal(p + q)
    return IlsProblem(name=name, A=A, b=b, p=p, q=q, xstar=xstar,
                      consistent=(noise == 0.0), tol=tol,
                      meta=dict(a2_scale=a2_scale, noise=noise, seed=seed))


def _haar(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """Haar-distributed orthonormal columns: QR of a Gaussian with the sign fix
    diag(R) > 0 (Mezzadri 2007)."""
    Z = rng.standard_normal((rows, cols))
    Q, R = np.linalg.qr(Z, mode="reduced")
    return Q * np.sign(np.diag(R))[None, :]


def make_ill_conditioned(p: int = 40000, q: int = 10000, n: int = 4000, seed: int = 0,
                         tol: float = 1e-8, name: str = "c2") -> IlsProblem:
    """BASELINE.json configs[2]: A1 = U diag(s) V^T, s log-spaced 1..1e3, U,V Haar;
    A2 = G * sqrt(0.9)/sigma_max(G) so lambda_max(A2^T A2) = 0.9 lambda_min(A1^T A1) = 0.9
    (the stated "rho about 0.9" is an upper bound; the oracle measures rho).
    x* ~ N(0,1), b = A x* (consistent)."""
    rng = _rng(seed)
    U = _haar(rng, p, n)
    V = _haar(rng, n, n)
    s = 10.0 ** (3.0 * np.arange(n) / max(n - 1, 1))
    A1 = (U * s[None, :]) @ V.T
    del U
    G = rng.standard_normal((q, n))
    # sigma_max(G)^2 = lambda_max(G^T G); a library eigen-routine, not the method
    lam = np.linalg.eigvalsh(G.T @ G)[-1]
    A2 = G * np.sqrt(0.9 / lam)
    xstar = rng.standard_normal(n)
    A = np.ascontiguousarray(np.vstack([A1, A2]))
    del A1, A2, G
    b = A @ xstar
    return IlsProblem(name=name, A=A, b=b, p=p, q=q, xstar=xstar, consistent=True,
                      tol=tol, meta=dict(seed=seed, smin=1.0, smax=1e3))


@dataclass
class SparseIls:
    """BASELINE.json configs[3]: A = [A1; A2] in CSR (row_ptr int64, col_idx int32 sorted within
    each row, vals float64), b = A x* + noise."""

    name: str
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    b: np.ndarray
    p: int
    q: int
    n: int
    xstar: np.ndarray
    tol: float
    meta: dict = field(default_factory=dict)

    consistent = False

    @property
    def m(self) -> int:
        return self.p + self.q

    @property
    def nnz(self) -> int:
        return int(self.vals.size)

    def scipy(self):
        """The same matrix as a scipy.sparse CSR matrix (test/oracle convenience)."""
        import scipy.sparse as sp
        return sp.csr_matrix((self.vals, self.col_idx, self.row_ptr), shape=(self.m, self.n))

    def dense(self) -> np.ndarray:
        return self.scipy().toarray()


def make_sparse(p: int = 500000, q: int = 100000, n: int = 20000, nnz_per_row: int = 10,
                a2_scale: float = 0.3, noise: float = 1e-3, seed: int = 0, tol: float = 1e-8,
                name: str = "c3") -> SparseIls:
    """BASELINE.json configs[3]: every row has nnz_per_row nonzeros at distinct uniform-random
    columns (sorted), values N(0,1) in A1 and a2_scale*N(0,1) in A2; x* ~ N(0,1);
    b = A x* + noise*N(0,1) on all m rows. Draw order: columns, values, x*, noise."""
    rng = _rng(seed)
    m = p + q
    k = min(nnz_per_row, n)
    cols = rng.integers(0, n, size=(m, k), dtype=np.int64)
    while True:   # redraw duplicated columns within a row until all k are distinct
        srt = np.sort(cols, axis=1)
        dup_rows = np.flatnonzero(np.any(srt[:, 1:] == srt[:, :-1], axis=1))
        if dup_rows.size == 0:
            break
        cols[dup_rows] = rng.integers(0, n, size=(dup_rows.size, k), dtype=np.int64)
    cols = np.sort(cols, axis=1)
    vals = rng.standard_normal((m, k))
    vals[p:] *= a2_scale
    xstar = rng.standard_normal(n)
    row_ptr = np.arange(0, (m + 1) * k, k, dtype=np.int64)
    col_idx = cols.reshape(-1).astype(np.int32)
    v = vals.reshape(-1)
    Ax = (vals * xstar[cols]).sum(axis=1)
    b = Ax + noise * rng.standard_normal(m) if noise > 0 else Ax
    return SparseIls(name=name, row_ptr=row_ptr, col_idx=col_idx, vals=np.ascontiguousarray(v), b=b, p=p, q=q,
                     n=n, xstar=xstar, tol=tol, meta=dict(seed=seed, nnz_per_row=k, a2_scale=a2_scale, noise=noise))


@dataclass
class BatchedIls:
    """BASELINE.json configs[4]: independent instances, instance i seeded base+i."""

    A: np.ndarray      # (batch, m, n)
    b: np.ndarray      # (batch, m)
    xstar: np.ndarray  # (batch, n)
    p: int
    q: int
    tol: float
    seeds: np.ndarray

    @property
    def batch(self) -> int:
        return self.A.shape[0]

    @property
    def n(self) -> int:
        return self.A.shape[2]


def make_batched(batch: int = 4096, p: int = 96, q: int = 32, n: int = 32,
                 a2_scale: float = 0.3, base_seed: int = 0, tol: float = 1e-10) -> BatchedIls:
    """Each instance generated as configs[0] (A1 N(0,1), A2 0.3 N(0,1), b = A x*)
    with seed = base_seed + instance id."""
    m = p + q
    A = np.empty((batch, m, n))
    b = np.empty((batch, m))
    xs = np.empty((batch, n))
    for i in range(batch):
        pr = make_dense(p, q, n, a2_scale, 0.0, seed=base_seed + i, tol=tol)
        A[i] = pr.A
        b[i] = pr.b
        xs[i] = pr.xstar
    return BatchedIls(A=A, b=b, xstar=xs, p=p, q=q, tol=tol,
                      seeds=base_seed + np.arange(batch))


CONFIGS = {
    "c0": dict(kind="dense", p=200, q=100, n=50, a2_scale=0.3, noise=0.0, tol=1e-10,
               max_inner=100000),
    "c1": dict(kind="dense", p=8000, q=2000, n=1000, a2_scale=0.5, noise=0.01, tol=1e-8),
    "c2": dict(kind="illcond", p=40000, q=10000, n=4000, tol=1e-8),
    "c3": dict(kind="sparse", p=500000, q=100000, n=20000, nnz_per_row=10,
               a2_scale=0.3, noise=1e-3, tol=1e-8),
    "c4": dict(kind="batched", batch=4096, p=96, q=32, n=32, a2_scale=0.3, tol=1e-10),
}


def make_paper(p: int, q: int, n: int, seed: int = 0, tol: float = 1e-6, name: str = "paper") -> IlsProblem:
    """The paper's own synthetic family.

    §5.2 (from Song's USSOR examples): A1 = rand(p,n), A2 = 7*eye(q,n),
    b1 = rand(p,1), b2 = rand(q,1); Tables 2-3 use p in {30000, 40000}, q = n in
    {13000, 14000, 15000}. §5.3 Minkowski: the same with q = 1 and
    p in {50000, 60000} (Tables 4-5). MATLAB's rand is uniform on (0,1); here numpy's
    Generator(Philox(seed)).random draws uniform [0,1) in the order A1, b1, b2 -- the same
    distribution, not MATLAB's stream. The problem is not consistent (b is random): there is no
    generating x*, so xstar is NaN and x_ref comes from a direct solve. tol is the paper's RR
    threshold 1e-6.
    """
    if q > n:
        raise ValueError("7*eye(q,n) with q > n has zero rows; the paper uses q = n or q = 1")
    rng = _rng(seed)
    m = p + q
    A = np.zeros((m, n))
    A[:p] = rng.random((p, n))
    A[p + np.arange(q), np.arange(q)] = 7.0
    b = np.empty(m)
    b[:p] = rng.random(p)
    b[p:] = rng.random(q)
    return IlsProblem(name=name, A=A, b=b, p=p, q=q, xstar=np.full(n, np.nan), consistent=False, tol=tol,
                      meta=dict(family="minkowski" if q == 1 else "song-ussor", seed=seed))


# Tables 2-5 of the paper: (table, p, q, n); q = "n" means q = n.
PAPER_TABLES = {
    "t2": [(30000, n, n) for n in (13000, 14000, 15000)],
    "t3": [(40000, n, n) for n in (13000, 14000, 15000)],
    "t4": [(50000, 1, n) for n in (13000, 14000, 15000)],
    "t5": [(60000, 1, n) for n in (13000, 14000, 15000)],
}


def make_problem(name: str, seed: int = 0, **overrides):
    """Build config `name` (c0..c4) with optional shape overrides (tests use
    reduced shapes with the same recipe)."""
    cfg = dict(CONFIGS[name])
    cfg.update(overrides)
    kind = cfg.pop("kind")
    if kind == "dense":
        return make_dense(cfg["p"], cfg["q"], cfg["n"], cfg["a2_scale"], cfg["noise"],
                          seed=seed, tol=cfg["tol"], name=name)
    if kind == "illcond":
        return make_ill_conditioned(cfg["p"], cfg["q"], cfg["n"], seed=seed,
                                    tol=cfg["tol"], name=name)
    if kind == "sparse":
        return make_sparse(cfg["p"], cfg["q"], cfg["n"], cfg["nnz_per_row"], cfg["a2_scale"], cfg["noise"],
                           seed=seed, tol=cfg["tol"], name=name)
    if kind == "batched":
        return make_batched(cfg["batch"], cfg["p"], cfg["q"], cfg["n"], cfg["a2_scale"],
                            base_seed=seed, tol=cfg["tol"])
    raise NotImplementedError(f"workload kind {kind!r} not generated yet")


def fingerprint(A, b: np.ndarray) -> str:
    """SHA-256 over the first/last 64 rows of A (dense) or its CSR arrays' heads and tails (sparse)
    and the head of b: ties a stored x_ref file (workloads/xref/, written by tools/make_xref.py
    from the oracle) to the generated data."""
    h = hashlib.sha256()
    if isinstance(A, np.ndarray):
        h.update(np.ascontiguousarray(A[:64]).tobytes())
        h.update(np.ascontiguousarray(A[-64:]).tobytes())
    else:
        for arr in (A.row_ptr, A.col_idx, A.vals):
            h.update(np.ascontiguousarray(arr[:640]).tobytes())
            h.update(np.ascontiguousarray(arr[-640:]).tobytes())
    h.update(np.ascontiguousarray(b[:64]).tobytes())
    return h.hexdigest()
