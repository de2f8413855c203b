"""Seeded synthetic ILS workloads (BASELINE.json configs c0..c4).

This package is the ONLY code shared by the CUDA path's callers (bench, tests)
and the CPU oracle. It draws random problem data and holds none of the
method's arithmetic (no splitting step, no sampling, no solve).
"""
from .configs import (  # noqa: F401
    CONFIGS,
    IlsProblem,
    make_problem,
    make_batched,
    make_dense,
    make_ill_conditioned,
    make_sparse,
    make_paper,
    PAPER_TABLES,
    SparseIls,
    fingerprint,
)
