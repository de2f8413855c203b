"""Thin ctypes binding of libils.so (include/ils.h). Argument marshalling only: every step of
the method runs in the CUDA kernels of libils. Arrays may be numpy arrays (host memory) or
torch tensors (host or CUDA); their data pointers are passed straight through.

The binding fails loudly if the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ILS_LIB_PATH") or os.path.join(_HERE, "lib", "libils.so")   # override: A/B builds

ILS_OK, ILS_NOT_CONVERGED = 0, 1
ILS_ERR_ARG, ILS_ERR_SHAPE, ILS_ERR_ZERO_COLUMN, ILS_ERR_NOT_SPD = -1, -2, -3, -4
ILS_ERR_CUDA, ILS_ERR_NOMEM, ILS_ERR_UNSUPPORTED = -5, -6, -7
ILS_STOP_XREF, ILS_STOP_RR, ILS_STOP_NONE = 0, 1, 2
ILS_FORMAT_DENSE, ILS_FORMAT_CSR = 0, 1
ILS_ALPHA_UNIFORM, ILS_ALPHA_FIXED = 0, 1
ILS_SP_FORM_AUTO = 3
ILS_SUBSET_EXACT = 0x10

EXPORTED = [
    "ils_default_opts", "ils_status_string", "ils_last_error", "ils_create", "ils_sp_solve",
    "ils_rk_solve", "ils_rgs_solve", "ils_destroy", "ils_direct_solve", "ils_relative_residual",
    "ils_get_sampling_tables", "ils_rk_indices", "ils_scd_subset", "ils_kernel_launch_count",
    "ils_comm_unique_id", "ils_comm_create", "ils_comm_destroy",
]


class IlsExt(C.Structure):
    _fields_ = [("format", C.c_int32), ("batch", C.c_int64), ("lda", C.c_int64), ("stream", C.c_void_p),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("nnz", C.c_int64), ("comm", C.c_void_p)]


class IlsOpts(C.Structure):
    _fields_ = [("stop", C.c_int32), ("x_ref", C.c_void_p), ("inner_tol", C.c_double),
                ("max_inner", C.c_int64), ("check_every", C.c_int64), ("seed", C.c_uint64),
                ("alpha_mode", C.c_int32), ("alpha_k", C.c_int32), ("weighted", C.c_int32),
                ("sp_form", C.c_int32), ("x_hist", C.c_void_p), ("inner_hist", C.c_void_p),
                ("expected_outer", C.c_int64)]


class IlsReport(C.Structure):
    _fields_ = [("outer_iters", C.c_int64), ("inner_iters_total", C.c_int64), ("converged", C.c_int32),
                ("final_metric", C.c_double), ("setup_ms", C.c_double), ("solve_ms", C.c_double),
                ("bytes_touched", C.c_double), ("kernel_launches", C.c_int64),
                ("hot_ms", C.c_double * 4), ("hot_work", C.c_double * 4), ("hot_launches", C.c_int64 * 4),
                ("inst_iters", C.c_void_p), ("inst_status", C.c_void_p), ("sp_form_used", C.c_int32)]

    def as_dict(self):
        d = {}
        for k, _ in self._fields_:
            if k in ("inst_iters", "inst_status"):
                continue
            v = getattr(self, k)
            d[k] = list(v) if k.startswith("hot_") else v
        return d


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libils.so. Raises (loudly) if it is missing -- there is no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libils.so not built ({path}); run python -m paper_2203_15340_b200.build "
                          "or __graft_entry__.build()")
    lib = C.CDLL(path)
    vp, i64, i32, dbl, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_uint64
    sig = {
        "ils_default_opts": (None, [C.POINTER(IlsOpts)]),
        "ils_status_string": (C.c_char_p, [C.c_int]),
        "ils_last_error": (C.c_char_p, []),
        "ils_create": (C.c_int, [C.POINTER(vp), vp, vp, i64, i64, i64, C.POINTER(IlsExt)]),
        "ils_sp_solve": (C.c_int, [vp, vp, vp, dbl, i64, C.POINTER(IlsOpts), C.POINTER(IlsReport)]),
        "ils_rk_solve": (C.c_int, [vp, vp, vp, dbl, i64, C.POINTER(IlsOpts), C.POINTER(IlsReport)]),
        "ils_rgs_solve": (C.c_int, [vp, vp, vp, dbl, i64, C.POINTER(IlsOpts), C.POINTER(IlsReport)]),
        "ils_destroy": (None, [vp]),
        "ils_direct_solve": (C.c_int, [vp, vp]),
        "ils_relative_residual": (C.c_int, [vp, vp, C.POINTER(C.c_double)]),
        "ils_get_sampling_tables": (C.c_int, [vp, vp, vp]),
        "ils_rk_indices": (C.c_int, [vp, u64, i64, i64, i64, vp, vp]),
        "ils_scd_subset": (C.c_int, [i64, u64, i64, i64, i32, i32, vp, vp]),
        "ils_kernel_launch_count": (C.c_int64, []),
        "ils_comm_unique_id": (C.c_int, [vp]),
        "ils_comm_create": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
        "ils_comm_destroy": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _ptr(a):
    """Raw data pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _arr(a, dtype, count, what):
    """Pointer of `a` after checking its element type and that it holds at least `count` elements
    (argument marshalling: a wrong dtype or a short buffer would make the library read past it)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        ok = a.dtype == np.dtype(dtype)
        size = a.size
    elif hasattr(a, "data_ptr"):
        import torch
        ok = a.dtype == {"float64": torch.float64, "int64": torch.int64, "int32": torch.int32}[dtype]
        size = a.numel()
    else:
        raise TypeError(f"{what}: unsupported array type {type(a)}")
    if not ok:
        raise TypeError(f"{what}: expected {dtype}, got {a.dtype}")
    if size < count:
        raise ValueError(f"{what}: {size} elements, the call reads {count}")
    return _ptr(a)


_shape = {}   # handle value -> (n, batch), for the solve-side length checks


class IlsError(RuntimeError):
    def __init__(self, status, where):
        lib = load_library()
        msg = lib.ils_status_string(status).decode()
        detail = lib.ils_last_error().decode()
        super().__init__(f"{where}: {msg} ({status}) {detail}")
        self.status = status


def _check(status, where):
    if status < 0:
        raise IlsError(status, where)
    return status


def ils_default_opts(**kw) -> IlsOpts:
    o = IlsOpts()
    load_library().ils_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def ils_create(A, b, p: int, q: int, n: int, batch: int = 1, lda: int = 0, stream=None, row_ptr=None,
               col_idx=None, comm=None):
    """ils_create(A, b, p, q, n, ext): A row-major (m x n) or [batch][m][n] fp64, b (m) or [batch][m].
    CSR input: A = values [nnz], row_ptr int64 [m+1], col_idx int32 [nnz] (ILS_FORMAT_CSR).
    comm (ils_comm_create): A, b are this rank's row block, p, q its local row counts."""
    lib = load_library()
    h = C.c_void_p()
    m = p + q
    if row_ptr is not None:
        nnz = int(A.numel() if hasattr(A, "numel") else A.size)
        ext = IlsExt(ILS_FORMAT_CSR, 1, 0, stream, _arr(row_ptr, "int64", m + 1, "row_ptr"),
                     _arr(col_idx, "int32", nnz, "col_idx"), nnz, comm)
        pa = _arr(A, "float64", nnz, "A (CSR values)")
    else:
        ext = IlsExt(ILS_FORMAT_DENSE, batch, lda, stream, None, None, 0, comm)
        ld = lda if lda else n
        pa = _arr(A, "float64", (batch * m - 1) * ld + n if m > 0 else 0, "A")
    pb = _arr(b, "float64", batch * m, "b")
    _check(lib.ils_create(C.byref(h), pa, pb, p, q, n, C.byref(ext)), "ils_create")
    _shape[h.value] = (n, batch)
    return h


def ils_destroy(h):
    _shape.pop(getattr(h, "value", None), None)
    load_library().ils_destroy(h)


def _solve(fn, name, h, x0, x, tol, max_iter, opts, inst_iters=None, inst_status=None):
    rep = IlsReport()
    n, batch = _shape.get(getattr(h, "value", None), (0, 1))
    rep.inst_iters = _arr(inst_iters, "int64", batch, "inst_iters")
    rep.inst_status = _arr(inst_status, "int32", batch, "inst_status")
    o = opts if opts is not None else ils_default_opts()
    st = _check(fn(h, _arr(x0, "float64", batch * n, "x0"), _arr(x, "float64", batch * n, "x"), float(tol),
                   int(max_iter), C.byref(o), C.byref(rep)), name)
    return st, rep


def ils_sp_solve(h, x0, x, tol, max_iter, opts=None, **kw):
    return _solve(load_library().ils_sp_solve, "ils_sp_solve", h, x0, x, tol, max_iter, opts, **kw)


def ils_rk_solve(h, x0, x, tol, max_iter, opts=None, **kw):
    return _solve(load_library().ils_rk_solve, "ils_rk_solve", h, x0, x, tol, max_iter, opts, **kw)


def ils_rgs_solve(h, x0, x, tol, max_iter, opts=None, **kw):
    return _solve(load_library().ils_rgs_solve, "ils_rgs_solve", h, x0, x, tol, max_iter, opts, **kw)


def ils_direct_solve(h, x):
    return _check(load_library().ils_direct_solve(h, _ptr(x)), "ils_direct_solve")


def ils_relative_residual(h, x) -> float:
    rr = C.c_double()
    _check(load_library().ils_relative_residual(h, _ptr(x), C.byref(rr)), "ils_relative_residual")
    return rr.value


def ils_get_sampling_tables(h, n: int):
    N = np.zeros(n)
    S = np.zeros(n, dtype=np.uint64)
    _check(load_library().ils_get_sampling_tables(h, _ptr(N), _ptr(S)), "ils_get_sampling_tables")
    return N, S


def ils_rk_indices(h, seed: int, k: int, t0: int, count: int):
    j1 = np.zeros(count, dtype=np.int32)
    j2 = np.zeros(count, dtype=np.int32)
    _check(load_library().ils_rk_indices(h, seed, k, t0, count, _ptr(j1), _ptr(j2)), "ils_rk_indices")
    return j1, j2


def ils_scd_subset(n: int, seed: int, k: int, t: int, alpha_mode: int = 0, alpha_k: int = 1):
    alpha = np.zeros(1, dtype=np.int32)
    mask = np.zeros(n, dtype=np.uint8)
    _check(load_library().ils_scd_subset(n, seed, k, t, alpha_mode, alpha_k, _ptr(alpha), _ptr(mask)),
           "ils_scd_subset")
    return int(alpha[0]), mask


def ils_kernel_launch_count() -> int:
    return int(load_library().ils_kernel_launch_count())


# ---- row sharding (include/ils.h "Row-sharded handles")
ILS_COMM_ID_BYTES = 128


def ils_comm_unique_id() -> bytes:
    buf = C.create_string_buffer(ILS_COMM_ID_BYTES)
    _check(load_library().ils_comm_unique_id(buf), "ils_comm_unique_id")
    return buf.raw


def ils_comm_create(uid: bytes, nranks: int, rank: int):
    if len(uid) != ILS_COMM_ID_BYTES:
        raise ValueError("communicator id must be ILS_COMM_ID_BYTES bytes")
    c = C.c_void_p()
    buf = C.create_string_buffer(uid, ILS_COMM_ID_BYTES)
    _check(load_library().ils_comm_create(buf, nranks, rank, C.byref(c)), "ils_comm_create")
    return c


def ils_comm_destroy(c):
    load_library().ils_comm_destroy(c)


def shard_rows(p: int, q: int, world: int, rank: int):
    """Contiguous row blocks of A1 and A2 for `rank` of `world`: ((p0, p1), (q0, q1)), the first
    p % world (q % world) ranks taking one extra row. Every rank gets >= 1 row of A1 (needs
    p >= world); the blocks tile [0, p) and [0, q) exactly."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world / rank")
    if p < world:
        raise ValueError("row sharding needs at least one A1 row per rank")

    def block(total):
        base, extra = divmod(total, world)
        lo = rank * base + min(rank, extra)
        return lo, lo + base + (1 if rank < extra else 0)

    return block(p), block(q)


def make_comm(rank: int, world: int, broadcast_object):
    """Create this rank's communicator: rank 0 draws the NCCL id, `broadcast_object(obj) -> obj`
    (e.g. a torch.distributed.broadcast_object_list wrapper) hands it to every rank."""
    uid = ils_comm_unique_id() if rank == 0 else None
    uid = broadcast_object(uid)
    return ils_comm_create(uid, world, rank)
