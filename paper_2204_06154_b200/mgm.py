"""Thin ctypes binding of libmgm's C ABI (include/mgm.h).  Argument marshalling only:
every step of the MGM path runs in libmgm's CUDA kernels.  There is no fallback; if
libmgm.so is missing or cannot be loaded this module raises.

Function names mirror the C ABI (``mgm_setup``, ``mgm_vcycle``, ``mgm_solve``, ...);
:class:`MGM` is a small convenience wrapper that owns a context and takes torch tensors
(device memory and streams come from PyTorch; the arithmetic does not).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmgm.so")

MGM_OK, MGM_ERR_ARG, MGM_ERR_UNISOLVENT, MGM_ERR_SINGULAR, MGM_ERR_BREAKDOWN, \
    MGM_ERR_CUDA, MGM_ERR_NCCL, MGM_ERR_OOM, MGM_ERR_INPUT = range(9)
OP_SPMV, OP_SWEEP, OP_RESIDUAL, OP_RESTRICT, OP_INTERP, OP_COARSE, OP_SWEEP_ZG, OP_PRECOND = range(8)
STATUS_NAMES = {0: "MGM_OK", 1: "MGM_ERR_ARG", 2: "MGM_ERR_UNISOLVENT", 3: "MGM_ERR_SINGULAR",
                4: "MGM_ERR_BREAKDOWN", 5: "MGM_ERR_CUDA", 6: "MGM_ERR_NCCL", 7: "MGM_ERR_OOM",
                8: "MGM_ERR_INPUT"}


class StencilParams(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("poly_degree", ctypes.c_int), ("phs_k", ctypes.c_int),
                ("stencil_n", ctypes.c_int), ("gfd_alpha", ctypes.c_double),
                ("problem", ctypes.c_int), ("mu", ctypes.c_double)]


class LevelParams(ctypes.Structure):
    _fields_ = [("num_levels", ctypes.c_int), ("n_min", ctypes.c_int),
                ("coarsen_factor", ctypes.c_int), ("interp_m", ctypes.c_int),
                ("nu1", ctypes.c_int), ("nu2", ctypes.c_int), ("smoother", ctypes.c_int),
                ("restart", ctypes.c_int)]


class Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("final_rel_residual", ctypes.c_double),
                ("history", ctypes.POINTER(ctypes.c_double)), ("history_cap", ctypes.c_int),
                ("lambda_", ctypes.c_double), ("setup_ms", ctypes.c_double),
                ("solve_ms", ctypes.c_double)]


_vp = ctypes.c_void_p
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
RELEASE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class Allocator(ctypes.Structure):
    """mgm_allocator: device allocations of a ctx (include/mgm.h)."""
    _fields_ = [("alloc", ALLOC_FN), ("release", RELEASE_FN), ("user", ctypes.c_void_p)]


_i64 = ctypes.c_int64
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "mgm_setup": ([_f64p, _f64p, _i64, ctypes.POINTER(StencilParams), ctypes.POINTER(LevelParams),
                   ctypes.POINTER(Allocator), _vp, ctypes.POINTER(_vp)], ctypes.c_int),
    "mgm_vcycle": ([_vp, _vp, _vp, _vp], ctypes.c_int),
    "mgm_solve": ([_vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                   ctypes.POINTER(Report), _vp], ctypes.c_int),
    "mgm_solve_host": ([_vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                        ctypes.POINTER(Report), _vp], ctypes.c_int),
    "mgm_destroy": ([_vp], ctypes.c_int),
    "mgm_nccl_unique_id": ([_vp], ctypes.c_int),
    "mgm_vcycle_batch": ([_vp, ctypes.c_int, _vp, _vp, _vp], ctypes.c_int),
    "mgm_solve_batch": ([_vp, ctypes.c_int, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                         ctypes.POINTER(Report), _vp], ctypes.c_int),
    "mgm_dist_attach": ([_vp, ctypes.c_int, ctypes.c_int, _vp], ctypes.c_int),
    "mgm_local_rows": ([_vp, _i64p, _i64p], ctypes.c_int),
    "mgm_dist_comm_time": ([_vp, ctypes.c_int, _f64p, _f64p, _vp], ctypes.c_int),
    "mgm_dist_info": ([_vp, ctypes.POINTER(ctypes.c_int), _i64p, _i64p], ctypes.c_int),
    "mgm_fake_group_create": ([ctypes.c_int, ctypes.POINTER(_vp)], ctypes.c_int),
    "mgm_fake_group_destroy": ([_vp], ctypes.c_int),
    "mgm_dist_attach_fake": ([_vp, ctypes.c_int, _vp], ctypes.c_int),
    "mgm_last_error": ([_vp, _i64p], ctypes.c_char_p),
    "mgm_num_levels": ([_vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "mgm_level_info": ([_vp, ctypes.c_int, _i64p, _i64p, _i64p, ctypes.POINTER(ctypes.c_int),
                        _i64p], ctypes.c_int),
    "mgm_export_level": ([_vp, ctypes.c_int, _i64p, _i64p, _i32p, _f64p, _i32p, _i64p, _i32p,
                          _f64p, _f64p], ctypes.c_int),
    "mgm_export_weights": ([_vp, _f64p, _i64p], ctypes.c_int),
    "mgm_apply": ([_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _vp], ctypes.c_int),
    "mgm_timing_enable": ([_vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "mgm_timing_read": ([_vp, ctypes.c_int, _f64p, _i64p, _f64p], ctypes.c_int),
    "mgm_bytes_model": ([_vp, _f64p, _f64p], ctypes.c_int),
    "mgm_vcycle_kernel_count": ([_vp, _i64p], ctypes.c_int),
    "mgm_trace_read": ([_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                        ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_int], ctypes.c_int),
    "mgm_bottom_trace_read": ([_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                               ctypes.POINTER(ctypes.c_int), _i32p], ctypes.c_int),
    "mgm_level_zg_nnz": ([_vp, ctypes.c_int, _i64p], ctypes.c_int),
    "mgm_dense_bottom_info": ([_vp, ctypes.POINTER(ctypes.c_int), _i64p, _i64p], ctypes.c_int),
    "mgm_bottom_ftrace_read": ([_vp, _i64p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "mgm_host_morton": ([_f64p, _i64, _i64p], ctypes.c_int),
    "mgm_host_knn": ([_f64p, _i64, _f64p, _i64, ctypes.c_int, _i32p], ctypes.c_int),
    "mgm_device_knn": ([_f64p, _i64, _f64p, _i64, ctypes.c_int, _i32p], ctypes.c_int),
    "mgm_host_wse": ([_f64p, _i64, _i64, _i64p], ctypes.c_int),
    "mgm_device_wse": ([_f64p, _i64, _i64, _i64p], ctypes.c_int),
    "mgm_host_colouring": ([_i64, _i64p, _i32p, _i32p, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "mgm_host_partition_level": ([_i64, _i64p, _i32p, _i32p, ctypes.c_int, _i32p, _i64, _i64p, _i32p, _i32p,
                                  _i64, _i64p, _i32p, _i32p, ctypes.c_int, ctypes.c_int,
                                  _i64p, _i64p, _i64p, _i64p, ctypes.POINTER(ctypes.c_int), _i32p, _i64p,
                                  _i64p, _i64p, _i64p, _i64p], ctypes.c_int),
}
EXPORTED = tuple(_SIGS)

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libmgm.so (raises OSError/RuntimeError if it is missing -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"libmgm.so not built ({path}); run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


class MGMError(RuntimeError):
    def __init__(self, status, msg, index):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg} (index {index})")
        self.status, self.index = status, index


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _check(status, ctx=None):
    if status != MGM_OK:
        idx = _i64(-1)
        msg = load_library().mgm_last_error(ctx, ctypes.byref(idx))
        raise MGMError(status, (msg or b"").decode(), idx.value)


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def torch_allocator():
    """An mgm_allocator that takes the ctx's device memory from PyTorch's caching allocator
    (marshalling only: the callbacks forward to torch.cuda.caching_allocator_alloc/_delete).
    Keep the returned object alive as long as the ctx."""
    import torch

    dev = torch.cuda.current_device()

    def _alloc(nbytes, user):
        try:
            return torch.cuda.caching_allocator_alloc(max(int(nbytes), 1), device=dev)
        except Exception:
            return None

    def _release(ptr, user):
        torch.cuda.caching_allocator_delete(ptr)

    a = Allocator(ALLOC_FN(_alloc), RELEASE_FN(_release), None)
    a._keep = (_alloc, _release)
    return a


# ---------------------------------------------------------------- ABI-named functions
def mgm_setup(points: np.ndarray, normals: np.ndarray, stencil: dict, levels: dict, stream=None,
              allocator: Allocator | None = None):
    """Returns an opaque ctx handle (c_void_p).  Raises MGMError on failure.  allocator: an
    :class:`Allocator` (e.g. :func:`torch_allocator`) or None for cudaMalloc."""
    lib = load_library()
    pts = np.ascontiguousarray(points, dtype=np.float64)
    nrm = np.ascontiguousarray(normals, dtype=np.float64)
    sp = StencilParams(method=stencil.get("method", 0), poly_degree=stencil.get("poly_degree", 2),
                       phs_k=stencil.get("phs_k", 1), stencil_n=stencil.get("stencil_n", 15),
                       gfd_alpha=stencil.get("gfd_alpha", 4.0), problem=stencil.get("problem", 0),
                       mu=stencil.get("mu", 1.0))
    lp = LevelParams(num_levels=levels.get("num_levels", 0), n_min=levels.get("n_min", 250),
                     coarsen_factor=levels.get("coarsen_factor", 4),
                     interp_m=levels.get("interp_m", 6), nu1=levels.get("nu1", 1),
                     nu2=levels.get("nu2", 1), smoother=levels.get("smoother", 0),
                     restart=levels.get("restart", 50))
    ctx = _vp()
    st = lib.mgm_setup(_ptr(pts, _f64p), _ptr(nrm, _f64p), len(pts), ctypes.byref(sp),
                       ctypes.byref(lp), ctypes.byref(allocator) if allocator is not None else None,
                       _vp(_stream_ptr(stream) if stream is not None else 0), ctypes.byref(ctx))
    if st != MGM_OK:
        idx = _i64(-1)
        msg = lib.mgm_last_error(None, ctypes.byref(idx)).decode()
        if ctx.value:
            lib.mgm_destroy(ctx)
        raise MGMError(st, msg, idx.value)
    return ctx


def mgm_destroy(ctx):
    load_library().mgm_destroy(ctx)


def mgm_vcycle(ctx, f, u, stream=None):
    _check(load_library().mgm_vcycle(ctx, _vp(f.data_ptr()), _vp(u.data_ptr()),
                                     _vp(_stream_ptr(stream))), ctx)


@dataclass
class SolveReport:
    iterations: int
    converged: bool
    final_rel_residual: float
    history: list
    lam: float
    setup_ms: float
    solve_ms: float


def _report(rep, hist):
    n = min(rep.iterations, len(hist))
    return SolveReport(rep.iterations, bool(rep.converged), rep.final_rel_residual,
                       list(hist[:n]), rep.lambda_, rep.setup_ms, rep.solve_ms)


def mgm_solve(ctx, rhs, x, tol=1e-10, maxit=500, krylov=1, stream=None, history_cap=1024, x0=None):
    """x0: initial guess (torch CUDA tensor, may be x itself) or None for x0 = 0."""
    hist = np.zeros(history_cap)
    rep = Report(history=_ptr(hist, _f64p), history_cap=history_cap)
    _check(load_library().mgm_solve(ctx, _vp(rhs.data_ptr()), _vp(x0.data_ptr()) if x0 is not None else None,
                                    _vp(x.data_ptr()), tol, maxit, krylov, ctypes.byref(rep),
                                    _vp(_stream_ptr(stream))), ctx)
    return _report(rep, hist)


def mgm_solve_host(ctx, rhs: np.ndarray, x: np.ndarray, tol=1e-10, maxit=500, krylov=1,
                   stream=None, history_cap=1024, x0: np.ndarray | None = None):
    """rhs / x / x0: host arrays (numpy, or pinned torch CPU tensors via .numpy())."""
    hist = np.zeros(history_cap)
    rep = Report(history=_ptr(hist, _f64p), history_cap=history_cap)
    assert rhs.dtype == np.float64 and x.dtype == np.float64 and x.flags.c_contiguous
    if x0 is not None:
        assert x0.dtype == np.float64 and x0.flags.c_contiguous
    _check(load_library().mgm_solve_host(ctx, _vp(rhs.ctypes.data), _vp(x0.ctypes.data) if x0 is not None else None,
                                         _vp(x.ctypes.data), tol, maxit, krylov, ctypes.byref(rep),
                                         _vp(_stream_ptr(stream))), ctx)
    return _report(rep, hist)


def mgm_vcycle_batch(ctx, K: int, f, u, stream=None):
    """f, u: torch CUDA float64 tensors of shape (K, N) (original order), u in place."""
    assert f.is_contiguous() and u.is_contiguous() and f.shape == u.shape and f.shape[0] == K
    _check(load_library().mgm_vcycle_batch(ctx, K, _vp(f.data_ptr()), _vp(u.data_ptr()),
                                           _vp(_stream_ptr(stream))), ctx)


def mgm_solve_batch(ctx, K: int, rhs, x, tol=1e-10, maxit=500, stream=None, history_cap=512, krylov=0):
    """K right-hand sides at once (rhs, x: (K, N) CUDA float64 tensors): standalone MGM
    (krylov=0) or K MGM-GMRES processes sharing every operator pass (krylov=1)."""
    assert rhs.is_contiguous() and x.is_contiguous() and rhs.shape == x.shape and rhs.shape[0] == K
    hists = [np.zeros(history_cap) for _ in range(K)]
    reps = (Report * K)()
    for k in range(K):
        reps[k].history = _ptr(hists[k], _f64p)
        reps[k].history_cap = history_cap
    _check(load_library().mgm_solve_batch(ctx, K, _vp(rhs.data_ptr()), _vp(x.data_ptr()), tol, maxit, krylov,
                                          reps, _vp(_stream_ptr(stream))), ctx)
    return [_report(reps[k], hists[k]) for k in range(K)]


def mgm_num_levels(ctx) -> int:
    p = ctypes.c_int(0)
    _check(load_library().mgm_num_levels(ctx, ctypes.byref(p)), ctx)
    return p.value


def mgm_level_info(ctx, level: int) -> dict:
    n, z, q, b = _i64(), _i64(), _i64(), _i64()
    c = ctypes.c_int()
    _check(load_library().mgm_level_info(ctx, level, ctypes.byref(n), ctypes.byref(z),
                                         ctypes.byref(q), ctypes.byref(c), ctypes.byref(b)), ctx)
    zg = _i64()
    _check(load_library().mgm_level_zg_nnz(ctx, level, ctypes.byref(zg)), ctx)
    return dict(n=n.value, nnz=z.value, nnz_P=q.value, colours=c.value, stored_bytes=b.value,
                nnz_zg=zg.value)


def mgm_export_level(ctx, level: int, poisson: bool = False) -> dict:
    info = mgm_level_info(ctx, level)
    n, z, q = info["n"], info["nnz"], info["nnz_P"]
    ids = np.empty(n, dtype=np.int64)
    Lp = np.empty(n + 1, dtype=np.int64)
    Lc = np.empty(z, dtype=np.int32)
    Lv = np.empty(z)
    col = np.empty(n, dtype=np.int32)
    Pp = np.empty(n + 1, dtype=np.int64)
    Pc = np.empty(max(q, 1), dtype=np.int32)
    Pv = np.empty(max(q, 1))
    bd = np.empty(n) if poisson else None
    _check(load_library().mgm_export_level(
        ctx, level, _ptr(ids, _i64p), _ptr(Lp, _i64p), _ptr(Lc, _i32p), _ptr(Lv, _f64p),
        _ptr(col, _i32p), _ptr(Pp, _i64p), _ptr(Pc, _i32p), _ptr(Pv, _f64p),
        _ptr(bd, _f64p) if poisson else None), ctx)
    out = dict(info, ids=ids, L_ptr=Lp, L_col=Lc, L_val=Lv, colour=col, border=bd)
    if q:
        out.update(P_ptr=Pp, P_col=Pc[:q], P_val=Pv[:q])
    return out


def mgm_export_weights(ctx, n_points: int, stencil_n: int):
    w = np.empty(n_points * stencil_n)
    s = np.empty(n_points * stencil_n, dtype=np.int64)
    _check(load_library().mgm_export_weights(ctx, _ptr(w, _f64p), _ptr(s, _i64p)), ctx)
    return w.reshape(n_points, stencil_n), s.reshape(n_points, stencil_n)


def mgm_apply(ctx, level: int, op: int, x, f=None, y=None, stream=None):
    _check(load_library().mgm_apply(ctx, level, op, _vp(x.data_ptr()),
                                    _vp(f.data_ptr()) if f is not None else None,
                                    _vp(y.data_ptr()), _vp(_stream_ptr(stream))), ctx)
    return y


def mgm_timing_enable(ctx, cls: int, enable: bool = True):
    _check(load_library().mgm_timing_enable(ctx, cls, 1 if enable else 0), ctx)


def mgm_timing_read(ctx, cls: int):
    t, n, b = ctypes.c_double(), _i64(), ctypes.c_double()
    _check(load_library().mgm_timing_read(ctx, cls, ctypes.byref(t), ctypes.byref(n),
                                          ctypes.byref(b)), ctx)
    return dict(total_ms=t.value, launches=n.value, alg_bytes=b.value)


def mgm_bytes_model(ctx):
    v, s = ctypes.c_double(), ctypes.c_double()
    _check(load_library().mgm_bytes_model(ctx, ctypes.byref(v), ctypes.byref(s)), ctx)
    return dict(vcycle_bytes=v.value, spmv_bytes=s.value)


def mgm_vcycle_kernel_count(ctx) -> int:
    c = _i64()
    _check(load_library().mgm_vcycle_kernel_count(ctx, ctypes.byref(c)), ctx)
    return c.value


def mgm_dense_bottom_info(ctx) -> dict:
    """{level J or -1, rows of B_J, bytes of B_J read per V-cycle}."""
    j, r, b = ctypes.c_int(), _i64(), _i64()
    _check(load_library().mgm_dense_bottom_info(ctx, ctypes.byref(j), ctypes.byref(r), ctypes.byref(b)), ctx)
    return dict(level=j.value, rows=r.value, bytes=b.value)


def mgm_nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().mgm_nccl_unique_id(buf), None)
    return buf.raw


def mgm_dist_attach(ctx, rank: int, nranks: int, nccl_id: bytes):
    buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
    _check(load_library().mgm_dist_attach(ctx, rank, nranks, buf), ctx)


def mgm_local_rows(ctx) -> np.ndarray:
    """Original point ids of the rows this rank owns, in the order of its local vectors."""
    n = _i64()
    _check(load_library().mgm_local_rows(ctx, ctypes.byref(n), None), ctx)
    ids = np.empty(n.value, dtype=np.int64)
    _check(load_library().mgm_local_rows(ctx, ctypes.byref(n), _ptr(ids, _i64p)), ctx)
    return ids


def mgm_dist_info(ctx) -> dict:
    d, g, h = ctypes.c_int(), _i64(), _i64()
    _check(load_library().mgm_dist_info(ctx, ctypes.byref(d), ctypes.byref(g), ctypes.byref(h)), ctx)
    return dict(dist_levels=d.value, ghosts=g.value, halo_values_per_vcycle=h.value)


def mgm_dist_comm_time(ctx, reps: int = 20, stream=None) -> dict:
    """Collective: device time of one V-cycle's halos + all-gather (no compute) and of one
    16-double allreduce, this rank."""
    h, a = ctypes.c_double(), ctypes.c_double()
    _check(load_library().mgm_dist_comm_time(ctx, reps, ctypes.byref(h), ctypes.byref(a),
                                             _vp(_stream_ptr(stream))), ctx)
    return dict(halo_ms_per_vcycle=h.value, allreduce_us=a.value)


def mgm_fake_group_create(nranks: int):
    g = _vp()
    _check(load_library().mgm_fake_group_create(nranks, ctypes.byref(g)))
    return g


def mgm_fake_group_destroy(group):
    load_library().mgm_fake_group_destroy(group)


def mgm_dist_attach_fake(ctx, rank: int, group):
    _check(load_library().mgm_dist_attach_fake(ctx, rank, group), ctx)


def mgm_trace_read(ctx):
    """Stage stamps of the last V-cycle (MGM_TRACE set at setup): list of (label, ns)."""
    buf = (ctypes.c_uint64 * 256)()
    n = ctypes.c_int()
    lab = ctypes.create_string_buffer(16384)
    _check(load_library().mgm_trace_read(ctx, buf, 256, ctypes.byref(n), lab, 16384), ctx)
    labels = lab.value.decode().split("\n")
    return [(labels[i], int(buf[i])) for i in range(n.value)]


def mgm_bottom_trace_read(ctx):
    """Phase start stamps of the one-kernel bottom (MGM_TRACE): (stamps ns, meta[n,4])."""
    buf = (ctypes.c_uint64 * 8192)()
    meta = np.zeros((4096, 4), dtype=np.int32)
    n = ctypes.c_int()
    _check(load_library().mgm_bottom_trace_read(ctx, buf, 8192, ctypes.byref(n), meta.ctypes.data_as(_i32p)), ctx)
    k = n.value
    return np.array(buf[:k], dtype=np.uint64), meta[:k]


def mgm_bottom_ftrace_read(ctx):
    """Fine per-phase clock timeline of the bottom kernel (MGM_TRACE=2): int64 [2, n, 8]."""
    cap = 1024
    clk = np.zeros((2, cap, 8), dtype=np.int64)
    n = ctypes.c_int()
    _check(load_library().mgm_bottom_ftrace_read(ctx, clk.ctypes.data_as(_i64p), cap, ctypes.byref(n)), ctx)
    return clk[:, :n.value]


def mgm_host_morton(points):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    perm = np.empty(len(pts), dtype=np.int64)
    _check(load_library().mgm_host_morton(_ptr(pts, _f64p), len(pts), _ptr(perm, _i64p)))
    return perm


def mgm_host_knn(points, queries, k):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    q = np.ascontiguousarray(queries, dtype=np.float64)
    out = np.empty((len(q), k), dtype=np.int32)
    _check(load_library().mgm_host_knn(_ptr(pts, _f64p), len(pts), _ptr(q, _f64p), len(q), k,
                                       _ptr(out, _i32p)))
    return out


def mgm_device_knn(points, queries, k):
    """The kNN lists of mgm_host_knn computed by the GPU path of mgm_setup (k <= 64)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    q = np.ascontiguousarray(queries, dtype=np.float64)
    out = np.empty((len(q), k), dtype=np.int32)
    _check(load_library().mgm_device_knn(_ptr(pts, _f64p), len(pts), _ptr(q, _f64p), len(q), k,
                                         _ptr(out, _i32p)))
    return out


def mgm_host_wse(points, nt):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    keep = np.empty(nt, dtype=np.int64)
    _check(load_library().mgm_host_wse(_ptr(pts, _f64p), len(pts), nt, _ptr(keep, _i64p)))
    return keep


def mgm_device_wse(points, nt):
    """The survivors of mgm_host_wse computed by the GPU path of mgm_setup."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    keep = np.empty(nt, dtype=np.int64)
    _check(load_library().mgm_device_wse(_ptr(pts, _f64p), len(pts), nt, _ptr(keep, _i64p)))
    return keep


def mgm_host_colouring(ptr, col):
    ptr = np.ascontiguousarray(ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    n = len(ptr) - 1
    c = np.empty(n, dtype=np.int32)
    nc = ctypes.c_int()
    _check(load_library().mgm_host_colouring(n, _ptr(ptr, _i64p), _ptr(col, _i32p), _ptr(c, _i32p),
                                             ctypes.byref(nc)))
    return c, nc.value


def mgm_host_partition_level(L_ptr, L_col, colour, ncol, owner, nranks, rank, P=None, owner_c=None,
                             Pf=None, owner_f=None):
    """Partition tables of one level (the host code of mgm_dist_attach).  L_ptr/L_col: pattern
    of L_j in lib order; P = (ptr, col, nc) of P_j with owner_c; Pf = (ptr, col, nf) of P_{j-1}
    with owner_f.  Returns a dict of numpy arrays (see include/mgm.h)."""
    i64a = lambda a: np.ascontiguousarray(a, dtype=np.int64)
    i32a = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    n = len(L_ptr) - 1
    Lp, Lc, col, ow = i64a(L_ptr), i32a(L_col), i32a(colour), i32a(owner)
    args = [n, _ptr(Lp, _i64p), _ptr(Lc, _i32p), _ptr(col, _i32p), int(ncol), _ptr(ow, _i32p)]
    keep = [Lp, Lc, col, ow]
    if P is not None:
        pp, pc, nc = i64a(P[0]), i32a(P[1]), int(P[2])
        oc = i32a(owner_c)
        keep += [pp, pc, oc]
        args += [nc, _ptr(pp, _i64p), _ptr(pc, _i32p), _ptr(oc, _i32p)]
    else:
        args += [0, None, None, None]
    if Pf is not None:
        fp, fc, nf = i64a(Pf[0]), i32a(Pf[1]), int(Pf[2])
        of = i32a(owner_f)
        keep += [fp, fc, of]
        args += [nf, _ptr(fp, _i64p), _ptr(fc, _i32p), _ptr(of, _i32p)]
    else:
        args += [0, None, None, None]
    nr, ng, npr = _i64(), _i64(), ctypes.c_int()
    rows = np.empty(n, dtype=np.int64)
    ghosts = np.empty(n, dtype=np.int64)
    peers = np.empty(nranks, dtype=np.int32)
    send_rows = np.empty(n, dtype=np.int64)
    soff = np.zeros(nranks + 1, dtype=np.int64)
    roff = np.zeros(nranks + 1, dtype=np.int64)
    scoff = np.zeros(nranks * (ncol + 1), dtype=np.int64)
    rcoff = np.zeros(nranks * (ncol + 1), dtype=np.int64)
    _check(load_library().mgm_host_partition_level(
        *args, nranks, rank, ctypes.byref(nr), _ptr(rows, _i64p), ctypes.byref(ng), _ptr(ghosts, _i64p),
        ctypes.byref(npr), _ptr(peers, _i32p), _ptr(send_rows, _i64p), _ptr(soff, _i64p), _ptr(roff, _i64p),
        _ptr(scoff, _i64p), _ptr(rcoff, _i64p)))
    k = npr.value
    return dict(rows=rows[:nr.value], ghosts=ghosts[:ng.value], peers=peers[:k], send_rows=send_rows[:soff[k]],
                send_off=soff[:k + 1], recv_off=roff[:k + 1], send_coff=scoff[:k * (ncol + 1)].reshape(k, ncol + 1),
                recv_coff=rcoff[:k * (ncol + 1)].reshape(k, ncol + 1))


# ---------------------------------------------------------------- convenience wrapper
class MGM:
    """Owns one libmgm context.  Vectors are torch CUDA float64 tensors in original order."""

    def __init__(self, points, normals, stencil: dict, levels: dict, torch_memory: bool = False):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("libmgm needs a CUDA device")
        self.n = len(points)
        self.stencil, self.levels = dict(stencil), dict(levels)
        self._alloc = torch_allocator() if torch_memory else None
        self.ctx = mgm_setup(points, normals, stencil, levels, allocator=self._alloc)
        self.p = mgm_num_levels(self.ctx)

    def close(self):
        if getattr(self, "ctx", None) is not None:
            mgm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def vcycle(self, f, u, stream=None):
        mgm_vcycle(self.ctx, f, u, stream)
        return u

    def solve(self, rhs, x=None, tol=1e-10, maxit=500, krylov=1, stream=None, x0=None):
        import torch

        if x is None:
            x = torch.empty_like(rhs)
        rep = mgm_solve(self.ctx, rhs, x, tol, maxit, krylov, stream, x0=x0)
        return x, rep

    def level_info(self):
        return [mgm_level_info(self.ctx, j) for j in range(self.p)]

    def attach_dist(self, group=None):
        """Make vcycle/solve collective over the torch.distributed process group (one rank
        per GPU; every rank built this MGM from the same cloud).  Rank 0 creates the NCCL id,
        torch.distributed broadcasts it (marshalling only), libmgm creates the communicator."""
        import torch.distributed as dist

        rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        obj = [mgm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        mgm_dist_attach(self.ctx, rank, nranks, obj[0])
        self.rank, self.nranks = rank, nranks
        self.local_ids = mgm_local_rows(self.ctx)

    def attach_fake(self, rank: int, group):
        """Test hook: join an in-process group of fake ranks on one GPU (mgm_dist_attach_fake)."""
        mgm_dist_attach_fake(self.ctx, rank, group)
        self.local_ids = mgm_local_rows(self.ctx)
