"""MGM oracle -- TEST INFRASTRUCTURE ONLY (arXiv 2204.06154, "Meshfree geometric multilevel").

A plain, slow, single-threaded CPU implementation of what the MGM solve path computes,
written from PAPER.md (cited as P:<line>) and the readings of DESIGN.md / SURVEY.md 8(c)
(cited as O1..O17).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It shares no code
with ``paper_2204_06154_b200`` (the CUDA library); the product path never calls it.

Layout: ``oracle/_core.c`` holds the C primitives (compiled -O2 -ffp-contract=off into
``oracle/_core.so``); this module strings them together in the paper's order:
Alg. 2 (preprocessing) in :class:`Oracle.__init__`, Alg. 3 (V-cycle)
in :meth:`Oracle.vcycle_level_order`, right-preconditioned GMRES in
:meth:`Oracle.gmres` and the standalone solver in :meth:`Oracle.standalone`.

Parity status: every function here is pinned by tests/test_oracle_*.py (see DESIGN.md
"Oracle pins"); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "_core.c")
_SO = os.path.join(_HERE, "_core.so")
_lib = None

i64p = ctypes.POINTER(ctypes.c_int64)
f64p = ctypes.POINTER(ctypes.c_double)
i32p = ctypes.POINTER(ctypes.c_int32)
u8p = ctypes.POINTER(ctypes.c_uint8)


def build_oracle(force: bool = False) -> str:
    """Compile oracle/_core.c -> oracle/_core.so (plain gcc, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c99",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        _lib = ctypes.CDLL(_SO)
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


class OracleError(RuntimeError):
    def __init__(self, code, index, msg):
        super().__init__(f"{msg} (code {code}, index {index})")
        self.code, self.index = code, index


# ----------------------------------------------------------------------------------------
# sparse matrices (CSR, int64 indices, columns ascending within each row)
# ----------------------------------------------------------------------------------------
@dataclass
class CSR:
    ptr: np.ndarray
    idx: np.ndarray
    val: np.ndarray
    shape: tuple

    @property
    def nnz(self):
        return int(self.ptr[-1])

    def dense(self):
        A = np.zeros(self.shape)
        for i in range(self.shape[0]):
            s, e = self.ptr[i], self.ptr[i + 1]
            A[i, self.idx[s:e]] += self.val[s:e]
        return A

    def matvec(self, x):
        y = np.empty(self.shape[0])
        lib().orc_spmv(ctypes.c_int64(self.shape[0]), _p(self.ptr, i64p), _p(self.idx, i64p),
                       _p(self.val, f64p), _p(np.ascontiguousarray(x, dtype=np.float64), f64p),
                       _p(y, f64p))
        return y

    def transpose(self):
        """Exact transpose (values copied bit for bit; P:205 restriction = interpolation^T)."""
        m, n = self.shape
        cnt = np.bincount(self.idx, minlength=n)
        ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(cnt, out=ptr[1:])
        rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(self.ptr))
        order = np.lexsort((rows, self.idx))
        return CSR(ptr, rows[order].copy(), self.val[order].copy(), (n, m))


def csr_from_rows(cols: np.ndarray, vals: np.ndarray, counts: np.ndarray, ncols: int) -> CSR:
    """Rows given as fixed-width lists with per-row lengths; sorted by column."""
    m, w = cols.shape
    ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    idx = np.empty(ptr[-1], dtype=np.int64)
    val = np.empty(ptr[-1])
    for i in range(m):
        c = counts[i]
        o = np.argsort(cols[i, :c], kind="stable")
        idx[ptr[i]:ptr[i + 1]] = cols[i, :c][o]
        val[ptr[i]:ptr[i + 1]] = vals[i, :c][o]
    return CSR(ptr, idx, val, (m, ncols))


def spgemm(A: CSR, B: CSR) -> CSR:
    """O10 symbolic+numeric product, full symbolic pattern (no zero dropping)."""
    m = A.shape[0]
    cp = np.zeros(m + 1, dtype=np.int64)
    L = lib()
    L.orc_spgemm(ctypes.c_int64(m), _p(A.ptr, i64p), _p(A.idx, i64p), _p(A.val, f64p),
                 ctypes.c_int64(B.shape[1]), _p(B.ptr, i64p), _p(B.idx, i64p), _p(B.val, f64p),
                 _p(cp, i64p), None, None)
    ci = np.empty(cp[-1], dtype=np.int64)
    cv = np.empty(cp[-1])
    L.orc_spgemm(ctypes.c_int64(m), _p(A.ptr, i64p), _p(A.idx, i64p), _p(A.val, f64p),
                 ctypes.c_int64(B.shape[1]), _p(B.ptr, i64p), _p(B.idx, i64p), _p(B.val, f64p),
                 _p(cp, i64p), _p(ci, i64p), _p(cv, f64p))
    return CSR(cp, ci, cv, (m, B.shape[1]))


# ----------------------------------------------------------------------------------------
# geometry primitives
# ----------------------------------------------------------------------------------------
def morton_perm(points: np.ndarray) -> np.ndarray:
    """O1: perm[new] = old (replaces RCM)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    perm = np.empty(len(pts), dtype=np.int64)
    rc = lib().orc_morton_perm(_p(pts, f64p), ctypes.c_int64(len(pts)), _p(perm, i64p))
    if rc:
        raise OracleError(rc, -1, "degenerate point cloud")
    return perm


def knn(points: np.ndarray, queries: np.ndarray, k: int) -> np.ndarray:
    """O2: the k nearest `points` of each query, ordered by (d2, index).
    Small cases: brute force.  Large: k-d tree candidates (scipy) re-ranked exactly by the
    O2 rule, with a brute-force fallback for any query whose k-th exact distance is not
    strictly inside the candidate radius."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    qry = np.ascontiguousarray(queries, dtype=np.float64)
    n, nq = len(pts), len(qry)
    out = np.empty((nq, k), dtype=np.int64)
    L = lib()
    if n * nq <= 4_000_000:
        L.orc_knn_brute(_p(pts, f64p), ctypes.c_int64(n), _p(qry, f64p), ctypes.c_int64(nq),
                        ctypes.c_int(k), _p(out, i64p))
        return out
    from scipy.spatial import cKDTree

    kc = min(n, k + 8)
    d, cand = cKDTree(pts).query(qry, k=kc, workers=-1)
    cand = np.ascontiguousarray(cand, dtype=np.int64)
    if kc < n:
        bound2 = (d[:, -1] * (1.0 - 1e-12)) ** 2
    else:
        bound2 = np.full(nq, np.inf)
    bound2 = np.ascontiguousarray(bound2)
    need = np.zeros(nq, dtype=np.uint8)
    L.orc_knn_rerank(_p(pts, f64p), ctypes.c_int64(n), _p(qry, f64p), ctypes.c_int64(nq),
                     ctypes.c_int(k), _p(cand, i64p), ctypes.c_int(kc), _p(bound2, f64p),
                     _p(out, i64p), _p(need, u8p))
    bad = np.flatnonzero(need)
    if len(bad):
        sub = np.ascontiguousarray(qry[bad])
        o2 = np.empty((len(bad), k), dtype=np.int64)
        L.orc_knn_brute(_p(pts, f64p), ctypes.c_int64(n), _p(sub, f64p),
                        ctypes.c_int64(len(bad)), ctypes.c_int(k), _p(o2, i64p))
        out[bad] = o2
    return out


def nn_dist2(points: np.ndarray) -> np.ndarray:
    """Squared distance (O2 rule) from each point to its nearest other point."""
    nb = knn(points, points, 2)
    d = points[nb[:, 1]] - points
    s = d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]
    return s + d[:, 2] * d[:, 2]


def tangent_project(points, normals, sten):
    pts = np.ascontiguousarray(points, dtype=np.float64)
    nrm = np.ascontiguousarray(normals, dtype=np.float64)
    st = np.ascontiguousarray(sten, dtype=np.int64)
    out = np.empty((st.shape[0], st.shape[1], 2))
    lib().orc_tangent_project(_p(pts, f64p), _p(nrm, f64p), _p(st, i64p),
                              ctypes.c_int64(st.shape[0]), ctypes.c_int(st.shape[1]),
                              _p(out, f64p))
    return out


def rbffd_weights(points, normals, sten, ell: int, k: int) -> np.ndarray:
    """O4 PHS RBF-FD Laplace-Beltrami weights."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    nrm = np.ascontiguousarray(normals, dtype=np.float64)
    st = np.ascontiguousarray(sten, dtype=np.int64)
    w = np.empty(st.shape)
    fail = ctypes.c_int64(-1)
    rc = lib().orc_rbffd_weights(_p(pts, f64p), _p(nrm, f64p), _p(st, i64p),
                                 ctypes.c_int64(st.shape[0]), ctypes.c_int(st.shape[1]),
                                 ctypes.c_int(ell), ctypes.c_int(k), _p(w, f64p),
                                 ctypes.byref(fail))
    if rc:
        raise OracleError(rc, fail.value, "RBF-FD stencil not unisolvent")
    return w


def stencil_radius(points, normals, sten) -> np.ndarray:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    nrm = np.ascontiguousarray(normals, dtype=np.float64)
    st = np.ascontiguousarray(sten, dtype=np.int64)
    rho = np.empty(st.shape[0])
    lib().orc_stencil_radius(_p(pts, f64p), _p(nrm, f64p), _p(st, i64p),
                             ctypes.c_int64(st.shape[0]), ctypes.c_int(st.shape[1]), _p(rho, f64p))
    return rho


def gfd_weights(points, normals, sten, ell: int, alpha: float) -> np.ndarray:
    """O5 GFD weights, QR of W^{1/2} P."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    nrm = np.ascontiguousarray(normals, dtype=np.float64)
    st = np.ascontiguousarray(sten, dtype=np.int64)
    rho = stencil_radius(pts, nrm, st)
    w = np.empty(st.shape)
    fail = ctypes.c_int64(-1)
    rc = lib().orc_gfd_weights(_p(pts, f64p), _p(nrm, f64p), _p(st, i64p),
                               ctypes.c_int64(st.shape[0]), ctypes.c_int(st.shape[1]),
                               ctypes.c_int(ell), ctypes.c_double(alpha), _p(rho, f64p),
                               _p(w, f64p), ctypes.byref(fail))
    if rc:
        raise OracleError(rc, fail.value, "GFD stencil rank deficient")
    return w


def wse(points: np.ndarray, nt: int) -> np.ndarray:
    """O8 weighted sample elimination to nt points; survivors in index order."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    nn2 = np.ascontiguousarray(nn_dist2(pts))
    keep = np.empty(nt, dtype=np.int64)
    rc = lib().orc_wse(_p(pts, f64p), ctypes.c_int64(len(pts)), ctypes.c_int64(nt),
                       _p(nn2, f64p), _p(keep, i64p))
    if rc:
        raise OracleError(rc, -1, "WSE failed")
    return keep


def interp_operator(fine: np.ndarray, coarse: np.ndarray, m: int) -> CSR:
    """O9 PHS (r + constant) interpolation I_H^h, N_h x N_H CSR."""
    fine = np.ascontiguousarray(fine, dtype=np.float64)
    coarse = np.ascontiguousarray(coarse, dtype=np.float64)
    st = knn(coarse, fine, m)
    w = np.empty(st.shape)
    cnt = np.empty(len(fine), dtype=np.int32)
    fail = ctypes.c_int64(-1)
    rc = lib().orc_interp_weights(_p(fine, f64p), ctypes.c_int64(len(fine)), _p(coarse, f64p),
                                  _p(st, i64p), ctypes.c_int(m), _p(w, f64p), _p(cnt, i32p),
                                  ctypes.byref(fail))
    if rc:
        raise OracleError(rc, fail.value, "singular transfer system")
    return csr_from_rows(st, w, cnt.astype(np.int64), len(coarse))


COLOUR_PASSES = 10   # O11: iterated-greedy passes after the first greedy pass


def greedy_colour(A: CSR, passes: int = COLOUR_PASSES):
    """O11 colouring of sym(pattern(A)) minus diagonal: DSATUR (largest saturation first, ties
    by larger degree then lower index; smallest free colour), then ``passes`` iterated-greedy
    passes (vertices by descending previous colour, ties by index; each gives the smallest
    colour unused by neighbours coloured earlier in the pass).  ``passes < 0``: plain greedy
    in index (Morton) order."""
    T = A.transpose()
    col = np.empty(A.shape[0], dtype=np.int32)
    nc = ctypes.c_int32(0)
    rc = lib().orc_greedy_colour(ctypes.c_int64(A.shape[0]), _p(A.ptr, i64p), _p(A.idx, i64p),
                                 _p(T.ptr, i64p), _p(T.idx, i64p), ctypes.c_int(passes), _p(col, i32p),
                                 ctypes.byref(nc))
    if rc:
        raise OracleError(rc, -1, "too many colours")
    return col, int(nc.value)


def rcm_order(A: CSR) -> np.ndarray:
    """Reverse Cuthill-McKee ordering of sym(pattern(A)) (scipy's implementation):
    the row order of the paper's lexicographic Gauss-Seidel (calibration variant)."""
    import scipy.sparse as sps
    from scipy.sparse.csgraph import reverse_cuthill_mckee

    n = A.shape[0]
    M = sps.csr_matrix((np.ones(len(A.idx)), A.idx, A.ptr), shape=(n, n))
    return np.ascontiguousarray(reverse_cuthill_mckee((M + M.T).tocsr(), symmetric_mode=True), dtype=np.int64)


def gs_sweep(A: CSR, order: np.ndarray, f, u, backward=False, c=None, lam=0.0):
    """O12 one GS sweep in the given row order, in place on u."""
    fail = ctypes.c_int64(-1)
    cptr = _p(c, f64p) if c is not None else None
    rc = lib().orc_gs_sweep(ctypes.c_int64(A.shape[0]), _p(A.ptr, i64p), _p(A.idx, i64p),
                            _p(A.val, f64p), _p(order, i64p), ctypes.c_int(1 if backward else 0),
                            _p(f, f64p), _p(u, f64p), cptr, ctypes.c_double(lam),
                            ctypes.byref(fail))
    if rc:
        raise OracleError(rc, fail.value, "zero or missing diagonal")


def dense_lu(A: np.ndarray):
    LU = np.ascontiguousarray(A, dtype=np.float64).copy()
    m = LU.shape[0]
    piv = np.empty(m, dtype=np.int32)
    fail = ctypes.c_int64(-1)
    rc = lib().orc_dense_lu(_p(LU, f64p), ctypes.c_int(m), _p(piv, i32p), ctypes.byref(fail))
    if rc:
        raise OracleError(rc, fail.value, "singular coarse matrix")
    return LU, piv


def dense_lu_solve(LU, piv, b):
    x = np.ascontiguousarray(b, dtype=np.float64).copy()
    lib().orc_dense_lu_solve(_p(LU, f64p), ctypes.c_int(LU.shape[0]), _p(piv, i32p), _p(x, f64p))
    return x


# ----------------------------------------------------------------------------------------
# hierarchy (Alg. 2) and cycle (Alg. 3)
# ----------------------------------------------------------------------------------------
@dataclass
class Level:
    X: np.ndarray            # points of this level, level (inherited Morton) order
    ids: np.ndarray          # original point index of each row
    L: CSR                   # operator L_j
    P: CSR | None = None     # I_{j+1}^j  (N_j x N_{j+1})
    R: CSR | None = None     # I_j^{j+1} = P^T
    colour: np.ndarray | None = None
    ncolours: int = 0
    order: np.ndarray | None = None   # colour-major GS row order
    c: np.ndarray | None = None       # Poisson border vector c_j (c_1 = 1)

    @property
    def N(self):
        return len(self.X)


@dataclass
class Report:
    iterations: int = 0
    converged: bool = False
    final_rel_residual: float = float("nan")
    history: list = field(default_factory=list)
    lam: float = 0.0


DEFAULT_STENCIL = dict(method=0, poly_degree=2, phs_k=1, stencil_n=15, gfd_alpha=4.0,
                       problem=0, mu=1.0)
DEFAULT_LEVELS = dict(num_levels=0, n_min=250, coarsen_factor=4, interp_m=6, nu1=1, nu2=1,
                      smoother=0, restart=50)


def assemble_operator(sten, W, n, problem, mu) -> CSR:
    """L_h = I - mu D_h (shifted) or D_h (Poisson), P:67-72 (O6)."""
    ns = sten.shape[1]
    if problem == 0:
        vals = -(mu * W)
        vals[:, 0] = 1.0 - mu * W[:, 0]       # sten[:,0] is the centre itself (O2)
    else:
        vals = W.copy()
    return csr_from_rows(sten, vals, np.full(n, ns, dtype=np.int64), n)


class Oracle:
    """Reference MGM hierarchy + solvers.  Vectors at the public API are in the caller's
    original point order (like the C ABI); internally level order is Morton (O1)."""

    def __init__(self, points, normals, stencil: dict | None = None, levels: dict | None = None,
                 fine_weights=None):
        sp = dict(DEFAULT_STENCIL, **(stencil or {}))
        lp = dict(DEFAULT_LEVELS, **(levels or {}))
        self.sp, self.lp = sp, lp
        points = np.ascontiguousarray(points, dtype=np.float64)
        normals = np.ascontiguousarray(normals, dtype=np.float64)
        N1 = len(points)
        # Alg. 2 lines 2-3: re-order (Morton instead of RCM)
        self.perm = morton_perm(points)
        X = points[self.perm]
        nrm = normals[self.perm]
        # level count (Alg. 2 line 4) unless given explicitly (O7)
        p = lp["num_levels"]
        if p <= 0:
            p = int(np.floor(np.log(N1 / lp["n_min"]) / np.log(lp["coarsen_factor"]))) + 1
            p = max(p, 1)
        self.p = p
        # fine operator L_1
        ns = sp["stencil_n"]
        sten = knn(X, X, ns)
        self.stencil = sten
        if fine_weights is not None:  # experiments with other weight readings (Morton order rows)
            W = np.ascontiguousarray(fine_weights(X, nrm, sten), dtype=np.float64)
        elif sp["method"] == 0:
            W = rbffd_weights(X, nrm, sten, sp["poly_degree"], sp["phs_k"])
        else:
            W = gfd_weights(X, nrm, sten, sp["poly_degree"], sp["gfd_alpha"])
        self.weights = W
        L1 = assemble_operator(sten, W, N1, sp["problem"], sp["mu"])
        self.levels = [Level(X=X, ids=self.perm.copy(), L=L1)]
        if sp["problem"] == 1:
            self.levels[0].c = np.ones(N1)
        # Alg. 2 lines 5-12
        for j in range(p - 1):
            lv = self.levels[j]
            Nt = lv.N // lp["coarsen_factor"]
            keep = wse(lv.X, Nt)                                   # line 6
            Xc = lv.X[keep]
            lv.P = interp_operator(lv.X, Xc, lp["interp_m"])       # line 7
            lv.R = lv.P.transpose()                                # line 8
            Lc = spgemm(lv.R, spgemm(lv.L, lv.P))                  # line 9
            nxt = Level(X=Xc, ids=lv.ids[keep], L=Lc)
            if sp["problem"] == 1:
                nxt.c = lv.R.matvec(lv.c)                          # border I_h^H b^T
            self.levels.append(nxt)
        for lv in self.levels[:-1]:
            lv.colour, lv.ncolours = greedy_colour(lv.L, lp.get("colour_passes", COLOUR_PASSES))
            if lp.get("gs_order", "colour") == "rcm":
                # the paper's own smoother (Alg. 2 lines 2-3 and 11-12):
                # lexicographic Gauss-Seidel in reverse Cuthill-McKee order of L_j
                lv.order = rcm_order(lv.L)
            else:
                lv.order = np.lexsort((np.arange(lv.N), lv.colour)).astype(np.int64)
        # coarsest factorisation (Alg. 2 line 13, P:293 / P:354-355), dense (O13)
        last = self.levels[-1]
        Ad = last.L.dense()
        if sp["problem"] == 1:
            n = last.N
            A2 = np.zeros((n + 1, n + 1))
            A2[:n, :n] = Ad
            A2[:n, n] = last.c
            A2[n, :n] = last.c
            Ad = A2
        self.coarse_LU, self.coarse_piv = dense_lu(Ad)

    # -- vector helpers (Poisson vectors carry lambda as a trailing entry) ----------------
    @property
    def poisson(self):
        return self.sp["problem"] == 1

    def _smooth(self, lv: Level, f, u, nsweep, backward):
        for _ in range(nsweep):
            if self.poisson:
                lam = float(u[lv.N])
                uu = np.ascontiguousarray(u[:lv.N])
                gs_sweep(lv.L, lv.order, np.ascontiguousarray(f[:lv.N]), uu, backward, lv.c, lam)
                u[:lv.N] = uu
            else:
                gs_sweep(lv.L, lv.order, f, u, backward)

    def _residual(self, lv: Level, f, u):
        if self.poisson:
            n = lv.N
            r = np.empty(n + 1)
            r[:n] = f[:n] - lv.L.matvec(u[:n]) - lv.c * u[n]
            r[n] = f[n] - lv.c @ u[:n]
            return r
        return f - lv.L.matvec(u)

    def _restrict(self, lv: Level, r):
        if self.poisson:
            return np.concatenate([lv.R.matvec(r[:lv.N]), r[lv.N:]])
        return lv.R.matvec(r)

    def _interp(self, lv: Level, e):
        if self.poisson:
            return np.concatenate([lv.P.matvec(e[:-1]), e[-1:]])
        return lv.P.matvec(e)

    def coarse_solve(self, r):
        return dense_lu_solve(self.coarse_LU, self.coarse_piv, r)

    def apply_A(self, u):
        """Fine operator (augmented in Poisson mode: [L u + lam*1; 1^T u])."""
        return self._apply_level(0, u)

    def _apply_level(self, j, u):
        lv = self.levels[j]
        if self.poisson:
            n = lv.N
            y = np.empty(n + 1)
            y[:n] = lv.L.matvec(u[:n]) + lv.c * u[n]
            y[n] = lv.c @ u[:n]
            return y
        return lv.L.matvec(u)

    def vcycle_level_order(self, f, u):
        """Alg. 3 in level-1 (Morton) order; returns the new u (copy).
        Reading: P:392's "r^1 = I_1^2(f^1 - L_1 u^h)" is r^2 computed from u^1."""
        p, lp = self.p, self.lp
        nu1, nu2 = lp["nu1"], lp["nu2"]
        pre_bwd = lp["smoother"] == 1
        post_bwd = lp["smoother"] in (1, 2)
        f = np.ascontiguousarray(f, dtype=np.float64)
        u = np.array(u, dtype=np.float64, copy=True)
        if p == 1:
            return self.coarse_solve(f)
        lv = self.levels
        r = [None] * p
        e = [None] * p
        self._smooth(lv[0], f, u, nu1, pre_bwd)                          # line 4
        r[1] = self._restrict(lv[0], self._residual(lv[0], f, u))       # line 5
        for j in range(1, p - 1):                                        # lines 6-9
            e[j] = np.zeros_like(r[j])
            self._smooth(lv[j], r[j], e[j], nu1, pre_bwd)
            r[j + 1] = self._restrict(lv[j], self._residual(lv[j], r[j], e[j]))
        e[p - 1] = self.coarse_solve(r[p - 1])                           # line 10
        for j in range(p - 2, 0, -1):                                    # lines 11-14
            e[j] = e[j] + self._interp(lv[j], e[j + 1])
            self._smooth(lv[j], r[j], e[j], nu2, post_bwd)
        u = u + self._interp(lv[0], e[1])                                # line 15
        self._smooth(lv[0], f, u, nu2, post_bwd)                         # line 16
        return u

    # -- public API in original order ----------------------------------------------------
    def to_level(self, v):
        v = np.asarray(v, dtype=np.float64)
        out = v[self.perm] if not self.poisson else np.concatenate([v[self.perm], [0.0]])
        return np.ascontiguousarray(out)

    def from_level(self, v):
        n = self.levels[0].N
        out = np.empty(n)
        out[self.perm] = v[:n]
        return out

    def vcycle(self, f, u):
        """One V-cycle on original-order vectors (Poisson: lambda starts at 0 and is dropped)."""
        return self.from_level(self.vcycle_level_order(self.to_level(f), self.to_level(u)))

    def precondition(self, v):
        """M(v): one V-cycle with zero initial guess, level order."""
        return self.vcycle_level_order(v, np.zeros_like(v))

    def gmres(self, b, tol=1e-10, restart=None, maxit=500, x0=None):
        """MGM-preconditioned GMRES on the fine operator, level order."""
        x, rep = gmres(self.apply_A, self.precondition, b, tol=tol,
                       restart=restart or self.lp["restart"], maxit=maxit, x0=x0)
        if self.poisson:
            rep.lam = float(x[-1])
        return x, rep

    def standalone(self, f, tol=1e-10, maxit=200, x0=None):
        """MGM as a standalone solver (O16): u <- V-cycle(f, u) from u = 0 (or from the
        initial guess x0, the applications' warm start from the previous step)."""
        f = np.ascontiguousarray(f, dtype=np.float64)
        u = np.zeros_like(f) if x0 is None else np.array(x0, dtype=np.float64)
        rep = Report()
        fn = float(np.linalg.norm(f))
        if fn == 0.0:
            rep.converged, rep.final_rel_residual = True, 0.0
            return np.zeros_like(f), rep
        for it in range(1, maxit + 1):
            u = self.vcycle_level_order(f, u)
            rel = float(np.linalg.norm(f - self.apply_A(u))) / fn
            rep.history.append(rel)
            rep.iterations = it
            if rel <= tol:
                rep.converged = True
                break
        rep.final_rel_residual = rep.history[-1]
        if self.poisson:
            rep.lam = float(u[-1])
        return u, rep

    def bicgstab(self, b, tol=1e-10, maxit=500, x0=None):
        """MGM-preconditioned BiCGSTAB on the fine operator, level order."""
        x, rep = bicgstab(self.apply_A, self.precondition, b, tol=tol, maxit=maxit, x0=x0)
        if self.poisson:
            rep.lam = float(x[-1])
        return x, rep

    def solve(self, rhs, tol=1e-10, maxit=500, krylov=1, x0=None):
        """Public solve on original-order vectors (mirrors mgm_solve: krylov 0 standalone,
        1 GMRES, 2 BiCGSTAB; x0 the initial guess or None for 0)."""
        b = self.to_level(rhs)
        g = None if x0 is None else self.to_level(x0)
        if krylov == 1:
            x, rep = self.gmres(b, tol=tol, maxit=maxit, x0=g)
        elif krylov == 2:
            x, rep = self.bicgstab(b, tol=tol, maxit=maxit, x0=g)
        else:
            x, rep = self.standalone(b, tol=tol, maxit=maxit, x0=g)
        return self.from_level(x), rep


def gmres(apply_A, precond, b, tol=1e-10, restart=50, maxit=500, x0=None):
    """Right-preconditioned restarted GMRES with modified Gram-Schmidt and Givens rotations
    (O15).  Stops when |g_{k+1}|/||b|| <= tol; restarts every `restart`
    steps from the current x (r0 recomputed).  Iterations = preconditioner applications
    inside Arnoldi; the final x = x0 + M(V y) costs one more application."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    rep = Report()
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        rep.converged, rep.final_rel_residual = True, 0.0
        return np.zeros_like(b), rep
    its = 0
    while True:
        r = b - apply_A(x)
        beta = float(np.linalg.norm(r))
        if beta / bnorm <= tol or its >= maxit:
            rep.converged = beta / bnorm <= tol
            break
        V = [r / beta]
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        k_done = 0
        stop = False
        for k in range(restart):
            z = precond(V[k])
            w = apply_A(z)
            its += 1
            for i in range(k + 1):                    # modified Gram-Schmidt
                H[i, k] = float(w @ V[i])
                w = w - H[i, k] * V[i]
            H[k + 1, k] = float(np.linalg.norm(w))
            for i in range(k):                        # apply previous rotations
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            den = float(np.hypot(H[k, k], H[k + 1, k]))
            cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
            hk1 = H[k + 1, k]
            H[k, k], H[k + 1, k] = den, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            rep.history.append(abs(g[k + 1]) / bnorm)
            k_done = k + 1
            if abs(g[k + 1]) / bnorm <= tol or its >= maxit or hk1 == 0.0:
                stop = True
                break
            V.append(w / hk1)
        y = np.zeros(k_done)
        for i in range(k_done - 1, -1, -1):          # back substitution, H upper triangular
            s = g[i] - H[i, i + 1:k_done] @ y[i + 1:k_done]
            y[i] = s / H[i, i]
        Vy = np.zeros_like(b)
        for i in range(k_done):
            Vy += y[i] * V[i]
        x = x + precond(Vy)
        if stop:
            rep.converged = abs(g[k_done]) / bnorm <= tol
            break
    rep.iterations = its
    rep.final_rel_residual = float(np.linalg.norm(b - apply_A(x))) / bnorm
    return x, rep


def bicgstab(apply_A, precond, b, tol=1e-10, maxit=500, x0=None):
    """Right-preconditioned BiCGSTAB ([Saad] Alg. 7.7 applied to A M, x = M z), in the
    algorithm's order.  Iterations are counted as preconditioner applications, two per full
    step; the relative residual ||r||/||b|| is recorded after each half step (||s||)
    and full step (||r||), and the iteration stops at the first one <= tol.  Breakdown
    (|rho| or |omega| < 1e-30 relative): restart once from the current iterate with
    r_hat = r, then report non-convergence (SPEC S:508-516 reading, O18)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    rep = Report()
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        rep.converged, rep.final_rel_residual = True, 0.0
        return np.zeros_like(b), rep
    its = 0
    restarts = 0
    r = b - apply_A(x)
    while True:
        r_hat = r.copy()
        rho_prev = alpha = omega = 1.0
        v = np.zeros_like(b)
        p = np.zeros_like(b)
        broke = False
        while its < maxit:
            rho = float(r_hat @ r)
            if abs(rho) < 1e-30 * bnorm * bnorm:
                broke = True
                break
            beta = (rho / rho_prev) * (alpha / omega)
            p = r + beta * (p - omega * v)
            p_hat = precond(p)
            its += 1
            v = apply_A(p_hat)
            alpha = rho / float(r_hat @ v)
            s = r - alpha * v
            rel_s = float(np.linalg.norm(s)) / bnorm
            rep.history.append(rel_s)
            if rel_s <= tol:
                x = x + alpha * p_hat
                r = s
                rep.converged = True
                break
            s_hat = precond(s)
            its += 1
            t = apply_A(s_hat)
            tt = float(t @ t)
            omega = float(t @ s) / tt if tt > 0.0 else 0.0
            x = x + alpha * p_hat + omega * s_hat
            r = s - omega * t
            rel = float(np.linalg.norm(r)) / bnorm
            rep.history.append(rel)
            if rel <= tol:
                rep.converged = True
                break
            if abs(omega) < 1e-30:
                broke = True
                break
            rho_prev = rho
        if rep.converged or its >= maxit or not broke or restarts >= 1:
            break
        restarts += 1
    rep.iterations = its
    rep.final_rel_residual = float(np.linalg.norm(b - apply_A(x))) / bnorm
    return x, rep
