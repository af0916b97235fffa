"""Pins of the oracle's operators: RBF-FD / GFD weights (O4/O5), PHS transfers
(O9), Galerkin product (O10), colouring + GS smoother (O11/O12,
P:285-291) and the dense coarse LU (O13)."""
import json
import os

import numpy as np
import pytest

import oracle as O
import mgm_inputs as MI

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _plane_stencil(offsets, h, normal_axis=2):
    off = np.asarray(offsets, dtype=np.float64) * h
    pts = np.zeros((len(off), 3))
    ax = [a for a in range(3) if a != normal_axis]
    pts[:, ax[0]] = off[:, 0]
    pts[:, ax[1]] = off[:, 1]
    nrm = np.zeros((len(off), 3))
    nrm[:, normal_axis] = 1.0
    return pts, nrm


# ---------------------------------------------------------------- weights (O4/O5)
@pytest.mark.parametrize("h", [1.0, 0.01])
def test_six_point_worked_example(h):
    g = GOLD["six_point_stencil"]
    pts, nrm = _plane_stencil(g["offsets"], h)
    sten = np.arange(6)[None, :]
    want = np.array(g["weights_times_h2"], dtype=np.float64) / h ** 2
    for k in (1, 2):
        w = O.rbffd_weights(pts, nrm, sten, 2, k)[0]
        # sten row 0 is centred at point 0; the saddle with n = L reduces to P^T c = Lap p
        assert np.abs(w - want).max() <= 1e-9 * np.abs(want).max()
    # GFD with n = L is interpolation: same weights
    allst = np.stack([np.arange(6)] * 6)
    wg = O.gfd_weights(pts, nrm, allst, 2, 4.0)[0]
    assert np.abs(wg - want).max() <= 1e-9 * np.abs(want).max()


def _monomials(xy, ell):
    cols = []
    for d in range(ell + 1):
        for i in range(d, -1, -1):
            cols.append(xy[..., 0] ** i * xy[..., 1] ** (d - i))
    return np.stack(cols, -1)


@pytest.mark.parametrize("method,ell,k,n", [("rbf", 2, 1, 15), ("rbf", 3, 2, 30),
                                            ("rbf", 4, 3, 50), ("gfd", 2, 0, 20)])
def test_polynomial_exactness_on_tangent_plane(method, ell, k, n):
    x, nrm = MI.fibonacci_sphere(3000, jitter=0.1, seed=7)
    st = O.knn(x, x, n)
    w = O.rbffd_weights(x, nrm, st, ell, k) if method == "rbf" else \
        O.gfd_weights(x, nrm, st, ell, 4.0)
    xh = O.tangent_project(x, nrm, st)
    Pm = _monomials(xh, ell)                       # (N, n, L)
    got = np.einsum("ij,ijl->il", w, Pm)
    want = np.zeros(Pm.shape[2])
    c = 0
    for d in range(ell + 1):
        for i in range(d, -1, -1):
            if d == 2 and i in (0, 2):
                want[c] = 2.0
            c += 1
    scale = np.einsum("ij,ijl->il", np.abs(w), np.abs(Pm)) + 1.0
    assert (np.abs(got - want) / scale).max() < 1e-10
    assert np.abs(w.sum(1)).max() < 1e-10 * np.abs(w).sum(1).max()   # zero row sums


def test_weights_invariant_under_rigid_rotation():
    x, nrm = MI.fibonacci_sphere(800, jitter=0.1, seed=1)
    st = O.knn(x, x, 30)
    w0 = O.rbffd_weights(x, nrm, st, 3, 2)
    rng = np.random.default_rng(2)
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    w1 = O.rbffd_weights(x @ Q.T, nrm @ Q.T, st, 3, 2)
    assert np.abs(w0 - w1).max() < 1e-8 * np.abs(w0).max()


def test_laplace_beltrami_consistency_on_sphere():
    """Delta_S Y_l^m = -l(l+1) Y_l^m (textbook; P:638 example Y_5^4): the discrete error
    decreases under refinement."""
    errs = []
    for N in (1024, 4096, 16384):
        x, nrm = MI.fibonacci_sphere(N)
        st = O.knn(x, x, 30)
        w = O.rbffd_weights(x, nrm, st, 3, 2)
        y = MI.sph_harm_cos(x, 5, 4)
        Dy = (w * y[st]).sum(1)
        errs.append(np.abs(Dy + 30.0 * y).max() / np.abs(30.0 * y).max())
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 1e-2
    assert errs[0] / errs[2] > 4.0       # at least ~first order in h


def test_y54_closed_form():
    rng = np.random.default_rng(0)
    x = rng.normal(size=(50, 3)); x /= np.linalg.norm(x, axis=1, keepdims=True)
    g = GOLD["y54"]
    ref = x[:, 2] * (x[:, 0] ** 4 - 6 * x[:, 0] ** 2 * x[:, 1] ** 2 + x[:, 1] ** 4)
    assert np.allclose(MI.sph_harm_cos(x, g["l"], g["m"]), g["scale_vs_generator"] * ref,
                       rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- transfers (O9)
def test_interp_closed_forms():
    # m = 2, x on the segment: linear interpolation d = (s2, s1)/r
    y = np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0]])
    x = np.array([[0.5, 0.0, 0.0]])
    P = O.interp_operator(x, y, 2).dense()[0]
    assert np.allclose(P, [1.5 / 2, 0.5 / 2], atol=1e-15)
    # m = 3, centroid of an equilateral triangle: 1/3 each
    y = np.array([[1.0, 0, 0], [-0.5, np.sqrt(3) / 2, 0], [-0.5, -np.sqrt(3) / 2, 0]])
    P = O.interp_operator(np.zeros((1, 3)), y, 3).dense()[0]
    assert np.allclose(P, 1.0 / 3.0, atol=1e-14)
    # coincident fine/coarse point reproduces the coarse value exactly
    P = O.interp_operator(y[1:2], y, 3)
    assert P.nnz == 1 and P.idx[0] == 1 and P.val[0] == 1.0


def test_interp_row_sums_and_transpose():
    x, _ = MI.fibonacci_sphere(2048, jitter=0.1, seed=3)
    keep = O.wse(x, 512)
    P = O.interp_operator(x, x[keep], 6)
    rs = np.add.reduceat(P.val, P.ptr[:-1])
    assert np.abs(rs - 1.0).max() < 1e-12
    R = P.transpose()
    assert np.array_equal(R.transpose().idx, P.idx) and np.array_equal(R.transpose().val, P.val)
    assert np.array_equal(R.dense(), P.dense().T)
    # coarse points are reproduced exactly (rows of kept points are unit vectors)
    Pd = P.dense()
    assert np.array_equal(Pd[keep], np.eye(512))


# ---------------------------------------------------------------- Galerkin (O10)
def _small_hierarchy(problem=0, N=1024, method=0):
    x, nrm = MI.fibonacci_sphere(N, jitter=0.1, seed=11)
    st = dict(method=method, poly_degree=2, phs_k=1, stencil_n=15, problem=problem, mu=1.0)
    if method == 1:
        st.update(stencil_n=20)
    return O.Oracle(x, nrm, st, dict(num_levels=4, interp_m=6))


def test_galerkin_equals_dense_triple_product():
    h = _small_hierarchy()
    for j in range(h.p - 1):
        lv, nx = h.levels[j], h.levels[j + 1]
        ref = lv.R.dense() @ lv.L.dense() @ lv.P.dense()
        got = nx.L.dense()
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
        # pattern = boolean product pattern (symbolic, nothing dropped)
        B = ((lv.R.dense() != 0).astype(int) @ (lv.L.dense() != 0).astype(int)
             @ (lv.P.dense() != 0).astype(int)) > 0
        pat = np.zeros_like(B)
        rows = np.repeat(np.arange(nx.N), np.diff(nx.L.ptr))
        pat[rows, nx.L.idx] = True
        assert np.array_equal(B, pat)


def test_galerkin_nullspace_invariants():
    hp = _small_hierarchy(problem=1)
    for lv in hp.levels:
        one = np.ones(lv.N)
        nrm = np.abs(lv.L.val).max()
        assert np.abs(lv.L.matvec(one)).max() < 1e-11 * nrm * 30
    hs = _small_hierarchy(problem=0)
    G = np.eye(hs.levels[0].N)
    for j, lv in enumerate(hs.levels):
        one = np.ones(lv.N)
        assert np.allclose(lv.L.matvec(one), G @ one, rtol=0, atol=1e-11 * np.abs(lv.L.val).max() * 30)
        if lv.P is not None:
            assert np.abs(lv.P.matvec(np.ones(lv.P.shape[1])) - 1.0).max() < 1e-12
            G = lv.R.dense() @ G @ lv.P.dense()


def test_poisson_border_vectors():
    hp = _small_hierarchy(problem=1)
    for j in range(hp.p - 1):
        lv, nx = hp.levels[j], hp.levels[j + 1]
        # coarse border I_h^H b_h^T = P^T c; total mass preserved: 1^T c_{j+1} = 1^T c_j
        assert np.allclose(nx.c, lv.P.dense().T @ lv.c, rtol=1e-14, atol=1e-14)
        assert abs(nx.c.sum() - lv.c.sum()) < 1e-9 * lv.N


# ---------------------------------------------------------------- colouring + GS (O11/O12)
def test_gs_hand_examples():
    g = GOLD["gs_hand_example"]
    A = O.CSR(np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([2., 1., 1., 2.]), (2, 2))
    u = np.zeros(2)
    O.gs_sweep(A, np.array([0, 1]), np.array(g["f"], dtype=float), u)
    assert np.array_equal(u, np.array(g["u"]))
    I = O.CSR(np.arange(4), np.arange(3), np.ones(3), (3, 3))
    u = np.array([5., -1., 2.])
    f = np.array([1., 2., 3.])
    O.gs_sweep(I, np.arange(3), f, u)
    assert np.array_equal(u, f)


def test_gs_lower_triangular_one_sweep():
    rng = np.random.default_rng(0)
    n = 30
    Ld = np.tril(rng.uniform(-1, 1, (n, n)) * (rng.uniform(size=(n, n)) < 0.3)) + 4 * np.eye(n)
    rows, cols = np.nonzero(Ld)
    ptr = np.zeros(n + 1, dtype=np.int64); np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    A = O.CSR(ptr, cols.astype(np.int64), Ld[rows, cols], (n, n))
    f = rng.normal(size=n)
    u = np.zeros(n)
    O.gs_sweep(A, np.arange(n, dtype=np.int64), f, u)
    assert np.allclose(u, np.linalg.solve(Ld, f), rtol=1e-13, atol=1e-13)


def _pattern_csr(n, edges):
    rows = [[i] for i in range(n)]
    for a, b in edges:
        rows[a].append(b)
    ptr = np.zeros(n + 1, dtype=np.int64)
    idx = []
    for i, r in enumerate(rows):
        r = sorted(set(r))
        idx += r
        ptr[i + 1] = len(idx)
    return O.CSR(ptr, np.array(idx, dtype=np.int64), np.ones(len(idx)), (n, n))


def test_dsatur_known_chromatic_numbers():
    """DSATUR is exact on bipartite graphs (Brelaz 1979): a 7x9 grid takes 2 colours, as does
    an even cycle; an odd cycle takes 3, the complete graph K_6 takes 6, a wheel with an odd
    rim (W_7) takes 4.  The iterated passes keep these counts."""
    grid = [(r * 9 + c, r * 9 + c + 1) for r in range(7) for c in range(8)] + \
           [(r * 9 + c, (r + 1) * 9 + c) for r in range(6) for c in range(9)]
    cases = [(63, grid, 2), (10, [(i, (i + 1) % 10) for i in range(10)], 2),
             (9, [(i, (i + 1) % 9) for i in range(9)], 3),
             (6, [(i, j) for i in range(6) for j in range(6) if i < j], 6),
             (8, [(i, (i % 7) + 1 if i < 7 else 1) for i in range(1, 8)] + [(0, i) for i in range(1, 8)], 4)]
    for n, edges, chi in cases:
        A = _pattern_csr(n, edges)   # one direction only: the colouring symmetrises the pattern
        for passes in (0, 10):
            col, nc = O.greedy_colour(A, passes=passes)
            assert nc == chi, (n, passes, nc)
            for a, b in edges:
                assert col[a] != col[b]


def test_colouring_proper_and_multicolour_gs_is_dense_gs():
    h = _small_hierarchy()
    for lv in h.levels[:-1]:
        A = lv.L.dense()
        S = (A != 0) | (A.T != 0)
        np.fill_diagonal(S, False)
        i, j = np.nonzero(S)
        assert not np.any(lv.colour[i] == lv.colour[j])          # proper
        # any greedy colouring (in whatever visiting order) is complete: a vertex of colour c
        # has neighbours of every colour 0..c-1 (it got c because those were taken)
        for v in range(lv.N):
            assert set(range(lv.colour[v])) <= set(lv.colour[S[v]].tolist())
        # plain greedy (passes < 0) in index (Morton) order: each vertex takes the smallest
        # colour not used by its lower-index neighbours
        c0, _ = O.greedy_colour(lv.L, passes=-1)
        for v in range(0, lv.N, 37):
            nb = np.flatnonzero(S[v]); nb = nb[nb < v]
            used = set(c0[nb].tolist())
            c = 0
            while c in used:
                c += 1
            assert c0[v] == c
        # iterated-greedy passes never add colours to the DSATUR colouring (Culberson)
        _, nd = O.greedy_colour(lv.L, passes=0)
        assert lv.ncolours <= nd and lv.ncolours == lv.colour.max() + 1
        # multicolour GS = forward GS on the colour-major permuted matrix (textbook form)
        rng = np.random.default_rng(1)
        f = rng.uniform(-1, 1, lv.N)
        u0 = rng.uniform(-1, 1, lv.N)
        u = u0.copy()
        O.gs_sweep(lv.L, lv.order, f, u)
        Pm = np.eye(lv.N)[lv.order]
        Ap = Pm @ A @ Pm.T
        ref = u0 + Pm.T @ np.linalg.solve(np.tril(Ap), Pm @ (f - A @ u0))
        assert np.abs(u - ref).max() <= 1e-12 * np.abs(ref).max()


def test_gs_reduces_residual_diagonally_dominant():
    rng = np.random.default_rng(4)
    n = 30
    Ad = rng.uniform(-1, 1, (n, n)) * (rng.uniform(size=(n, n)) < 0.3)
    Ad += np.diag(np.abs(Ad).sum(1) + 1.0)
    rows, cols = np.nonzero(Ad)
    ptr = np.zeros(n + 1, dtype=np.int64); np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    A = O.CSR(ptr, cols.astype(np.int64), Ad[rows, cols], (n, n))
    f = rng.normal(size=n)
    u = np.zeros(n)
    prev = np.linalg.norm(f)
    for _ in range(5):
        O.gs_sweep(A, np.arange(n, dtype=np.int64), f, u)
        r = np.linalg.norm(f - Ad @ u)
        assert r < prev
        prev = r


def test_dense_lu_examples():
    LU, piv = O.dense_lu(np.array([[2., 1.], [1., 3.]]))
    assert np.allclose(O.dense_lu_solve(LU, piv, np.array([3., 4.])), [1., 1.], atol=1e-15)
    rng = np.random.default_rng(0)
    A = rng.normal(size=(50, 50)) + 10 * np.eye(50)
    b = rng.normal(size=50)
    LU, piv = O.dense_lu(A)
    x = O.dense_lu_solve(LU, piv, b)
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12
    with pytest.raises(O.OracleError):
        O.dense_lu(np.array([[1., 2.], [2., 4.]]))
