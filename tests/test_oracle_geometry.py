"""Pins of the oracle's discrete geometry: Morton order (O1), kNN (O2), tangent
projection (O3) and weighted sample elimination (O8)."""
import json
import os

import numpy as np
import pytest

import oracle as O
import mgm_inputs as MI

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


# ---------------------------------------------------------------- Morton (O1)
def _octant_sort(idx, pts, lo, size, depth):
    """Textbook recursive Z-order: split the cube into octants ordered by (x,y,z) bits
    (x most significant), recurse.  Independent of bit interleaving."""
    if depth == 0 or len(idx) <= 1:
        return list(sorted(idx))
    half = size / 2.0
    out = []
    for ox in (0, 1):
        for oy in (0, 1):
            for oz in (0, 1):
                c = lo + half * np.array([ox, oy, oz])
                sel = [i for i in idx if all(c[a] <= pts[i, a] < c[a] + half for a in range(3))]
                out += _octant_sort(sel, pts, c, half, depth - 1)
    return out


def test_morton_matches_recursive_octant_order():
    rng = np.random.default_rng(5)
    g = np.stack(np.meshgrid(*[np.arange(8)] * 3, indexing="ij"), -1).reshape(-1, 3)
    g = g[rng.permutation(len(g))].astype(np.float64)
    # grid on [0,7]^3, ext = 7 -> cells of width 7/2^21; compare with octant order on [0,8)
    pts = g.copy()
    perm = O.morton_perm(pts)
    # the quantisation maps coordinate c to floor(c/7*2^21); its top 3 bits equal the
    # octant bits of c on [0, 8) scaled by 8/7, so compare on the scaled cube
    ref = _octant_sort(list(range(len(pts))), pts * (8.0 / 7.0) * (1 - 1e-12), np.zeros(3), 8.0, 3)
    assert list(perm) == ref


def test_morton_corners_and_bijection():
    c = np.array([[x, y, z] for x in (0., 1.) for y in (0., 1.) for z in (0., 1.)])
    rng = np.random.default_rng(0)
    sh = rng.permutation(8)
    perm = O.morton_perm(c[sh])
    # Z-order of the unit cube corners is 4x + 2y + z
    codes = (4 * c[sh][perm, 0] + 2 * c[sh][perm, 1] + c[sh][perm, 2]).astype(int)
    assert list(codes) == list(range(8))
    x, _ = MI.fibonacci_sphere(3000)
    p = O.morton_perm(x)
    assert sorted(p) == list(range(3000))


# ---------------------------------------------------------------- kNN (O2)
def test_knn_grid_hand_example():
    g = np.stack(np.meshgrid(np.arange(10.), np.arange(10.), indexing="ij"), -1).reshape(-1, 2)
    pts = np.concatenate([g, np.zeros((100, 1))], 1)
    i = 4 * 10 + 5
    nb = O.knn(pts, pts[i:i + 1], 5)[0]
    assert nb[0] == i
    assert sorted(nb[1:]) == sorted([i - 10, i + 10, i - 1, i + 1])
    assert list(nb[1:]) == sorted(nb[1:])  # ties broken by index


def test_knn_tree_path_equals_brute_force():
    x, _ = MI.fibonacci_sphere(2500, jitter=0.1, seed=4)
    brute = np.empty((len(x), 12), dtype=np.int64)
    import ctypes
    O.lib().orc_knn_brute(O._p(x, O.f64p), ctypes.c_int64(len(x)), O._p(x, O.f64p),
                          ctypes.c_int64(len(x)), ctypes.c_int(12), O._p(brute, O.i64p))
    tree = O.knn(x, x, 12)   # 6.25e6 pairs > threshold -> k-d tree + exact re-rank
    assert np.array_equal(brute, tree)
    # independent brute force in numpy on a few rows
    for q in (0, 17, 1234, 2499):
        d = ((x - x[q]) ** 2).sum(1)
        ref = np.lexsort((np.arange(len(x)), d))[:12]
        assert np.array_equal(ref, brute[q])


# ---------------------------------------------------------------- tangent plane (O3)
def test_tangent_projection_centre_and_isometry():
    rng = np.random.default_rng(1)
    n = rng.normal(size=3)
    n /= np.linalg.norm(n)
    a = np.cross(n, [1.0, 0, 0]); a /= np.linalg.norm(a)
    b = np.cross(n, a)
    uv = rng.uniform(-1, 1, size=(10, 2))
    pts = 0.3 + uv[:, :1] * a + uv[:, 1:] * b           # planar stencil orthogonal to n
    nrm = np.tile(n, (10, 1))
    sten = np.arange(10)[None, :]
    xh = O.tangent_project(pts, nrm, sten)[0]
    assert np.allclose(xh[0], 0.0, atol=0.0)
    D3 = np.linalg.norm(pts[:, None] - pts[None], axis=2)
    D2 = np.linalg.norm(xh[:, None] - xh[None], axis=2)
    assert np.abs(D3 - D2).max() < 1e-14


def test_tangent_projection_contracts_on_sphere():
    x, nrm = MI.fibonacci_sphere(500)
    st = O.knn(x, x, 10)
    xh = O.tangent_project(x, nrm, st)
    d3 = np.linalg.norm(x[st] - x[:, None, :], axis=2)
    d2 = np.linalg.norm(xh, axis=2)
    assert (d2 <= d3 + 1e-15).all()


# ---------------------------------------------------------------- WSE (O8)
def _wse_brute(pts, nt):
    """Literal O(N^2) weighted sample elimination on tiny inputs (no grid, no heap), O8:
    integer weights (2^40 fixed point), ties to the lowest index, and a pass that would
    eliminate a zero-weight point restarts with R * 1.25."""
    n = len(pts)
    d = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(2))
    dd = d + np.diag(np.full(n, np.inf))
    nn = np.sort(dd.min(1))
    rh = 0.5 * nn[(n - 1) // 2]
    R = 2.0 * rh * np.sqrt(n / nt)
    for _ in range(16):
        W = [[0] * n for _ in range(n)]
        for i in range(n):
            for j in range(n):
                if i != j and d[i, j] < R:
                    u = 1.0 - d[i, j] / R
                    u2 = u * u
                    u4 = u2 * u2
                    W[i][j] = int(np.floor(u4 * u4 * 2.0 ** 40 + 0.5))
        weight = [sum(row) for row in W]
        alive = [True] * n
        ok = True
        for _ in range(n - nt):
            best = max((i for i in range(n) if alive[i]), key=lambda i: (weight[i], -i))  # ties: lowest index
            if weight[best] == 0:
                ok = False
                break
            alive[best] = False
            for i in range(n):
                weight[i] -= W[i][best]
        if ok:
            return np.flatnonzero(alive)
        R *= 1.25
    raise RuntimeError("no pass")


@pytest.mark.parametrize("n", [60, 157, 300])
def test_wse_equals_brute_force(n):
    rng = np.random.default_rng(n)
    x = rng.normal(size=(n, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    # distances computed by numpy differ from the O2 rule only in the last bit; these
    # random clouds have no near-ties at that level
    assert np.array_equal(O.wse(x, n // 4), _wse_brute(x, n // 4))


def test_wse_sizes_and_removal_of_max_weight():
    for N, NH in GOLD["wse_sizes"]["pairs"]:
        assert N // 4 == NH
    x, _ = MI.fibonacci_sphere(2000, jitter=0.2, seed=9)
    keep = O.wse(x, 2000 // 4)
    assert len(keep) == 500 and np.all(np.diff(keep) > 0)
    # N_t = N - 1 removes exactly the point of maximal weight
    rng = np.random.default_rng(3)
    y = rng.normal(size=(80, 3)); y /= np.linalg.norm(y, axis=1, keepdims=True)
    k1 = O.wse(y, 79)
    assert np.array_equal(k1, _wse_brute(y, 79))


def test_wse_separation_beats_random_subsets():
    x, _ = MI.fibonacci_sphere(4000, jitter=0.3, seed=2)
    keep = O.wse(x, 1000)

    def sep(ix):
        from scipy.spatial import cKDTree
        d, _ = cKDTree(x[ix]).query(x[ix], k=2)
        return d[:, 1].min(), d[:, 1].max()

    s, smax = sep(keep)
    rng = np.random.default_rng(0)
    best_rand = max(sep(np.sort(rng.choice(4000, 1000, replace=False)))[0] for _ in range(100))
    assert s > best_rand
    assert smax / s < 4.0   # quasi-uniformity


def test_level_rule_examples():
    for N, nmin, p in GOLD["level_rule_examples"]["cases"]:
        assert int(np.floor(np.log(N / nmin) / np.log(4))) + 1 == p
        Np = N // 4 ** (p - 1)
        assert nmin <= Np < 4 * nmin


def test_wse_covers_irregular_cloud():
    """O8 degenerate passes: on the quartic cloud (cfg4 recipe) the median-spacing radius is
    too small, the elimination reaches points with no live neighbour (zero weight) and index
    ties then wiped out the lowest-Morton corner (a 38-spacing hole).  The restart rule
    (R *= 1.25) keeps the coarse set covering the surface (quasi-uniform subsets)."""
    from scipy.spatial import cKDTree

    w = MI.make_workload(4, n=16384)
    x = w.points[O.morton_perm(w.points)]
    keep = O.wse(x, len(x) // 4)
    d, _ = cKDTree(x[keep]).query(x)
    dn, _ = cKDTree(x).query(x, k=2)
    assert d.max() < 5.0 * np.median(dn[:, 1])
