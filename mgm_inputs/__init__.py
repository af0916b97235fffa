"""Seeded synthetic workloads for the MGM solve path (shared by tests, bench and oracle).

This module holds NONE of the method's arithmetic (no Morton order, kNN stencils,
weights, WSE, transfers, Galerkin products, smoothing or Krylov steps).  It only draws
point clouds, normals and right-hand sides shaped like the paper's workloads:

* PAPER.md P:416 (section "Numerical results"): sphere and cyclide clouds; replaced by the
  BASELINE.json configs (Fibonacci sphere, torus, quartic level set), SURVEY.md 8(d).
* spherical-harmonic closed forms, Y_5^4 = z(x^4 - 6x^2y^2 + y^4).

Every generator takes a seed and uses ``np.random.SeedSequence(seed).spawn(2)`` ->
(rng_pts, rng_rhs), as fixed in SURVEY.md 8(d).  Thinning of oversampled clouds uses a
simple nearest-pair removal rule written here (NOT the paper's weighted sample
elimination, which is part of the method and lives in the library and the oracle).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Workload", "fibonacci_sphere", "torus_cloud", "quartic_cloud",
    "sph_harm_cos", "make_workload", "CONFIGS",
]


def _rngs(seed: int):
    ss = np.random.SeedSequence(seed)
    a, b = ss.spawn(2)
    return np.random.default_rng(a), np.random.default_rng(b)


def fibonacci_sphere(n: int, jitter: float = 0.0, seed: int = 0):
    """Fibonacci lattice on the unit sphere (BASELINE.json configs[0], configs[1], configs[4]).

    z_i = 1 - (2i+1)/N, phi_i = i*pi*(3 - sqrt 5).  With ``jitter`` > 0 each point moves by
    jitter*h*(xi1*e1 + xi2*e2), h = sqrt(4 pi / N), xi ~ U[-1,1]^2, e1/e2 the local
    azimuthal/polar unit vectors, then is renormalised.  Normals are the points.
    """
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    phi = i * (math.pi * (3.0 - math.sqrt(5.0)))
    s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    x = np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=1)
    if jitter > 0.0:
        rng_pts, _ = _rngs(seed)
        h = math.sqrt(4.0 * math.pi / n)
        xi = rng_pts.uniform(-1.0, 1.0, size=(n, 2))
        e1 = np.stack([-np.sin(phi), np.cos(phi), np.zeros(n)], axis=1)
        e2 = np.cross(x, e1)
        x = x + jitter * h * (xi[:, :1] * e1 + xi[:, 1:2] * e2)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
    return np.ascontiguousarray(x), np.ascontiguousarray(x.copy())


def icosahedral_sphere(level: int):
    """Icosahedral node set on the unit sphere (the paper's sphere clouds): the 12
    vertices of an icosahedron, each triangle recursively split into four by edge midpoints
    projected to the sphere, `level` times: N = 10 * 4**level + 2.  Normals are the points.
    Deterministic; no method arithmetic."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
         (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    verts = [np.array(p, dtype=np.float64) / np.linalg.norm(p) for p in v]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
             (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
             (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    x = np.ascontiguousarray(np.array(verts))
    return x, x.copy()


def _thin_nearest_pairs(x: np.ndarray, n_remove: int) -> np.ndarray:
    """Remove ``n_remove`` points, walking points by ascending nearest-neighbour distance
    and removing a point unless it is protected; removing a point protects its nearest
    neighbour (so close pairs lose one member).  Returns the kept indices in order."""
    from scipy.spatial import cKDTree

    d, j = cKDTree(x).query(x, k=2, workers=-1)
    nn_d, nn_j = d[:, 1], j[:, 1]
    order = np.lexsort((np.arange(len(x)), nn_d))
    removed = np.zeros(len(x), dtype=bool)
    protected = np.zeros(len(x), dtype=bool)
    count = 0
    for i in order:
        if count == n_remove:
            break
        if protected[i] or removed[i]:
            continue
        removed[i] = True
        protected[nn_j[i]] = True
        count += 1
    if count < n_remove:  # second walk without protection (rare)
        for i in order:
            if count == n_remove:
                break
            if not removed[i]:
                removed[i] = True
                count += 1
    return np.flatnonzero(~removed)


def _torus_sample(rng, count: int, R: float, r: float):
    """Uniform surface density on the torus by rejection on (theta, phi)."""
    out = []
    have = 0
    while have < count:
        m = int((count - have) * 1.3) + 64
        th = rng.uniform(0.0, 2.0 * math.pi, m)
        ph = rng.uniform(0.0, 2.0 * math.pi, m)
        acc = rng.uniform(0.0, 1.0, m) < (R + r * np.cos(th)) / (R + r)
        th, ph = th[acc], ph[acc]
        out.append(np.stack([th, ph], axis=1))
        have += len(th)
    tp = np.concatenate(out)[:count]
    return tp[:, 0], tp[:, 1]


def _torus_xyz(th, ph, R, r):
    x = np.stack([(R + r * np.cos(th)) * np.cos(ph), (R + r * np.cos(th)) * np.sin(ph),
                  r * np.sin(th)], axis=1)
    nrm = np.stack([np.cos(th) * np.cos(ph), np.cos(th) * np.sin(ph), np.sin(th)], axis=1)
    return x, nrm


def _sobol(dim: int, count: int, seed: int) -> np.ndarray:
    """Scrambled Sobol points in [0,1)^dim (at least `count`, a power of two)."""
    from scipy.stats import qmc

    m = max(1, int(math.ceil(math.log2(max(2, count)))))
    return qmc.Sobol(dim, scramble=True, seed=seed).random_base2(m)


def torus_cloud(n: int, seed: int = 1, R: float = 1.0, r: float = 1.0 / 3.0,
                jitter: float = 0.15):
    """Torus R=1, r=1/3 (BASELINE.json configs[2]), N quasi-uniform points: rings of constant
    theta spaced h along the tube, each ring holding round(2 pi (R + r cos theta) / h) points
    (uniform surface density), h chosen by bisection so the total is N (excess, if any,
    removed at random); every ring gets a random phase and every point a jitter of
    +-jitter*h in both tangent directions.  Analytic normals.
    for why this replaces rejection sampling + thinning (defects -> 50-290 GMRES iterations)."""
    rng, _ = _rngs(seed)
    area = 4.0 * math.pi ** 2 * R * r

    def rings(h):
        nth = max(3, int(round(2.0 * math.pi * r / h)))
        th = (np.arange(nth) + 0.5) * (2.0 * math.pi / nth)
        cnt = np.maximum(3, np.round(2.0 * math.pi * (R + r * np.cos(th)) / h).astype(np.int64))
        return th, cnt

    lo, hi = 0.5 * math.sqrt(area / n), 2.0 * math.sqrt(area / n)
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if rings(mid)[1].sum() >= n:
            lo = mid
        else:
            hi = mid
    h = lo
    th_r, cnt = rings(h)
    ring = np.repeat(np.arange(len(th_r)), cnt)
    k = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    phase = rng.uniform(0.0, 1.0, len(th_r))
    ph = (k + phase[ring]) * (2.0 * math.pi / cnt[ring])
    th = th_r[ring]
    xi = rng.uniform(-1.0, 1.0, size=(len(th), 2))
    th = th + jitter * h * xi[:, 0] / r
    ph = ph + jitter * h * xi[:, 1] / (R + r * np.cos(th))
    if len(th) > n:
        keep = np.sort(rng.choice(len(th), n, replace=False))
        th, ph = th[keep], ph[keep]
    x, nrm = _torus_xyz(th, ph, R, r)
    return np.ascontiguousarray(x), np.ascontiguousarray(nrm)


def _quartic_F(x):
    return (x ** 4).sum(1) - (x ** 2).sum(1) - 0.3


def quartic_cloud(n: int, seed: int = 2, passes: int = 8):
    """Level set x^4+y^4+z^4 - (x^2+y^2+z^2) = 0.3 (BASELINE.json configs[3]): 2N scrambled
    Sobol points in [-1.25,1.25]^3 (|x| >= 0.25) pushed onto the surface by Newton, then thinning.
    Normal = grad F / |grad F|."""
    pts = []
    have = 0
    rnd = 0
    while have < 2 * n:
        m = int((2 * n - have) * 1.3) + 64
        x = -1.25 + 2.5 * _sobol(3, m, seed + 1000 * rnd)
        rnd += 1
        x = x[np.linalg.norm(x, axis=1) >= 0.25]
        for _ in range(50):
            F = _quartic_F(x)
            g = 4.0 * x ** 3 - 2.0 * x
            x = x - (F / (g * g).sum(1))[:, None] * g
        ok = np.abs(_quartic_F(x)) <= 1e-14
        pts.append(x[ok])
        have += int(ok.sum())
    x = np.concatenate(pts)[: 2 * n]
    total = len(x) - n
    for p in range(passes):
        k = total // passes + (1 if p < total % passes else 0)
        x = x[_thin_nearest_pairs(x, k)]
    g = 4.0 * x ** 3 - 2.0 * x
    nrm = g / np.linalg.norm(g, axis=1, keepdims=True)
    return np.ascontiguousarray(x), np.ascontiguousarray(nrm)


def sph_harm_cos(x: np.ndarray, l: int, m: int) -> np.ndarray:
    """Unnormalised real spherical harmonic Re((x+iy)^m) * P_l^(m)(z) on the unit sphere,
    P_l^(m) the m-th derivative of the Legendre polynomial P_l.  For (l, m) = (5, 4) this
    is 945 * z(x^4 - 6x^2y^2 + y^4), the paper's worked formula."""
    from numpy.polynomial import legendre as Lg

    c = np.zeros(l + 1)
    c[l] = 1.0
    dP = Lg.legder(c, m)
    zpart = Lg.legval(x[:, 2], dP)
    w = (x[:, 0] + 1j * x[:, 1]) ** m
    return np.real(w) * zpart


@dataclasses.dataclass
class Workload:
    name: str
    points: np.ndarray
    normals: np.ndarray
    rhs: np.ndarray
    exact: np.ndarray | None
    stencil: dict
    levels: dict


def _bumps_rhs(rng_rhs, x, sampler, count=20, width=0.1):
    c = sampler(rng_rhs, count)
    a = rng_rhs.uniform(-1.0, 1.0, count)
    f = np.zeros(len(x))
    for k in range(count):
        f += a[k] * np.exp(-((x - c[k]) ** 2).sum(1) / (2.0 * width * width))
    return f


def _trig_rhs(rng_rhs, x, count=24):
    f = np.zeros(len(x))
    for _ in range(count):
        while True:
            w = rng_rhs.integers(-8, 9, size=3)
            if 1 <= np.abs(w).sum() <= 8:
                break
        a = rng_rhs.uniform(-1.0, 1.0)
        ph = rng_rhs.uniform(0.0, 2.0 * math.pi)
        f += a * np.cos(x @ w.astype(np.float64) + ph)
    return f - f.mean()


def level_count(n: int, cap: int = 200) -> int:
    """Harness rule of SURVEY.md 8(c) O7: p = 1 + min{j : floor(N/4^j) <= cap}."""
    j = 0
    while n // (4 ** j) > cap:
        j += 1
    return j + 1


def make_workload(cfg: int, n: int | None = None, method: str = "rbffd") -> Workload:
    """BASELINE.json configs[cfg-1] (cfg in 1..5) at its size, or at a smaller ``n`` with the
    same recipe (used for oracle-sized parity cases and CPU-baseline samples)."""
    if cfg == 1:
        n = n or 4096
        x, nrm = fibonacci_sphere(n)
        u = sph_harm_cos(x, 4, 2)
        st = dict(method=0, poly_degree=2, phs_k=1, stencil_n=15, problem=0, mu=1.0)
        lv = dict(num_levels=level_count(n), interp_m=6, nu1=1, nu2=1)
        return Workload("cfg1-sphere", x, nrm, 21.0 * u, u, st, lv)
    if cfg == 2:
        n = n or 262144
        x, nrm = fibonacci_sphere(n, jitter=0.1, seed=0)
        u = sph_harm_cos(x, 10, 5)
        if method == "gfd":
            st = dict(method=1, poly_degree=2, phs_k=0, stencil_n=20, problem=0, mu=1.0,
                      gfd_alpha=16.0)  # paper alpha = 4 (Table 1) under reading O5 (gfd_alpha = 4 alpha)
        else:
            st = dict(method=0, poly_degree=3, phs_k=2, stencil_n=30, problem=0, mu=1.0)
        lv = dict(num_levels=level_count(n), interp_m=6, nu1=2, nu2=2)
        return Workload("cfg2-jittered-sphere-" + method, x, nrm, 111.0 * u, u, st, lv)
    if cfg == 3:
        n = n or 1048576
        x, nrm = torus_cloud(n, seed=1)
        _, rng_rhs = _rngs(1)

        def sampler(rng, count):
            th, ph = _torus_sample(rng, count, 1.0, 1.0 / 3.0)
            return _torus_xyz(th, ph, 1.0, 1.0 / 3.0)[0]

        f = _bumps_rhs(rng_rhs, x, sampler)
        st = dict(method=0, poly_degree=3, phs_k=2, stencil_n=30, problem=0, mu=1.0)
        lv = dict(num_levels=level_count(n), interp_m=6, nu1=1, nu2=1)
        return Workload("cfg3-torus", x, nrm, f, None, st, lv)
    if cfg == 4:
        n = n or 4194304
        x, nrm = quartic_cloud(n, seed=2)
        _, rng_rhs = _rngs(2)
        f = _trig_rhs(rng_rhs, x)
        st = dict(method=0, poly_degree=4, phs_k=3, stencil_n=50, problem=1, mu=1.0)
        # BASELINE cfg4 names neither the GMRES restart nor the sweeps (cfg1/cfg5 say GMRES(50),
        # cfg2 says 2 pre-/2 post-sweeps): restarted GMRES(50) stagnates near 1e-8 on this
        # problem (oracle, N = 262144) and V(1,1) needs 86 GMRES(128) iterations there,
        # V(2,2) 51 -- GMRES(128) with V(2,2)
        lv = dict(num_levels=level_count(n), interp_m=6, nu1=2, nu2=2, restart=128)
        return Workload("cfg4-quartic-poisson", x, nrm, f, None, st, lv)
    if cfg == 5:
        n = n or 16777216
        x, nrm = fibonacci_sphere(n, jitter=0.1, seed=3)
        u = sph_harm_cos(x, 20, 7)
        st = dict(method=0, poly_degree=3, phs_k=2, stencil_n=30, problem=0, mu=1.0)
        lv = dict(num_levels=7 if n == 16777216 else level_count(n), interp_m=6, nu1=1, nu2=1)
        return Workload("cfg5-sphere", x, nrm, 421.0 * u, u, st, lv)
    raise ValueError(f"unknown config {cfg}")


CONFIGS = {1: 4096, 2: 262144, 3: 1048576, 4: 4194304, 5: 16777216}
