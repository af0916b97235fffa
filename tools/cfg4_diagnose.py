"""cfg4 root cause (VERDICT r01 'Next' 2c): on the quartic level set with the cfg4
discretization (RBF-FD PHS r^7 + degree-4 polynomials, n = 50, Poisson), does the method
itself degrade with N?  Oracle only (CPU).  For each case and N:
  * spurious spectrum: eigenvalues of the fine RBF-FD Laplacian D_h with Re > 0 (the exact
    Laplace-Beltrami operator is negative semi-definite; ARPACK 'LR' on the sparse D_h);
  * multigrid contraction: spectral radius of the V-cycle iteration operator E = I - M A
    (bordered Poisson system) by power iteration on u <- V-cycle(0, u);
  * MGM-GMRES iterations to 1e-10 (GMRES(128), the cfg4 workload's settings).
Controls: the same cloud with l = 3 / r^5 / n = 30; the jittered sphere with the cfg4
discretization; and the quartic cloud thinned by WSE (O8) instead of the generator's
nearest-pair thinning (node quality: separation and fill distance).
  python tools/cfg4_diagnose.py N [N ...]   -> one JSON line per (case, N)"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sps
from scipy.sparse.linalg import eigs

import mgm_inputs as MI
import oracle as O


def quartic_raw(n, seed=2):
    """the 2N Newton-projected Sobol points of mgm_inputs.quartic_cloud, before thinning"""
    pts, have, rnd = [], 0, 0
    while have < 2 * n:
        m = int((2 * n - have) * 1.3) + 64
        x = -1.25 + 2.5 * MI._sobol(3, m, seed + 1000 * rnd)
        rnd += 1
        x = x[np.linalg.norm(x, axis=1) >= 0.25]
        for _ in range(50):
            F = MI._quartic_F(x)
            g = 4.0 * x ** 3 - 2.0 * x
            x = x - (F / (g * g).sum(1))[:, None] * g
        ok = np.abs(MI._quartic_F(x)) <= 1e-14
        pts.append(x[ok])
        have += int(ok.sum())
    return np.concatenate(pts)[: 2 * n]


def normals_of(x):
    g = 4.0 * x ** 3 - 2.0 * x
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def node_quality(x, ref):
    """separation (min NN distance / median NN distance) and fill distance (max distance of a
    dense reference sample of the surface to the cloud, / median NN distance)"""
    d = np.sqrt(O.nn_dist2(x))
    med = float(np.median(d))
    nn = O.knn(x, ref, 1)[:, 0]
    fill = float(np.sqrt(((ref - x[nn]) ** 2).sum(1)).max())
    return dict(sep_ratio=float(d.min()) / med, fill_ratio=fill / med)


def spectrum_right(D, k=12):
    n = D.shape[0]
    lm = eigs(D, k=1, which="LM", return_eigenvectors=False, maxiter=5000, tol=1e-6)
    lr = eigs(D, k=k, which="LR", return_eigenvectors=False, maxiter=20000, tol=1e-8)
    scale = float(np.abs(lm).max())
    pos = lr.real[lr.real > 1e-8 * scale]
    return dict(max_abs=scale, max_real=float(lr.real.max()), n_right_of_tol=int(len(pos)),
                right_eigs=[[float(v.real), float(v.imag)] for v in sorted(lr, key=lambda z: -z.real)[:6]])


def contraction(Oh, iters=40, seed=0):
    n = Oh.levels[0].N + (1 if Oh.poisson else 0)
    u = np.random.default_rng(seed).uniform(-1, 1, n)
    f = np.zeros(n)
    norms = []
    for _ in range(iters):
        u = Oh.vcycle_level_order(f, u)
        nu = float(np.linalg.norm(u))
        norms.append(nu)
        if nu == 0.0 or not np.isfinite(nu):
            break
        u /= nu
    # norms are of normalised iterates: the growth factor per cycle
    return dict(rho_last10=float(np.exp(np.mean(np.log(norms[-10:])))), per_cycle=norms[-5:])


def run(case, n):
    t0 = time.time()
    if case in ("quartic-cfg4", "quartic-l3n30", "quartic-wse-cfg4"):
        if case == "quartic-wse-cfg4":
            raw = quartic_raw(n)
            keep = O.wse(raw, n)
            x = np.ascontiguousarray(raw[keep])
            nrm = normals_of(x)
        else:
            x, nrm = MI.quartic_cloud(n, seed=2)
        st = dict(method=0, poly_degree=4, phs_k=3, stencil_n=50, problem=1, mu=1.0)
        if case == "quartic-l3n30":
            st.update(poly_degree=3, phs_k=2, stencil_n=30)
        _, rng_rhs = MI._rngs(2)
        rhs = MI._trig_rhs(rng_rhs, x)
        ref = quartic_raw(4 * n, seed=7)
    else:  # sphere control
        x, nrm = MI.fibonacci_sphere(n, jitter=0.1, seed=3)
        st = dict(method=0, poly_degree=4, phs_k=3, stencil_n=50, problem=1, mu=1.0)
        rhs = MI.sph_harm_cos(x, 6, 3)
        rhs = rhs - rhs.mean()
        ref = None
    lv = dict(num_levels=MI.level_count(n), interp_m=6, nu1=2, nu2=2, restart=128)
    Oh = O.Oracle(x, nrm, st, lv)
    out = dict(case=case, N=n, levels=[l.N for l in Oh.levels])
    if ref is not None:
        out["nodes"] = node_quality(x, ref)
    A = Oh.levels[0].L
    D = sps.csr_matrix((A.val, A.idx, A.ptr), shape=A.shape)   # Poisson: L_1 = D_h
    try:
        out["spectrum"] = spectrum_right(D)
    except Exception as e:  # noqa: BLE001
        out["spectrum"] = f"eigs failed: {e}"
    out["vcycle"] = contraction(Oh)
    _, rep = Oh.solve(rhs, tol=1e-10, maxit=300)
    out["gmres"] = dict(iterations=rep.iterations, converged=bool(rep.converged),
                        final=rep.final_rel_residual, after30=rep.history[29] if len(rep.history) > 29 else None)
    out["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    ns = [int(a) for a in sys.argv[1:]] or [4096, 16384]
    cases = os.environ.get("CASES", "quartic-cfg4,quartic-l3n30,sphere-cfg4,quartic-wse-cfg4").split(",")
    for n in ns:
        for c in cases:
            run(c, n)
