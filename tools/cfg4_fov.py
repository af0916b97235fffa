"""cfg4 root cause, part 3: field of values.  D_h's eigenvalues lie in the left half-plane,
but a non-normal D_h's field of values W(D) = {x*Dx / x*x} can reach into the right half-plane
(lambda_max of the symmetric part H = (D + D^T)/2 > 0).  The Galerkin coarse operator
P^T D P has its eigenvalues inside W(P^T D P) subset of W(D) only up to the scaling by P, so
with lambda_max(H) > 0 the coarse operators may acquire right-half-plane eigenvalues and
the coarse-grid correction I - P (P^T D P)^{-1} P^T D loses its stability.  For each case:
lambda_max(H) relative to |lambda(D)|_max, the departure ||D - D^T||_F / ||D + D^T||_F, and
the right-most eigenvalues of every Galerkin level.
  python tools/cfg4_fov.py N"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sps
from scipy.sparse.linalg import eigs, eigsh

import mgm_inputs as MI
import oracle as O


def analyse(name, x, nrm, st, n):
    lvl = dict(num_levels=MI.level_count(n), interp_m=6, nu1=1, nu2=1)
    Oh = O.Oracle(x, nrm, st, lvl)
    out = dict(case=name, N=n)
    for j, lv in enumerate(Oh.levels[:-1]):
        A = sps.csr_matrix((lv.L.val, lv.L.idx, lv.L.ptr), shape=lv.L.shape)
        H = (A + A.T) * 0.5
        S = (A - A.T) * 0.5
        hmax = float(eigsh(H, k=1, which="LA", return_eigenvectors=False, maxiter=20000, tol=1e-8)[0])
        amax = float(np.abs(eigs(A, k=1, which="LM", return_eigenvectors=False, maxiter=20000, tol=1e-6)).max())
        lr = eigs(A, k=6, which="LR", return_eigenvectors=False, maxiter=50000, tol=1e-8)
        out[f"L{j}"] = dict(n=lv.N, sym_part_max=hmax, sym_part_max_rel=hmax / amax,
                            skew_over_sym=float(sps.linalg.norm(S) / sps.linalg.norm(H)),
                            rightmost=[[float(v.real), float(v.imag)] for v in sorted(lr, key=lambda z: -z.real)[:3]])
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    cfg4 = dict(method=0, poly_degree=4, phs_k=3, stencil_n=50, problem=1, mu=1.0)
    x, nrm = MI.quartic_cloud(n, seed=2)
    analyse("quartic-cfg4", x, nrm, cfg4, n)
    analyse("quartic-l3n30", x, nrm, dict(cfg4, poly_degree=3, phs_k=2, stencil_n=30), n)
    xs, ns = MI.fibonacci_sphere(n, jitter=0.1, seed=3)
    analyse("sphere-cfg4", xs, ns, cfg4, n)
