"""cfg4 root cause, part 2: which component of the V-cycle amplifies the error on the quartic
cloud (oracle, CPU)?  For N given: spectral radius (power iteration, 40 steps) of
  * the multicolour Gauss-Seidel sweep alone on A = D_h (f = 0, mean removed each step),
  * the two-grid cycle (p = 2, exact coarse solve), V(1,1),
  * the full V-cycle with the paper's own smoother (lexicographic GS in RCM order),
  * the full V-cycle with k = ell (the paper's PHS order): r^9 instead of r^7,
  * the full V-cycle with m = 3 interpolation points (Table 1) instead of 6.
  python tools/cfg4_smoother.py N"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import mgm_inputs as MI
import oracle as O


def rho_power(step, n, iters=40, seed=0, project=None):
    u = np.random.default_rng(seed).uniform(-1, 1, n)
    gs = []
    for _ in range(iters):
        if project:
            u = project(u)
        u /= np.linalg.norm(u)
        u = step(u)
        if project:
            u = project(u)
        gs.append(float(np.linalg.norm(u)))
    return float(np.exp(np.mean(np.log(gs[-10:]))))


def main(n):
    x, nrm = MI.quartic_cloud(n, seed=2)
    base = dict(method=0, poly_degree=4, phs_k=3, stencil_n=50, problem=1, mu=1.0)
    lvl = dict(num_levels=MI.level_count(n), interp_m=6, nu1=1, nu2=1, restart=128)
    out = {"N": n}
    Oh = O.Oracle(x, nrm, base, lvl)
    L0 = Oh.levels[0]
    mean0 = lambda v: v - v.mean()

    def gs_step(u):
        u = u.copy()
        O.gs_sweep(L0.L, L0.order, np.zeros(L0.N), u, False)
        return u
    out["gs_sweep_rho"] = rho_power(gs_step, L0.N, project=mean0)
    nb = L0.N + 1
    out["vcycle_V11_rho"] = rho_power(lambda u: Oh.vcycle_level_order(np.zeros(nb), u), nb)
    for name, st, lv in [("two_grid_V11", base, dict(lvl, num_levels=2)),
                         ("vcycle_V22", base, dict(lvl, nu1=2, nu2=2)),
                         ("vcycle_symmetric_GS", base, dict(lvl, smoother=2)),
                         ("vcycle_rcm_lexicographic_GS", base, dict(lvl, gs_order="rcm")),
                         ("vcycle_k_eq_ell_r9", dict(base, phs_k=4), lvl),
                         ("vcycle_m3", base, dict(lvl, interp_m=3))]:
        try:
            Ov = O.Oracle(x, nrm, st, lv)
            out[name] = rho_power(lambda u: Ov.vcycle_level_order(np.zeros(nb), u), nb)
        except Exception as e:  # noqa: BLE001
            out[name] = f"failed: {e}"
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 16384)
