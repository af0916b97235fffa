"""WSE coverage of the cfg4 quartic cloud at a given N (library host WSE, level 0 -> 1),
and the MGM-GMRES residual after 30 iterations on the GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from scipy.spatial import cKDTree

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM
from paper_2204_06154_b200.mgm import mgm_host_morton, mgm_host_wse

for n in [int(a) for a in sys.argv[1:]]:
    t = time.time()
    w = MI.make_workload(4, n=n)
    print("n", n, "gen", round(time.time() - t, 1), flush=True)
    X = w.points[mgm_host_morton(w.points)]
    for lvl in range(2):
        keep = mgm_host_wse(X, len(X) // 4)
        d, _ = cKDTree(X[keep]).query(X, workers=-1)
        dn, _ = cKDTree(X).query(X, k=2, workers=-1)
        sp = np.median(dn[:, 1])
        print("  level", lvl, "max dist/sp %.1f" % (d.max() / sp), "far", int((d > 5 * sp).sum()), flush=True)
        X = X[keep]
    m = MGM(w.points, w.normals, w.stencil, w.levels)
    x, rep = m.solve(torch.from_numpy(w.rhs).cuda(), tol=1e-10, maxit=30)
    print("  gmres 30 its rel", rep.final_rel_residual, "levels", [l["n"] for l in m.level_info()], flush=True)
    m.close()
