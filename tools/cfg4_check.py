"""Convergence of MGM-GMRES on the cfg4 recipe (bordered Poisson, l=4, r^7, n=50) at several
sizes, GPU vs oracle residual histories for the first iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
import oracle as O
from paper_2204_06154_b200 import MGM

for n in [int(a) for a in sys.argv[1:]] or [6000, 16384, 65536]:
    w = MI.make_workload(4, n=n)
    g = MGM(w.points, w.normals, w.stencil, w.levels)
    x, rep = g.solve(torch.from_numpy(w.rhs).cuda(), tol=1e-10, maxit=15)
    o = O.Oracle(w.points, w.normals, w.stencil, w.levels)
    xr, rr = o.solve(w.rhs, tol=1e-10, maxit=15)
    print(n, "levels", [lv["n"] for lv in g.level_info()])
    print("  gpu   ", np.round(rep.history[:15], 4).tolist())
    print("  oracle", np.round(rr.history[:15], 4).tolist(), flush=True)
    g.close()
