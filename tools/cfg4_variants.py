"""MGM-GMRES residual after 30 iterations for cfg4 variants at a given N (GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM

n = int(sys.argv[1])
w4 = MI.make_workload(4, n=n)
w1 = MI.make_workload(1, n=n)
cases = [
    ("quartic poisson (cfg4)", w4, {}, w4.rhs),
    ("quartic shifted", w4, dict(problem=0, mu=1.0), w4.rhs),
    ("quartic poisson l3 k2 n30", w4, dict(poly_degree=3, phs_k=2, stencil_n=30), w4.rhs),
    ("sphere poisson l4 k3 n50", w1, dict(problem=1, poly_degree=4, phs_k=3, stencil_n=50), w1.rhs - w1.rhs.mean()),
]
for name, w, over, rhs in cases:
    st = dict(w.stencil, **over)
    m = MGM(w.points, w.normals, st, w.levels)
    x, rep = m.solve(torch.from_numpy(np.ascontiguousarray(rhs)).cuda(), tol=1e-10, maxit=30)
    print(n, name, "rel after", rep.iterations, rep.final_rel_residual, flush=True)
    m.close()
