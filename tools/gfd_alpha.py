"""cfg2-GFD (BASELINE configs[1], N = 262144) with the GFD weight exponent alpha of P:185-187
taken literally: alpha = 4 (the paper's Table 1 value) and alpha = 16 (the workload's choice,
DESIGN.md O5).  Prints MGM-GMRES / standalone iterations and convergence (GPU)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
w = MI.make_workload(2, n=n, method="gfd")
rhs = torch.from_numpy(w.rhs).cuda()
for alpha in (4.0, 16.0):
    m = MGM(w.points, w.normals, dict(w.stencil, gfd_alpha=alpha), w.levels)
    out = {"N": n, "gfd_alpha": alpha}
    for name, kr in (("gmres", 1), ("standalone", 0)):
        x, rep = m.solve(rhs, tol=1e-10, krylov=kr, maxit=300)
        err = float(np.abs(x.cpu().numpy() - w.exact).max() / np.abs(w.exact).max())
        out[name] = dict(iterations=rep.iterations, converged=bool(rep.converged),
                         final_rel_residual=rep.final_rel_residual, solve_ms=rep.solve_ms, rel_err_vs_Y10_5=err)
    print(json.dumps(out), flush=True)
    m.close()
