"""Standalone MGM (krylov=0) solve time at cfg3: median of 5 (CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM

w = MI.make_workload(int(os.environ.get("MGM_CFG", "3")))
m = MGM(w.points, w.normals, w.stencil, w.levels)
rhs = torch.from_numpy(w.rhs).cuda()
x = torch.empty_like(rhs)
ts = []
for k in range(7):
    _, rep = m.solve(rhs, x, tol=1e-10, krylov=0)
    if k >= 2:
        ts.append(rep.solve_ms)
ts.sort()
print(json.dumps({"variant": os.environ.get("MGM_NO_MODE3", "mode3"), "standalone_ms": ts[2], "its": rep.iterations,
                  "final": rep.final_rel_residual}))
