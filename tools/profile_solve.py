"""One MGM-GMRES solve of the bench workload inside a cudaProfilerStart/Stop window, for ncu
(--profile-from-start off).  MGM_CFG / MGM_N select the workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM

cfg = int(os.environ.get("MGM_CFG", "3"))
n = int(os.environ["MGM_N"]) if "MGM_N" in os.environ else None
w = MI.make_workload(cfg, n=n)
m = MGM(w.points, w.normals, w.stencil, w.levels)
rhs = torch.from_numpy(w.rhs).cuda()
x = torch.empty_like(rhs)
for _ in range(2):
    m.solve(rhs, x, tol=1e-10)
torch.cuda.synchronize()
torch.cuda.profiler.start()
_, rep = m.solve(rhs, x, tol=1e-10)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iterations", rep.iterations, "solve_ms", rep.solve_ms)
m.close()
