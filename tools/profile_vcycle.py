"""Run one V-cycle (and one GMRES Arnoldi-step's worth of kernels) of the bench workload
inside a cudaProfilerStart/Stop window, for ncu (--profile-from-start off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM

cfg = int(os.environ.get("MGM_CFG", "3"))
n = int(os.environ["MGM_N"]) if "MGM_N" in os.environ else None
w = MI.make_workload(cfg, n=n)
m = MGM(w.points, w.normals, w.stencil, w.levels)
f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, len(w.points))).cuda()
u = torch.zeros_like(f)
for _ in range(3):
    m.vcycle(f, u)
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.vcycle(f, u)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("levels", m.level_info())
m.close()
