"""Debug helper: set up configs[0] (sphere N=4096) through the C ABI and run one solve."""
import faulthandler
import os
import sys

faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM

torch.cuda.set_device(0)
w = MI.make_workload(int(os.environ.get("MGM_CFG", "1")))
print("setup...", flush=True)
m = MGM(w.points, w.normals, w.stencil, w.levels)
print("levels", m.level_info(), flush=True)
rhs = torch.from_numpy(w.rhs).cuda()
x, rep = m.solve(rhs, tol=1e-10)
torch.cuda.synchronize()
print("solve", rep, flush=True)
m.close()
