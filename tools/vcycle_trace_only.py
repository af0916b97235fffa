"""V-cycle time (graph, 50 replays) and traced stages only (no solve) at cfg3 -- for timing
experiments whose numerics are deliberately wrong."""
import json
import os
import sys

os.environ["MGM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_trace_read

w = MI.make_workload(int(os.environ.get("MGM_CFG", "3")))
m = MGM(w.points, w.normals, w.stencil, w.levels)
n = len(w.points)
f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
u = torch.zeros_like(f)
for _ in range(5):
    u.zero_()
    m.vcycle(f, u)
torch.cuda.synchronize()
acc, tr = None, None
for _ in range(20):
    u.zero_()
    m.vcycle(f, u)
    torch.cuda.synchronize()
    tr = mgm_trace_read(m.ctx)
    d = np.diff([t for _, t in tr]) / 1e3
    acc = d if acc is None else acc + d
st = {lab: round(float(x) / 20, 1) for (lab, _), x in zip(tr[1:], acc)}
print(json.dumps({"variant": os.environ.get("VARIANT", ""), "stages": st, "total_us": round(float(acc.sum()) / 20, 1)}))
