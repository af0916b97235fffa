"""Traced stages of the ZERO-GUESS V-cycle (the Krylov preconditioner M v, vgraph0: the graph
MGM-GMRES replays every iteration) at the bench workload (MGM_TRACE=1 stamps in the graph)."""
import json
import os
import sys

os.environ["MGM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_apply, mgm_trace_read

w = MI.make_workload(int(os.environ.get("MGM_CFG", "3")))
m = MGM(w.points, w.normals, w.stencil, w.levels)
n = len(w.points)
v = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
y = torch.empty_like(v)
for _ in range(3):
    mgm_apply(m.ctx, 0, 7, v, None, y)
acc, tr = None, None
for _ in range(20):
    mgm_apply(m.ctx, 0, 7, v, None, y)
    torch.cuda.synchronize()
    tr = mgm_trace_read(m.ctx)
    d = np.diff([t for _, t in tr]) / 1e3
    acc = d if acc is None else acc + d
st = {lab: round(float(x) / 20, 1) for (lab, _), x in zip(tr[1:], acc)}
print(json.dumps({"zero_guess_vcycle_stages_us": st, "total_us": round(float(acc.sum()) / 20, 1)}))
