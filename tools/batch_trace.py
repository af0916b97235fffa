"""Traced stages of one batched (multi-RHS) V-cycle of cfg3 (MGM_TRACE=1 stamps in the graph)."""
import os
import sys

os.environ["MGM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_trace_read, mgm_vcycle_batch

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = MI.make_workload(3)
m = MGM(w.points, w.normals, w.stencil, w.levels)
N = len(w.points)
F = torch.from_numpy(np.random.default_rng(K).uniform(-1, 1, (K, N))).cuda()
U = torch.zeros_like(F)
for _ in range(3):
    mgm_vcycle_batch(m.ctx, K, F, U)
acc = None
for _ in range(10):
    mgm_vcycle_batch(m.ctx, K, F, U)
    torch.cuda.synchronize()
    tr = mgm_trace_read(m.ctx)
    d = np.diff([t for _, t in tr]) / 1e3
    acc = d if acc is None else acc + d
print("K", K, {lab: round(float(v) / 10, 1) for (lab, _), v in zip(tr[1:], acc)}, "total", round(float(acc.sum()) / 10, 1))
