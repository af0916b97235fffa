"""Multi-RHS throughput at the bench workload: batched V-cycle and batched standalone MGM for
K = 1, 2, 4, 8 right-hand sides (CUDA events; K = 1 is the single-RHS path)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_solve_batch, mgm_vcycle_batch

w = MI.make_workload(int(os.environ.get("MGM_CFG", "3")))
m = MGM(w.points, w.normals, w.stencil, w.levels)
n = len(w.points)
rng = np.random.default_rng(0)
out = {}
for K in (1, 2, 4, 8):
    F = torch.from_numpy(rng.uniform(-1, 1, (K, n))).cuda()
    U = torch.zeros_like(F)
    run = (lambda: m.vcycle(F[0], U[0])) if K == 1 else (lambda: mgm_vcycle_batch(m.ctx, K, F, U))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    vc = e0.elapsed_time(e1) / 20
    R = torch.from_numpy(np.stack([w.rhs] * K)).cuda()
    X = torch.zeros_like(R)
    if K == 1:
        m.solve(R[0], X[0], tol=1e-10, krylov=0)
    else:
        mgm_solve_batch(m.ctx, K, R, X, tol=1e-10)
    torch.cuda.synchronize()
    e0.record()
    if K == 1:
        _, rep = m.solve(R[0], X[0], tol=1e-10, krylov=0)
        its = rep.iterations
    else:
        reps = mgm_solve_batch(m.ctx, K, R, X, tol=1e-10)
        its = max(r.iterations for r in reps)
    e1.record()
    torch.cuda.synchronize()
    sm = e0.elapsed_time(e1)
    out[K] = dict(vcycle_ms=round(vc, 3), vcycle_ms_per_rhs=round(vc / K, 3), standalone_ms=round(sm, 2),
                  standalone_ms_per_rhs=round(sm / K, 2), iterations=its)
    print(K, out[K], flush=True)
print(json.dumps(out))
