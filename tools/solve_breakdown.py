"""Where the MGM-GMRES solve time goes: V-cycles (CUDA events around each preconditioner
graph launch, timing class 2) vs the rest (SpMV, CGS2, host Givens / synchronisation)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_timing_enable, mgm_timing_read

w = MI.make_workload(int(os.environ.get("MGM_CFG", "3")))
m = MGM(w.points, w.normals, w.stencil, w.levels)
rhs = torch.from_numpy(w.rhs).cuda()
x = torch.empty_like(rhs)
for kr in (1, 2):
    for _ in range(2):
        m.solve(rhs, x, tol=1e-10, krylov=kr)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, rep = m.solve(rhs, x, tol=1e-10, krylov=kr)
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1)
    mgm_timing_enable(m.ctx, 2, True)
    m.solve(rhs, x, tol=1e-10, krylov=kr)
    torch.cuda.synchronize()
    t = mgm_timing_read(m.ctx, 2)
    mgm_timing_enable(m.ctx, 2, False)
    print(f"krylov={kr}: solve {total:.2f} ms, {rep.iterations} its; V-cycles (events) {t['total_ms']:.2f} ms "
          f"over {t['launches']} launches = {t['total_ms'] / max(1, t['launches']):.3f} ms each; "
          f"rest {total - t['total_ms']:.2f} ms = {(total - t['total_ms']) / max(1, rep.iterations):.3f} ms/iteration")
