"""Fine per-phase timeline of the one-kernel V-cycle bottom (MGM_TRACE=2): for thread 0 of
the first and last CTA of the cluster, SM clocks at the steps of each phase, averaged over
10 V-cycles and grouped by (op, local, rows, threads per row)."""
import os
import sys

os.environ["MGM_TRACE"] = "2"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_bottom_ftrace_read, mgm_bottom_trace_read

w = MI.make_workload(int(os.environ.get("MGM_CFG", "3")))
f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, len(w.points))).cuda()
m = MGM(w.points, w.normals, w.stencil, w.levels)
u = torch.zeros_like(f)
for _ in range(3):
    m.vcycle(f, u)
acc = None
for _ in range(10):
    m.vcycle(f, u)
    torch.cuda.synchronize()
    c = mgm_bottom_ftrace_read(m.ctx).astype(np.float64)
    acc = c if acc is None else acc + c
acc /= 10
_, meta = mgm_bottom_trace_read(m.ctx)
names = ["ZERO", "GS", "RES", "MVZ", "ADD", "MV", "STORE"]
# slot order in time: 0 start, 7 rows in registers, 1 row sum, 2 broadcast value, 3 stores
# issued, 4 arrive done, 5 next loads issued, 6 wait done (= next start)
steps = [(7, "regs"), (1, "rowsum"), (2, "value"), (3, "stores"), (4, "arrive"), (5, "ld-issue"), (6, "wait")]
for cta in (0, 1):
    a = acc[cta]
    groups = {}
    for q in range(len(meta)):
        if a[q, 0] == 0 or a[q, 6] == 0:
            continue
        key = (names[meta[q, 0]], int(meta[q, 1]), int(meta[q, 3]))
        prev = a[q, 0]
        d = []
        for s, _ in steps:
            d.append(a[q, s] - prev if a[q, s] > 0 else np.nan)
            if a[q, s] > 0:
                prev = a[q, s]
        groups.setdefault(key, []).append(d)
    print(f"CTA {'first' if cta == 0 else 'last'}: cycles per step (mean over phases of the group)")
    print("   op    local tpr  count | " + " ".join(f"{n:>8s}" for _, n in steps) + " |  total")
    for k, v in sorted(groups.items()):
        v = np.array(v)
        mu = np.nanmean(v, axis=0)
        print(f"   {k[0]:5s} {k[1]:5d} {k[2]:3d} {len(v):6d} | " + " ".join(f"{x:8.0f}" for x in mu) +
              f" | {np.nansum(mu):6.0f}")
m.close()
