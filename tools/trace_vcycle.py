"""Per-stage timeline of one graph-replayed V-cycle (MGM_TRACE stamps) for the bench workload,
averaged over 20 V-cycles, under setup-time env variants (VARIANTS json list)."""
import json
import os
import sys

os.environ["MGM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_trace_read

cfg = int(os.environ.get("MGM_CFG", "3"))
n = int(os.environ["MGM_N"]) if "MGM_N" in os.environ else None
w = MI.make_workload(cfg, n=n)
variants = json.loads(os.environ.get("VARIANTS", "[{}]"))
f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, len(w.points))).cuda()
for var in variants:
    for k in ("MGM_BOT_MAX", "MGM_BOT_LOCAL", "MGM_NO_PDL", "MGM_L0_TPR", "MGM_LJ_TPR", "MGM_L0_STPR", "MGM_LJ_STPR", "MGM_GS_BLOCK_SMALL", "MGM_GS_BLOCK_L0", "MGM_BOT_CS", "MGM_NO_PIPE", "MGM_PIPE_CTAS", "MGM_RTPR", "MGM_BOT_TPR_MAX", "MGM_PF_DIST", "MGM_PF_CAP_MB", "MGM_PF_BOT_MB", "MGM_PF_LATE", "MGM_PF_NOF", "MGM_PF_L0ONLY", "MGM_MORTON_T_MIN", "MGM_UPPER_RES_MIN", "MGM_NO_ZG", "MGM_BOT_GEMV_MIN", "MGM_NO_C0_FUSE"):
        os.environ.pop(k, None)
    os.environ.update(var)
    m = MGM(w.points, w.normals, w.stencil, w.levels)
    u = torch.zeros_like(f)
    for _ in range(3):
        m.vcycle(f, u)
    acc = None
    for _ in range(20):
        m.vcycle(f, u)
        torch.cuda.synchronize()
        tr = mgm_trace_read(m.ctx)
        d = np.diff([t for _, t in tr]) / 1e3
        acc = d if acc is None else acc + d
    acc /= 20
    print(json.dumps(var), f"total {acc.sum():.1f} us")
    for (lab, _), dt in zip(tr[1:], acc):
        print(f"   {dt:8.1f} us  {lab}")
    m.close()

# per-phase costs of the one-kernel bottom (last variant), grouped by (op, local, rows, tpr)
if os.environ.get("BOTTOM_PHASES"):
    from paper_2204_06154_b200 import mgm_bottom_trace_read
    os.environ.update(variants[-1])
    m = MGM(w.points, w.normals, w.stencil, w.levels)
    u = torch.zeros_like(f)
    m.vcycle(f, u)
    acc = None
    for _ in range(10):
        m.vcycle(f, u)
        torch.cuda.synchronize()
        st, meta = mgm_bottom_trace_read(m.ctx)
        d = np.diff(st.astype(np.float64)) / 1e3
        acc = d if acc is None else acc + d
    acc /= 10
    names = ["ZERO", "GS", "RES", "MVZ", "ADD", "MV", "STORE"]
    print("bottom phases:", len(st), "sum of phase gaps", acc.sum(), "us")
    rows = {}
    for q, dt in enumerate(acc):
        k = (names[meta[q, 0]], int(meta[q, 1]), int(meta[q, 2]) if meta[q, 0] != 1 else -1, int(meta[q, 3]))
        rows.setdefault(k, []).append(dt)
    for k, v in sorted(rows.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {k}: n={len(v)} mean {np.mean(v):.2f} us total {np.sum(v):.1f} us")
    m.close()
