"""Time graph-replayed V-cycles of the bench workload under setup-time variants (env knobs
read at mgm_setup: MGM_TAIL_MAX, MGM_NO_TAIL, MGM_NO_PDL)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_bytes_model

cfg = int(os.environ.get("MGM_CFG", "3"))
n = int(os.environ["MGM_N"]) if "MGM_N" in os.environ else None
w = MI.make_workload(cfg, n=n)
variants = json.loads(os.environ.get("VARIANTS", '[{"MGM_TAIL_MAX": "65536"}, {"MGM_TAIL_MAX": "16384"}, '
                                      '{"MGM_TAIL_MAX": "4096"}, {"MGM_TAIL_MAX": "1024"}, {"MGM_NO_TAIL": "1"}]'))
knobs = {"MGM_TAIL_MAX", "MGM_NO_TAIL", "MGM_NO_PDL"}
f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, len(w.points))).cuda()
for var in variants:
    for k in knobs:
        os.environ.pop(k, None)
    os.environ.update(var)
    m = MGM(w.points, w.normals, w.stencil, w.levels)
    u = torch.zeros_like(f)
    for _ in range(5):
        m.vcycle(f, u)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        m.vcycle(f, u)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    bm = mgm_bytes_model(m.ctx)
    print(json.dumps({"variant": var, "vcycle_ms": ms, "GBps": bm["vcycle_bytes"] / ms / 1e6}), flush=True)
    m.close()
