"""One batched (multi-RHS) V-cycle of cfg3 between cudaProfilerStart/Stop (for an ncu launch
list: ncu --profile-from-start off --metrics gpu__time_duration.sum ...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM, mgm_vcycle_batch

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = MI.make_workload(3)
m = MGM(w.points, w.normals, w.stencil, w.levels)
N = len(w.points)
F = torch.from_numpy(np.random.default_rng(K).uniform(-1, 1, (K, N))).cuda()
U = torch.zeros_like(F)
for _ in range(3):
    mgm_vcycle_batch(m.ctx, K, F, U)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    mgm_vcycle_batch(m.ctx, K, F, U)
e1.record()
torch.cuda.synchronize()
print("K", K, "vcycle_ms", e0.elapsed_time(e1) / 10, flush=True)
torch.cuda.profiler.start()
mgm_vcycle_batch(m.ctx, K, F, U)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
