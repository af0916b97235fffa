# usage: bash tools/setup_timing.sh CFG  -> gpurun_out/setup_timing_cfgCFG.log (MGM_SETUP_TIMING stages)
mkdir -p gpurun_out
MGM_SETUP_TIMING=1 python -c "
import sys, time; sys.path.insert(0, '.')
t = time.time()
import mgm_inputs as MI
w = MI.make_workload($1)
print('workload_s', time.time() - t, flush=True)
import torch
from paper_2204_06154_b200 import MGM
torch.zeros(1, device='cuda'); torch.cuda.synchronize()
t = time.time(); m = MGM(w.points, w.normals, w.stencil, w.levels); print('setup_s', time.time() - t, flush=True)
x, rep = m.solve(torch.from_numpy(w.rhs).cuda(), tol=1e-10)
print('solve its', rep.iterations if hasattr(rep, 'iterations') else rep, flush=True)
" > gpurun_out/setup_timing_cfg$1.log 2>&1
