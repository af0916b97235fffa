mkdir -p gpurun_out
MGM_SETUP_TIMING=1 python -c "
import sys, time; sys.path.insert(0, '.')
t = time.time()
import mgm_inputs as MI
w = MI.make_workload(5)
print('workload_s', time.time() - t, flush=True)
from paper_2204_06154_b200 import MGM
t = time.time(); m = MGM(w.points, w.normals, w.stencil, w.levels); print('setup_s', time.time() - t, flush=True)
" > gpurun_out/setup_timing_cfg5.log 2>&1
