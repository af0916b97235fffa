# round 2: GPU tests, setup timing, cfg2-GFD alpha, cfg5 bench (outputs small)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
MGM_SETUP_TIMING=1 python -c "
import sys, time; sys.path.insert(0, '.')
import mgm_inputs as MI
from paper_2204_06154_b200 import MGM
w = MI.make_workload(3)
t = time.time(); m = MGM(w.points, w.normals, w.stencil, w.levels); print('setup_s', time.time() - t)
" > gpurun_out/setup_timing_cfg3.log 2>&1
python tools/gfd_alpha.py > gpurun_out/gfd_alpha.log 2>&1
timeout 1800 python bench.py --cfg 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
echo "cfg5 rc=$?" >> gpurun_out/bench_cfg5.log
echo done
