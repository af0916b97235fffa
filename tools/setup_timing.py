"""Host wall time per setup phase (MGM_SETUP_TIMING) for the given BASELINE configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MGM_SETUP_TIMING"] = "1"
import torch  # noqa: F401

import mgm_inputs as MI
from paper_2204_06154_b200 import MGM

for c in [int(a) for a in sys.argv[1:]] or [3]:
    t0 = time.perf_counter()
    w = MI.make_workload(c)
    t1 = time.perf_counter()
    print(f"cfg{c}: inputs {t1 - t0:.1f} s, N={len(w.points)}, threads={os.cpu_count()}", flush=True)
    m = MGM(w.points, w.normals, w.stencil, w.levels)
    t2 = time.perf_counter()
    print(f"cfg{c}: mgm_setup {t2 - t1:.1f} s", flush=True)
    m.close()
