"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/mgm.h
declares, rejects bad arguments without touching a GPU, and its host-side setup steps
(Morton order, kNN, WSE, greedy colouring) equal the oracle's exactly."""
import ctypes
import os
import re

import numpy as np
import pytest

import mgm_inputs as MI
import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mgm.h")).read()
    return sorted(set(re.findall(r"^(?:mgm_status|const char\*)\s+(mgm_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    import paper_2204_06154_b200 as P

    lib = ctypes.CDLL(P.LIB_PATH)
    names = _declared()
    assert len(names) >= 19
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(P.EXPORTED) == names          # the binding covers the whole ABI


def test_setup_rejects_null_arguments():
    import paper_2204_06154_b200 as P

    lib = P.load_library()
    ctx = ctypes.c_void_p()
    st = lib.mgm_setup(None, None, 0, None, None, None, None, ctypes.byref(ctx))
    assert st == P.mgm.MGM_ERR_ARG and not ctx.value
    assert lib.mgm_vcycle(None, None, None, None) == P.mgm.MGM_ERR_ARG


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2204_06154_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "_core.c" not in txt and "orc_" not in txt, f


@pytest.mark.parametrize("n,seed", [(3000, 1), (20000, 2)])
def test_host_morton_and_knn_equal_oracle(n, seed):
    from paper_2204_06154_b200.mgm import mgm_host_knn, mgm_host_morton

    x, _ = MI.fibonacci_sphere(n, jitter=0.2, seed=seed)
    assert np.array_equal(mgm_host_morton(x), O.morton_perm(x))
    for k in (2, 15, 30):
        assert np.array_equal(mgm_host_knn(x, x, k).astype(np.int64), O.knn(x, x, k))
    y = x[::4].copy()
    assert np.array_equal(mgm_host_knn(y, x, 6).astype(np.int64), O.knn(y, x, 6))


def test_host_knn_torus_and_grid_ties():
    from paper_2204_06154_b200.mgm import mgm_host_knn

    x, _ = MI.torus_cloud(6000, seed=3)
    assert np.array_equal(mgm_host_knn(x, x, 30).astype(np.int64), O.knn(x, x, 30))
    g = np.stack(np.meshgrid(np.arange(12.), np.arange(12.), np.arange(3.), indexing="ij"), -1)
    g = g.reshape(-1, 3)                                   # many exact distance ties
    assert np.array_equal(mgm_host_knn(g, g, 19).astype(np.int64), O.knn(g, g, 19))


@pytest.mark.parametrize("maker", [lambda: MI.fibonacci_sphere(8000, jitter=0.1, seed=0)[0],
                                   lambda: MI.torus_cloud(10000, seed=1)[0],
                                   lambda: MI.quartic_cloud(5000, seed=2)[0]])
def test_host_wse_equals_oracle(maker):
    from paper_2204_06154_b200.mgm import mgm_host_wse

    x = maker()
    for nt in (len(x) // 4, len(x) - 1):
        assert np.array_equal(mgm_host_wse(x, nt), O.wse(x, nt))


def test_host_colouring_equals_oracle():
    from paper_2204_06154_b200.mgm import mgm_host_colouring

    w = MI.make_workload(1, n=2000)
    h = O.Oracle(w.points, w.normals, w.stencil, dict(w.levels, num_levels=3))
    for lv in h.levels[:-1]:
        c, nc = mgm_host_colouring(lv.L.ptr, lv.L.idx.astype(np.int32))
        assert nc == lv.ncolours and np.array_equal(c, lv.colour)
