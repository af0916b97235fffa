#!/usr/bin/env python
"""Benchmark of the MGM solve path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[2], the metric's N=1M case): torus R=1, r=1/3,
N = 1,048,576 quasi-uniform points, shifted surface Poisson (mu = 1), RBF-FD PHS r^5 + degree-3
polynomials, n = 30, m = 6, V(1,1), 8 levels, right-preconditioned GMRES(50) to 1e-10.
A step = one full MGM-GMRES solve from a zero initial guess (every V-cycle, SpMV and
Krylov step of the hot path); setup (hierarchy construction) is untimed, as in the paper
(P:588).  The hierarchy (~2.6 GB) and Krylov basis are far larger than L2 (126 MB), so no
L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--cfg 3] [--n N]

--impl reference times the oracle (oracle/, plain single-thread C + numpy) on the SAME
workload (N = 1,048,576), one pinned host core, setup untimed: one warm-up, then the
median of up to 3 solves (about 1.5 min including the oracle's ~45 s setup).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MGM-GMRES solve time to 1e-10 at N=1M (torus, RBF-FD n=30, V(1,1)); V-cycle HBM GB/s"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _cpu_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def oracle_worker(steps: int, warmup: int, n: int | None):
    """(child process, pinned to one core) The oracle as it stands on the benched workload:
    setup (untimed, as the paper), then `warmup` + `steps` MGM-GMRES solves to 1e-10;
    prints one JSON line with the median solve time."""
    import mgm_inputs as MI
    import oracle as O

    w = MI.make_workload(3, n=n)
    t0 = time.perf_counter()
    h = O.Oracle(w.points, w.normals, w.stencil, w.levels)
    setup_s = time.perf_counter() - t0
    times, its = [], []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        _, rep = h.solve(w.rhs, tol=1e-10)
        dt = time.perf_counter() - t0
        assert rep.converged, rep
        if s >= warmup:
            times.append(dt)
            its.append(rep.iterations)
    print(json.dumps({"ms": statistics.median(times) * 1e3, "times_ms": [t * 1e3 for t in times],
                      "iterations": its, "setup_s": setup_s, "N": len(w.points)}), flush=True)
    return 0


def oracle_full(steps: int, warmup: int, n: int | None = None):
    """Time the oracle on the SAME workload as the GPU arm (BASELINE configs[2], N = 1,048,576)
    on one host core: a child process under `taskset -c <core>` with single-threaded BLAS,
    3 solves (median) after one warm-up by default.  Returns (ms per solve, cpu_baseline dict)."""
    core = sorted(os.sched_getaffinity(0))[0] if hasattr(os, "sched_getaffinity") else 0
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.abspath(__file__), "--oracle-worker", "--steps", str(steps),
           "--warmup", str(warmup)] + (["--n", str(n)] if n else [])
    try:
        subprocess.run(["taskset", "-c", "0", "true"], check=True, capture_output=True)
        cmd = ["taskset", "-c", str(core)] + cmd
        pinned = True
    except Exception:
        pinned = False
    r = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if r.returncode != 0:
        raise RuntimeError("oracle worker failed: " + r.stderr[-2000:])
    d = json.loads(r.stdout.strip().splitlines()[-1])
    ms = d["ms"]
    cpu = dict(kind="oracle", cores=1, value=ms, unit="ms", pinned_core=core if pinned else None,
               sample=(f"the benched workload itself: torus N={d['N']} (BASELINE configs[2]), one MGM-GMRES "
                       f"solve to 1e-10 ({d['iterations'][0]} iterations), median of {len(d['times_ms'])} "
                       f"after {warmup} warm-up; oracle setup {d['setup_s']:.1f} s untimed (P:588)"),
               times_ms=d["times_ms"], iterations=d["iterations"], setup_s=d["setup_s"], **_cpu_info())
    return ms, cpu


def stage_breakdown(w, f, hbm):
    """Stage times of the V-cycle graph (MGM_TRACE instance, 20 cycles averaged) with the
    algorithmic bytes of each stage (DESIGN.md section 6 byte model) and the one-kernel
    bottom's share; the bottom is latency-bound, its GB/s is reported against HBM anyway."""
    import numpy as np
    import torch
    from paper_2204_06154_b200 import MGM, mgm_trace_read

    os.environ["MGM_TRACE"] = "1"
    try:
        mt = MGM(w.points, w.normals, w.stencil, w.levels)
    finally:
        os.environ.pop("MGM_TRACE", None)
    lv = mt.level_info()
    u = torch.zeros_like(f)
    for _ in range(3):
        mt.vcycle(f, u)
    acc = None
    for _ in range(20):
        mt.vcycle(f, u)
        torch.cuda.synchronize()
        tr = mgm_trace_read(mt.ctx)
        d = np.diff([t for _, t in tr]) / 1e3
        acc = d if acc is None else acc + d
    acc = acc / 20
    labels = [lab for lab, _ in tr[1:]]
    nu1, nu2 = w.levels.get("nu1", 1), w.levels.get("nu2", 1)

    def sweep_b(j, nsw):
        return nsw * (12.0 * lv[j]["nnz"] + 24.0 * lv[j]["n"])

    # level 0 of the traced (general) V-cycle: the last presmooth and postsmooth write their
    # increments d (8 B/row each) and the residual reads the later-colour entries only, from d
    # (libmgm dpre_ok / mode3_ok: shifted problem, forward sweeps, level >= 131072 rows)
    smoother = w.levels.get("smoother", 0)
    d0 = (os.environ.get("MGM_NO_MODE3") is None and w.stencil.get("problem", 0) == 0 and smoother == 0
          and lv[0]["nnz_zg"] < lv[0]["nnz"] and lv[0]["n"] >= 131072 and len(lv) > 1)

    def bytes_of(lab):
        name, jl = lab.rsplit(" L", 1)
        j = int(jl)
        if name == "presmooth":
            return sweep_b(j, nu1) + (8.0 * lv[j]["n"] if d0 and j == 0 else 0.0)
        if name == "residual":  # reads L, u, f; writes t (12 z + 24 N)
            if d0 and j == 0:  # later-colour entries only, from the presmooth's increments
                return 12.0 * (lv[j]["nnz"] - lv[j]["nnz_zg"]) + 24.0 * lv[j]["n"]
            return 12.0 * lv[j]["nnz"] + 24.0 * lv[j]["n"]
        if name == "restrict":
            return 12.0 * lv[j]["nnz_P"] + 8.0 * lv[j]["n"] + 8.0 * lv[j + 1]["n"]
        if name == "zero+presmooth":  # first sweep from the zero guess: diag + earlier colours, no fill
            if lv[j]["nnz_zg"] < lv[j]["nnz"] and nu1 >= 1:
                return 12.0 * lv[j]["nnz_zg"] + 16.0 * lv[j]["n"] + sweep_b(j, nu1 - 1)
            return 8.0 * lv[j]["n"] + sweep_b(j, nu1)
        if name == "residual+restrict":
            res = 12.0 * lv[j]["nnz"] + 24.0 * lv[j]["n"]
            # after the zero-guess sweep (coarse levels always start from zero) or, on level 0 of
            # the traced general V-cycle, from the presmooth's increments d (d0)
            if (d0 and j == 0) or (j > 0 and lv[j]["nnz_zg"] < lv[j]["nnz"] and nu1 == 1 and lv[j]["n"] >= 131072):
                res = 12.0 * (lv[j]["nnz"] - lv[j]["nnz_zg"]) + 24.0 * lv[j]["n"]
            return res + 12.0 * lv[j]["nnz_P"] + 8.0 * lv[j]["n"] + 8.0 * lv[j + 1]["n"]
        if name == "interp":
            return 12.0 * lv[j]["nnz_P"] + 8.0 * lv[j + 1]["n"] + 16.0 * lv[j]["n"]
        if name == "interp+postsmooth":
            return 12.0 * lv[j]["nnz_P"] + 8.0 * lv[j + 1]["n"] + 16.0 * lv[j]["n"] + sweep_b(j, nu2)
        if name == "postsmooth":
            return sweep_b(j, nu2) + (8.0 * lv[j]["n"] if d0 and j == 0 else 0.0)
        if name == "bottom":  # levels j..p-1: sweeps, residuals, transfers, dense coarse solve
            b = 0.0
            for q in range(j, len(lv) - 1):
                b += sweep_b(q, nu1 + nu2) + 12.0 * lv[q]["nnz"] + 32.0 * lv[q]["n"]
                b += 2 * (12.0 * lv[q]["nnz_P"] + 8.0 * lv[q + 1]["n"]) + 24.0 * lv[q]["n"]
            nc = lv[-1]["n"]
            return b + 12.0 * nc * nc + 16.0 * nc
        return 0.0

    from paper_2204_06154_b200 import mgm_dense_bottom_info
    dinfo = mgm_dense_bottom_info(mt.ctx)
    total = float(acc.sum())
    out, bottom = [], None
    for lab, us in zip(labels, acc):
        b = bytes_of(lab)
        gbs = b / (us * 1e-6) / 1e9 if us > 0 else None
        out.append({"stage": lab, "us": round(float(us), 2), "share": round(float(us) / total, 4),
                    "alg_MB": round(b / 1e6, 2), "GBps": round(gbs, 1) if gbs else None})
        if lab.startswith("bottom") and dinfo["level"] >= 0:
            # the dense bottom B_J: one HBM-bound apply; its bytes are B_J's plus r_J / e_J
            db = dinfo["bytes"] + 16.0 * dinfo["rows"]
            g2 = db / (us * 1e-6) / 1e9 if us > 0 else None
            out[-1]["dense_MB"] = round(db / 1e6, 2)
            out[-1]["dense_GBps"] = round(g2, 1) if g2 else None
            bottom = {"bound": "hbm", "kernel": "k_dense_apply<1> (B_J r_J, levels >= J as one dense operator)",
                      "level": dinfo["level"], "rows": dinfo["rows"], "bytes_per_launch": db,
                      "achieved": g2, "peak": hbm, "unit": "GB/s", "frac": g2 / hbm if g2 else None,
                      "share_of_vcycle": float(us) / total, "us": float(us),
                      "alg3_bytes_replaced": b}
        elif lab.startswith("bottom"):
            bottom = {"bound": "latency (cluster barrier per colour step)", "kernel": "k_vcycle_bottom",
                      "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm if gbs else None,
                      "share_of_vcycle": float(us) / total, "us": float(us)}
    mt.close()
    return out, bottom


def run_reference(args):
    """--impl reference: the oracle (this tier's reference arm) on the GPU arm's workload and
    metric, one pinned host core; rank 0 only (the other ranks exit without work)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    steps = max(1, min(args.steps, 3))
    warm = min(args.warmup, 1)
    ms, cpu = oracle_full(steps, warm, args.n)
    line = {"metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg3 torus N={args.n or 1048576}", "gmres_iterations": cpu["iterations"][0],
                       "parallelism": "oracle, 1 pinned host core"},
            "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mgm")
    ap.add_argument("--cfg", type=int, default=3)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--method", default="rbffd", choices=["rbffd", "gfd"], help="cfg 2 only: RBF-FD or GFD")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--oracle-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-stages", action="store_true", help="skip the traced per-stage V-cycle breakdown")
    ap.add_argument("--parallel", choices=["replicas", "dist"], default="dist",
                    help="N>1: one solve partitioned across the ranks (mgm_dist_attach: Morton row "
                         "blocks + ghost halos, strong scaling; the default) or independent replicas")
    args = ap.parse_args()
    if args.oracle_worker:
        return oracle_worker(args.steps, args.warmup, args.n)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import mgm_inputs as MI
    from paper_2204_06154_b200 import (MGM, mgm_bytes_model, mgm_solve_host, mgm_timing_enable,
                                       mgm_timing_read, mgm_vcycle_kernel_count)

    ws, rank, local = _dist()
    if args.warmup < 3:
        print(f"bench.py: --warmup {args.warmup} < 3 (the timing rules ask for >= 3)", file=sys.stderr)
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    w = MI.make_workload(args.cfg, n=args.n, method=args.method)
    N = len(w.points)
    t0 = time.perf_counter()
    m = MGM(w.points, w.normals, w.stencil, w.levels)
    setup_s = time.perf_counter() - t0
    dist_mode = ws > 1 and args.parallel == "dist"
    dinfo = None
    ids = np.arange(N)
    if dist_mode:  # this rank's Morton block: its rows of every vector (mgm_local_rows order)
        from paper_2204_06154_b200 import mgm_dist_info
        m.attach_dist()
        ids = m.local_ids
        dinfo = mgm_dist_info(m.ctx)
    NL = len(ids)
    st = torch.cuda.current_stream()
    rhs = torch.from_numpy(np.ascontiguousarray(w.rhs[ids])).cuda()
    x = torch.empty_like(rhs)

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        rep = m.solve(rhs, x, tol=1e-10)[1]
    barrier()
    clk = ClockSampler(local)
    clk.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    its = []
    prof = bool(os.environ.get("MGM_BENCH_PROFILE"))  # ncu --profile-from-start off: timed region only
    if prof:
        torch.cuda.profiler.start()
    ev0.record(st)
    for _ in range(args.steps):
        _, rep = m.solve(rhs, x, tol=1e-10)
        its.append(rep.iterations)
    ev1.record(st)
    if prof:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    assert rep.converged and rep.final_rel_residual <= 1e-10, rep

    # ---- end to end through the public API with pinned host buffers
    rhs_h = torch.from_numpy(np.ascontiguousarray(w.rhs[ids])).pin_memory()
    x_h = torch.empty(NL, dtype=torch.float64).pin_memory()
    rn, xn = rhs_h.numpy(), x_h.numpy()
    mgm_solve_host(m.ctx, rn, xn, tol=1e-10)
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        mgm_solve_host(m.ctx, rn, xn, tol=1e-10)
    e1.record(st)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / args.steps

    # ---- the other solvers of the path on the same system (context, not the metric):
    # MGM-BiCGSTAB (iterations = preconditioner applications) and standalone MGM
    others = {}
    for name, kr in (("bicgstab", 2), ("standalone", 0)):
        m.solve(rhs, x, tol=1e-10, krylov=kr, maxit=300)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _, rk = m.solve(rhs, x, tol=1e-10, krylov=kr, maxit=300)
        e1.record(st)
        barrier()
        others[name] = {"ms": e0.elapsed_time(e1), "iterations": rk.iterations, "converged": bool(rk.converged),
                        "final_rel_residual": rk.final_rel_residual}

    # ---- multi-right-hand-side throughput: K columns per operator pass
    multi = {}
    if ws == 1 and not args.no_stages:
        from paper_2204_06154_b200 import mgm_solve_batch, mgm_vcycle_batch

        for K in (4, 8):
            FK = torch.from_numpy(np.random.default_rng(K).uniform(-1, 1, (K, N))).cuda()
            UK = torch.zeros_like(FK)
            for _ in range(3):
                mgm_vcycle_batch(m.ctx, K, FK, UK)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10):
                mgm_vcycle_batch(m.ctx, K, FK, UK)
            e1.record(st)
            barrier()
            vck = e0.elapsed_time(e1) / 10
            RK = torch.from_numpy(np.stack([w.rhs] * K)).cuda()
            XK = torch.zeros_like(RK)
            e0.record(st)
            reps = mgm_solve_batch(m.ctx, K, RK, XK, tol=1e-10, maxit=300)
            e1.record(st)
            barrier()
            sa_ms = e0.elapsed_time(e1)
            RG = torch.from_numpy(np.stack([w.rhs] + [np.random.default_rng(100 + k).uniform(-1, 1, N)
                                                      for k in range(K - 1)])).cuda()
            XG = torch.zeros_like(RG)
            mgm_solve_batch(m.ctx, K, RG, XG, tol=1e-10, maxit=300, krylov=1)  # (allocates the basis)
            barrier()
            e0.record(st)
            repg = mgm_solve_batch(m.ctx, K, RG, XG, tol=1e-10, maxit=300, krylov=1)
            e1.record(st)
            barrier()
            multi[K] = {"vcycle_ms": vck, "vcycle_ms_per_rhs": vck / K,
                        "standalone_ms": sa_ms, "standalone_ms_per_rhs": sa_ms / K,
                        "iterations": max(r.iterations for r in reps),
                        "all_converged": all(r.converged for r in reps),
                        "gmres_ms": e0.elapsed_time(e1), "gmres_ms_per_rhs": e0.elapsed_time(e1) / K,
                        "gmres_iterations": [r.iterations for r in repg],
                        "gmres_all_converged": all(r.converged for r in repg)}

    # ---- V-cycle throughput (graph-replayed V-cycles on device vectors)
    bm = mgm_bytes_model(m.ctx)
    f = torch.from_numpy(np.ascontiguousarray(np.random.default_rng(0).uniform(-1, 1, N)[ids])).cuda()
    u = torch.zeros_like(f)
    for _ in range(5):
        m.vcycle(f, u)
    nv = 50
    barrier()
    e0.record(st)
    for _ in range(nv):
        m.vcycle(f, u)
    e1.record(st)
    barrier()
    vc_ms = e0.elapsed_time(e1) / nv
    peaks = _peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    vc_gbs = bm["vcycle_bytes"] / (vc_ms * 1e-3) / 1e9

    # ---- dominant kernel class: the level-0 colour GS kernels (k_gs_colour).  CUDA events on
    # the library stream bracket each whole level-0 sweep (its colour kernels keep their PDL
    # overlap inside); achieved = algorithmic bytes / (sweep time / colour launches).
    # class 0 = full sweeps (postsmooth; presmooth outside the Krylov preconditioner), class 3 =
    # the first presmooth from the zero guess inside the Krylov solvers (reads the diagonal and
    # earlier-colour entries only: fewer algorithmic bytes per row, reported beside it)
    mgm_timing_enable(m.ctx, 0, True)
    mgm_timing_enable(m.ctx, 3, True)
    for _ in range(args.steps):
        m.solve(rhs, x, tol=1e-10)
    torch.cuda.synchronize()
    tk = mgm_timing_read(m.ctx, 0)
    tz = mgm_timing_read(m.ctx, 3)
    mgm_timing_enable(m.ctx, 0, False)
    mgm_timing_enable(m.ctx, 3, False)
    zg_gbs = tz["alg_bytes"] / (tz["total_ms"] * 1e-3) / 1e9 if tz["total_ms"] > 0 else None
    gs_gbs = tk["alg_bytes"] / (tk["total_ms"] * 1e-3) / 1e9 if tk["total_ms"] > 0 else None
    launch_avg_us = tk["total_ms"] * 1e3 / max(1, tk["launches"])
    alg_per_launch = tk["alg_bytes"] / max(1, tk["launches"])
    traffic = None
    try:  # dram bytes per launch of the same kernel from one ncu --set full capture (profiles/)
        prof = json.load(open(os.path.join(ROOT, "profiles", "r02_ncu_gs_colour_l0.json")))
        traffic = prof["dram_bytes_per_launch"]
    except Exception:
        pass

    # ---- per-stage V-cycle breakdown (a second, traced instance: %globaltimer stamps between
    # the stages of Alg. 3 inside the graph), with each stage's algorithmic bytes
    stages, bottom = None, None
    if not args.no_stages and ws == 1:
        stages, bottom = stage_breakdown(w, f, hbm)

    comm = None
    if dist_mode:  # communication-only replay of one V-cycle's halos + one allreduce (max over ranks)
        from paper_2204_06154_b200 import mgm_dist_comm_time
        c = mgm_dist_comm_time(m.ctx, 20)
        t = torch.tensor([c["halo_ms_per_vcycle"], c["allreduce_us"], vc_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        comm = {"halo_ms_per_vcycle": float(t[0]), "allreduce16_us": float(t[1]),
                "vcycle_ms": float(t[2]), "note": "device times, max over ranks"}
    vk = mgm_vcycle_kernel_count(m.ctx)
    # kernels per solve: per Arnoldi step the V-cycle graph (vk) + SpMV + 5 CGS2 kernels;
    # start: dot + scale; end: lincomb + V-cycle + axpby, true residual SpMV + axpby + dot
    per_step = its[-1] * (vk + 6) + 2 + (vk + 2) + 3
    levels = m.level_info()

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and args.cfg == 3 and ws == 1:
            _, cpu = oracle_full(3, 0, args.n)  # median of 3 solves, one pinned core
        line = {
            "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong" if dist_mode else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded torus cloud, BASELINE configs[2] recipe)",
            "config": {"workload": f"{w.name} N={N}", "levels": [lv["n"] for lv in levels],
                       "nnz": [lv["nnz"] for lv in levels],
                       "colours": [lv["colours"] for lv in levels],
                       "gmres_iterations": its[-1], "restart": w.levels.get("restart", 50), "tol": 1e-10,
                       "parallelism": (f"dist{ws}: Morton row blocks on levels 0..{dinfo['dist_levels'] - 1} "
                                       f"+ ghost halos (NCCL), replicated bottom" if dist_mode else
                                       f"replicas{ws}" if ws > 1 else "single GPU"),
                       "dist_rank0": dinfo, "comm": comm,
                       "l2": "inputs larger than L2 (hierarchy %.2f GB)" %
                             (sum(lv["stored_bytes"] for lv in levels) / 1e9),
                       "setup_s": round(setup_s, 2)},
            "vcycle": {"ms": vc_ms, "alg_bytes_rank0": bm["vcycle_bytes"], "GBps_rank0": vc_gbs,
                       "frac_of_measured_hbm": vc_gbs / hbm, "vcycles_per_s": 1e3 / vc_ms,
                       "Mrows_per_s": N * 1e-3 / vc_ms, "kernels": vk},
            "roofline": {"bound": "hbm", "kernel": "k_gs_colour (level-0 multicolour GS, one launch per colour)",
                         "achieved": gs_gbs, "peak": hbm, "peak_source": peak_src,
                         "unit": "GB/s", "frac": (gs_gbs / hbm) if gs_gbs else None,
                         "traffic": traffic, "alg_bytes_per_launch": alg_per_launch,
                         "launches_timed": tk["launches"], "avg_launch_us": launch_avg_us},
            "roofline_zero_guess_sweep": {
                "bound": "hbm", "kernel": "k_gs_colour<ZG> (level-0 first presmooth from the zero guess)",
                "achieved": zg_gbs, "peak": hbm, "unit": "GB/s", "frac": (zg_gbs / hbm) if zg_gbs else None,
                "alg_bytes_per_launch": tz["alg_bytes"] / max(1, tz["launches"]),
                "launches_timed": tz["launches"],
                "avg_launch_us": tz["total_ms"] * 1e3 / max(1, tz["launches"])},
            "other_solvers": others,
            "vcycle_stages": stages,
            "multi_rhs": multi,
            "roofline_bottom": bottom,
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 8 * N,
                    "d2h_bytes_per_step": 8 * N, "note": "all ranks together (each copies its own rows)"},
            "gpu_launches": per_step * args.steps,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    m.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
