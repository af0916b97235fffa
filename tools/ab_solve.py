"""A/B timing of the cfg3 (or other) solve path under environment variants (each variant
in its own process, since libmgm reads its knobs at load / setup time).

  python tools/ab_solve.py [--cfg 3] [--n N] VAR=VAL,VAR2=VAL ...   ('-' = no variables)
Prints one JSON line per variant: V-cycle ms (graph, 50 replays), zero-guess preconditioner
ms, MGM-GMRES solve ms (median of 5) and iterations, traced stage times."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, n):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import mgm_inputs as MI
    from paper_2204_06154_b200 import MGM, mgm_apply, mgm_trace_read

    w = MI.make_workload(cfg, n=n)
    m = MGM(w.points, w.normals, w.stencil, w.levels)
    N = len(w.points)
    f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, N)).cuda()
    u = torch.zeros_like(f)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        m.vcycle(f, u)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(50):
        m.vcycle(f, u)
    e1.record(st)
    torch.cuda.synchronize()
    vc = e0.elapsed_time(e1) / 50
    rhs = torch.from_numpy(w.rhs).cuda()
    x = torch.empty_like(rhs)
    ts, its = [], None
    for k in range(7):
        _, rep = m.solve(rhs, x, tol=1e-10)
        if k >= 2:
            ts.append(rep.solve_ms)
        its = rep.iterations
    ts.sort()
    out = {"vcycle_ms": vc, "solve_ms": ts[len(ts) // 2], "its": its, "final": rep.final_rel_residual}
    if os.environ.get("MGM_TRACE"):
        for _ in range(3):
            m.vcycle(f, u)
        acc = None
        for _ in range(10):
            m.vcycle(f, u)
            torch.cuda.synchronize()
            tr = mgm_trace_read(m.ctx)
            d = np.diff([t for _, t in tr]) / 1e3
            acc = d if acc is None else acc + d
        out["stages"] = {lab: round(float(v) / 10, 1) for (lab, _), v in zip(tr[1:], acc)}
    print("RESULT " + json.dumps(out), flush=True)


def main():
    args = sys.argv[1:]
    cfg, n = 3, None
    if args and args[0] == "--child":
        child(int(args[1]), None if args[2] == "None" else int(args[2]))
        return
    while args and args[0].startswith("--"):
        if args[0] == "--cfg":
            cfg = int(args[1]); args = args[2:]
        elif args[0] == "--n":
            n = int(args[1]); args = args[2:]
    for var in args or ["-"]:
        env = dict(os.environ)
        if var != "-":
            for kv in var.split(","):
                k, v = kv.split("=", 1)
                env[k] = v
        r = subprocess.run([sys.executable, __file__, "--child", str(cfg), str(n)], env=env,
                           capture_output=True, text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        print(json.dumps({"variant": var, **(json.loads(line[0][7:]) if line else {"error": r.stderr[-1500:]})}),
              flush=True)


if __name__ == "__main__":
    main()
