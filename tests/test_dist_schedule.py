"""Multi-GPU decomposition, checked on CPU with gloo,
world_size 2: every rank holds the full hierarchy and full vectors; each level-0 operator
application (every colour of the GS sweep, the residual, the restriction, the
interpolation) is split into `nranks` contiguous row pieces -- a colour's rows are Morton
ordered, so each piece is a Morton block of that colour -- rank q computes piece q and the
pieces are exchanged by broadcasts from their owners; the lower levels run redundantly.
This is the schedule libmgm executes with NCCL (mgm_dist_attach).  The distributed V-cycle
must equal the sequential one (oracle, Alg. 3) bitwise: same arithmetic per row, and
same-colour rows never read each other (O12).  The oracle is only the reference here."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import mgm_inputs as MI

WORLD = 2


def piece(lo, hi, R, q):
    """rows [a, b) of piece q of [lo, hi) (the rule of libmgm's piece())"""
    n = hi - lo
    return lo + n * q // R, lo + n * (q + 1) // R


def exchange(v, lo, hi, R):
    for q in range(R):
        a, b = piece(lo, hi, R, q)
        if b > a:
            t = torch.from_numpy(np.ascontiguousarray(v[a:b]))
            dist.broadcast(t, src=q)
            v[a:b] = t.numpy()


def dist_vcycle(O, f, u, rank, R):
    """Alg. 3 with level 0 split across ranks (mirrors enqueue_vcycle with dist_levels = 1)."""
    lv, p, lp = O.levels, O.p, O.lp
    L0 = lv[0]
    A = L0.L
    order = L0.order
    cols = L0.colour[order]
    bounds = np.concatenate([[0], np.cumsum(np.bincount(cols, minlength=L0.ncolours))])

    def sweep(u, backward):
        cs = range(L0.ncolours - 1, -1, -1) if backward else range(L0.ncolours)
        for c in cs:
            a, b = piece(bounds[c], bounds[c + 1], R, rank)
            for i in order[a:b]:   # this rank's Morton block of colour c (O12 row update)
                s0, s1 = A.ptr[i], A.ptr[i + 1]
                cols, vals = A.idx[s0:s1], A.val[s0:s1]
                aii = vals[cols == i][0]
                r = f[i] - aii * u[i]
                for cj, v in zip(cols, vals):
                    if cj != i:
                        r = r - v * u[cj]
                u[i] = u[i] + r / aii
            exchange_rows(u, order, bounds[c], bounds[c + 1])

    def exchange_rows(v, rows, lo, hi):
        for q in range(R):
            a, b = piece(lo, hi, R, q)
            if b > a:
                idx = rows[a:b]
                t = torch.from_numpy(np.ascontiguousarray(v[idx]))
                dist.broadcast(t, src=q)
                v[idx] = t.numpy()

    u = u.copy()
    for _ in range(lp["nu1"]):
        sweep(u, lp["smoother"] == 1)
    # residual and restriction, split by rows (lib order of level 0 / of level 1)
    t = np.zeros_like(f)
    a, b = piece(0, L0.N, R, rank)
    rows = order[a:b]
    t[rows] = (f - L0.L.matvec(u))[rows]   # the residual rows of this piece
    exchange_rows(t, order, 0, L0.N)
    L1 = lv[1]
    r1 = np.zeros(L1.N)
    o1 = L1.order if L1.order is not None else np.arange(L1.N)
    a, b = piece(0, L1.N, R, rank)
    full = L0.R.matvec(t)
    r1[o1[a:b]] = full[o1[a:b]]
    exchange_rows(r1, o1, 0, L1.N)
    # levels >= 1: redundant on every rank (oracle steps of Alg. 3 lines 6-14)
    r = [None] * p
    e = [None] * p
    r[1] = r1
    for j in range(1, p - 1):
        e[j] = np.zeros_like(r[j])
        O._smooth(lv[j], r[j], e[j], lp["nu1"], lp["smoother"] == 1)
        r[j + 1] = O._restrict(lv[j], O._residual(lv[j], r[j], e[j]))
    e[p - 1] = O.coarse_solve(r[p - 1])
    for j in range(p - 2, 0, -1):
        e[j] = e[j] + O._interp(lv[j], e[j + 1])
        O._smooth(lv[j], r[j], e[j], lp["nu2"], lp["smoother"] in (1, 2))
    # interpolation + correction split by rows, then the post-sweep
    corr = O._interp(L0, e[1])
    a, b = piece(0, L0.N, R, rank)
    rows = order[a:b]
    un = u.copy()
    un[rows] = u[rows] + corr[rows]
    exchange_rows(un, order, 0, L0.N)
    for _ in range(lp["nu2"]):
        sweep(un, lp["smoother"] in (1, 2))
    return un


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import oracle as orc

        w = MI.make_workload(3, n=2000)
        O = orc.Oracle(w.points, w.normals, w.stencil, w.levels)
        rng = np.random.default_rng(11)
        f = rng.uniform(-1, 1, len(w.points))
        u0 = rng.uniform(-1, 1, len(w.points))
        ud = dist_vcycle(O, f, u0, rank, WORLD)
        us = O.vcycle_level_order(f, u0)
        # every rank holds the same replicated vector, bitwise equal to the sequential cycle
        other = torch.from_numpy(ud.copy())
        dist.broadcast(other, src=0)
        q.put((rank, bool(np.array_equal(ud, us)), bool(np.array_equal(ud, other.numpy()))))
    finally:
        dist.destroy_process_group()


def test_dist_vcycle_gloo_world2():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    res = sorted(q.get(timeout=5) for _ in range(WORLD))
    for p in procs:
        assert p.exitcode == 0
    assert all(eq_seq and eq_rank for _, eq_seq, eq_rank in res), res
