"""Multi-GPU decomposition, checked on CPU with gloo,
world_size 2, driven by the partition tables libmgm itself computes (mgm_host_partition_level:
the host code mgm_dist_attach runs).

Each rank owns a Morton block of rows on every distributed level and keeps every other row
NaN except its ghosts; the V-cycle runs the oracle's per-row arithmetic on the owned rows
only (orc_gs_sweep on the rank's rows of one colour, the oracle's SpMV / transfer routines
restricted to owned rows) and refreshes ghosts with gloo send/recv of exactly the library's
send lists, in the library's schedule: after each colour of a sweep (that colour's slice),
after interpolation + correction and before the restriction (all ghosts); the first
replicated level is all-gathered.  A ghost missing from the tables, a colour slice at the
wrong offset or a halo missing from the schedule reads a NaN and fails the bitwise comparison
with the sequential oracle V-cycle (Alg. 3).  The oracle is only the reference
arithmetic here; the tables come from the library (no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import mgm_inputs as MI

WORLD = 2


def _level_tables(O, j, owner, nranks, rank, D):
    """The library's partition tables of level j (lib order = colour-major, Morton within a
    colour, the library's rule) plus the lib <-> Morton maps."""
    from paper_2204_06154_b200.mgm import mgm_host_partition_level

    lv = O.levels[j]
    order = lv.order                         # lib row -> Morton row
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    A = lv.L
    rows = order
    cnt = np.diff(A.ptr)[rows]
    Lp = np.concatenate([[0], np.cumsum(cnt)])
    Lc = np.concatenate([inv[A.idx[A.ptr[r]:A.ptr[r + 1]]] for r in rows])
    col = lv.colour[order]
    P = Pf = None
    oc = of = None
    if j + 1 < O.p:
        nxt = O.levels[j + 1]
        inv_c = np.empty_like(nxt.order) if nxt.order is not None else np.arange(nxt.N)
        if nxt.order is not None:
            inv_c[nxt.order] = np.arange(nxt.N)
        Pm = lv.P
        pc = np.diff(Pm.ptr)[rows]
        P = (np.concatenate([[0], np.cumsum(pc)]),
             np.concatenate([inv_c[Pm.idx[Pm.ptr[r]:Pm.ptr[r + 1]]] for r in rows]), nxt.N)
        oc = owner[j + 1]
    if j > 0:
        prv = O.levels[j - 1]
        Pm = prv.P
        pr = prv.order
        pc = np.diff(Pm.ptr)[pr]
        Pf = (np.concatenate([[0], np.cumsum(pc)]),
              np.concatenate([inv[Pm.idx[Pm.ptr[r]:Pm.ptr[r + 1]]] for r in pr]), prv.N)
        of = owner[j - 1]
    T = mgm_host_partition_level(Lp, Lc, col, lv.ncolours, owner[j], nranks, rank, P, oc, Pf, of)
    T["order"] = order
    return T


def _owners(O, nranks, D):
    """owner of every lib row on levels 0..D: the level-0 Morton block of its point (lib order)."""
    N = O.levels[0].N
    mor0 = np.empty(N, dtype=np.int64)
    mor0[O.levels[0].ids] = np.arange(N)              # level 0 rows are in Morton order
    starts = np.array([q * N // nranks for q in range(nranks + 1)])
    out = []
    for j in range(D + 1):
        lv = O.levels[j]
        order = lv.order if lv.order is not None else np.arange(lv.N)
        m0 = mor0[lv.ids[order]]
        out.append((np.searchsorted(starts, m0, side="right") - 1).astype(np.int32))
    return out


def _exchange(v, T, colour=None):
    """send this rank's slice (colour c or all) to every peer, receive into the ghost rows"""
    order = T["order"]
    reqs, bufs = [], []
    for i, p in enumerate(T["peers"]):
        if colour is None:
            s0, s1 = T["send_off"][i], T["send_off"][i + 1]
            g0, g1 = T["recv_off"][i], T["recv_off"][i + 1]
        else:
            s0, s1 = T["send_coff"][i][colour], T["send_coff"][i][colour + 1]
            g0, g1 = T["recv_coff"][i][colour], T["recv_coff"][i][colour + 1]
        if s1 > s0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(v[order[T["send_rows"][s0:s1]]])), int(p)))
        if g1 > g0:
            buf = torch.empty(g1 - g0, dtype=torch.float64)
            reqs.append(dist.irecv(buf, int(p)))
            bufs.append((buf, g0, g1))
    for r in reqs:
        r.wait()
    for buf, g0, g1 in bufs:
        v[order[T["ghosts"][g0:g1]]] = buf.numpy()


def _sweep_rows(OR, A, rows, f, u):
    """the oracle's O12 row update (orc_gs_sweep) on the given rows only, in their order"""
    import ctypes

    fail = ctypes.c_int64(-1)
    rc = OR.lib().orc_gs_sweep(ctypes.c_int64(len(rows)), OR._p(A.ptr, OR.i64p), OR._p(A.idx, OR.i64p),
                               OR._p(A.val, OR.f64p), OR._p(rows, OR.i64p), ctypes.c_int(0), OR._p(f, OR.f64p),
                               OR._p(u, OR.f64p), None, ctypes.c_double(0.0), ctypes.byref(fail))
    assert rc == 0


def dist_vcycle(O, f, u, rank, nranks, D):
    """Alg. 3 with levels 0..D-1 partitioned (owned rows + ghosts, NaN elsewhere), levels >= D
    replicated (the oracle's routines on full vectors)."""
    import oracle as OR

    lp = O.lp
    nu1, nu2 = lp["nu1"], lp["nu2"]
    owner = _owners(O, nranks, D)
    T = [_level_tables(O, j, owner, nranks, rank, D) for j in range(D)]
    mine = [T[j]["order"][T[j]["rows"]] for j in range(D)]          # my rows (Morton index)

    def local(v, j, ghosts_too=True):
        out = np.full_like(v, np.nan)
        out[mine[j]] = v[mine[j]]
        if ghosts_too:
            g = T[j]["order"][T[j]["ghosts"]]
            out[g] = v[g]
        return out

    def sweep(j, fj, uj):
        lv = O.levels[j]
        for c in range(lv.ncolours):
            rows = np.sort(mine[j][lv.colour[mine[j]] == c])
            if len(rows):
                _sweep_rows(OR, lv.L, np.ascontiguousarray(rows, dtype=np.int64), fj, uj)
            _exchange(uj, T[j], c)

    def own(vals, j):  # keep only this rank's rows of a full-length result
        out = np.full_like(vals, np.nan)
        out[mine[j]] = vals[mine[j]]
        return out

    p = O.p
    r, e = [None] * p, [None] * p
    u = local(u, 0)
    f = local(f, 0, ghosts_too=False)
    for _ in range(nu1):                                              # line 4
        sweep(0, f, u)
    for j in range(p - 1):                                            # lines 5-9
        lv = O.levels[j]
        fj, uj = (f, u) if j == 0 else (r[j], e[j])
        if j < D:
            t = own(fj - lv.L.matvec(uj), j)
            _exchange(t, T[j])                                        # restriction reads t ghosts
            rc = lv.R.matvec(t)
            if j + 1 < D:
                r[j + 1] = own(rc, j + 1)
            else:                                                     # all-gather the replicated level
                mask = owner[j + 1] == rank
                nxt = O.levels[j + 1]
                ordr = nxt.order if nxt.order is not None else np.arange(nxt.N)
                vals = np.where(np.isin(np.arange(nxt.N), ordr[np.nonzero(mask)[0]]), rc, 0.0)
                tt = torch.from_numpy(vals)
                dist.all_reduce(tt)                                   # (disjoint shares: a gather)
                r[j + 1] = tt.numpy().copy()
        else:
            r[j + 1] = O._restrict(lv, O._residual(lv, fj, uj))
        if j + 1 < p - 1:
            nj = j + 1
            if nj < D:
                e[nj] = np.full(O.levels[nj].N, np.nan)
                e[nj][mine[nj]] = 0.0
                e[nj][T[nj]["order"][T[nj]["ghosts"]]] = 0.0         # ghosts start at 0 too
                for _ in range(nu1):
                    sweep(nj, r[nj], e[nj])
            else:
                e[nj] = np.zeros(O.levels[nj].N)
                O._smooth(O.levels[nj], r[nj], e[nj], nu1, False)
    e[p - 1] = O.coarse_solve(r[p - 1])                                # line 10
    for j in range(p - 2, -1, -1):                                   # lines 11-16
        lv = O.levels[j]
        uj = u if j == 0 else e[j]
        fj = f if j == 0 else r[j]
        if j < D:
            corr = own(lv.P.matvec(e[j + 1]), j)
            uj[mine[j]] = uj[mine[j]] + corr[mine[j]]
            _exchange(uj, T[j])
            for _ in range(nu2):
                sweep(j, fj, uj)
        else:
            uj += O._interp(lv, e[j + 1])
            O._smooth(lv, fj, uj, nu2, False)
    return u[mine[0]], mine[0]


def _worker(rank, port, result_q, D):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import traceback
    try:
        import oracle as O

        w = MI.make_workload(1, n=2000)
        lv = dict(w.levels, num_levels=4)
        Oh = O.Oracle(w.points, w.normals, w.stencil, lv)
        rng = np.random.default_rng(3)
        n = len(w.points)
        f, u0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        um, rows = dist_vcycle(Oh, f, u0, rank, WORLD, D)
        ref = Oh.vcycle_level_order(f, u0)
        ok = np.array_equal(um, ref[rows]) and np.isfinite(um).all()
        counts = torch.tensor([len(rows)])
        dist.all_reduce(counts)
        result_q.put((rank, bool(ok), int(counts.item()), n, float(np.nanmax(np.abs(um - ref[rows])))))
    except Exception:
        result_q.put((rank, False, -1, -1, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("D", [1, 2, 3])
def test_distributed_vcycle_equals_sequential(D):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q, D)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(WORLD)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, ok, total, n, diff in res:
        assert total == n                      # the ranks' rows tile level 0
        assert ok, (rank, diff)


def test_partition_tables_properties():
    """The tables of every rank of a 3-way split: owned rows tile the level, ghosts are
    exactly the non-owned rows the operators read, every ghost is sent by its owner (the
    send list of q to p equals p's ghosts owned by q, in the same order), colour slices are
    contiguous and ordered."""
    import oracle as O
    from paper_2204_06154_b200.mgm import mgm_host_partition_level  # noqa: F401

    w = MI.make_workload(1, n=3000)
    Oh = O.Oracle(w.points, w.normals, w.stencil, dict(w.levels, num_levels=3))
    R = 3
    owner = _owners(Oh, R, 2)
    for j in range(2):
        Ts = [_level_tables(Oh, j, owner, R, q, 2) for q in range(R)]
        n = Oh.levels[j].N
        allrows = np.sort(np.concatenate([T["rows"] for T in Ts]))
        assert np.array_equal(allrows, np.arange(n))
        col = Oh.levels[j].colour[Ts[0]["order"]]
        for q, T in enumerate(Ts):
            assert (owner[j][T["rows"]] == q).all()
            assert (owner[j][T["ghosts"]] != q).all()
            for i, p in enumerate(T["peers"]):
                s = T["send_rows"][T["send_off"][i]:T["send_off"][i + 1]]
                Tp = Ts[p]
                k = list(Tp["peers"]).index(q)
                g = Tp["ghosts"][Tp["recv_off"][k]:Tp["recv_off"][k + 1]]
                assert np.array_equal(s, g)                 # what q sends is what p receives
                sc = T["send_coff"][i]
                assert (np.diff(sc) >= 0).all() and sc[0] == T["send_off"][i] and sc[-1] == T["send_off"][i + 1]
                for c in range(len(sc) - 1):
                    assert (col[s[sc[c] - T["send_off"][i]:sc[c + 1] - T["send_off"][i]]] == c).all()
