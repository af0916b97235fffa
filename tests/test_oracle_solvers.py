"""Pins of the oracle's cycle and solvers: Alg. 3 V-cycle (O14) against the
textbook dense recursion, GMRES (O15) against dense solves, standalone MGM
(O16), and end-to-end closed forms (O17)."""
import numpy as np
import pytest

import oracle as O
import mgm_inputs as MI


def _hier(problem=0, N=1024, p=4, nu=(1, 1), smoother=0, method=0, seed=11):
    x, nrm = MI.fibonacci_sphere(N, jitter=0.1, seed=seed)
    st = dict(method=method, poly_degree=2, phs_k=1, stencil_n=15 if method == 0 else 20,
              problem=problem, mu=1.0, gfd_alpha=16.0)
    return O.Oracle(x, nrm, st, dict(num_levels=p, interp_m=6, nu1=nu[0], nu2=nu[1],
                                     smoother=smoother))


def _dense_vcycle(h, f, u):
    """Textbook recursive V(nu1,nu2) with dense matrices: S(u) = u + B^{-1}(f - A u),
    B = lower (forward) or upper (backward) triangle of the colour-permuted A; the coarse
    problem is solved by the same cycle from a zero guess; coarsest exact."""
    lv = h.levels
    nu1, nu2 = h.lp["nu1"], h.lp["nu2"]
    pre_b = h.lp["smoother"] == 1
    post_b = h.lp["smoother"] in (1, 2)
    A = [l.L.dense() for l in lv]
    poisson = h.poisson

    def aug(j):
        if not poisson:
            return A[j]
        n = lv[j].N
        M = np.zeros((n + 1, n + 1)); M[:n, :n] = A[j]; M[:n, n] = lv[j].c; M[n, :n] = lv[j].c
        return M

    def smooth(j, f, u, back):
        n = lv[j].N
        Pm = np.eye(n)[lv[j].order]
        Ap = Pm @ A[j] @ Pm.T
        B = np.triu(Ap) if back else np.tril(Ap)
        if poisson:
            lam = u[n]
            r = f[:n] - A[j] @ u[:n] - lv[j].c * lam
            u = u.copy(); u[:n] = u[:n] + Pm.T @ np.linalg.solve(B, Pm @ r)
            return u
        return u + Pm.T @ np.linalg.solve(B, Pm @ (f - A[j] @ u))

    def P_(j, e):
        return np.concatenate([lv[j].P.dense() @ e[:-1], e[-1:]]) if poisson else lv[j].P.dense() @ e

    def R_(j, r):
        n = lv[j].N
        return np.concatenate([lv[j].R.dense() @ r[:n], r[n:]]) if poisson else lv[j].R.dense() @ r

    def cyc(j, f, u):
        if j == h.p - 1:
            return np.linalg.solve(aug(j), f)
        for _ in range(nu1):
            u = smooth(j, f, u, pre_b)
        rc = R_(j, f - aug(j) @ u)
        ec = cyc(j + 1, rc, np.zeros_like(rc))
        u = u + P_(j, ec)
        for _ in range(nu2):
            u = smooth(j, f, u, post_b)
        return u

    return cyc(0, f, u)


@pytest.mark.parametrize("problem,nu,smoother,p", [(0, (1, 1), 0, 4), (0, (2, 2), 2, 3),
                                                   (1, (1, 1), 0, 4), (0, (1, 2), 1, 2)])
def test_vcycle_equals_textbook_dense_recursion(problem, nu, smoother, p):
    h = _hier(problem=problem, N=700, p=p, nu=nu, smoother=smoother)
    rng = np.random.default_rng(0)
    n = h.levels[0].N + (1 if problem else 0)
    f = rng.uniform(-1, 1, n)
    u = rng.uniform(-1, 1, n)
    if problem:
        u[-1] = 0.3
    got = h.vcycle_level_order(f, u)
    ref = _dense_vcycle(h, f, u)
    assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()


def test_vcycle_linear_and_contracting():
    h = _hier(N=1024, p=4)
    rng = np.random.default_rng(1)
    r1, r2 = rng.uniform(-1, 1, (2, 1024))
    M = h.precondition
    assert np.abs(M(r1 + 2 * r2) - M(r1) - 2 * M(r2)).max() < 1e-11 * np.abs(M(r1)).max()
    assert np.array_equal(M(np.zeros(1024)), np.zeros(1024))
    # error propagation E e = e - M(A e); spectral radius < 1 via power iteration (S:464 idea)
    e = rng.uniform(-1, 1, 1024)
    rho = 0.0
    for _ in range(50):
        e2 = e - M(h.apply_A(e))
        rho = np.linalg.norm(e2) / np.linalg.norm(e)
        e = e2 / np.linalg.norm(e2)
    assert rho < 0.5


def test_p1_is_direct_solve():
    h = _hier(N=180, p=1)
    rng = np.random.default_rng(2)
    f = rng.uniform(-1, 1, 180)
    u = h.vcycle_level_order(f, np.zeros(180))
    assert np.linalg.norm(h.apply_A(u) - f) < 1e-12 * np.linalg.norm(f) * 1e2


# ---------------------------------------------------------------- GMRES (O15)
def test_gmres_dense_cases():
    rng = np.random.default_rng(0)
    b = rng.normal(size=10)
    x, rep = O.gmres(lambda v: v, lambda v: v, b, tol=1e-12)
    assert rep.iterations == 1 and np.allclose(x, b, atol=1e-14)
    A = rng.normal(size=(10, 10)) + 5 * np.eye(10)
    x, rep = O.gmres(lambda v: A @ v, lambda v: v, b, tol=1e-13)
    assert np.linalg.norm(x - np.linalg.solve(A, b)) / np.linalg.norm(x) < 1e-10
    assert rep.iterations <= 10
    assert all(a >= b_ - 1e-15 for a, b_ in zip(rep.history, rep.history[1:]))   # monotone
    Ai = np.linalg.inv(A)
    x, rep = O.gmres(lambda v: A @ v, lambda v: Ai @ v, b, tol=1e-10)
    assert rep.iterations == 1
    # restarted GMRES still converges and the recurrence matches the true residual
    x, rep = O.gmres(lambda v: A @ v, lambda v: v, b, tol=1e-12, restart=3, maxit=200)
    assert rep.converged
    assert rep.final_rel_residual < 10 * 1e-12
    x, rep = O.gmres(lambda v: A @ v, lambda v: v, np.zeros(10))
    assert rep.iterations == 0 and not x.any()


def test_mgm_gmres_matches_dense_direct_solve():
    for problem in (0, 1):
        h = _hier(problem=problem, N=900, p=3)
        rng = np.random.default_rng(5)
        f = rng.uniform(-1, 1, 900)
        if problem:
            f -= f.mean()
        x, rep = h.solve(f, tol=1e-12)
        assert rep.converged and rep.iterations < 40
        A = h.levels[0].L.dense()
        if problem:
            n = 900
            M = np.zeros((n + 1, n + 1)); M[:n, :n] = A; M[:n, n] = 1.0; M[n, :n] = 1.0
            ref = np.linalg.solve(M, np.concatenate([f[h.perm], [0.0]]))[:n]
            xr = np.empty(n); xr[h.perm] = ref
            assert abs(x.sum()) < 1e-8 * n                    # mean-zero constraint
        else:
            xr = np.empty(900); xr[h.perm] = np.linalg.solve(A, f[h.perm])
        assert np.linalg.norm(x - xr) / np.linalg.norm(xr) < 1e-9


def test_standalone_and_gmres_agree_cfg1():
    w = MI.make_workload(1)
    h = O.Oracle(w.points, w.normals, w.stencil, w.levels)
    assert [lv.N for lv in h.levels] == [4096, 1024, 256, 64]
    x1, r1 = h.solve(w.rhs, tol=1e-10, krylov=1)
    x0, r0 = h.solve(w.rhs, tol=1e-10, krylov=0)
    assert r1.converged and r0.converged
    assert r1.final_rel_residual <= 1e-10 and r0.final_rel_residual <= 1e-10
    assert r1.iterations < r0.iterations
    assert all(b < a for a, b in zip(r0.history, r0.history[1:]))
    assert np.linalg.norm(x1 - x0) / np.linalg.norm(x1) < 1e-8


def test_closed_form_solution_converges_under_refinement():
    """-Delta_S u + u = f with u = Y_4^2, f = 21 u (BASELINE cfg1 recipe, O17)."""
    errs = []
    for N in (1024, 4096, 16384):
        w = MI.make_workload(1, n=N)
        h = O.Oracle(w.points, w.normals, w.stencil, w.levels)
        x, rep = h.solve(w.rhs, tol=1e-10)
        assert rep.converged
        errs.append(np.abs(x - w.exact).max() / np.abs(w.exact).max())
    assert errs[0] > errs[1] > errs[2]
    assert errs[0] / errs[2] > 3.0


def test_gfd_alpha_reading():
    """DESIGN.md reading O5: the exponent written at P:187 with the full projected-stencil
    radii gives spurious left-half-plane eigenvalues of L = I - D at the paper's alpha = 4;
    the calibrated reading (gfd_alpha = 4 x the paper's alpha = 16) gives none."""
    x, nrm = MI.fibonacci_sphere(1200, jitter=0.1, seed=11)
    st = O.knn(x, x, 20)
    neg = []
    for a in (4.0, 16.0):
        W = O.gfd_weights(x, nrm, st, 2, a)
        ev = np.linalg.eigvals(O.assemble_operator(st, W, 1200, 0, 1.0).dense())
        neg.append(int((ev.real < 0).sum()))
    assert neg[0] > 0 and neg[1] == 0


@pytest.mark.parametrize("ell,alpha_paper,paper_gmres,paper_bicgstab", [
    (3, 4.0, 10, 10),
    (5, 4.0, 14, 14),
    (7, 5.0, 20, 21),
])
def test_paper_table3_gfd_iteration_counts(ell, alpha_paper, paper_gmres, paper_bicgstab):
    """GFD calibration against Table 3 (sphere, N = 10242): the paper's settings
    (as in the Table 2 test) with alpha from Table 1 (4 or 5) and the O5 reading
    gfd_alpha = 4 alpha reproduce the MGM GMRES / BiCGSTAB counts within one iteration."""
    x, nrm = MI.icosahedral_sphere(5)
    n = (ell + 1) * (ell + 2)
    st = dict(method=1, poly_degree=ell, phs_k=0, stencil_n=n, problem=0, mu=1.0,
              gfd_alpha=4.0 * alpha_paper)
    lv = dict(num_levels=0, n_min=250, interp_m=3, nu1=1, nu2=1, smoother=0, gs_order="rcm")
    h = O.Oracle(x, nrm, st, lv)
    f = np.random.default_rng(0).uniform(-1, 1, len(x))
    _, rg = h.solve(f, tol=1e-12, krylov=1)
    _, rb = h.solve(f, tol=1e-12, krylov=2)
    assert rg.converged and rb.converged
    assert abs(rg.iterations - paper_gmres) <= 1, rg.iterations
    assert abs(rb.iterations - paper_bicgstab) <= 1, rb.iterations


def test_gfd_hierarchy_solves():
    h = _hier(method=1, N=1500, p=3)
    rng = np.random.default_rng(8)
    f = rng.uniform(-1, 1, 1500)
    x, rep = h.solve(f, tol=1e-10)
    assert rep.converged
    assert rep.final_rel_residual <= 1e-10


# ------------------------------------------------------------------ BiCGSTAB
def test_bicgstab_dense_cases():
    """A = I converges at the first half step; a diagonally dominant SPD 20x20 system with
    M = I matches the dense solve; an exact preconditioner converges in one
    application; iterations count preconditioner applications."""
    rng = np.random.default_rng(3)
    b = rng.normal(size=20)
    x, rep = O.bicgstab(lambda v: v, lambda v: v, b, tol=1e-12)
    assert rep.converged and rep.iterations == 1 and np.allclose(x, b, atol=1e-14)
    B = rng.normal(size=(20, 20))
    A = B @ B.T / 20 + 4 * np.eye(20)
    x, rep = O.bicgstab(lambda v: A @ v, lambda v: v, b, tol=1e-13)
    assert rep.converged
    assert np.linalg.norm(x - np.linalg.solve(A, b)) / np.linalg.norm(x) < 1e-10
    assert len(rep.history) == rep.iterations              # one residual per application
    Ai = np.linalg.inv(A)
    x, rep = O.bicgstab(lambda v: A @ v, lambda v: Ai @ v, b, tol=1e-10)
    assert rep.converged and rep.iterations == 1
    x, rep = O.bicgstab(lambda v: A @ v, lambda v: v, np.zeros(20))
    assert rep.iterations == 0 and not x.any()
    # non-symmetric, non-normal: still the dense solution
    C = rng.normal(size=(20, 20)) + 8 * np.eye(20)
    x, rep = O.bicgstab(lambda v: C @ v, lambda v: v, b, tol=1e-13, maxit=400)
    assert rep.converged and np.linalg.norm(x - np.linalg.solve(C, b)) / np.linalg.norm(x) < 1e-10


def test_mgm_bicgstab_matches_dense_direct_solve_and_gmres():
    """MGM-BiCGSTAB (shifted and bordered Poisson) reaches the dense direct solution, and
    needs about as many preconditioner applications as MGM-GMRES."""
    for problem in (0, 1):
        h = _hier(problem=problem, N=900, p=3)
        rng = np.random.default_rng(5)
        f = rng.uniform(-1, 1, 900)
        if problem:
            f -= f.mean()
        x, rep = h.solve(f, tol=1e-12, krylov=2)
        xg, repg = h.solve(f, tol=1e-12, krylov=1)
        assert rep.converged and rep.final_rel_residual <= 1e-11
        assert rep.iterations <= 2 * repg.iterations + 2
        A = h.levels[0].L.dense()
        if problem:
            n = 900
            M = np.zeros((n + 1, n + 1)); M[:n, :n] = A; M[:n, n] = 1.0; M[n, :n] = 1.0
            ref = np.linalg.solve(M, np.concatenate([f[h.perm], [0.0]]))[:n]
            xr = np.empty(n); xr[h.perm] = ref
        else:
            xr = np.empty(900); xr[h.perm] = np.linalg.solve(A, f[h.perm])
        assert np.linalg.norm(x - xr) / np.linalg.norm(xr) < 1e-9


# ------------------------------------------------------------------ paper calibration (Table 2)
@pytest.mark.parametrize("level,ell,paper_gmres,paper_bicgstab", [
    (5, 3, 18, 19),     # N = 10242
    (5, 5, 18, 18),
    (6, 3, 19, 19),     # N = 40962
])
def test_paper_table2_iteration_counts(level, ell, paper_gmres, paper_bicgstab):
    """The oracle with the paper's OWN settings (Table 1):
    icosahedral sphere nodes, RBF-FD with k = l and n = (l+1)(l+2),
    m = 3, N_min = 250, one forward Gauss-Seidel sweep pre and post in RCM
    order, shifted Poisson (mu = 1, O6), tolerance 1e-12 --
    reproduces the MGM columns of Table 2, GMRES iterations and BiCGSTAB
    preconditioner applications, within one iteration (the right-hand side is not stated;
    a seeded uniform one is used)."""
    x, nrm = MI.icosahedral_sphere(level)
    n = (ell + 1) * (ell + 2)
    st = dict(method=0, poly_degree=ell, phs_k=ell, stencil_n=n, problem=0, mu=1.0)
    lv = dict(num_levels=0, n_min=250, interp_m=3, nu1=1, nu2=1, smoother=0, gs_order="rcm")
    h = O.Oracle(x, nrm, st, lv)
    f = np.random.default_rng(0).uniform(-1, 1, len(x))
    _, rg = h.solve(f, tol=1e-12, krylov=1)
    _, rb = h.solve(f, tol=1e-12, krylov=2)
    assert rg.converged and rb.converged
    assert abs(rg.iterations - paper_gmres) <= 1, rg.iterations
    assert abs(rb.iterations - paper_bicgstab) <= 1, rb.iterations


def test_icosahedral_nodes():
    """N = 10 * 4^level + 2 distinct unit vectors."""
    for level in (0, 1, 3):
        x, nrm = MI.icosahedral_sphere(level)
        assert len(x) == 10 * 4 ** level + 2
        assert np.allclose(np.linalg.norm(x, axis=1), 1.0, atol=1e-15)
        assert len(np.unique(np.round(x, 12), axis=0)) == len(x)
