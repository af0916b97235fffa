"""Independent pin of the oracle's GFD weight function (O5; section 2.3
"GFD", eq. wls_fd_approx_system and eq. wls_fd_lap).

The paper defines the stencil weights as c = W P (P^T W P)^{-1} (Lap p) (eq. wls_fd_lap)
with W = diag(w(x_i)), w(x_i) = exp(-alpha |x_1 - x_i|^2 / (rho_1^2 + rho_i^2)),
rho_k the radius of the minimum ball centred at point k that encloses ITS OWN projected stencil
(P:187).  The oracle computes the same vector through a Householder QR of W^{1/2} P with
coordinates scaled by rho_1 (the "QR of WP" remark at P:198).  Every other GFD pin (polynomial
exactness, zero row sums, the n = L six-point case) holds for ANY positive weight function, so
this file evaluates eq. wls_fd_lap literally -- numpy normal equations, a different tangent
basis, a different polynomial scaling, rho computed basis-free from 3-D geometry -- and
requires agreement to 1e-10 on stencils with n > L.  Mutations of the weight function
(rho_i in place of the neighbour's own rho, W instead of W^{1/2} inside the QR, i.e. W^2 in
the normal equations) are shown to move the weights by far more than the tolerance, so the pin
discriminates them.  The alpha passed here is the alpha of the formula as written (the
cfg2-GFD workload passes 16 into it, O5).
"""
import numpy as np
import pytest

import mgm_inputs as MI
import oracle as O


def _tangent_rotated(n, angle):
    """An orthonormal tangent basis at normal n, rotated by `angle` (independent of the
    oracle's O3 choice; the weights are invariant under rotations of the tangent plane)."""
    a = np.array([1.0, 0.0, 0.0]) if abs(n[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    t1 = a - (a @ n) * n
    t1 /= np.linalg.norm(t1)
    t2 = np.cross(n, t1)
    c, s = np.cos(angle), np.sin(angle)
    return c * t1 + s * t2, -s * t1 + c * t2


def _own_radius(x, nrm, sten):
    """rho_k = max_j |tangential part of (x_j - x_k)| over k's own stencil, basis-free."""
    d = x[sten] - x[:, None, :]
    dn = np.einsum("ijk,ik->ij", d, nrm)
    tang = d - dn[..., None] * nrm[:, None, :]
    return np.sqrt((tang ** 2).sum(-1)).max(1)


def _lap_monomials(ell, s):
    """Lap of the monomials q_a(x, y) = (x/s)^i (y/s)^(d-i) at the origin: 2/s^2 for x^2, y^2."""
    out = []
    for d in range(ell + 1):
        for i in range(d, -1, -1):
            out.append(2.0 / s ** 2 if d == 2 and i in (0, 2) else 0.0)
    return np.array(out)


def _mono(xy, ell, s):
    cols = []
    for d in range(ell + 1):
        for i in range(d, -1, -1):
            cols.append((xy[:, 0] / s) ** i * (xy[:, 1] / s) ** (d - i))
    return np.stack(cols, 1)


def literal_gfd(x, nrm, sten, ell, alpha, rho_mode="own", wpow=1.0, seed=0):
    """eq. wls_fd_lap, c = W P (P^T W P)^{-1} Lap p, evaluated by the normal equations."""
    rng = np.random.default_rng(seed)
    rho = _own_radius(x, nrm, sten)
    s = float(np.median(rho))  # a global polynomial scale (the LS projector is basis independent)
    W_out = np.empty(sten.shape)
    for i in range(len(sten)):
        t1, t2 = _tangent_rotated(nrm[i], rng.uniform(0, 2 * np.pi))
        d = x[sten[i]] - x[i]
        xy = np.stack([d @ t1, d @ t2], 1)
        r2 = (xy ** 2).sum(1)          # |x_1 - x_j|^2, the centre projects to the origin
        rj = rho[sten[i]] if rho_mode == "own" else np.full(len(sten[i]), rho[i])
        w = np.exp(-alpha * r2 / (rho[i] ** 2 + rj ** 2)) ** wpow
        P = _mono(xy, ell, s)
        G = P.T @ (w[:, None] * P)
        W_out[i] = w * (P @ np.linalg.solve(G, _lap_monomials(ell, s)))
    return W_out


CASES = [(2, 20, 4.0), (2, 20, 16.0), (3, 30, 4.0), (3, 30, 16.0)]


@pytest.mark.parametrize("ell,n,alpha", CASES)
def test_gfd_weights_equal_eq_wls_fd_lap(ell, n, alpha):
    x, nrm = MI.fibonacci_sphere(600, jitter=0.1, seed=11)
    st = O.knn(x, x, n)
    sel = np.random.default_rng(5).choice(len(x), 40, replace=False)
    got = O.gfd_weights(x, nrm, st, ell, alpha)[sel]
    want = literal_gfd(x, nrm, st, ell, alpha)[sel]
    scale = np.abs(want).max(1, keepdims=True)
    assert (np.abs(got - want) / scale).max() <= 1e-10


@pytest.mark.parametrize("ell,n,alpha", [(2, 20, 16.0), (3, 30, 16.0)])
def test_gfd_pin_discriminates_weight_mutations(ell, n, alpha):
    """The pin above would catch a wrong weight function: rho_i used twice (instead of the
    neighbour's own rho_j) or W in place of W^{1/2} in the QR (W^2 in the normal equations)."""
    x, nrm = MI.fibonacci_sphere(600, jitter=0.1, seed=11)
    st = O.knn(x, x, n)
    sel = np.random.default_rng(5).choice(len(x), 40, replace=False)
    got = O.gfd_weights(x, nrm, st, ell, alpha)[sel]
    for kw in (dict(rho_mode="centre"), dict(wpow=2.0), dict(wpow=0.5)):
        mut = literal_gfd(x, nrm, st, ell, alpha, **kw)[sel]
        scale = np.abs(mut).max(1, keepdims=True)
        assert (np.abs(got - mut) / scale).max() > 1e-6, kw


def test_gfd_hand_case_neighbour_radius_matters():
    """A planar stencil (normal e_z) whose neighbours have stencils of different radii: the
    weights with the neighbour's own rho_j differ from those with rho_1 everywhere, and
    the oracle follows the former."""
    rng = np.random.default_rng(3)
    # centre + 9 near points on a ring, plus far points that only enter the OUTER points' stencils
    inner = [(0.0, 0.0)] + [(np.cos(t), np.sin(t)) for t in np.linspace(0, 2 * np.pi, 10)[:-1]]
    inner = np.array(inner) * 0.1 + rng.uniform(-0.01, 0.01, (10, 2)) * np.r_[0, np.ones(9)][:, None]
    far = np.array([(np.cos(t), np.sin(t)) for t in np.linspace(0, 2 * np.pi, 13)[:-1]]) * 0.5
    xy = np.vstack([inner, far])
    x = np.c_[xy, np.zeros(len(xy))]
    nrm = np.tile([0.0, 0.0, 1.0], (len(x), 1))
    n = 10
    st = O.knn(x, x, n)
    rho = _own_radius(x, nrm, st)
    assert rho[st[0]].max() > 1.5 * rho[0]        # neighbours' own radii differ from the centre's
    got = O.gfd_weights(x, nrm, st, 2, 4.0)[0]
    want = literal_gfd(x, nrm, st, 2, 4.0)[0]
    mut = literal_gfd(x, nrm, st, 2, 4.0, rho_mode="centre")[0]
    assert np.abs(got - want).max() <= 1e-10 * np.abs(want).max()
    assert np.abs(got - mut).max() > 1e-3 * np.abs(want).max()
