/*
 * oracle/_core.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded C primitives of the MGM method (arXiv 2204.06154), used by
 * oracle/__init__.py to build the reference hierarchy and run the reference V-cycle/GMRES.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this file's shared object.  It shares no code with the CUDA library
 * (paper_2204_06154_b200/csrc); both implement the same written-down rules of DESIGN.md.
 *
 * Compiled with -O2 -ffp-contract=off (no FMA contraction), fp64 throughout.
 * Citations: P:n = /root/reference/PAPER.md line n; O-numbers = SURVEY.md 8(c) readings.
 * Every routine returns 0 on success, a negative code on bad arguments, or a positive
 * code with *fail set to the offending index.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* ------------------------------------------------------------------------------------
 * O1  Morton (Z-order) ordering -- replaces RCM per BASELINE north star.
 * lo = per-axis min; ext = max over axes of (max - min); q_a = min(floor(((x_a-lo_a)/ext)*2^21), 2^21-1);
 * key interleaves bits x:3b+2, y:3b+1, z:3b.  Sorted by (key, original index).
 * perm[new] = old.
 * ---------------------------------------------------------------------------------- */
typedef struct { uint64_t key; i64 idx; } keyidx;
static int cmp_keyidx(const void* a, const void* b) {
    const keyidx* x = (const keyidx*)a; const keyidx* y = (const keyidx*)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    return (x->idx < y->idx) ? -1 : (x->idx > y->idx);
}
int orc_morton_perm(const double* pts, i64 n, i64* perm) {
    if (n <= 0) return -1;
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) { lo[a] = pts[a]; hi[a] = pts[a]; }
    for (i64 i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            double v = pts[3 * i + a];
            if (v < lo[a]) lo[a] = v;
            if (v > hi[a]) hi[a] = v;
        }
    double ext = 0.0;
    for (int a = 0; a < 3; ++a) if (hi[a] - lo[a] > ext) ext = hi[a] - lo[a];
    if (!(ext > 0.0)) return -2;
    keyidx* ki = (keyidx*)malloc(sizeof(keyidx) * (size_t)n);
    for (i64 i = 0; i < n; ++i) {
        uint64_t q[3];
        for (int a = 0; a < 3; ++a) {
            double t = (pts[3 * i + a] - lo[a]) / ext;
            double s = floor(t * 2097152.0);
            i64 qi = (i64)s;
            if (qi > 2097151) qi = 2097151;
            if (qi < 0) qi = 0;
            q[a] = (uint64_t)qi;
        }
        uint64_t key = 0;
        for (int b = 0; b < 21; ++b) {
            key |= ((q[0] >> b) & 1ull) << (3 * b + 2);
            key |= ((q[1] >> b) & 1ull) << (3 * b + 1);
            key |= ((q[2] >> b) & 1ull) << (3 * b);
        }
        ki[i].key = key; ki[i].idx = i;
    }
    qsort(ki, (size_t)n, sizeof(keyidx), cmp_keyidx);
    for (i64 i = 0; i < n; ++i) perm[i] = ki[i].idx;
    free(ki);
    return 0;
}

/* ------------------------------------------------------------------------------------
 * O2  Squared distance rule used by every neighbour decision:
 *     d2 = (dx*dx + dy*dy) + dz*dz, dx = y - x, no FMA.  Order = (d2, index).
 * ---------------------------------------------------------------------------------- */
static inline double dist2(const double* x, const double* y) {
    double dx = y[0] - x[0], dy = y[1] - x[1], dz = y[2] - x[2];
    double s = dx * dx + dy * dy;
    return s + dz * dz;
}

/* insert (d, j) into sorted lists of length k (ascending by (d, j)) */
static void knn_insert(double* bd, i64* bj, int k, double d, i64 j) {
    if (d > bd[k - 1] || (d == bd[k - 1] && j > bj[k - 1])) return;
    int p = k - 1;
    while (p > 0 && (bd[p - 1] > d || (bd[p - 1] == d && bj[p - 1] > j))) {
        bd[p] = bd[p - 1]; bj[p] = bj[p - 1]; --p;
    }
    bd[p] = d; bj[p] = j;
}

/* Brute-force kNN of each query among candidates `pts` (O(n*nq)). */
int orc_knn_brute(const double* pts, i64 n, const double* qry, i64 nq, int k, i64* out) {
    if (k <= 0 || k > n) return -1;
    double* bd = (double*)malloc(sizeof(double) * k);
    i64* bj = (i64*)malloc(sizeof(i64) * k);
    for (i64 q = 0; q < nq; ++q) {
        for (int t = 0; t < k; ++t) { bd[t] = INFINITY; bj[t] = INT64_MAX; }
        for (i64 j = 0; j < n; ++j) knn_insert(bd, bj, k, dist2(qry + 3 * q, pts + 3 * j), j);
        for (int t = 0; t < k; ++t) out[q * k + t] = bj[t];
    }
    free(bd); free(bj);
    return 0;
}

/* Exact re-rank of candidate lists (ncand >= k+1 per query, e.g. from a k-d tree).
 * A query is flagged (need_brute[q] = 1) unless its exact k-th distance is strictly
 * below every non-selected candidate AND below `bound2[q]` (a lower bound, supplied by
 * the caller, on the squared distance of any point not in the candidate list). */
int orc_knn_rerank(const double* pts, i64 n, const double* qry, i64 nq, int k,
                   const i64* cand, int ncand, const double* bound2, i64* out, uint8_t* need_brute) {
    if (k <= 0 || ncand < k) return -1;
    double* bd = (double*)malloc(sizeof(double) * k);
    i64* bj = (i64*)malloc(sizeof(i64) * k);
    for (i64 q = 0; q < nq; ++q) {
        for (int t = 0; t < k; ++t) { bd[t] = INFINITY; bj[t] = INT64_MAX; }
        for (int c = 0; c < ncand; ++c) {
            i64 j = cand[q * ncand + c];
            if (j < 0 || j >= n) continue;
            knn_insert(bd, bj, k, dist2(qry + 3 * q, pts + 3 * j), j);
        }
        need_brute[q] = (bj[k - 1] == INT64_MAX || !(bd[k - 1] < bound2[q])) ? 1 : 0;
        for (int t = 0; t < k; ++t) out[q * k + t] = bj[t];
    }
    free(bd); free(bj);
    return 0;
}

/* ------------------------------------------------------------------------------------
 * O3  Tangent-plane projection (eq. tp_pts):  xhat_j = R^T (x_j - x_1),
 * R = [t1 t2].  t1 = normalised (e_a - n_a n) with a = argmin_a |n_a| (lowest a on ties),
 * t2 = n x t1.
 * ---------------------------------------------------------------------------------- */
static void tangent_basis(const double* n, double* t1, double* t2) {
    int a = 0;
    if (fabs(n[1]) < fabs(n[a])) a = 1;
    if (fabs(n[2]) < fabs(n[a])) a = 2;
    for (int b = 0; b < 3; ++b) t1[b] = (b == a ? 1.0 : 0.0) - n[a] * n[b];
    double s = t1[0] * t1[0] + t1[1] * t1[1];
    s = s + t1[2] * t1[2];
    double nn = sqrt(s);
    for (int b = 0; b < 3; ++b) t1[b] = t1[b] / nn;
    t2[0] = n[1] * t1[2] - n[2] * t1[1];
    t2[1] = n[2] * t1[0] - n[0] * t1[2];
    t2[2] = n[0] * t1[1] - n[1] * t1[0];
}
static void project(const double* xc, const double* t1, const double* t2, const double* xj,
                    double* out) {
    double d0 = xj[0] - xc[0], d1 = xj[1] - xc[1], d2 = xj[2] - xc[2];
    double a = t1[0] * d0 + t1[1] * d1; a = a + t1[2] * d2;
    double b = t2[0] * d0 + t2[1] * d1; b = b + t2[2] * d2;
    out[0] = a; out[1] = b;
}
int orc_tangent_project(const double* pts, const double* nrm, const i64* sten, i64 n, int ns,
                        double* out /* n*ns*2 */) {
    for (i64 i = 0; i < n; ++i) {
        double t1[3], t2[3];
        tangent_basis(nrm + 3 * i, t1, t2);
        for (int j = 0; j < ns; ++j)
            project(pts + 3 * i, t1, t2, pts + 3 * sten[i * ns + j], out + 2 * (i * ns + j));
    }
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Dense LU with partial pivoting (ties -> lowest row), RHS eliminated alongside,
 * back substitution x_i = (b_i - sum_{j=m-1 down to i+1} M_ij x_j) / M_ii (the sum taken
 * in descending j).  M is m x m row-major, overwritten.
 * Returns the failing pivot column + 1 if |pivot| <= tol * max|M|, else 0.
 * ---------------------------------------------------------------------------------- */
static int lu_solve_inplace(double* M, double* b, int m, double tol) {
    double amax = 0.0;
    for (int i = 0; i < m * m; ++i) if (fabs(M[i]) > amax) amax = fabs(M[i]);
    for (int k = 0; k < m; ++k) {
        int p = k;
        double pv = fabs(M[k * m + k]);
        for (int i = k + 1; i < m; ++i)
            if (fabs(M[i * m + k]) > pv) { pv = fabs(M[i * m + k]); p = i; }
        if (!(pv > tol * amax)) return k + 1;
        if (p != k) {
            for (int j = 0; j < m; ++j) { double t = M[k * m + j]; M[k * m + j] = M[p * m + j]; M[p * m + j] = t; }
            double t = b[k]; b[k] = b[p]; b[p] = t;
        }
        double piv = M[k * m + k];
        for (int i = k + 1; i < m; ++i) {
            double l = M[i * m + k] / piv;
            M[i * m + k] = l;
            for (int j = k + 1; j < m; ++j) M[i * m + j] = M[i * m + j] - l * M[k * m + j];
            b[i] = b[i] - l * b[k];
        }
    }
    for (int i = m - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = m - 1; j > i; --j) s = s - M[i * m + j] * b[j];
        b[i] = s / M[i * m + i];
    }
    return 0;
}

/* graded monomials x^i y^(d-i), d = 0..ell, i = d..0 ("standard bivariate monomials") */
static int n_monomials(int ell) { return (ell + 1) * (ell + 2) / 2; }
static void monomials(double x, double y, int ell, double* out) {
    double xp[16], yp[16];
    xp[0] = 1.0; yp[0] = 1.0;
    for (int t = 1; t <= ell; ++t) { xp[t] = xp[t - 1] * x; yp[t] = yp[t - 1] * y; }
    int c = 0;
    for (int d = 0; d <= ell; ++d)
        for (int i = d; i >= 0; --i) out[c++] = xp[i] * yp[d - i];
}
/* Laplacian of each monomial at the origin: 2 for x^2 and y^2, else 0 */
static void monomial_lap0(int ell, double* out) {
    int c = 0;
    for (int d = 0; d <= ell; ++d)
        for (int i = d; i >= 0; --i) out[c++] = (d == 2 && (i == 2 || i == 0)) ? 2.0 : 0.0;
}

/* ------------------------------------------------------------------------------------
 * O4  PHS RBF-FD weights (eqs. phs_interp, rbf_fd_interp_system, rbf_fd_lap).
 * Per centre i: project (O3); rho = max_j |xhat_j|; z = xhat / rho (scale covariance of
 * PHS + polynomials, reading of DESIGN.md); saddle [A P; P^T 0][c; lam] = [Lap s; Lap p]
 * with A_ab = |z_a - z_b|^(2k+1), (Lap s)_a = (2k+1)^2 |z_a|^(2k-1), (Lap p) from
 * monomial_lap0; LU with partial pivoting; weights = c / (rho*rho).
 * ---------------------------------------------------------------------------------- */
static double phs(double r2, int k) {      /* r^(2k+1) = r * (r2)^k */
    double r = sqrt(r2), v = r;
    for (int t = 0; t < k; ++t) v = v * r2;
    return v;
}
static double phs_lap(double r2, int k) {  /* (2k+1)^2 r^(2k-1), k >= 1 */
    double r = sqrt(r2), v = r;
    for (int t = 0; t < k - 1; ++t) v = v * r2;
    return (double)((2 * k + 1) * (2 * k + 1)) * v;
}
int orc_rbffd_weights(const double* pts, const double* nrm, const i64* sten, i64 n, int ns,
                      int ell, int kphs, double* w, i64* fail) {
    if (kphs < 1 || ell < 0 || ell > 8) return -1;
    int L = n_monomials(ell), m = ns + L;
    double* M = (double*)malloc(sizeof(double) * m * m);
    double* b = (double*)malloc(sizeof(double) * m);
    double* z = (double*)malloc(sizeof(double) * 2 * ns);
    double* pm = (double*)malloc(sizeof(double) * L);
    double lap0[64];
    monomial_lap0(ell, lap0);
    for (i64 i = 0; i < n; ++i) {
        double t1[3], t2[3];
        tangent_basis(nrm + 3 * i, t1, t2);
        double rho = 0.0;
        for (int j = 0; j < ns; ++j) {
            project(pts + 3 * i, t1, t2, pts + 3 * sten[i * ns + j], z + 2 * j);
            double r = sqrt(z[2 * j] * z[2 * j] + z[2 * j + 1] * z[2 * j + 1]);
            if (r > rho) rho = r;
        }
        for (int j = 0; j < 2 * ns; ++j) z[j] = z[j] / rho;
        memset(M, 0, sizeof(double) * m * m);
        for (int a = 0; a < ns; ++a) {
            for (int c = 0; c < ns; ++c) {
                double dx = z[2 * a] - z[2 * c], dy = z[2 * a + 1] - z[2 * c + 1];
                M[a * m + c] = phs(dx * dx + dy * dy, kphs);
            }
            monomials(z[2 * a], z[2 * a + 1], ell, pm);
            for (int c = 0; c < L; ++c) { M[a * m + ns + c] = pm[c]; M[(ns + c) * m + a] = pm[c]; }
            b[a] = phs_lap(z[2 * a] * z[2 * a] + z[2 * a + 1] * z[2 * a + 1], kphs);
        }
        for (int c = 0; c < L; ++c) b[ns + c] = lap0[c];
        if (lu_solve_inplace(M, b, m, 1e-14)) { *fail = i; free(M); free(b); free(z); free(pm); return 2; }
        double rr = rho * rho;
        for (int j = 0; j < ns; ++j) w[i * ns + j] = b[j] / rr;
    }
    free(M); free(b); free(z); free(pm);
    return 0;
}

/* ------------------------------------------------------------------------------------
 * O5  GFD weights (eqs. wls_fd_approx_system, wls_fd_lap; QR remark P:198).
 * rho_i = own projected-stencil radius of point i (pre-pass over all points);
 * W_j = exp(-alpha |xhat_j|^2 / (rho_i^2 + rho_{sigma_j}^2));  c = W^{1/2} Q R^{-T} Lap p
 * with W^{1/2} P(z) = QR (Householder), z = xhat / rho_i, final c / rho_i^2.
 * ---------------------------------------------------------------------------------- */
int orc_stencil_radius(const double* pts, const double* nrm, const i64* sten, i64 n, int ns,
                       double* rho_out) {
    for (i64 i = 0; i < n; ++i) {
        double t1[3], t2[3], xh[2];
        tangent_basis(nrm + 3 * i, t1, t2);
        double rho = 0.0;
        for (int j = 0; j < ns; ++j) {
            project(pts + 3 * i, t1, t2, pts + 3 * sten[i * ns + j], xh);
            double r = sqrt(xh[0] * xh[0] + xh[1] * xh[1]);
            if (r > rho) rho = r;
        }
        rho_out[i] = rho;
    }
    return 0;
}
int orc_gfd_weights(const double* pts, const double* nrm, const i64* sten, i64 n, int ns,
                    int ell, double alpha, const double* rho_all, double* w, i64* fail) {
    int L = n_monomials(ell);
    if (ns < L || ell > 8) return -1;
    double* B = (double*)malloc(sizeof(double) * ns * L);  /* row-major ns x L */
    double* V = (double*)malloc(sizeof(double) * ns * L);  /* Householder vectors, column k */
    double* tau = (double*)malloc(sizeof(double) * L);
    double* xh = (double*)malloc(sizeof(double) * 2 * ns);
    double* sw = (double*)malloc(sizeof(double) * ns);
    double* q = (double*)malloc(sizeof(double) * ns);
    double pm[64], lap0[64], y[64];
    monomial_lap0(ell, lap0);
    for (i64 i = 0; i < n; ++i) {
        double t1[3], t2[3];
        tangent_basis(nrm + 3 * i, t1, t2);
        double rho = rho_all[i];
        double rr = rho * rho;
        for (int j = 0; j < ns; ++j) {
            i64 g = sten[i * ns + j];
            project(pts + 3 * i, t1, t2, pts + 3 * g, xh + 2 * j);
            double d2 = xh[2 * j] * xh[2 * j] + xh[2 * j + 1] * xh[2 * j + 1];
            double rg = rho_all[g];
            sw[j] = sqrt(exp(-alpha * d2 / (rr + rg * rg)));
            monomials(xh[2 * j] / rho, xh[2 * j + 1] / rho, ell, pm);
            for (int c = 0; c < L; ++c) B[j * L + c] = sw[j] * pm[c];
        }
        /* Householder QR: B = Q R, R upper L x L stored in B's top rows */
        double rmax = 0.0;
        for (int k = 0; k < L; ++k) {
            double s = 0.0;
            for (int r = k; r < ns; ++r) s = s + B[r * L + k] * B[r * L + k];
            double nx = sqrt(s);
            double x0 = B[k * L + k];
            double alph = (x0 >= 0.0) ? -nx : nx;
            for (int r = 0; r < ns; ++r) V[r * L + k] = 0.0;
            if (nx == 0.0) { tau[k] = 0.0; continue; }
            V[k * L + k] = x0 - alph;
            for (int r = k + 1; r < ns; ++r) V[r * L + k] = B[r * L + k];
            double vv = 0.0;
            for (int r = k; r < ns; ++r) vv = vv + V[r * L + k] * V[r * L + k];
            tau[k] = 2.0 / vv;
            for (int c = k; c < L; ++c) {          /* B := (I - tau v v^T) B */
                double d = 0.0;
                for (int r = k; r < ns; ++r) d = d + V[r * L + k] * B[r * L + c];
                d = tau[k] * d;
                for (int r = k; r < ns; ++r) B[r * L + c] = B[r * L + c] - d * V[r * L + k];
            }
            if (fabs(B[k * L + k]) > rmax) rmax = fabs(B[k * L + k]);
        }
        for (int k = 0; k < L; ++k)
            if (!(fabs(B[k * L + k]) > 1e-12 * rmax)) {
                *fail = i; free(B); free(V); free(tau); free(xh); free(sw); free(q); return 2;
            }
        /* y = R^{-T} lap0 (forward substitution with R^T) */
        for (int k = 0; k < L; ++k) {
            double s = lap0[k];
            for (int c = 0; c < k; ++c) s = s - B[c * L + k] * y[c];
            y[k] = s / B[k * L + k];
        }
        /* q = Q [y; 0] = H_0 H_1 ... H_{L-1} [y; 0] */
        for (int r = 0; r < ns; ++r) q[r] = (r < L) ? y[r] : 0.0;
        for (int k = L - 1; k >= 0; --k) {
            double d = 0.0;
            for (int r = k; r < ns; ++r) d = d + V[r * L + k] * q[r];
            d = tau[k] * d;
            for (int r = k; r < ns; ++r) q[r] = q[r] - d * V[r * L + k];
        }
        for (int j = 0; j < ns; ++j) w[i * ns + j] = (sw[j] * q[j]) / rr;
    }
    free(B); free(V); free(tau); free(xh); free(sw); free(q);
    return 0;
}

/* ------------------------------------------------------------------------------------
 * O9  PHS interpolation weights (eq. rbf_fd_interp): per fine point x
 * with coarse stencil y_1..y_m (O2 order): if |x - y_1| = 0 the row is e_1 (one entry);
 * else [A 1; 1^T 0][d; lam] = [s; 1], A_ab = |y_a - y_b|, s_a = |x - y_a|.
 * Output: w (nf x m), cnt[i] = number of pattern entries of row i (1 or m).
 * ---------------------------------------------------------------------------------- */
int orc_interp_weights(const double* fine, i64 nf, const double* coarse, const i64* sten, int m,
                       double* w, int32_t* cnt, i64* fail) {
    int mm = m + 1;
    double M[64 * 64], b[64];
    if (mm > 64) return -1;
    for (i64 i = 0; i < nf; ++i) {
        const double* x = fine + 3 * i;
        if (dist2(x, coarse + 3 * sten[i * m]) == 0.0) {
            for (int a = 0; a < m; ++a) w[i * m + a] = (a == 0) ? 1.0 : 0.0;
            cnt[i] = 1;
            continue;
        }
        for (int a = 0; a < m; ++a) {
            const double* ya = coarse + 3 * sten[i * m + a];
            for (int c = 0; c < m; ++c) M[a * mm + c] = sqrt(dist2(ya, coarse + 3 * sten[i * m + c]));
            M[a * mm + m] = 1.0;
            M[m * mm + a] = 1.0;
            b[a] = sqrt(dist2(x, ya));
        }
        M[m * mm + m] = 0.0;
        b[m] = 1.0;
        if (lu_solve_inplace(M, b, mm, 1e-14)) { *fail = i; return 3; }
        for (int a = 0; a < m; ++a) w[i * m + a] = b[a];
        cnt[i] = m;
    }
    return 0;
}

/* ------------------------------------------------------------------------------------
 * O8  Weighted sample elimination (Yuksel 2015 via P:260), reading of DESIGN.md:
 *   r_h = 0.5 * sorted(nn distance)[floor((N-1)/2)];  r_max = r_h*sqrt(N/Nt);  R = 2 r_max;
 *   pairs with d < R get W_ab = floor((1 - d/R)^8 * 2^40 + 0.5) (int64, exact sums);
 *   remove the live point of maximal weight (ties -> lowest index) N - Nt times,
 *   subtracting W_ab from its live neighbours.  Survivors returned in index order.
 * nn2[i] = squared distance to the nearest other point (from kNN, k=2).
 * ---------------------------------------------------------------------------------- */
static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x < y) ? -1 : (x > y);
}
typedef int64_t wse_w;  /* O8: fixed-point weights, 2^40 per unit */
typedef struct { wse_w w; i64 idx; } heapent;
/* max-heap on (w desc, idx asc) */
static int he_less(heapent a, heapent b) {  /* a has lower priority than b */
    if (a.w != b.w) return a.w < b.w;
    return a.idx > b.idx;
}
static void heap_push(heapent* h, i64* sz, heapent e) {
    i64 p = (*sz)++;
    h[p] = e;
    while (p > 0) {
        i64 q = (p - 1) / 2;
        if (he_less(h[q], h[p])) { heapent t = h[q]; h[q] = h[p]; h[p] = t; p = q; } else break;
    }
}
static heapent heap_pop(heapent* h, i64* sz) {
    heapent top = h[0];
    h[0] = h[--(*sz)];
    i64 p = 0;
    for (;;) {
        i64 l = 2 * p + 1, r = l + 1, best = p;
        if (l < *sz && he_less(h[best], h[l])) best = l;
        if (r < *sz && he_less(h[best], h[r])) best = r;
        if (best == p) break;
        heapent t = h[p]; h[p] = h[best]; h[best] = t; p = best;
    }
    return top;
}
/* One elimination pass with weight radius R.  Returns 0 (keep filled), 1 if the pass had to
 * eliminate a point of zero weight (no live neighbour within R: the weight no longer ranks
 * the points and index ties would decide, wiping out the lowest-index region), -3 on error. */
static int wse_pass(const double* pts, i64 n, i64 nt, double R, i64* keep) {
    /* uniform grid with cell size >= R: all pairs with d < R lie in adjacent cells */
    double lo[3] = {pts[0], pts[1], pts[2]}, hi[3] = {pts[0], pts[1], pts[2]};
    for (i64 i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            if (pts[3 * i + a] < lo[a]) lo[a] = pts[3 * i + a];
            if (pts[3 * i + a] > hi[a]) hi[a] = pts[3 * i + a];
        }
    double vol = 1.0;
    for (int a = 0; a < 3; ++a) vol *= (hi[a] - lo[a] > R ? hi[a] - lo[a] : R);
    double side = cbrt(vol / (double)n);
    if (side < R) side = R;
    i64 dims[3];
    double csz[3];
    for (int a = 0; a < 3; ++a) {
        dims[a] = (i64)floor((hi[a] - lo[a]) / side);
        if (dims[a] < 1) dims[a] = 1;
        csz[a] = (hi[a] - lo[a]) / (double)dims[a];   /* >= side >= R */
    }
    i64 ncell = dims[0] * dims[1] * dims[2];
    i64* cell = (i64*)malloc(sizeof(i64) * n);
    i64* cstart = (i64*)calloc((size_t)ncell + 1, sizeof(i64));
    i64* clist = (i64*)malloc(sizeof(i64) * n);
    for (i64 i = 0; i < n; ++i) {
        i64 c[3];
        for (int a = 0; a < 3; ++a) {
            c[a] = (csz[a] > 0.0) ? (i64)floor((pts[3 * i + a] - lo[a]) / csz[a]) : 0;
            if (c[a] >= dims[a]) c[a] = dims[a] - 1;
            if (c[a] < 0) c[a] = 0;
        }
        cell[i] = (c[2] * dims[1] + c[1]) * dims[0] + c[0];
        cstart[cell[i] + 1]++;
    }
    for (i64 c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
    i64* fillp = (i64*)malloc(sizeof(i64) * ncell);
    memcpy(fillp, cstart, sizeof(i64) * ncell);
    for (i64 i = 0; i < n; ++i) clist[fillp[cell[i]]++] = i;
    free(fillp);
    /* neighbour lists (CSR), W_ab */
    i64 cap = 32 * n, nnz = 0;
    i64* nptr = (i64*)malloc(sizeof(i64) * (n + 1));
    i64* nidx = (i64*)malloc(sizeof(i64) * cap);
    wse_w* nw = (wse_w*)malloc(sizeof(wse_w) * cap);
    wse_w* weight = (wse_w*)calloc((size_t)n, sizeof(wse_w));
    for (i64 i = 0; i < n; ++i) {
        nptr[i] = nnz;
        i64 cx = cell[i] % dims[0], cy = (cell[i] / dims[0]) % dims[1], cz = cell[i] / (dims[0] * dims[1]);
        for (i64 z = cz - 1; z <= cz + 1; ++z) {
            if (z < 0 || z >= dims[2]) continue;
            for (i64 y = cy - 1; y <= cy + 1; ++y) {
                if (y < 0 || y >= dims[1]) continue;
                for (i64 x = cx - 1; x <= cx + 1; ++x) {
                    if (x < 0 || x >= dims[0]) continue;
                    i64 c = (z * dims[1] + y) * dims[0] + x;
                    for (i64 t = cstart[c]; t < cstart[c + 1]; ++t) {
                        i64 j = clist[t];
                        if (j == i) continue;
                        double d = sqrt(dist2(pts + 3 * i, pts + 3 * j));
                        if (!(d < R)) continue;
                        double u = 1.0 - d / R;
                        double u2 = u * u, u4 = u2 * u2, u8 = u4 * u4;
                        wse_w W = (wse_w)floor(u8 * 1099511627776.0 + 0.5);  /* 2^40 */
                        if (nnz == cap) {
                            cap *= 2;
                            nidx = (i64*)realloc(nidx, sizeof(i64) * cap);
                            nw = (wse_w*)realloc(nw, sizeof(wse_w) * cap);
                        }
                        nidx[nnz] = j; nw[nnz] = W; ++nnz;
                        weight[i] += W;
                    }
                }
            }
        }
    }
    nptr[n] = nnz;
    free(cell); free(cstart); free(clist);
    /* lazy max-heap elimination */
    heapent* h = (heapent*)malloc(sizeof(heapent) * (n + nnz + 1));
    i64 hs = 0;
    uint8_t* dead = (uint8_t*)calloc((size_t)n, 1);
    for (i64 i = 0; i < n; ++i) { heapent e = {weight[i], i}; heap_push(h, &hs, e); }
    i64 removed = 0;
    while (removed < n - nt) {
        heapent e = heap_pop(h, &hs);
        if (dead[e.idx] || e.w != weight[e.idx]) continue;  /* stale entry */
        if (e.w == 0) {  /* degenerate: R too small for this cloud (O8) */
            free(h); free(dead); free(nptr); free(nidx); free(nw); free(weight);
            return 1;
        }
        dead[e.idx] = 1;
        ++removed;
        for (i64 t = nptr[e.idx]; t < nptr[e.idx + 1]; ++t) {
            i64 j = nidx[t];
            if (dead[j]) continue;
            weight[j] -= nw[t];
            heapent f = {weight[j], j};
            heap_push(h, &hs, f);
        }
    }
    i64 c = 0;
    for (i64 i = 0; i < n; ++i) if (!dead[i]) keep[c++] = i;
    free(h); free(dead); free(nptr); free(nidx); free(nw); free(weight);
    return (c == nt) ? 0 : -3;
}

int orc_wse(const double* pts, i64 n, i64 nt, const double* nn2, i64* keep /* nt */) {
    if (nt <= 0 || nt > n) return -1;
    if (nt == n) { for (i64 i = 0; i < n; ++i) keep[i] = i; return 0; }
    double* s = (double*)malloc(sizeof(double) * n);
    for (i64 i = 0; i < n; ++i) s[i] = sqrt(nn2[i]);
    qsort(s, (size_t)n, sizeof(double), cmp_double);
    double rh = 0.5 * s[(n - 1) / 2];
    free(s);
    double rmax = rh * sqrt((double)n / (double)nt);
    /* O8: R = 2 r_max; if a pass degenerates (zero-weight elimination), R *= 1.25 and restart */
    double R = 2.0 * rmax;
    for (int attempt = 0; attempt < 16; ++attempt, R *= 1.25) {
        int rc = wse_pass(pts, n, nt, R, keep);
        if (rc != 1) return rc;
    }
    return -4;
}

/* ------------------------------------------------------------------------------------
 * CSR helpers (row pointers i64, columns i64 ascending within a row).
 * ---------------------------------------------------------------------------------- */

/* O10 Galerkin product L_H = R (L P) (eq. galerkin), symbolic pattern
 * kept in full (no zero dropping).  Two-call protocol: with cols==NULL it fills ptr (n_out+1)
 * only; then with allocated cols/vals it fills values.  Inner sums in the order
 * (L P)_kj = sum_{l ascending} L_kl P_lj ;  (R (LP))_ij = sum_{k ascending} R_ik (LP)_kj. */
int orc_spgemm(i64 nra, const i64* ap, const i64* ai, const double* av,
               i64 ncb, const i64* bp, const i64* bi, const double* bv,
               i64* cp, i64* ci, double* cv) {
    i64* mark = (i64*)malloc(sizeof(i64) * ncb);
    double* acc = (double*)calloc((size_t)ncb, sizeof(double));
    i64* list = (i64*)malloc(sizeof(i64) * ncb);
    for (i64 j = 0; j < ncb; ++j) mark[j] = -1;
    i64 nnz = 0;
    for (i64 i = 0; i < nra; ++i) {
        i64 cnt = 0;
        for (i64 t = ap[i]; t < ap[i + 1]; ++t) {
            i64 k = ai[t];
            for (i64 s = bp[k]; s < bp[k + 1]; ++s) {
                i64 j = bi[s];
                if (mark[j] != i) { mark[j] = i; list[cnt++] = j; acc[j] = 0.0; }
                if (cv) acc[j] = acc[j] + av[t] * bv[s];
            }
        }
        /* sort column list ascending (insertion sort: rows are short) */
        for (i64 a = 1; a < cnt; ++a) {
            i64 v = list[a], b = a - 1;
            while (b >= 0 && list[b] > v) { list[b + 1] = list[b]; --b; }
            list[b + 1] = v;
        }
        if (ci) for (i64 a = 0; a < cnt; ++a) { ci[cp[i] + a] = list[a]; cv[cp[i] + a] = acc[list[a]]; }
        else cp[i] = nnz;
        nnz += cnt;
    }
    if (!ci) cp[nra] = nnz;
    free(mark); free(acc); free(list);
    return 0;
}

/* O11 greedy colouring of pattern(A) U pattern(A^T) minus the diagonal, vertices visited in
 * index order, colour = smallest non-negative integer unused by coloured neighbours.
 * at_p/at_i = transpose pattern.  Returns number of colours in *ncol. */
/* One greedy pass (O11): visit vertices in `order`, give each the smallest colour not used by
 * a neighbour (sym(pattern) minus the diagonal) already coloured in this pass. */
static int greedy_pass(i64 n, const i64* ap, const i64* ai, const i64* tp, const i64* ti, const i64* order,
                       int32_t* colour, int32_t* used, int32_t* ncol) {
    int32_t maxc = 0;
    for (i64 i = 0; i < n; ++i) colour[i] = -1;
    for (i64 q = 0; q < n; ++q) {
        i64 i = order[q];
        for (i64 t = ap[i]; t < ap[i + 1]; ++t) {
            i64 j = ai[t];
            if (j != i && colour[j] >= 0) used[colour[j]] = (int32_t)q;
        }
        for (i64 t = tp[i]; t < tp[i + 1]; ++t) {
            i64 j = ti[t];
            if (j != i && colour[j] >= 0) used[colour[j]] = (int32_t)q;
        }
        int32_t c = 0;
        while (used[c] == (int32_t)q) ++c;
        if (c >= 4095) return -1;
        colour[i] = c;
        if (c + 1 > maxc) maxc = c + 1;
    }
    *ncol = maxc;
    return 0;
}

/* DSATUR (Brelaz 1979), O11: repeatedly colour the uncoloured vertex of largest saturation
 * (number of distinct colours among its neighbours in sym(pattern) minus the diagonal), ties
 * by larger degree (distinct neighbours), then lower index, with the smallest colour unused
 * by its neighbours.  Returns -2 if a colour index reaches 256 (caller falls back). */
typedef struct { int32_t sat, deg; i64 v; } ds_ent;
static int cmp_i64(const void* a, const void* b) {
    i64 x = *(const i64*)a, y = *(const i64*)b;
    return (x > y) - (x < y);
}
static int ds_less(ds_ent a, ds_ent b) { /* a has lower priority than b */
    if (a.sat != b.sat) return a.sat < b.sat;
    if (a.deg != b.deg) return a.deg < b.deg;
    return a.v > b.v;
}
static int dsatur(i64 n, const i64* ap, const i64* ai, const i64* tp, const i64* ti, int32_t* colour, int32_t* ncol) {
    /* distinct-neighbour lists (merge of the row and column patterns) */
    i64* np = (i64*)malloc(sizeof(i64) * (size_t)(n + 1));
    i64 cap = (ap[n] + tp[n]) > 0 ? (ap[n] + tp[n]) : 1;
    i64* nb = (i64*)malloc(sizeof(i64) * (size_t)cap);
    np[0] = 0;
    for (i64 i = 0; i < n; ++i) { /* row and column patterns, sorted, deduplicated, no diagonal */
        i64 o = np[i], q = np[i];
        for (i64 t = ap[i]; t < ap[i + 1]; ++t) if (ai[t] != i) nb[o++] = ai[t];
        for (i64 t = tp[i]; t < tp[i + 1]; ++t) if (ti[t] != i) nb[o++] = ti[t];
        qsort(nb + np[i], (size_t)(o - np[i]), sizeof(i64), cmp_i64);
        for (i64 t = np[i]; t < o; ++t) if (q == np[i] || nb[q - 1] != nb[t]) nb[q++] = nb[t];
        np[i + 1] = q;
    }
    uint64_t* bits = (uint64_t*)calloc((size_t)n * 4, sizeof(uint64_t));
    int32_t* sat = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    i64 hcap = n + np[n] + 1, hn = 0;
    ds_ent* h = (ds_ent*)malloc(sizeof(ds_ent) * (size_t)hcap);
    int rc = 0;
    int32_t maxc = 0;
#define DS_PUSH(E) do { i64 k_ = hn++; h[k_] = (E); \
        while (k_ > 0 && ds_less(h[(k_ - 1) / 2], h[k_])) { ds_ent t_ = h[k_]; h[k_] = h[(k_ - 1) / 2]; h[(k_ - 1) / 2] = t_; k_ = (k_ - 1) / 2; } } while (0)
    for (i64 i = 0; i < n; ++i) { colour[i] = -1; ds_ent e = {0, (int32_t)(np[i + 1] - np[i]), i}; DS_PUSH(e); }
    for (i64 done = 0; done < n;) {
        ds_ent top = h[0];
        h[0] = h[--hn];
        for (i64 k = 0;;) { /* sift down */
            i64 l = 2 * k + 1, r = l + 1, m = k;
            if (l < hn && ds_less(h[m], h[l])) m = l;
            if (r < hn && ds_less(h[m], h[r])) m = r;
            if (m == k) break;
            ds_ent t = h[k]; h[k] = h[m]; h[m] = t; k = m;
        }
        i64 v = top.v;
        if (colour[v] >= 0 || top.sat != sat[v]) continue; /* stale entry */
        int32_t c = 0;
        while (c < 256 && (bits[v * 4 + (c >> 6)] >> (c & 63) & 1ull)) ++c;
        if (c >= 256) { rc = -2; break; }
        colour[v] = c;
        if (c + 1 > maxc) maxc = c + 1;
        ++done;
        for (i64 t = np[v]; t < np[v + 1]; ++t) {
            i64 w = nb[t];
            if (colour[w] >= 0 || (bits[w * 4 + (c >> 6)] >> (c & 63) & 1ull)) continue;
            bits[w * 4 + (c >> 6)] |= 1ull << (c & 63);
            sat[w]++;
            ds_ent e = {sat[w], (int32_t)(np[w + 1] - np[w]), w};
            DS_PUSH(e);
        }
    }
#undef DS_PUSH
    *ncol = maxc;
    free(h); free(sat); free(bits); free(nb); free(np);
    return rc;
}

/* O11: DSATUR colouring, then `passes` iterated-greedy passes (Culberson): each visits the
 * vertices by descending colour of the previous pass, ties by index; a pass never increases
 * the number of colours.  passes < 0: plain greedy in index (Morton) order (reference). */
int orc_greedy_colour(i64 n, const i64* ap, const i64* ai, const i64* tp, const i64* ti, int passes,
                      int32_t* colour, int32_t* ncol) {
    int32_t* used = (int32_t*)malloc(sizeof(int32_t) * 4096);
    i64* order = (i64*)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    i64* cnt = (i64*)malloc(sizeof(i64) * 4097);
    int rc = 0;
    for (int c = 0; c < 4096; ++c) used[c] = -1;
    for (i64 i = 0; i < n; ++i) order[i] = i;
    /* first colouring: DSATUR, or greedy in index order if DSATUR needed >= 256 colours
       (passes < 0: plain greedy, no DSATUR and no iterated passes) */
    if (passes < 0 || dsatur(n, ap, ai, tp, ti, colour, ncol) != 0)
        rc = greedy_pass(n, ap, ai, tp, ti, order, colour, used, ncol);
    for (int r = 0; r < passes && rc == 0; ++r) {
        /* vertices by descending colour, ascending index within a colour */
        int32_t K = *ncol;
        for (int32_t c = 0; c <= K; ++c) cnt[c] = 0;
        for (i64 i = 0; i < n; ++i) cnt[K - 1 - colour[i] + 1]++;
        for (int32_t c = 0; c < K; ++c) cnt[c + 1] += cnt[c];
        for (i64 i = 0; i < n; ++i) order[cnt[K - 1 - colour[i]]++] = i;
        for (int c = 0; c < 4096; ++c) used[c] = -1;
        rc = greedy_pass(n, ap, ai, tp, ti, order, colour, used, ncol);
    }
    free(cnt);
    free(order);
    free(used);
    return rc;
}

/* y = A x, row sums in stored (ascending column) order */
int orc_spmv(i64 n, const i64* ap, const i64* ai, const double* av, const double* x, double* y) {
    for (i64 i = 0; i < n; ++i) {
        double s = 0.0;
        for (i64 t = ap[i]; t < ap[i + 1]; ++t) s = s + av[t] * x[ai[t]];
        y[i] = s;
    }
    return 0;
}

/* O12 one Gauss-Seidel sweep u <- u + B^{-1}(f - A u - c*lam) (eq. smoother P:288;
 * Poisson variant P:348-352) in the row order `order` (colour-major: forward = colours
 * ascending, rows ascending within a colour; backward = reverse of that list).
 * Row update: r = f_i - a_ii u_i - sum_{j != i, ascending} a_ij u_j [- c_i lam];  u_i += r / a_ii.
 * c may be NULL (no border term). */
int orc_gs_sweep(i64 n, const i64* ap, const i64* ai, const double* av, const i64* order,
                 int backward, const double* f, double* u, const double* c, double lam, i64* fail) {
    for (i64 s = 0; s < n; ++s) {
        i64 i = backward ? order[n - 1 - s] : order[s];
        double aii = 0.0;
        int has = 0;
        for (i64 t = ap[i]; t < ap[i + 1]; ++t) if (ai[t] == i) { aii = av[t]; has = 1; }
        if (!has || aii == 0.0) { *fail = i; return 4; }
        double r = f[i] - aii * u[i];
        for (i64 t = ap[i]; t < ap[i + 1]; ++t) if (ai[t] != i) r = r - av[t] * u[ai[t]];
        if (c) r = r - c[i] * lam;
        u[i] = u[i] + r / aii;
    }
    return 0;
}

/* O13 dense LU with partial pivoting (ties -> lowest row): A (m x m row-major) overwritten
 * by L\U, piv[k] = row swapped with k.  Solve uses the stored factors. */
int orc_dense_lu(double* A, int m, int32_t* piv, i64* fail) {
    double amax = 0.0;
    for (i64 i = 0; i < (i64)m * m; ++i) if (fabs(A[i]) > amax) amax = fabs(A[i]);
    for (int k = 0; k < m; ++k) {
        int p = k;
        double pv = fabs(A[(i64)k * m + k]);
        for (int i = k + 1; i < m; ++i) if (fabs(A[(i64)i * m + k]) > pv) { pv = fabs(A[(i64)i * m + k]); p = i; }
        if (!(pv > 1e-14 * amax)) { *fail = k; return 3; }
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < m; ++j) { double t = A[(i64)k * m + j]; A[(i64)k * m + j] = A[(i64)p * m + j]; A[(i64)p * m + j] = t; }
        double d = A[(i64)k * m + k];
        for (int i = k + 1; i < m; ++i) {
            double l = A[(i64)i * m + k] / d;
            A[(i64)i * m + k] = l;
            for (int j = k + 1; j < m; ++j) A[(i64)i * m + j] = A[(i64)i * m + j] - l * A[(i64)k * m + j];
        }
    }
    return 0;
}
int orc_dense_lu_solve(const double* LU, int m, const int32_t* piv, double* b) {
    for (int k = 0; k < m; ++k) if (piv[k] != k) { double t = b[k]; b[k] = b[piv[k]]; b[piv[k]] = t; }
    for (int i = 0; i < m; ++i) {
        double s = b[i];
        for (int j = 0; j < i; ++j) s = s - LU[(i64)i * m + j] * b[j];
        b[i] = s;
    }
    for (int i = m - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < m; ++j) s = s - LU[(i64)i * m + j] * b[j];
        b[i] = s / LU[(i64)i * m + i];
    }
    return 0;
}
