// Device setup kernels of libmgm (compiled with -fmad=false: every multiply and add is
// rounded separately, so the operation sequences written in DESIGN.md give the same bits
// as a sequential host loop).
//   * batched tangent-plane PHS RBF-FD weights, one warp per stencil
//   * batched GFD weights, one warp per stencil, Householder QR
//   * batched PHS interpolation weights, one thread per fine point
//   * SpGEMM for the Galerkin product, one CTA per output row, sort-based
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include <climits>
#include <cstdint>
#include <string>
#include <vector>

#include "mgm_internal.h"

#include <cub/cub.cuh>

namespace mgm {

#define FULL 0xffffffffu

// ---------------------------------------------------------------------------------------
// shared device helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void tangent_basis_dev(const double* n, double* t1, double* t2) {
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

__device__ __forceinline__ void project_dev(const double* xc, const double* t1, const double* t2,
                                            const double* xj, double& u, double& v) {
    double d0 = xj[0] - xc[0], d1 = xj[1] - xc[1], d2 = xj[2] - xc[2];
    double a = t1[0] * d0 + t1[1] * d1;
    a = a + t1[2] * d2;
    double b = t2[0] * d0 + t2[1] * d1;
    b = b + t2[2] * d2;
    u = a;
    v = b;
}

__device__ __forceinline__ double dist2_dev(const double* x, const double* y) {
    double dx = y[0] - x[0], dy = y[1] - x[1], dz = y[2] - x[2];
    double s = dx * dx + dy * dy;
    return s + dz * dz;
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

// monomial x^i y^(d-i) in graded order; value by repeated multiplication (as DESIGN.md)
__device__ __forceinline__ double monomial_dev(double x, double y, int col) {
    int d = 0, c = col;
    while (c > d) { c -= d + 1; ++d; }
    int i = d - c;  // within degree d: i = d, d-1, ..., 0
    double xp = 1.0, yp = 1.0;
    for (int t = 0; t < i; ++t) xp = xp * x;
    for (int t = 0; t < d - i; ++t) yp = yp * y;
    return xp * yp;
}
__device__ __forceinline__ double monomial_lap0_dev(int col) {
    int d = 0, c = col;
    while (c > d) { c -= d + 1; ++d; }
    int i = d - c;
    return (d == 2 && (i == 2 || i == 0)) ? 2.0 : 0.0;
}

// Warp LU with partial pivoting on M (m x m, row-major in smem) and RHS b; the update
// order of every entry equals the sequential right-looking algorithm; back substitution
// column-oriented (descending j).  Returns false if |pivot| <= tol * max|M|.
__device__ bool warp_lu_solve(double* M, double* b, double* lcol, int m, double tol) {
    const int lane = threadIdx.x & 31;
    double amax = 0.0;
    for (int e = lane; e < m * m; e += 32) amax = fmax(amax, fabs(M[e]));
    amax = warp_max(amax);
    for (int k = 0; k < m; ++k) {
        // pivot: max |M[i][k]|, lowest i on ties
        double pv = -1.0;
        int pi = INT_MAX;
        for (int i = k + lane; i < m; i += 32) {
            double v = fabs(M[i * m + k]);
            if (v > pv) { pv = v; pi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(FULL, pv, o);
            int oi = __shfl_xor_sync(FULL, pi, o);
            if (ov > pv || (ov == pv && oi < pi)) { pv = ov; pi = oi; }
        }
        if (!(pv > tol * amax)) return false;
        if (pi != k) {
            for (int j = lane; j < m; j += 32) {
                double t = M[k * m + j];
                M[k * m + j] = M[pi * m + j];
                M[pi * m + j] = t;
            }
            if (lane == 0) { double t = b[k]; b[k] = b[pi]; b[pi] = t; }
        }
        __syncwarp();
        double piv = M[k * m + k];
        for (int i = k + 1 + lane; i < m; i += 32) {
            double l = M[i * m + k] / piv;
            lcol[i] = l;
            M[i * m + k] = l;
            b[i] = b[i] - l * b[k];
        }
        __syncwarp();
        for (int j = k + 1 + lane; j < m; j += 32) {
            double mk = M[k * m + j];
            for (int i = k + 1; i < m; ++i) M[i * m + j] = M[i * m + j] - lcol[i] * mk;
        }
        __syncwarp();
    }
    for (int i = m - 1; i >= 0; --i) {
        if (lane == 0) b[i] = b[i] / M[i * m + i];
        __syncwarp();
        double xi = b[i];
        for (int r = lane; r < i; r += 32) b[r] = b[r] - M[r * m + i] * xi;
        __syncwarp();
    }
    return true;
}

// ---------------------------------------------------------------------------------------
// O4: PHS RBF-FD weights, one warp per stencil
// smem per warp: M[m*m], b[m], lcol[m], z[2*ns]
// ---------------------------------------------------------------------------------------
__global__ void k_rbffd_weights(const double* __restrict__ pts, const double* __restrict__ nrm,
                                const i32* __restrict__ sten, i64 n, int ns, int ell, int kphs,
                                double* __restrict__ w, i64* fail) {
    extern __shared__ double smem[];
    const int L = (ell + 1) * (ell + 2) / 2, m = ns + L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int per_warp = m * m + 2 * m + 2 * ns;
    double* M = smem + (size_t)warp * per_warp;
    double* b = M + m * m;
    double* lcol = b + m;
    double* z = lcol + m;
    const int wpb = blockDim.x >> 5;
    for (i64 i = (i64)blockIdx.x * wpb + warp; i < n; i += (i64)gridDim.x * wpb) {
        double t1[3], t2[3];
        tangent_basis_dev(nrm + 3 * i, t1, t2);
        double rho = 0.0;
        for (int j = lane; j < ns; j += 32) {
            double u, v;
            project_dev(pts + 3 * i, t1, t2, pts + 3 * (i64)sten[i * ns + j], u, v);
            z[2 * j] = u;
            z[2 * j + 1] = v;
            rho = fmax(rho, sqrt(u * u + v * v));
        }
        rho = warp_max(rho);
        __syncwarp();
        for (int j = lane; j < 2 * ns; j += 32) z[j] = z[j] / rho;
        __syncwarp();
        for (int e = lane; e < m * m; e += 32) {
            int a = e / m, c = e % m;
            double v;
            if (a < ns && c < ns) {
                double dx = z[2 * a] - z[2 * c], dy = z[2 * a + 1] - z[2 * c + 1];
                double r2 = dx * dx + dy * dy;
                double r = sqrt(r2);
                v = r;
                for (int t = 0; t < kphs; ++t) v = v * r2;
            } else if (a < ns) {
                v = monomial_dev(z[2 * a], z[2 * a + 1], c - ns);
            } else if (c < ns) {
                v = monomial_dev(z[2 * c], z[2 * c + 1], a - ns);
            } else {
                v = 0.0;
            }
            M[e] = v;
        }
        for (int a = lane; a < m; a += 32) {
            double v;
            if (a < ns) {
                double r2 = z[2 * a] * z[2 * a] + z[2 * a + 1] * z[2 * a + 1];
                double r = sqrt(r2);
                v = r;
                for (int t = 0; t < kphs - 1; ++t) v = v * r2;
                v = (double)((2 * kphs + 1) * (2 * kphs + 1)) * v;
            } else {
                v = monomial_lap0_dev(a - ns);
            }
            b[a] = v;
        }
        __syncwarp();
        bool ok = warp_lu_solve(M, b, lcol, m, 1e-14);
        if (!ok) {
            if (lane == 0) atomicMin((unsigned long long*)fail, (unsigned long long)i);
            for (int j = lane; j < ns; j += 32) w[i * ns + j] = 0.0;
        } else {
            double rr = rho * rho;
            for (int j = lane; j < ns; j += 32) w[i * ns + j] = b[j] / rr;
        }
        __syncwarp();
    }
}

int launch_rbffd_weights(const double* pts, const double* nrm, const i32* sten, i64 n, int ns,
                         int ell, int k, double* w, i64* fail_dev, void* stream) {
    int L = (ell + 1) * (ell + 2) / 2, m = ns + L;
    size_t per_warp = (size_t)(m * m + 2 * m + 2 * ns) * sizeof(double);
    int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per_warp));
    size_t smem = per_warp * wpb;
    cudaFuncSetAttribute(k_rbffd_weights, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    i64 blocks = std::min<i64>((n + wpb - 1) / wpb, 148 * 16);
    k_rbffd_weights<<<(unsigned)blocks, 32 * wpb, smem, (cudaStream_t)stream>>>(pts, nrm, sten, n, ns,
                                                                                 ell, k, w, fail_dev);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// O5: GFD weights.  rho of every point first (own projected stencil radius).
// ---------------------------------------------------------------------------------------
__global__ void k_stencil_radius(const double* __restrict__ pts, const double* __restrict__ nrm,
                                 const i32* __restrict__ sten, i64 n, int ns, double* rho_out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
    for (i64 i = (i64)blockIdx.x * wpb + warp; i < n; i += (i64)gridDim.x * wpb) {
        double t1[3], t2[3];
        tangent_basis_dev(nrm + 3 * i, t1, t2);
        double rho = 0.0;
        for (int j = lane; j < ns; j += 32) {
            double u, v;
            project_dev(pts + 3 * i, t1, t2, pts + 3 * (i64)sten[i * ns + j], u, v);
            rho = fmax(rho, sqrt(u * u + v * v));
        }
        rho = warp_max(rho);
        if (lane == 0) rho_out[i] = rho;
    }
}

int launch_stencil_radius(const double* pts, const double* nrm, const i32* sten, i64 n, int ns,
                          double* rho, void* stream) {
    i64 blocks = std::min<i64>((n + 7) / 8, 148 * 32);
    k_stencil_radius<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(pts, nrm, sten, n, ns, rho);
    return (int)cudaGetLastError();
}

// smem per warp: B[ns*L], V[ns*L], tau[L], sw[ns], q[ns], y[L]
__global__ void k_gfd_weights(const double* __restrict__ pts, const double* __restrict__ nrm,
                              const i32* __restrict__ sten, i64 n, int ns, int ell, double alpha,
                              const double* __restrict__ rho_all, double* __restrict__ w, i64* fail) {
    extern __shared__ double smem[];
    const int L = (ell + 1) * (ell + 2) / 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const int per_warp = 2 * ns * L + 2 * L + 2 * ns;
    double* B = smem + (size_t)warp * per_warp;
    double* V = B + ns * L;
    double* tau = V + ns * L;
    double* y = tau + L;
    double* sw = y + L;
    double* q = sw + ns;
    for (i64 i = (i64)blockIdx.x * wpb + warp; i < n; i += (i64)gridDim.x * wpb) {
        double t1[3], t2[3];
        tangent_basis_dev(nrm + 3 * i, t1, t2);
        const double rho = rho_all[i];
        const double rr = rho * rho;
        for (int j = lane; j < ns; j += 32) {
            i64 g = sten[i * ns + j];
            double u, v;
            project_dev(pts + 3 * i, t1, t2, pts + 3 * g, u, v);
            double d2 = u * u + v * v;
            double rg = rho_all[g];
            double s = sqrt(exp(-alpha * d2 / (rr + rg * rg)));
            sw[j] = s;
            double zx = u / rho, zy = v / rho;
            for (int c = 0; c < L; ++c) B[j * L + c] = s * monomial_dev(zx, zy, c);
        }
        __syncwarp();
        double rmax = 0.0;
        bool ok = true;
        for (int k = 0; k < L; ++k) {
            // column norm by one lane (sequential order), reflector v
            double nx = 0.0, x0 = 0.0;
            if (lane == 0) {
                double s = 0.0;
                for (int r = k; r < ns; ++r) s = s + B[r * L + k] * B[r * L + k];
                nx = sqrt(s);
                x0 = B[k * L + k];
            }
            nx = __shfl_sync(FULL, nx, 0);
            x0 = __shfl_sync(FULL, x0, 0);
            double alph = (x0 >= 0.0) ? -nx : nx;
            for (int r = lane; r < ns; r += 32)
                V[r * L + k] = (r < k) ? 0.0 : (r == k ? x0 - alph : B[r * L + k]);
            __syncwarp();
            if (nx == 0.0) {
                if (lane == 0) tau[k] = 0.0;
                __syncwarp();
                continue;
            }
            if (lane == 0) {
                double vv = 0.0;
                for (int r = k; r < ns; ++r) vv = vv + V[r * L + k] * V[r * L + k];
                tau[k] = 2.0 / vv;
            }
            __syncwarp();
            for (int c = k + lane; c < L; c += 32) {
                double d = 0.0;
                for (int r = k; r < ns; ++r) d = d + V[r * L + k] * B[r * L + c];
                d = tau[k] * d;
                for (int r = k; r < ns; ++r) B[r * L + c] = B[r * L + c] - d * V[r * L + k];
            }
            __syncwarp();
            rmax = fmax(rmax, fabs(B[k * L + k]));
        }
        for (int k = 0; k < L; ++k)
            if (!(fabs(B[k * L + k]) > 1e-12 * rmax)) ok = false;
        if (!ok) {
            if (lane == 0) atomicMin((unsigned long long*)fail, (unsigned long long)i);
            for (int j = lane; j < ns; j += 32) w[i * ns + j] = 0.0;
            __syncwarp();
            continue;
        }
        if (lane == 0) {
            for (int k = 0; k < L; ++k) {  // y = R^{-T} Lap p
                double s = monomial_lap0_dev(k);
                for (int c = 0; c < k; ++c) s = s - B[c * L + k] * y[c];
                y[k] = s / B[k * L + k];
            }
            for (int r = 0; r < ns; ++r) q[r] = (r < L) ? y[r] : 0.0;
            for (int k = L - 1; k >= 0; --k) {  // q = H_0 ... H_{L-1} [y; 0]
                double d = 0.0;
                for (int r = k; r < ns; ++r) d = d + V[r * L + k] * q[r];
                d = tau[k] * d;
                for (int r = k; r < ns; ++r) q[r] = q[r] - d * V[r * L + k];
            }
        }
        __syncwarp();
        for (int j = lane; j < ns; j += 32) w[i * ns + j] = (sw[j] * q[j]) / rr;
        __syncwarp();
    }
}

int launch_gfd_weights(const double* pts, const double* nrm, const i32* sten, i64 n, int ns,
                       int ell, double alpha, const double* rho, double* w, i64* fail_dev,
                       void* stream) {
    int L = (ell + 1) * (ell + 2) / 2;
    size_t per_warp = (size_t)(2 * ns * L + 2 * L + 2 * ns) * sizeof(double);
    int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / per_warp));
    size_t smem = per_warp * wpb;
    cudaFuncSetAttribute(k_gfd_weights, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    i64 blocks = std::min<i64>((n + wpb - 1) / wpb, 148 * 16);
    k_gfd_weights<<<(unsigned)blocks, 32 * wpb, smem, (cudaStream_t)stream>>>(pts, nrm, sten, n, ns, ell,
                                                                              alpha, rho, w, fail_dev);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// O9: PHS interpolation weights, one thread per fine point.
// ---------------------------------------------------------------------------------------
__global__ void k_interp_weights(const double* __restrict__ fine, i64 nf,
                                 const double* __restrict__ coarse, const i32* __restrict__ sten,
                                 int m, double* __restrict__ w, i32* __restrict__ cnt, i64* fail) {
    double M[17 * 17], b[17];
    const int mm = m + 1;
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += (i64)gridDim.x * blockDim.x) {
        const double* x = fine + 3 * i;
        if (dist2_dev(x, coarse + 3 * (i64)sten[i * m]) == 0.0) {
            for (int a = 0; a < m; ++a) w[i * m + a] = (a == 0) ? 1.0 : 0.0;
            cnt[i] = 1;
            continue;
        }
        for (int a = 0; a < m; ++a) {
            const double* ya = coarse + 3 * (i64)sten[i * m + a];
            for (int c = 0; c < m; ++c) M[a * mm + c] = sqrt(dist2_dev(ya, coarse + 3 * (i64)sten[i * m + c]));
            M[a * mm + m] = 1.0;
            M[m * mm + a] = 1.0;
            b[a] = sqrt(dist2_dev(x, ya));
        }
        M[m * mm + m] = 0.0;
        b[m] = 1.0;
        // sequential LU, same operation order as the warp version
        double amax = 0.0;
        for (int e = 0; e < mm * mm; ++e) amax = fmax(amax, fabs(M[e]));
        bool ok = true;
        for (int k = 0; k < mm && ok; ++k) {
            int p = k;
            double pv = fabs(M[k * mm + k]);
            for (int r = k + 1; r < mm; ++r)
                if (fabs(M[r * mm + k]) > pv) { pv = fabs(M[r * mm + k]); p = r; }
            if (!(pv > 1e-14 * amax)) { ok = false; break; }
            if (p != k) {
                for (int j = 0; j < mm; ++j) { double t = M[k * mm + j]; M[k * mm + j] = M[p * mm + j]; M[p * mm + j] = t; }
                double t = b[k]; b[k] = b[p]; b[p] = t;
            }
            double piv = M[k * mm + k];
            for (int r = k + 1; r < mm; ++r) {
                double l = M[r * mm + k] / piv;
                M[r * mm + k] = l;
                for (int j = k + 1; j < mm; ++j) M[r * mm + j] = M[r * mm + j] - l * M[k * mm + j];
                b[r] = b[r] - l * b[k];
            }
        }
        if (!ok) {
            atomicMin((unsigned long long*)fail, (unsigned long long)i);
            for (int a = 0; a < m; ++a) w[i * m + a] = 0.0;
            cnt[i] = m;
            continue;
        }
        for (int r = mm - 1; r >= 0; --r) {
            double s = b[r];
            for (int j = mm - 1; j > r; --j) s = s - M[r * mm + j] * b[j];
            b[r] = s / M[r * mm + r];
        }
        for (int a = 0; a < m; ++a) w[i * m + a] = b[a];
        cnt[i] = m;
    }
}

int launch_interp_weights(const double* fine, i64 nf, const double* coarse, const i32* sten,
                          int m, double* w, i32* cnt, i64* fail_dev, void* stream) {
    if (m > 16) return (int)cudaErrorInvalidValue;
    i64 blocks = std::min<i64>((nf + 127) / 128, 148 * 32);
    k_interp_weights<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(fine, nf, coarse, sten, m, w,
                                                                         cnt, fail_dev);
    return (int)cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// O10: SpGEMM C = A B, one CTA per output row (grid-stride).  Products of row i are laid
// out in canonical order (A entries by ascending column, then B entries by ascending
// column), keyed (col << 32 | product index), bitonic-sorted in shared memory; each run
// of equal columns is summed sequentially in product order, as the host loop would.
// ---------------------------------------------------------------------------------------
__global__ void k_row_products(const i64* __restrict__ ap, const i32* __restrict__ ai,
                               const i64* __restrict__ bp, i64 nrows, i64* __restrict__ cnt) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += (i64)gridDim.x * blockDim.x) {
        i64 s = 0;
        for (i64 t = ap[i]; t < ap[i + 1]; ++t) s += bp[ai[t] + 1] - bp[ai[t]];
        cnt[i] = s;
    }
}

__device__ void block_bitonic_sort(unsigned long long* keys, int n2) {
    for (int size = 2; size <= n2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (n2 >> 1); t += blockDim.x) {
                int lo = 2 * stride * (t / stride) + (t % stride);
                int hi = lo + stride;
                bool up = ((lo & size) == 0);
                unsigned long long a = keys[lo], b = keys[hi];
                if ((a > b) == up) { keys[lo] = b; keys[hi] = a; }
            }
            __syncthreads();
        }
    }
}

// flag[0 .. total) in {0, 1} -> flag[p] = flag[p] ? (number of ones before p) : -1 and
// flag[total] = number of ones: contiguous runs per thread, block scan of the run sums.
// blockDim.x a multiple of 32, <= 1024.
__device__ void block_rank_flags(int* flag, int total) {
    __shared__ int wsum[32];
    const int nthr = blockDim.x, per = (total + nthr - 1) / nthr;
    const int b = threadIdx.x * per, e = min(total, b + per);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int s = 0;
    for (int p = b; p < e; ++p) s += flag[p];
    int incl = s;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        const int v = lane < (nthr >> 5) ? wsum[lane] : 0;
        int vi = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, vi, o);
            if (lane >= o) vi += u;
        }
        if (lane < (nthr >> 5)) wsum[lane] = vi - v;
    }
    __syncthreads();
    int run = wsum[w] + incl - s;
    for (int p = b; p < e; ++p) {
        const int f = flag[p];
        flag[p] = f ? run : -1;
        run += f;
    }
    if (threadIdx.x == nthr - 1) flag[total] = run;
    __syncthreads();
}

// numeric == false: write the unique-column count of each row to cnt.
// numeric == true : write columns/values at cptr[i].
template <bool NUMERIC>
__global__ void k_spgemm_rows(i64 nrows, const i64* __restrict__ ap, const i32* __restrict__ ai,
                              const double* __restrict__ av, const i64* __restrict__ bp,
                              const i32* __restrict__ bi, const double* __restrict__ bv, int n2,
                              i64* __restrict__ cnt, const i64* __restrict__ cptr,
                              i32* __restrict__ ci, double* __restrict__ cv,
                              const unsigned char* __restrict__ skip) {
    extern __shared__ unsigned long long sm[];
    unsigned long long* keys = sm;                          // n2
    double* vals = (double*)(keys + n2);                    // n2
    int* flag = (int*)(vals + n2);                          // n2 + 1 (scan)
    __shared__ i64 off_s[1025];
    __shared__ int total_s;
    for (i64 i = blockIdx.x; i < nrows; i += gridDim.x) {
        if (skip[i]) continue;  // long rows: spgemm_long_rows (sorted products, same order)
        const i64 a0 = ap[i], a1 = ap[i + 1];
        const int na = (int)(a1 - a0);
        // offsets of each A entry's products: warp 0, shuffle scan over chunks of 32 entries
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            i64 carry = 0;
            for (int base = 0; base < na; base += 32) {
                const int t = base + lane;
                i64 len = 0;
                if (t < na) {
                    const i32 k = ai[a0 + t];
                    len = bp[k + 1] - bp[k];
                }
                i64 inc = len;
                for (int o = 1; o < 32; o <<= 1) {
                    const i64 v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += v;
                }
                if (t < na) off_s[t] = carry + inc - len;
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
            if (lane == 0) {
                off_s[na] = carry;
                total_s = (int)carry;
            }
        }
        __syncthreads();
        const int total = total_s;
        for (int t = 0; t < na; ++t) {
            i32 k = ai[a0 + t];
            i64 b0 = bp[k], b1 = bp[k + 1];
            double a = NUMERIC ? av[a0 + t] : 0.0;
            for (i64 s = b0 + threadIdx.x; s < b1; s += blockDim.x) {
                int pidx = (int)(off_s[t] + (s - b0));
                keys[pidx] = ((unsigned long long)(unsigned)bi[s] << 32) | (unsigned)pidx;
                if (NUMERIC) vals[pidx] = __dmul_rn(a, bv[s]);
            }
        }
        for (int p = total + threadIdx.x; p < n2; p += blockDim.x) keys[p] = ~0ull;
        __syncthreads();
        block_bitonic_sort(keys, n2);
        // segment starts and their ranks (exclusive scan, serial over warps for simplicity)
        for (int p = threadIdx.x; p < total; p += blockDim.x)
            flag[p] = (p == 0 || (keys[p] >> 32) != (keys[p - 1] >> 32)) ? 1 : 0;
        __syncthreads();
        block_rank_flags(flag, total);
        if (!NUMERIC) {
            if (threadIdx.x == 0) cnt[i] = flag[total];
        } else {
            const i64 base = cptr[i];
            for (int p = threadIdx.x; p < total; p += blockDim.x) {
                int rank = flag[p];
                if (rank < 0) continue;
                unsigned col = (unsigned)(keys[p] >> 32);
                double s = 0.0;
                for (int q = p; q < total && (unsigned)(keys[q] >> 32) == col; ++q)
                    s = __dadd_rn(s, vals[(unsigned)(keys[q] & 0xffffffffu)]);
                ci[base + rank] = (i32)col;
                cv[base + rank] = s;
            }
        }
        __syncthreads();
    }
}

static inline int next_pow2(i64 v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// ---------------------------------------------------------------------------------------
// Long rows (products beyond the shared-memory buffer, or > 1024 A entries), on the GPU in
// the same canonical order: every product of the long rows is written with the key
// (long-row slot << 32 | column) and its global product index, the pairs are radix-sorted
// (stable: equal keys keep ascending product index = the canonical product order), and each
// run of equal keys is summed sequentially in that order with the same correctly rounded
// multiply and add as k_spgemm_rows -- bit-identical to the shared-memory path.
// ---------------------------------------------------------------------------------------
__global__ void k_long_offsets(i64 nl, const i64* __restrict__ rows, const i64* __restrict__ ap,
                               const i32* __restrict__ ai, const i64* __restrict__ bp, const i64* __restrict__ loff,
                               i64* __restrict__ aoff /* per long row: product offset of each A entry */,
                               const i64* __restrict__ aoff_base) {
    for (i64 q = (i64)blockIdx.x * blockDim.x + threadIdx.x; q < nl; q += (i64)gridDim.x * blockDim.x) {
        const i64 i = rows[q], a0 = ap[i], a1 = ap[i + 1];
        i64 o = loff[q];
        for (i64 t = a0; t < a1; ++t) {
            aoff[aoff_base[q] + (t - a0)] = o;
            const i32 k = ai[t];
            o += bp[k + 1] - bp[k];
        }
    }
}
__global__ void k_long_products(i64 nl, const i64* __restrict__ rows, const i64* __restrict__ ap,
                                const i32* __restrict__ ai, const double* __restrict__ av,
                                const i64* __restrict__ bp, const i32* __restrict__ bi,
                                const double* __restrict__ bv, const i64* __restrict__ aoff,
                                const i64* __restrict__ aoff_base, unsigned long long* __restrict__ key,
                                i64* __restrict__ pidx, double* __restrict__ val) {
    for (i64 q = blockIdx.x; q < nl; q += gridDim.x) {
        const i64 i = rows[q], a0 = ap[i], a1 = ap[i + 1];
        for (i64 t = a0; t < a1; ++t) {
            const i32 k = ai[t];
            const i64 b0 = bp[k], b1 = bp[k + 1], o = aoff[aoff_base[q] + (t - a0)];
            const double a = av[t];
            for (i64 s = b0 + threadIdx.x; s < b1; s += blockDim.x) {
                key[o + (s - b0)] = ((unsigned long long)q << 32) | (unsigned)bi[s];
                pidx[o + (s - b0)] = o + (s - b0);
                val[o + (s - b0)] = __dmul_rn(a, bv[s]);
            }
        }
    }
}
__global__ void k_long_heads(i64 np, const unsigned long long* __restrict__ key, int* __restrict__ head) {
    for (i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (i64)gridDim.x * blockDim.x)
        head[p] = (p == 0 || key[p] != key[p - 1]) ? 1 : 0;
}
// segment sums (sequential in product order) and per-long-row unique counts
__global__ void k_long_sums(i64 np, const unsigned long long* __restrict__ key, const i64* __restrict__ pidx,
                            const double* __restrict__ val, const int* __restrict__ head,
                            const int* __restrict__ rank, i32* __restrict__ ocol, double* __restrict__ oval,
                            int* __restrict__ row_first) {
    for (i64 p = (i64)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (i64)gridDim.x * blockDim.x) {
        if (!head[p]) continue;
        const unsigned long long k = key[p];
        double s = 0.0;
        for (i64 r = p; r < np && key[r] == k; ++r) s = __dadd_rn(s, val[pidx[r]]);
        ocol[rank[p]] = (i32)(unsigned)(k & 0xffffffffull);
        oval[rank[p]] = s;
        if (p == 0 || (key[p - 1] >> 32) != (k >> 32)) row_first[k >> 32] = rank[p];
    }
}

struct LongRows {
    i64 nl = 0, np = 0, nout = 0;
    std::vector<i64> rows, first;  // first[q] .. first[q+1]: unique columns of long row q in ocol/oval
    i32* ocol = nullptr;
    double* oval = nullptr;
};

template <class T>
static cudaError_t dalloc_n(T** p, i64 n) { return dev_malloc((void**)p, sizeof(T) * (size_t)std::max<i64>(n, 1)); }

static int spgemm_long_rows(const DevCSR& A, const DevCSR& B, const std::vector<i64>& longs,
                            const std::vector<i64>& cnt, const std::vector<i64>& aptr, LongRows& LR,
                            cudaStream_t st, std::string& err) {
    LR.nl = (i64)longs.size();
    LR.rows = longs;
    if (LR.nl == 0) return 0;
    std::vector<i64> loff(LR.nl + 1, 0), abase(LR.nl + 1, 0);
    for (i64 q = 0; q < LR.nl; ++q) {
        loff[q + 1] = loff[q] + cnt[longs[q]];
        abase[q + 1] = abase[q] + (aptr[longs[q] + 1] - aptr[longs[q]]);
    }
    const i64 np = loff[LR.nl];
    LR.np = np;
    i64 *d_rows = nullptr, *d_loff = nullptr, *d_abase = nullptr, *d_aoff = nullptr, *d_pidx = nullptr,
        *d_pidx2 = nullptr;
    unsigned long long *d_key = nullptr, *d_key2 = nullptr;
    double* d_val = nullptr;
    int *d_head = nullptr, *d_rank = nullptr, *d_first = nullptr;
    void* d_tmp = nullptr;
    auto cleanup = [&]() {
        for (void* ptr : {(void*)d_rows, (void*)d_loff, (void*)d_abase, (void*)d_aoff, (void*)d_pidx, (void*)d_pidx2,
                          (void*)d_key, (void*)d_key2, (void*)d_val, (void*)d_head, (void*)d_rank, (void*)d_first,
                          d_tmp})
            if (ptr) dev_free(ptr);
    };
    cudaError_t e = dalloc_n(&d_rows, LR.nl);
    if (!e) e = dalloc_n(&d_loff, LR.nl + 1);
    if (!e) e = dalloc_n(&d_abase, LR.nl + 1);
    if (!e) e = dalloc_n(&d_aoff, abase[LR.nl]);
    if (!e) e = dalloc_n(&d_pidx, np);
    if (!e) e = dalloc_n(&d_pidx2, np);
    if (!e) e = dalloc_n(&d_key, np);
    if (!e) e = dalloc_n(&d_key2, np);
    if (!e) e = dalloc_n(&d_val, np);
    if (!e) e = dalloc_n(&d_head, np);
    if (!e) e = dalloc_n(&d_rank, np);
    if (!e) e = dalloc_n(&d_first, LR.nl + 1);
    if (e) { cleanup(); err = "cudaMalloc (long SpGEMM rows)"; return (int)e; }
    cudaMemcpyAsync(d_rows, longs.data(), sizeof(i64) * LR.nl, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_loff, loff.data(), sizeof(i64) * (LR.nl + 1), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_abase, abase.data(), sizeof(i64) * (LR.nl + 1), cudaMemcpyHostToDevice, st);
    const unsigned g = (unsigned)std::min<i64>(148 * 8, std::max<i64>(1, (LR.nl + 127) / 128));
    k_long_offsets<<<g, 128, 0, st>>>(LR.nl, d_rows, A.ptr, A.col, B.ptr, d_loff, d_aoff, d_abase);
    k_long_products<<<(unsigned)std::min<i64>(LR.nl, 148 * 8), 256, 0, st>>>(
        LR.nl, d_rows, A.ptr, A.col, A.val, B.ptr, B.col, B.val, d_aoff, d_abase, d_key, d_pidx, d_val);
    // stable radix sort of (row slot, column) keys carrying the product index
    int hi_bit = 33;
    while ((1ll << (hi_bit - 32)) <= LR.nl) ++hi_bit;
    size_t tmp_bytes = 0, tmp2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_key, d_key2, d_pidx, d_pidx2, (int)np, 0, hi_bit, st);
    cub::DeviceScan::ExclusiveSum(nullptr, tmp2, d_head, d_rank, (int)np, st);
    tmp_bytes = std::max(tmp_bytes, tmp2);
    if ((e = dev_malloc(&d_tmp, std::max<size_t>(tmp_bytes, 1)))) { cleanup(); err = "cudaMalloc (sort)"; return (int)e; }
    cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_key, d_key2, d_pidx, d_pidx2, (int)np, 0, hi_bit, st);
    const unsigned gp = (unsigned)std::min<i64>(148 * 16, std::max<i64>(1, (np + 255) / 256));
    k_long_heads<<<gp, 256, 0, st>>>(np, d_key2, d_head);
    cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_head, d_rank, (int)np, st);
    int last_head = 0, last_rank = 0;
    cudaMemcpyAsync(&last_head, d_head + np - 1, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&last_rank, d_rank + np - 1, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    LR.nout = (i64)last_rank + last_head;
    if ((e = dalloc_n(&LR.ocol, LR.nout)) || (e = dalloc_n(&LR.oval, LR.nout))) {
        cleanup();
        err = "cudaMalloc (long rows out)";
        return (int)e;
    }
    k_long_sums<<<gp, 256, 0, st>>>(np, d_key2, d_pidx2, d_val, d_head, d_rank, LR.ocol, LR.oval, d_first);
    std::vector<int> first(LR.nl);
    cudaMemcpyAsync(first.data(), d_first, sizeof(int) * LR.nl, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    cleanup();
    if (e) { err = "long SpGEMM rows"; return (int)e; }
    LR.first.assign(LR.nl + 1, LR.nout);
    for (i64 q = 0; q < LR.nl; ++q) LR.first[q] = first[q];  // (every long row has >= 1 product)
    return 0;
}

// ---------------------------------------------------------------------------------------
// Exact grid kNN on the device (O2; the same lists as host_setup.cpp knn_grid: the k
// smallest (squared distance, index) pairs, ascending).  A dense cell table over the
// bounding box (cells grown until it holds at most 4n + 64 cells, then shrunk towards ~k/2
// points per occupied cell); one thread per query expands Chebyshev shells of cells and
// stops once the k-th best squared distance is below the squared distance to every
// unvisited cell (1e-9 relative margin).  The result does not depend on the cell size.
// ---------------------------------------------------------------------------------------
struct DevGrid {
    double lo[3], cell;
    i64 dims[3];
};

__device__ __forceinline__ void grid_coords(const DevGrid& g, const double* x, i64* c) {
    for (int a = 0; a < 3; ++a) {
        const i64 v = (i64)floor((x[a] - g.lo[a]) / g.cell);
        c[a] = min(max(v, (i64)0), g.dims[a] - 1);
    }
}

__global__ void k_grid_count(DevGrid g, const double* __restrict__ pts, i64 n, i64* __restrict__ cid,
                             int* __restrict__ cnt) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        i64 c[3];
        grid_coords(g, pts + 3 * i, c);
        const i64 id = (c[2] * g.dims[1] + c[1]) * g.dims[0] + c[0];
        cid[i] = id;
        atomicAdd(&cnt[id], 1);
    }
}

__global__ void k_grid_fill(i64 n, const i64* __restrict__ cid, int* __restrict__ fill, i32* __restrict__ items) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        items[atomicAdd(&fill[cid[i]], 1)] = (i32)i;
}

__global__ void k_count_occupied(i64 total, const int* __restrict__ cnt, unsigned long long* __restrict__ occ) {
    unsigned long long c = 0;
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < total; i += (i64)gridDim.x * blockDim.x)
        c += cnt[i] > 0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(FULL, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(occ, c);
}

template <int KMAX>
__global__ void __launch_bounds__(128) k_knn(DevGrid g, const double* __restrict__ pts, const int* __restrict__ start,
                                             const i32* __restrict__ items, const double* __restrict__ qry, i64 nq,
                                             int k, i32* __restrict__ out) {
    double bd[KMAX];
    int bj[KMAX];
    const i64 maxr = max(g.dims[0], max(g.dims[1], g.dims[2]));
    for (i64 qi = blockIdx.x * (i64)blockDim.x + threadIdx.x; qi < nq; qi += (i64)gridDim.x * blockDim.x) {
        const double x[3] = {qry[3 * qi], qry[3 * qi + 1], qry[3 * qi + 2]};
        int count = 0;
        i64 c[3];
        grid_coords(g, x, c);
        for (i64 r = 0; r <= maxr; ++r) {
            for (i64 z = c[2] - r; z <= c[2] + r; ++z) {
                if (z < 0 || z >= g.dims[2]) continue;
                const bool zface = (z == c[2] - r || z == c[2] + r);
                for (i64 y = c[1] - r; y <= c[1] + r; ++y) {
                    if (y < 0 || y >= g.dims[1]) continue;
                    const bool yface = zface || (y == c[1] - r || y == c[1] + r);
                    for (i64 xx = c[0] - r; xx <= c[0] + r; ++xx) {
                        if (xx < 0 || xx >= g.dims[0]) continue;
                        if (!yface && xx != c[0] - r && xx != c[0] + r) {
                            xx = c[0] + r - 1;  // skip the interior run of this row
                            continue;
                        }
                        const i64 cell = (z * g.dims[1] + y) * g.dims[0] + xx;
                        for (int t = start[cell]; t < start[cell + 1]; ++t) {
                            const i32 j = items[t];
                            const double* yv = pts + 3 * (i64)j;
                            const double dx = yv[0] - x[0], dy = yv[1] - x[1], dz = yv[2] - x[2];
                            const double dd = (dx * dx + dy * dy) + dz * dz;  // O2 (no FMA: -fmad=false)
                            if (count == k && (dd > bd[k - 1] || (dd == bd[k - 1] && j > bj[k - 1]))) continue;
                            int p = count < k ? count++ : k - 1;
                            while (p > 0 && (bd[p - 1] > dd || (bd[p - 1] == dd && bj[p - 1] > j))) {
                                bd[p] = bd[p - 1];
                                bj[p] = bj[p - 1];
                                --p;
                            }
                            bd[p] = dd;
                            bj[p] = j;
                        }
                    }
                }
            }
            if (count == k) {
                double dmin = INFINITY;
                bool all = true;
                for (int a = 0; a < 3; ++a) {
                    const double lo_face = g.lo[a] + (double)(c[a] - r) * g.cell;
                    const double hi_face = g.lo[a] + (double)(c[a] + r + 1) * g.cell;
                    if (c[a] - r > 0) { dmin = fmin(dmin, x[a] - lo_face); all = false; }
                    if (c[a] + r + 1 < g.dims[a]) { dmin = fmin(dmin, hi_face - x[a]); all = false; }
                }
                if (all) break;
                if (dmin > 0) {
                    const double b2 = dmin * dmin * (1.0 - 1e-9);
                    if (bd[k - 1] < b2) break;
                }
            }
        }
        for (int t = 0; t < k; ++t) out[qi * k + t] = t < count ? bj[t] : -1;
    }
}

int knn_device(const double* h_pts, const double* d_pts, i64 n, const double* d_qry, i64 nq, int k, i32* d_out,
               void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (k < 1 || k > 64 || n < 1) return (int)cudaErrorInvalidValue;
    DevGrid g;
    double hi[3];
    for (int a = 0; a < 3; ++a) g.lo[a] = hi[a] = h_pts[a];
    for (i64 i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            g.lo[a] = std::min(g.lo[a], h_pts[3 * i + a]);
            hi[a] = std::max(hi[a], h_pts[3 * i + a]);
        }
    double cell;
    {  // volumetric start: ~k/4 points per cell of the box
        const double ext = std::max(hi[0] - g.lo[0], std::max(hi[1] - g.lo[1], hi[2] - g.lo[2]));
        double vol = 1.0;
        for (int a = 0; a < 3; ++a) vol *= std::max(hi[a] - g.lo[a], 1e-3 * ext);
        cell = std::cbrt(vol * std::max(1, k / 4) / (double)n);
        if (!(cell > 0)) cell = 1.0;
    }
    i64* cid = nullptr;
    int *cnt = nullptr, *fill = nullptr;
    i32* items = nullptr;
    unsigned long long* occ = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    i64 cap = 0;
    auto release = [&] {
        dev_free(cid);
        dev_free(cnt);
        dev_free(fill);
        dev_free(items);
        dev_free(occ);
        dev_free(tmp);
    };
    cudaError_t e = dev_malloc((void**)&cid, sizeof(i64) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&items, sizeof(i32) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&occ, sizeof(unsigned long long));
    if (e != cudaSuccess) { release(); return (int)e; }
    const unsigned nb = (unsigned)std::min<i64>((n + 255) / 256, 148 * 16);
    for (int pass = 0; pass < 2; ++pass) {
        g.cell = cell;
        i64 total = 1;
        auto dims_for = [&] {
            total = 1;
            for (int a = 0; a < 3; ++a) {
                g.dims[a] = std::max<i64>(1, (i64)std::floor((hi[a] - g.lo[a]) / g.cell) + 1);
                total *= g.dims[a];
            }
        };
        dims_for();
        while (total > 4 * n + 64) {  // bounded dense table (cells only grow)
            g.cell *= 1.26;
            dims_for();
        }
        if (total + 1 > cap) {
            dev_free(cnt);
            dev_free(fill);
            dev_free(tmp);
            cnt = fill = nullptr;
            tmp = nullptr;
            cap = total + 1;
            e = dev_malloc((void**)&cnt, sizeof(int) * cap);
            if (e == cudaSuccess) e = dev_malloc((void**)&fill, sizeof(int) * cap);
            tmp_bytes = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, fill, (int)cap, st);
            if (e == cudaSuccess) e = dev_malloc(&tmp, std::max<size_t>(tmp_bytes, 16));
            if (e != cudaSuccess) { release(); return (int)e; }
        }
        cudaMemsetAsync(cnt, 0, sizeof(int) * (total + 1), st);
        k_grid_count<<<nb, 256, 0, st>>>(g, d_pts, n, cid, cnt);
        if (pass == 0) {  // surface clouds fill few cells of the box: shrink the cells
            cudaMemsetAsync(occ, 0, sizeof(unsigned long long), st);
            k_count_occupied<<<(unsigned)std::min<i64>((total + 255) / 256, 148 * 16), 256, 0, st>>>(total, cnt, occ);
            unsigned long long h_occ = 1;
            cudaMemcpyAsync(&h_occ, occ, sizeof(h_occ), cudaMemcpyDeviceToHost, st);
            e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) { release(); return (int)e; }
            const double per = (double)n / (double)std::max<unsigned long long>(h_occ, 1);
            if (per > 2.0 * k) {
                cell = g.cell * std::sqrt(0.5 * k / per);
                continue;
            }
        }
        size_t tb = tmp_bytes;
        cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, fill, (int)(total + 1), st);
        cudaMemcpyAsync(cnt, fill, sizeof(int) * (total + 1), cudaMemcpyDeviceToDevice, st);  // cnt := start
        k_grid_fill<<<nb, 256, 0, st>>>(n, cid, fill, items);
        const unsigned qb = (unsigned)std::max<i64>(1, std::min<i64>((nq + 127) / 128, 148 * 64));
        if (k <= 16) k_knn<16><<<qb, 128, 0, st>>>(g, d_pts, cnt, items, d_qry, nq, k, d_out);
        else if (k <= 32) k_knn<32><<<qb, 128, 0, st>>>(g, d_pts, cnt, items, d_qry, nq, k, d_out);
        else k_knn<64><<<qb, 128, 0, st>>>(g, d_pts, cnt, items, d_qry, nq, k, d_out);
        break;
    }
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    release();
    return (int)e;
}

// Squared distance to the nearest other point (host_setup.cpp nearest_other, the same
// arithmetic): from the 3 nearest (O2 order) of every point, the first entry that is not the
// point itself.  dup: the smallest index with a zero distance (a duplicate), or n.
__global__ void k_nearest_other(i64 n, const double* __restrict__ pts, const i32* __restrict__ nb,
                                double* __restrict__ nn2, unsigned long long* __restrict__ dup) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const i32 j = nb[3 * i] == (i32)i ? nb[3 * i + 1] : nb[3 * i];
        const double* x = pts + 3 * i;
        const double* y = pts + 3 * (i64)j;
        const double dx = y[0] - x[0], dy = y[1] - x[1], dz = y[2] - x[2];
        const double d2 = (dx * dx + dy * dy) + dz * dz;
        nn2[i] = d2;
        if (d2 == 0.0) atomicMin(dup, (unsigned long long)i);
    }
}

i64 nearest_other_device(const double* h_pts, const double* d_pts, i64 n, std::vector<double>& nn2, void* stream,
                         int* err) {
    cudaStream_t st = (cudaStream_t)stream;
    *err = 0;
    if (n < 3) { *err = (int)cudaErrorInvalidValue; return -1; }
    i32* nb = nullptr;
    double* d_nn2 = nullptr;
    unsigned long long* d_dup = nullptr;
    cudaError_t e = dev_malloc((void**)&nb, sizeof(i32) * 3 * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&d_nn2, sizeof(double) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&d_dup, sizeof(unsigned long long));
    unsigned long long h_dup = (unsigned long long)n;
    if (e == cudaSuccess) e = (cudaError_t)knn_device(h_pts, d_pts, n, d_pts, n, 3, nb, stream);
    if (e == cudaSuccess) {
        cudaMemcpyAsync(d_dup, &h_dup, sizeof(h_dup), cudaMemcpyHostToDevice, st);
        k_nearest_other<<<(unsigned)std::min<i64>((n + 255) / 256, 148 * 16), 256, 0, st>>>(n, d_pts, nb, d_nn2, d_dup);
        nn2.resize(n);
        cudaMemcpyAsync(nn2.data(), d_nn2, sizeof(double) * n, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(&h_dup, d_dup, sizeof(h_dup), cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
    }
    dev_free(nb);
    dev_free(d_nn2);
    dev_free(d_dup);
    if (e != cudaSuccess) { *err = (int)e; return -1; }
    return h_dup < (unsigned long long)n ? (i64)h_dup : -1;
}

// ---------------------------------------------------------------------------------------
// Weighted sample elimination on the device (O8).  The same result as
// host_setup.cpp's wse_pass, step for step:
//   * neighbour sets {j != i : sqrt(d2) < R} with d2 = (dx^2 + dy^2) + dz^2 (-fmad=false: the
//     host's rounding), W_ij = floor((1 - d/R)^8 2^40 + 0.5) as int64 and weight_i = sum_j W_ij
//     (exact integers: the order of the neighbour lists does not matter);
//   * rounds of local maxima: every live point of positive weight whose priority (weight
//     desc, index asc) beats all its live neighbours' pops in this round with its current
//     weight, then its live neighbours' weights drop by W (integer atomics commute);
//   * the n - nt highest pop priorities are eliminated (stable radix sort, index order ties),
//     or the pass is degenerate (fewer positive pops) and R grows by 1.25.
// A dense cell table over the bounding box (cell side >= R, grown until it holds at most
// 4n + 64 cells); one thread per point scans the cells that meet the box of half side R.
// ---------------------------------------------------------------------------------------
template <bool FILL>
__global__ void __launch_bounds__(128) k_wse_nbrs(DevGrid g, const double* __restrict__ pts, const int* __restrict__ start,
                                                  const i32* __restrict__ items, i64 n, double R,
                                                  i64* __restrict__ cnt, const i64* __restrict__ ptr,
                                                  i32* __restrict__ adj, i64* __restrict__ adjw,
                                                  i64* __restrict__ weight) {
    const double R2far = R * R * (1.0 + 1e-6);
    const double Rm = R * (1.0 + 1e-6);
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        const double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
        i64 lo[3], hi[3];
        for (int a = 0; a < 3; ++a) {
            lo[a] = max((i64)floor((x[a] - Rm - g.lo[a]) / g.cell), (i64)0);
            hi[a] = min((i64)floor((x[a] + Rm - g.lo[a]) / g.cell), g.dims[a] - 1);
        }
        i64 c = 0, o = FILL ? ptr[i] : 0, wsum = 0;
        for (i64 z = lo[2]; z <= hi[2]; ++z)
            for (i64 y = lo[1]; y <= hi[1]; ++y)
                for (i64 xx = lo[0]; xx <= hi[0]; ++xx) {
                    const i64 cell = (z * g.dims[1] + y) * g.dims[0] + xx;
                    for (int t = start[cell]; t < start[cell + 1]; ++t) {
                        const i32 j = items[t];
                        if (j == (i32)i) continue;
                        const double* yv = pts + 3 * (i64)j;
                        const double dx = yv[0] - x[0], dy = yv[1] - x[1], dz = yv[2] - x[2];
                        const double d2 = (dx * dx + dy * dy) + dz * dz;
                        if (d2 > R2far) continue;  // sqrt(d2) > R for certain
                        const double d = sqrt(d2);
                        if (!(d < R)) continue;
                        if (FILL) {
                            const double u = 1.0 - d / R;
                            const double u2 = u * u;
                            const double u4 = u2 * u2;
                            const double u8 = u4 * u4;
                            const i64 w = (i64)floor(u8 * 1099511627776.0 + 0.5);  // 2^40
                            adj[o] = j;
                            adjw[o] = w;
                            ++o;
                            wsum += w;
                        } else {
                            ++c;
                        }
                    }
                }
        if (FILL) weight[i] = wsum;
        else cnt[i] = c;
    }
}

// All rounds in one cooperative launch (grid barriers between the phases), the work of a
// round limited to its candidates as in the host loop: round 0 every point of positive
// weight, later rounds the live points within two hops of the previous round's pops (only
// their neighbourhoods changed).  dead[x]: 0 live, r + 1 popped in round r (live at the start
// of round r: 0 or > r).  Per round:
//   A. each live candidate of positive weight that beats every live neighbour (weight desc,
//      index asc) pops: dead = r + 1, popw = its weight, appended to pops;
//   B. each pop lowers its live neighbours' weights by W (int64 atomics: the updates commute)
//      and queues its live 1- and 2-hop neighbours (stamp: once per round) for round r + 1.
// Ends after a round without pops; *total = the number of pops.
struct WseRounds {
    i64 n;
    const i64* ptr;
    const i32* adj;
    const i64* adjw;
    i64* weight;
    int* dead;
    int* stamp;
    unsigned long long* popw;
    i32* cand[2];
    i32* pops;
    unsigned long long* cnt;  // [0..1] candidates per parity, [2..3] pops per parity, [4] total
};

__global__ void __launch_bounds__(256) k_wse_rounds(WseRounds a) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const i64 tid = blockIdx.x * (i64)blockDim.x + threadIdx.x, nth = (i64)gridDim.x * blockDim.x;
    volatile unsigned long long* cnt = a.cnt;
    for (int r = 0;; ++r) {
        const int p = r & 1;
        const i64 nc = (i64)cnt[p];
        const i32* cand = a.cand[p];
        if (tid == 0) cnt[p ^ 1] = 0;  // round r + 1's candidates (round r - 1 read them)
        for (i64 q = tid; q < nc; q += nth) {
            const i32 x = cand[q];
            if (a.dead[x] != 0) continue;
            const i64 wx = a.weight[x];
            if (wx <= 0) continue;
            bool top = true;
            for (i64 t = a.ptr[x]; t < a.ptr[x + 1] && top; ++t) {
                const i32 y = a.adj[t];
                const int dy = *(volatile int*)&a.dead[y];
                if (dy != 0 && dy <= r) continue;  // popped in an earlier round
                const i64 wy = a.weight[y];
                if (wy > wx || (wy == wx && y < x)) top = false;
            }
            if (top) {
                a.dead[x] = r + 1;
                a.popw[x] = (unsigned long long)wx;
                a.pops[atomicAdd(&a.cnt[2 + p], 1ull)] = x;
            }
        }
        grid.sync();
        const i64 np = (i64)cnt[2 + p];
        if (np == 0) break;
        if (tid == 0) {
            cnt[2 + (p ^ 1)] = 0;
            cnt[4] += (unsigned long long)np;
        }
        i32* next = a.cand[p ^ 1];
        auto queue = [&](i32 y) {
            if (atomicExch(&a.stamp[y], r) != r) next[atomicAdd(&a.cnt[p ^ 1], 1ull)] = y;
        };
        for (i64 q = tid; q < np; q += nth) {
            const i32 x = a.pops[q];
            for (i64 t = a.ptr[x]; t < a.ptr[x + 1]; ++t) {
                const i32 y = a.adj[t];
                if (a.dead[y] != 0) continue;
                atomicAdd((unsigned long long*)&a.weight[y], (unsigned long long)(-a.adjw[t]));
                queue(y);
                for (i64 t2 = a.ptr[y]; t2 < a.ptr[y + 1]; ++t2)
                    if (a.dead[a.adj[t2]] == 0) queue(a.adj[t2]);
            }
        }
        grid.sync();
    }
}

__global__ void k_wse_cand0(i64 n, const i64* __restrict__ weight, i32* __restrict__ cand,
                            unsigned long long* __restrict__ cnt) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
        if (weight[i] > 0) cand[atomicAdd(cnt, 1ull)] = (i32)i;
}

__global__ void k_iota_i32(i64 n, i32* __restrict__ v) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) v[i] = (i32)i;
}

__global__ void k_wse_mark(i64 ne, const i32* __restrict__ order, uint8_t* __restrict__ elim) {
    for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < ne; q += (i64)gridDim.x * blockDim.x)
        elim[order[q]] = 1;
}

int wse_device(const double* d_pts, const double* h_pts, i64 n, i64 nt, const std::vector<double>& nn2,
               std::vector<i64>& keep, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    keep.clear();
    if (nt >= n) {
        for (i64 i = 0; i < n; ++i) keep.push_back(i);
        return 0;
    }
    if (n >= ((i64)1 << 31)) return (int)cudaErrorInvalidValue;
    const i64 ne = n - nt;
    double lo3[3], hi3[3];
    for (int a = 0; a < 3; ++a) lo3[a] = hi3[a] = h_pts[a];
    for (i64 i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            lo3[a] = std::min(lo3[a], h_pts[3 * i + a]);
            hi3[a] = std::max(hi3[a], h_pts[3 * i + a]);
        }
    i64 *cid = nullptr, *cnt = nullptr, *ptr = nullptr, *adjw = nullptr, *weight = nullptr;
    int *gcnt = nullptr, *gfill = nullptr, *dead = nullptr;
    i32 *items = nullptr, *adj = nullptr, *ord_in = nullptr, *ord_out = nullptr, *candA = nullptr, *candB = nullptr,
        *pops = nullptr;
    int* stamp = nullptr;
    unsigned long long *popw = nullptr, *popw_out = nullptr, *npop = nullptr;
    uint8_t* elim = nullptr;
    void* tmp = nullptr;
    size_t tmp_cap = 0;
    auto release = [&] {
        dev_free(cid); dev_free(cnt); dev_free(ptr); dev_free(adjw); dev_free(weight);
        dev_free(gcnt); dev_free(gfill); dev_free(dead); dev_free(items); dev_free(adj);
        dev_free(ord_in); dev_free(ord_out); dev_free(popw); dev_free(popw_out); dev_free(npop);
        dev_free(elim); dev_free(tmp); dev_free(candA); dev_free(candB); dev_free(pops); dev_free(stamp);
    };
    auto need_tmp = [&](size_t b) -> cudaError_t {
        if (b <= tmp_cap) return cudaSuccess;
        dev_free(tmp);
        tmp = nullptr;
        tmp_cap = b;
        return dev_malloc(&tmp, b);
    };
    cudaError_t e = dev_malloc((void**)&cid, sizeof(i64) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&items, sizeof(i32) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&cnt, sizeof(i64) * (n + 1));
    if (e == cudaSuccess) e = dev_malloc((void**)&ptr, sizeof(i64) * (n + 1));
    if (e == cudaSuccess) e = dev_malloc((void**)&weight, sizeof(i64) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&dead, sizeof(int) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&popw, sizeof(unsigned long long) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&popw_out, sizeof(unsigned long long) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&ord_in, sizeof(i32) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&ord_out, sizeof(i32) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&npop, sizeof(unsigned long long) * 5);
    if (e == cudaSuccess) e = dev_malloc((void**)&elim, n);
    if (e == cudaSuccess) e = dev_malloc((void**)&candA, sizeof(i32) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&candB, sizeof(i32) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&pops, sizeof(i32) * n);
    if (e == cudaSuccess) e = dev_malloc((void**)&stamp, sizeof(int) * n);
    if (e != cudaSuccess) { release(); return (int)e; }
    const unsigned nb = (unsigned)std::min<i64>((n + 255) / 256, 148 * 16);
    const unsigned nbq = (unsigned)std::min<i64>((n + 127) / 128, 148 * 64);
    double R = wse_initial_radius(nn2, n, nt);
    bool done = false;
    for (int attempt = 0; attempt < 16 && !done; ++attempt, R *= 1.25) {
        // cell table, side >= R
        DevGrid g;
        for (int a = 0; a < 3; ++a) g.lo[a] = lo3[a];
        g.cell = R * (1.0 + 1e-6);
        i64 total = 1;
        for (;;) {
            total = 1;
            for (int a = 0; a < 3; ++a) {
                g.dims[a] = std::max<i64>(1, (i64)std::floor((hi3[a] - g.lo[a]) / g.cell) + 1);
                total *= g.dims[a];
            }
            if (total <= std::min<i64>(4 * n + 64, (i64)1 << 30)) break;  // (int cell offsets)
            g.cell *= 1.26;
        }
        dev_free(gcnt);
        dev_free(gfill);
        gcnt = gfill = nullptr;
        e = dev_malloc((void**)&gcnt, sizeof(int) * (total + 1));
        if (e == cudaSuccess) e = dev_malloc((void**)&gfill, sizeof(int) * (total + 1));
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, gcnt, gfill, (int)(total + 1), st);
        if (e == cudaSuccess) e = need_tmp(std::max<size_t>(tb, 16));
        if (e != cudaSuccess) { release(); return (int)e; }
        cudaMemsetAsync(gcnt, 0, sizeof(int) * (total + 1), st);
        k_grid_count<<<nb, 256, 0, st>>>(g, d_pts, n, cid, gcnt);
        tb = tmp_cap;
        cub::DeviceScan::ExclusiveSum(tmp, tb, gcnt, gfill, (int)(total + 1), st);
        cudaMemcpyAsync(gcnt, gfill, sizeof(int) * (total + 1), cudaMemcpyDeviceToDevice, st);  // gcnt := start
        k_grid_fill<<<nb, 256, 0, st>>>(n, cid, gfill, items);
        // neighbour CSR
        k_wse_nbrs<false><<<nbq, 128, 0, st>>>(g, d_pts, gcnt, items, n, R, cnt, nullptr, nullptr, nullptr, nullptr);
        cudaMemsetAsync(cnt + n, 0, sizeof(i64), st);
        tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, ptr, n + 1, st);
        e = need_tmp(tb);
        if (e != cudaSuccess) { release(); return (int)e; }
        tb = tmp_cap;
        cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, ptr, n + 1, st);
        i64 nnz = 0;
        cudaMemcpyAsync(&nnz, ptr + n, sizeof(i64), cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { release(); return (int)e; }
        dev_free(adj);
        dev_free(adjw);
        adj = nullptr;
        adjw = nullptr;
        e = dev_malloc((void**)&adj, sizeof(i32) * std::max<i64>(nnz, 1));
        if (e == cudaSuccess) e = dev_malloc((void**)&adjw, sizeof(i64) * std::max<i64>(nnz, 1));
        if (e != cudaSuccess) { release(); return (int)e; }
        k_wse_nbrs<true><<<nbq, 128, 0, st>>>(g, d_pts, gcnt, items, n, R, nullptr, ptr, adj, adjw, weight);
        // rounds of local maxima until a round pops nothing (one cooperative launch)
        cudaMemsetAsync(dead, 0, sizeof(int) * n, st);
        cudaMemsetAsync(stamp, 0xff, sizeof(int) * n, st);  // -1
        cudaMemsetAsync(popw, 0, sizeof(unsigned long long) * n, st);
        cudaMemsetAsync(npop, 0, sizeof(unsigned long long) * 5, st);
        k_wse_cand0<<<nb, 256, 0, st>>>(n, weight, candA, npop);
        {
            WseRounds wr{n, ptr, adj, adjw, weight, dead, stamp, popw, {candA, candB}, pops, npop};
            int dev = 0, per_sm = 0, nsm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_wse_rounds, 256, 0);
            const i64 want = (n + 255) / 256;
            const unsigned grid = (unsigned)std::max<i64>(1, std::min<i64>(want, (i64)std::max(per_sm, 1) * nsm));
            void* args[] = {&wr};
            e = cudaLaunchCooperativeKernel((const void*)k_wse_rounds, grid, 256, args, 0, st);
            if (e != cudaSuccess) { release(); return (int)e; }
        }
        unsigned long long popped = 0;
        cudaMemcpyAsync(&popped, npop + 4, sizeof(popped), cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { release(); return (int)e; }
        if ((i64)popped < ne) continue;  // degenerate: R too small for this cloud (O8)
        // the ne highest pop priorities (weight desc, index asc; unpopped points have key 0)
        k_iota_i32<<<nb, 256, 0, st>>>(n, ord_in);
        tb = 0;
        cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, popw, popw_out, ord_in, ord_out, (int)n, 0, 64, st);
        e = need_tmp(tb);
        if (e != cudaSuccess) { release(); return (int)e; }
        tb = tmp_cap;
        cub::DeviceRadixSort::SortPairsDescending(tmp, tb, popw, popw_out, ord_in, ord_out, (int)n, 0, 64, st);
        cudaMemsetAsync(elim, 0, n, st);
        k_wse_mark<<<nb, 256, 0, st>>>(ne, ord_out, elim);
        std::vector<uint8_t> h_elim(n);
        cudaMemcpyAsync(h_elim.data(), elim, n, cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { release(); return (int)e; }
        keep.reserve(nt);
        for (i64 i = 0; i < n; ++i)
            if (!h_elim[i]) keep.push_back(i);
        done = true;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    release();
    if (e == cudaSuccess && !done) {  // 16 degenerate passes: the host loop's outcome (keep empty)
        keep.clear();
    }
    return (int)e;
}

// ---------------------------------------------------------------------------------------
// Iterated-greedy colouring passes on the device (O11; host_setup.cpp greedy_colouring):
// each pass visits the previous colour classes by descending colour and gives every vertex
// the smallest colour unused by its neighbours already coloured in this pass.  A class is an
// independent set of sym(pattern), so its vertices are coloured by one launch with the
// sequential visit's result.  Classes: stable 8-bit radix sort of (ncol - 1 - colour) with
// the vertex indices (ascending within a class).  Plain cudaMalloc on a private stream: this
// runs on the setup's background colouring threads.
// ---------------------------------------------------------------------------------------
__global__ void k_ig_keys(i64 n, const i32* __restrict__ colour, int ncol, uint8_t* __restrict__ key,
                          i32* __restrict__ idx, int* __restrict__ cnt) {
    for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        key[i] = (uint8_t)(ncol - 1 - colour[i]);
        idx[i] = (i32)i;
        atomicAdd(&cnt[colour[i]], 1);
    }
}

__global__ void k_ig_class(i64 len, const i32* __restrict__ ord, const i64* __restrict__ np,
                           const i32* __restrict__ nb, i32* colour, int* __restrict__ maxc) {
    int m = 0;
    for (i64 q = blockIdx.x * (i64)blockDim.x + threadIdx.x; q < len; q += (i64)gridDim.x * blockDim.x) {
        const i32 i = ord[q];
        uint64_t used[4] = {0, 0, 0, 0};
        for (i64 t = np[i]; t < np[i + 1]; ++t) {
            const int c = colour[nb[t]];
            if (c >= 0) used[c >> 6] |= 1ull << (c & 63);
        }
        int c = 0;
        for (int w = 0; w < 4; ++w)
            if (~used[w]) {
                c = 64 * w + __ffsll((long long)~used[w]) - 1;
                break;
            }
        colour[i] = c;
        m = max(m, c + 1);
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxc, m);
}

int ig_passes_device(i64 n, const i64* h_np, const i32* h_nb, i32* h_colour, int ncol, int passes, int device) {
    if (ncol < 1 || ncol > 255 || n >= ((i64)1 << 31)) return -(int)cudaErrorInvalidValue;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return -(int)e;
    cudaStream_t st = nullptr;
    e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return -(int)e;
    const i64 nnz = h_np[n];
    i64* np = nullptr;
    i32 *nb = nullptr, *cp = nullptr, *cn = nullptr, *idx = nullptr, *ord = nullptr;
    uint8_t *key = nullptr, *key2 = nullptr;
    int* cnt = nullptr;  // [256] class sizes, [256] max colour
    void* tmp = nullptr;
    size_t tb = 0;
    auto release = [&] {
        cudaFree(np); cudaFree(nb); cudaFree(cp); cudaFree(cn); cudaFree(idx); cudaFree(ord);
        cudaFree(key); cudaFree(key2); cudaFree(cnt); cudaFree(tmp);
        cudaStreamDestroy(st);
    };
    e = cudaMalloc(&np, sizeof(i64) * (n + 1));
    if (e == cudaSuccess) e = cudaMalloc(&nb, sizeof(i32) * std::max<i64>(nnz, 1));
    if (e == cudaSuccess) e = cudaMalloc(&cp, sizeof(i32) * n);
    if (e == cudaSuccess) e = cudaMalloc(&cn, sizeof(i32) * n);
    if (e == cudaSuccess) e = cudaMalloc(&idx, sizeof(i32) * n);
    if (e == cudaSuccess) e = cudaMalloc(&ord, sizeof(i32) * n);
    if (e == cudaSuccess) e = cudaMalloc(&key, n);
    if (e == cudaSuccess) e = cudaMalloc(&key2, n);
    if (e == cudaSuccess) e = cudaMalloc(&cnt, sizeof(int) * 257);
    if (e == cudaSuccess) cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, idx, ord, (int)n, 0, 8, st);
    if (e == cudaSuccess) e = cudaMalloc(&tmp, std::max<size_t>(tb, 16));
    if (e != cudaSuccess) { release(); return -(int)e; }
    cudaMemcpyAsync(np, h_np, sizeof(i64) * (n + 1), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(nb, h_nb, sizeof(i32) * nnz, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(cp, h_colour, sizeof(i32) * n, cudaMemcpyHostToDevice, st);
    const unsigned nb1 = (unsigned)std::min<i64>((n + 255) / 256, 148 * 16);
    std::vector<int> h_cnt(257);
    for (int pass = 1; pass <= passes; ++pass) {
        cudaMemsetAsync(cnt, 0, sizeof(int) * 257, st);
        k_ig_keys<<<nb1, 256, 0, st>>>(n, cp, ncol, key, idx, cnt);
        size_t t2 = tb;
        cub::DeviceRadixSort::SortPairs(tmp, t2, key, key2, idx, ord, (int)n, 0, 8, st);
        cudaMemcpyAsync(h_cnt.data(), cnt, sizeof(int) * ncol, cudaMemcpyDeviceToHost, st);
        cudaMemsetAsync(cn, 0xff, sizeof(i32) * n, st);  // -1: not yet coloured in this pass
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { release(); return -(int)e; }
        i64 off = 0;
        for (int k = 0; k < ncol; ++k) {  // class k = previous colour ncol - 1 - k
            const i64 len = h_cnt[ncol - 1 - k];
            if (len > 0) {
                const unsigned g = (unsigned)std::min<i64>((len + 127) / 128, 148 * 16);
                k_ig_class<<<g, 128, 0, st>>>(len, ord + off, np, nb, cn, cnt + 256);
            }
            off += len;
        }
        int nc = 0;
        cudaMemcpyAsync(&nc, cnt + 256, sizeof(int), cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) { release(); return -(int)e; }
        std::swap(cp, cn);
        ncol = nc;
    }
    e = cudaMemcpyAsync(h_colour, cp, sizeof(i32) * n, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    release();
    return e == cudaSuccess ? ncol : -(int)e;
}

int spgemm_device(const DevCSR& A, const DevCSR& B, DevCSR& C, void* stream, std::string& err) {
    cudaStream_t st = (cudaStream_t)stream;
    C = DevCSR();
    C.nrows = A.nrows;
    C.ncols = B.ncols;
    i64 n = A.nrows;
    i64* d_cnt = nullptr;
    unsigned char* d_skip = nullptr;
    cudaError_t e = dev_malloc((void**)&d_cnt, sizeof(i64) * (n + 1));
    if (e == cudaSuccess) e = dev_malloc((void**)&d_skip, std::max<i64>(1, n));
    if (e != cudaSuccess) { err = "cudaMalloc"; return (int)e; }
    k_row_products<<<(unsigned)std::min<i64>((n + 255) / 256, 148 * 16), 256, 0, st>>>(A.ptr, A.col, B.ptr, n, d_cnt);
    std::vector<i64> cnt(n), aptr(n + 1);
    cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(i64) * n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(aptr.data(), A.ptr, sizeof(i64) * (n + 1), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    // shared-memory row buffer: the largest power of two <= 8192 covering the typical rows;
    // longer rows (and rows with > 1024 A entries) go to spgemm_long_rows
    i64 cap = 8192;
    if (const char* e = std::getenv("MGM_SPGEMM_CAP")) cap = std::max<i64>(2, std::atoll(e));  // test hook
    i64 mx = 2;
    std::vector<unsigned char> skip(n, 0);
    std::vector<i64> longs;
    const std::vector<i64> pcnt = cnt;  // products per row
    for (i64 r = 0; r < n; ++r) {
        if (cnt[r] > cap || aptr[r + 1] - aptr[r] > 1024) {
            skip[r] = 1;
            longs.push_back(r);
        } else {
            mx = std::max(mx, cnt[r]);
        }
    }
    cudaMemcpyAsync(d_skip, skip.data(), std::max<i64>(1, n), cudaMemcpyHostToDevice, st);
    int n2 = next_pow2(mx);
    size_t smem = (size_t)n2 * (8 + 8 + 4) + 8;
    cudaFuncSetAttribute(k_spgemm_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_spgemm_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned grid = (unsigned)std::min<i64>(n, 148 * 8);
    int threads = n2 >= 2048 ? 512 : 256;
    k_spgemm_rows<false><<<grid, threads, smem, st>>>(n, A.ptr, A.col, A.val, B.ptr, B.col, B.val, n2, d_cnt,
                                                      nullptr, nullptr, nullptr, d_skip);
    cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(i64) * n, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    LongRows LR;
    {
        std::vector<i64> pc(n);  // products per row (the count pass above overwrote d_cnt for short rows)
        for (size_t q = 0; q < longs.size(); ++q) pc[longs[q]] = pcnt[longs[q]];
        const int rc = spgemm_long_rows(A, B, longs, pc, aptr, LR, st, err);
        if (rc) { dev_free(d_cnt); dev_free(d_skip); return rc; }
        for (i64 q = 0; q < LR.nl; ++q) cnt[longs[q]] = LR.first[q + 1] - LR.first[q];
    }
    std::vector<i64> ptr(n + 1, 0);
    for (i64 r = 0; r < n; ++r) ptr[r + 1] = ptr[r] + cnt[r];
    C.nnz = ptr[n];
    e = dev_malloc((void**)&C.ptr, sizeof(i64) * (n + 1));
    if (e == cudaSuccess) e = dev_malloc((void**)&C.col, sizeof(i32) * std::max<i64>(1, C.nnz));
    if (e == cudaSuccess) e = dev_malloc((void**)&C.val, sizeof(double) * std::max<i64>(1, C.nnz));
    if (e != cudaSuccess) { dev_free(d_cnt); dev_free(d_skip); err = "cudaMalloc (SpGEMM output)"; return (int)e; }
    cudaMemcpyAsync(C.ptr, ptr.data(), sizeof(i64) * (n + 1), cudaMemcpyHostToDevice, st);
    k_spgemm_rows<true><<<grid, threads, smem, st>>>(n, A.ptr, A.col, A.val, B.ptr, B.col, B.val, n2, nullptr,
                                                     C.ptr, C.col, C.val, d_skip);
    for (i64 q = 0; q < LR.nl; ++q) {  // long rows: device-to-device into place
        const i64 o = ptr[longs[q]], c0 = LR.first[q], c1 = LR.first[q + 1];
        cudaMemcpyAsync(C.col + o, LR.ocol + c0, sizeof(i32) * (c1 - c0), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(C.val + o, LR.oval + c0, sizeof(double) * (c1 - c0), cudaMemcpyDeviceToDevice, st);
    }
    e = cudaStreamSynchronize(st);
    if (LR.ocol) dev_free(LR.ocol);
    if (LR.oval) dev_free(LR.oval);
    dev_free(d_cnt);
    dev_free(d_skip);
    if (e != cudaSuccess) { err = "SpGEMM kernel"; return (int)e; }
    return (int)cudaGetLastError();
}

void free_dev_csr(DevCSR& M) {
    if (M.ptr) dev_free(M.ptr);
    if (M.col) dev_free(M.col);
    if (M.val) dev_free(M.val);
    M = DevCSR();
}

int upload_csr(const HostCSR& H, DevCSR& D, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    D.nrows = H.nrows;
    D.ncols = H.ncols;
    D.nnz = H.nnz();
    cudaError_t e = dev_malloc((void**)&D.ptr, sizeof(i64) * (H.nrows + 1));
    if (e == cudaSuccess) e = dev_malloc((void**)&D.col, sizeof(i32) * std::max<i64>(1, D.nnz));
    if (e == cudaSuccess) e = dev_malloc((void**)&D.val, sizeof(double) * std::max<i64>(1, D.nnz));
    if (e != cudaSuccess) return (int)e;
    cudaMemcpyAsync(D.ptr, H.ptr.data(), sizeof(i64) * (H.nrows + 1), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(D.col, H.col.data(), sizeof(i32) * D.nnz, cudaMemcpyHostToDevice, st);
    if (!H.val.empty()) cudaMemcpyAsync(D.val, H.val.data(), sizeof(double) * D.nnz, cudaMemcpyHostToDevice, st);
    return (int)cudaStreamSynchronize(st);
}

int download_csr(const DevCSR& D, HostCSR& H, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    H.nrows = D.nrows;
    H.ncols = D.ncols;
    H.ptr.resize(D.nrows + 1);
    H.col.resize(D.nnz);
    H.val.resize(D.nnz);
    cudaMemcpyAsync(H.ptr.data(), D.ptr, sizeof(i64) * (D.nrows + 1), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(H.col.data(), D.col, sizeof(i32) * D.nnz, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(H.val.data(), D.val, sizeof(double) * D.nnz, cudaMemcpyDeviceToHost, st);
    return (int)cudaStreamSynchronize(st);
}

}  // namespace mgm
