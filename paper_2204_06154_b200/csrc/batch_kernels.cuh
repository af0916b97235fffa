// Multi-right-hand-side (batched) solve kernels: one pass over an
// operator serves K right-hand sides.  Batched vectors are interleaved, row-major [row][K]
// in lib order, so the K values a gather needs are contiguous (one 32-byte sector for K = 4).
// The arithmetic per (row, right-hand side) is exactly that of the single-RHS kernels
// (same threads-per-row split, same summation order), so a batched V-cycle reproduces K
// single V-cycles.  Shifted problems only.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "solve_kernels.cuh"

namespace mgm {

// ---- Colour sweep / SpMV / interpolation for K right-hand sides (K even), split over the
// right-hand sides: KS = K/2 threads per (row, slot part), each owning the pair of
// right-hand sides (2 kk, 2 kk + 1).  A gather of column j by the KS threads of a row
// reads the K contiguous values of u[j][*] as ONE coalesced 16 * KS-byte segment (instead of
// K/2 16-byte loads by one thread, each warp load touching 32 scattered lines); the operator
// entry (same address for the KS threads) is one broadcast load.  Per (row, right-hand side)
// the slots are summed exactly as the single-RHS kernels sum them with TPR threads per row
// (TPR slot parts, then the group sum over the parts).  One thread gathering all K values of
// a column (round 1) measured 3.88 ms per K = 8 V-cycle at cfg3 against 3.06 split.
template <int TPR, int KS>
__device__ __forceinline__ double part_sum(double v) {
#pragma unroll
    for (int o = (TPR * KS) >> 1; o >= KS; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <int TPR, int CH, int K, bool ZG = false>
__global__ void __launch_bounds__(256) k_gs_colour_bs(int r0, int r1, int Wu, const int64_t* __restrict__ sptr,
                                                      const int* __restrict__ scol, const double* __restrict__ sval,
                                                      const double* __restrict__ f, double* u,
                                                      const int* __restrict__ slw, const uint8_t* __restrict__ nlow,
                                                      double* __restrict__ dlt) {
    constexpr int KS = K / 2;
    pdl_trigger();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = (r0 & ~31) + g / (TPR * KS);
    const int kk = g % KS, part = (g / KS) % TPR;
    const bool live = (r >= r0 && r < r1);
    RowFrag<TPR, CH> fr;
    int w = 0;
    int64_t base = 0;
    double d = 1.0;
    if (live) {
        if (Wu > 0) {
            w = Wu;
            base = (int64_t)(r >> 5) * 32 * Wu + (r & 31);
        } else {
            const int64_t s0 = sptr[r >> 5];
            w = (int)((sptr[(r >> 5) + 1] - s0) >> 5);
            base = s0 + (r & 31);
        }
        int lim = 0;
        if (ZG) {
            w = slw[r >> 5];
            lim = 1 + (int)nlow[r];
        }
        fr.load(sval + base, scol + base, ZG ? lim : w, part);
        if (ZG) {
#pragma unroll
            for (int q = 0; q < CH; ++q)
                if (part + q * TPR == 0 || part + q * TPR >= lim) fr.c[q] = -1;
            w = lim;
        }
        d = ld_stream_f64(sval + base);
    } else {
        fr.load(sval, scol, 0, 0);
    }
    pdl_wait();
    const double2* u2 = reinterpret_cast<const double2*>(u);
    double2 fv = make_double2(0.0, 0.0), uv = make_double2(0.0, 0.0);
    double a0 = 0.0, a1 = 0.0;
    if (live && part == 0) {
        fv = reinterpret_cast<const double2*>(f)[(int64_t)r * KS + kk];
        if (!ZG) uv = u2[(int64_t)r * KS + kk];
    }
    for (int k0 = part;; k0 += TPR * CH) {
        if (k0 != part) fr.load(sval + base, scol + base, w, k0);
#pragma unroll
        for (int q = 0; q < CH; ++q)
            if (fr.c[q] >= 0) {
                const double2 v = u2[(int64_t)fr.c[q] * KS + kk];
                a0 = fma(fr.a[q], v.x, a0);
                a1 = fma(fr.a[q], v.y, a1);
            }
        if (k0 + TPR * CH >= w) break;
    }
    a0 = part_sum<TPR, KS>(a0);
    a1 = part_sum<TPR, KS>(a1);
    if (live && part == 0)
    {
        const double d0 = (fv.x - a0) / d, d1 = (fv.y - a1) / d;
        reinterpret_cast<double2*>(u)[(int64_t)r * KS + kk] = make_double2(uv.x + d0, uv.y + d1);
        if (dlt) reinterpret_cast<double2*>(dlt)[(int64_t)r * KS + kk] = make_double2(d0, d1);  // increments (MODE 3)
    }
}
// MODE 0: y = A x; MODE 1: y = f - A x; MODE 3: y = f + (later-colour part of A) x (A u after
// a forward sweep that added x to u); MODE 2: y = -(later-colour part of A) x, the residual
// right after a forward sweep from a zero guess (k_sell_spmv MODE 2: from the slice's first
// later-colour slot sluw, masked below the row's own 1 + nlow).  yperm: output row of each
// input row (the residual written in Morton order for the restriction's Morton columns).
template <int MODE, int TPR, int CH, int K>
__global__ void __launch_bounds__(256) k_sell_spmv_bs(int r0, int r1, const int64_t* __restrict__ sptr,
                                                      const int* __restrict__ scol, const double* __restrict__ sval,
                                                      const double* __restrict__ x, const double* __restrict__ f,
                                                      double* __restrict__ y, const int* __restrict__ sluw,
                                                      const uint8_t* __restrict__ nlow, const int* __restrict__ yperm) {
    constexpr int KS = K / 2;
    pdl_trigger();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = (r0 & ~31) + g / (TPR * KS);
    const int kk = g % KS, part = (g / KS) % TPR;
    const bool live = r >= r0 && r < r1;
    RowFrag<TPR, CH> fr;
    int w = 0, k1 = part, lim = 0, yr = r;
    int64_t base = 0;
    if (live) {
        if (yperm) yr = yperm[r];
        const int64_t s0 = sptr[r >> 5];
        w = (int)((sptr[(r >> 5) + 1] - s0) >> 5);
        base = s0 + (r & 31);
        if (MODE >= 2) {
            k1 = sluw[r >> 5] + part;
            lim = 1 + (int)nlow[r];
        }
        fr.load(sval + base, scol + base, w, k1);
    } else {
        fr.load(sval, scol, 0, 0);
    }
    if (MODE >= 2) {
#pragma unroll
        for (int q = 0; q < CH; ++q)
            if (k1 + q * TPR < lim) fr.c[q] = -1;
    }
    pdl_wait();
    const double2* x2 = reinterpret_cast<const double2*>(x);
    double a0 = 0.0, a1 = 0.0;
    for (int k0 = k1;; k0 += TPR * CH) {
        if (k0 != k1) {
            fr.load(sval + base, scol + base, w, k0);
            if (MODE >= 2) {
#pragma unroll
                for (int q = 0; q < CH; ++q)
                    if (k0 + q * TPR < lim) fr.c[q] = -1;
            }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q)
            if (fr.c[q] >= 0) {
                const double2 v = x2[(int64_t)fr.c[q] * KS + kk];
                a0 = fma(fr.a[q], v.x, a0);
                a1 = fma(fr.a[q], v.y, a1);
            }
        if (k0 + TPR * CH >= w) break;
    }
    a0 = part_sum<TPR, KS>(a0);
    a1 = part_sum<TPR, KS>(a1);
    if (live && part == 0) {
        double2 o = make_double2(a0, a1);
        if (MODE == 1) {
            const double2 fv = reinterpret_cast<const double2*>(f)[(int64_t)r * KS + kk];
            o = make_double2(fv.x - a0, fv.y - a1);
        } else if (MODE == 2) {
            o = make_double2(-a0, -a1);
        } else if (MODE == 3) {  // A u after a forward sweep that added x to u (k_sell_spmv MODE 3)
            const double2 fv = reinterpret_cast<const double2*>(f)[(int64_t)r * KS + kk];
            o = make_double2(fv.x + a0, fv.y + a1);
        }
        reinterpret_cast<double2*>(y)[(int64_t)yr * KS + kk] = o;
    }
}
template <int M, int K>
__global__ void __launch_bounds__(256) k_interp_correct_bs(int n, int m, const int* __restrict__ pcol,
                                                           const double* __restrict__ pval,
                                                           const double* __restrict__ ec, double* __restrict__ e) {
    constexpr int KS = K / 2;
    pdl_trigger();
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = g / KS, kk = g % KS;
    int cidx[M];
    double a[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
        const bool ok = r < n && q < m;
        cidx[q] = ok ? ld_stream_i32(pcol + (int64_t)q * n + r) : -1;
        a[q] = ok ? ld_stream_f64(pval + (int64_t)q * n + r) : 0.0;
    }
    pdl_wait();
    if (r >= n) return;
    const double2* ec2 = reinterpret_cast<const double2*>(ec);
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int q = 0; q < M; ++q)
        if (cidx[q] >= 0) {
            const double2 v = ec2[(int64_t)cidx[q] * KS + kk];
            a0 = fma(a[q], v.x, a0);
            a1 = fma(a[q], v.y, a1);
        }
    double2* e2 = reinterpret_cast<double2*>(e);
    double2 o = e2[(int64_t)r * KS + kk];
    o.x += a0;
    o.y += a1;
    e2[(int64_t)r * KS + kk] = o;
}

// coarsest level: y = A^{-1} x for K right-hand sides with the explicit inverse (row-major)
template <int K>
__global__ void k_dense_mv_b(int m, const double* __restrict__ Ainv, const double* __restrict__ x,
                             double* __restrict__ y) {
    pdl_trigger();
    pdl_wait();
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m * K; t += gridDim.x * blockDim.x) {
        const int i = t / K, k = t % K;
        double acc = 0.0;
        for (int j = 0; j < m; ++j) acc = fma(Ainv[(int64_t)i * m + j], x[(int64_t)j * K + k], acc);
        y[t] = acc;
    }
}

// column-major user vectors (K x N, original order) <-> interleaved lib order of width KK >= K
// (columns K..KK-1 of the interleaved layout are zero)
__global__ void k_gather_b(int n, int K, int KK, const int* __restrict__ idx, const double* __restrict__ in,
                           double* __restrict__ out) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * KK;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / KK, k = t % KK;
        out[t] = k < K ? in[k * n + idx[r]] : 0.0;
    }
}
__global__ void k_scatter_b(int n, int K, int KK, const int* __restrict__ idx, const double* __restrict__ in,
                            double* __restrict__ out) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)n * KK;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / KK, k = t % KK;
        if (k < K) out[k * n + idx[r]] = in[t];
    }
}

// y[r][k] = (acc ? y[r][k] : 0) + sgn * sum_{j < nv} c[j*K + k] V_j[r][k]   (V_j = V + j*stride)
template <int K>
__global__ void k_blincomb(int64_t n, int nv, const double* __restrict__ V, int64_t stride,
                           const double* __restrict__ c, double sgn, int acc, double* y) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(t % K);
        double s = acc ? y[t] : 0.0;
        for (int j = 0; j < nv; ++j) s = fma(sgn * c[j * K + k], V[j * stride + t], s);
        y[t] = s;
    }
}
// y[r][k] = x[r][k] * c[k]
template <int K>
__global__ void k_bscale(int64_t n, const double* __restrict__ x, const double* __restrict__ c, double* __restrict__ y) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * K; t += (int64_t)gridDim.x * blockDim.x)
        y[t] = x[t] * c[t % K];
}

// out[k] = sum_r a[r*K+k] b[r*K+k], deterministic (block partials in fixed order, last-block finish)
template <int K>
__global__ void __launch_bounds__(RED_THREADS) k_bdot_fin(int64_t n, const double* __restrict__ a,
                                                          const double* __restrict__ b, double* __restrict__ partials,
                                                          unsigned* ticket, double* out) {
    __shared__ double red[RED_THREADS / 32][K];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x)
#pragma unroll
        for (int k = 0; k < K; ++k) s[k] = fma(a[i * K + k], b[i * K + k], s[k]);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double t = warp_sum(s[k]);
        if (lane == 0) red[warp][k] = t;
    }
    __syncthreads();
    if (threadIdx.x < K) {
        double t = 0.0;
        for (int ww = 0; ww < RED_THREADS / 32; ++ww) t += red[ww][threadIdx.x];
        partials[(int64_t)blockIdx.x * K + threadIdx.x] = t;
    }
    finish_partials(partials, K, ticket, out, nullptr);
}

// out[j K + k] = sum_r V_j[r][k] w[r][k] for j < k1 (V_j = V + j stride): every basis vector of
// a batched CGS2 pass in ONE launch (w read once per group of G vectors instead of once per
// vector).  Same block chunks, per-thread order, warp / block / last-block sums as
// k_bdot_fin<K> on (V_j, w), so each output is bitwise that kernel's.  partials holds
// gridDim.x * k1 * K doubles.
template <int K, int G>
__global__ void __launch_bounds__(RED_THREADS) k_bmultidot_fin(int64_t n, const double* __restrict__ V, int64_t stride,
                                                               int k1, const double* __restrict__ w,
                                                               double* __restrict__ partials, unsigned* ticket,
                                                               double* out) {
    __shared__ double red[RED_THREADS / 32][G * K];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nout = k1 * K;
    for (int g = 0; g < k1; g += G) {
        const int gn = min(G, k1 - g);
        double s[G][K];
#pragma unroll
        for (int q = 0; q < G; ++q)
#pragma unroll
            for (int k = 0; k < K; ++k) s[q][k] = 0.0;
        for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
            double wr[K];
#pragma unroll
            for (int k = 0; k < K; ++k) wr[k] = w[i * K + k];
#pragma unroll
            for (int q = 0; q < G; ++q)
                if (q < gn) {
                    const double* a = V + (int64_t)(g + q) * stride + i * K;
#pragma unroll
                    for (int k = 0; k < K; ++k) s[q][k] = fma(a[k], wr[k], s[q][k]);
                }
        }
#pragma unroll
        for (int q = 0; q < G; ++q)
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const double t = warp_sum(s[q][k]);
                if (lane == 0) red[warp][q * K + k] = t;
            }
        __syncthreads();
        if (threadIdx.x < gn * K) {
            double t = 0.0;
            for (int ww = 0; ww < RED_THREADS / 32; ++ww) t += red[ww][threadIdx.x];
            partials[(int64_t)blockIdx.x * nout + g * K + threadIdx.x] = t;
        }
        __syncthreads();
    }
    finish_partials(partials, nout, ticket, out, nullptr);
}

}  // namespace mgm
