// The bottom of the V-cycle as ONE dense operator.
//
// Alg. 3 enters every level j >= 2 with e_j = 0 (line 6) and touches the levels
// below j only through r_j (line 8 restricts, line 11 interpolates back).  Lines 6-14 for the
// levels J..p-1 are therefore a LINEAR map r_J -> e_J: presmooth from zero, residual,
// restriction, the same recursively, the coarse solve L_p^{-1} (line 10), interpolation +
// correction and postsmoothing back up to J.  Its matrix B_J (n_J x n_J, Poisson: the
// bordered n_J + 1) is built once at setup by applying those lines -- the library's own
// per-level kernels -- to the unit vectors (mgm.cu setup_dense_bottom), so each V-cycle
// replaces ~2 sum_{j>=J} nu C_j dependent colour steps (cfg3: ~230, ~325 us, latency bound)
// by one HBM-bound dense apply e_J = B_J r_J (4096^2 fp64 = 134 MB, ~21 us at 6.5 TB/s).
// Same result up to rounding (the sums run in another order), like the explicit coarse
// inverse of O13.
//
// k_dense_apply<K>: Y[r][k] = sum_i B[r][i] X[i][k] for K interleaved right-hand sides
// (K = 1: the V-cycle; 2/4/8: the multi-RHS V-cycle).  B is row-major with a padded leading
// dimension ld (multiple of 64, zero columns), read once with streaming loads; X is staged
// through shared memory in chunks of 4096/K rows (32 KB); one warp per output row, eight
// rows per CTA.  B does not depend on the predecessor kernel, so with PDL each warp issues
// its first loads of B before griddepcontrol.wait.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "solve_kernels.cuh"

namespace mgm {

constexpr int DENSE_ROWS_PER_CTA = 8;
constexpr int DENSE_THREADS = 32 * DENSE_ROWS_PER_CTA;

__device__ __forceinline__ double2 ld_stream_f64x2(const double* p) {
    double2 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
        : "=d"(v.x), "=d"(v.y)
        : "l"(p), "l"(policy_evict_first()));
    return v;
}

template <int K>
__global__ void __launch_bounds__(DENSE_THREADS) k_dense_apply(int m, int ld, const double* __restrict__ B,
                                                               const double* __restrict__ X, double* __restrict__ Y) {
    constexpr int CR = 4096 / K;  // X rows per staged chunk (32 KB)
    constexpr int U = 8;          // double2 loads in flight per lane
    __shared__ __align__(16) double xs[CR * K];
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * DENSE_ROWS_PER_CTA + warp;
    const bool live = row < m;
    const double* a = B + (int64_t)(live ? row : 0) * ld;
    // prologue: the first U pairs of this lane's slice of the row (independent of X)
    double2 v[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const int c = 2 * (lane + 32 * q);
        v[q] = (live && c < ld && c < CR) ? ld_stream_f64x2(a + c) : make_double2(0.0, 0.0);
    }
    pdl_wait();
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.0;
    for (int c0 = 0; c0 < ld; c0 += CR) {
        const int cn = min(CR, ld - c0);
        if (c0 > 0) __syncthreads();
        for (int t = threadIdx.x; t < cn * K; t += DENSE_THREADS) {
            const int i = c0 + t / K;
            xs[t] = i < m ? X[(int64_t)c0 * K + t] : 0.0;
        }
        __syncthreads();
        if (!live) continue;
        // pairs of this lane: columns c0 + 2*(lane + 32 q), q = 0 .. cn/64 - 1, U at a time
        for (int q0 = 0; q0 < cn / 64; q0 += U) {
            if (c0 > 0 || q0 > 0) {
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int c = 2 * (lane + 32 * (q0 + q));
                    v[q] = (c < cn) ? ld_stream_f64x2(a + c0 + c) : make_double2(0.0, 0.0);
                }
            }
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int c = 2 * (lane + 32 * (q0 + q));
                if (c < cn) {
                    if (K == 1) {
                        const double2 x2 = *reinterpret_cast<const double2*>(xs + c);
                        acc[0] = fma(v[q].x, x2.x, acc[0]);
                        acc[0] = fma(v[q].y, x2.y, acc[0]);
                    } else {  // (K even: the K values of a column are 16-byte pairs in shared memory)
#pragma unroll
                        for (int k2 = 0; k2 < K / 2; ++k2) {
                            const double2 a2 = *reinterpret_cast<const double2*>(xs + c * K + 2 * k2);
                            acc[2 * k2] = fma(v[q].x, a2.x, acc[2 * k2]);
                            acc[2 * k2 + 1] = fma(v[q].x, a2.y, acc[2 * k2 + 1]);
                        }
#pragma unroll
                        for (int k2 = 0; k2 < K / 2; ++k2) {
                            const double2 b2 = *reinterpret_cast<const double2*>(xs + (c + 1) * K + 2 * k2);
                            acc[2 * k2] = fma(v[q].y, b2.x, acc[2 * k2]);
                            acc[2 * k2 + 1] = fma(v[q].y, b2.y, acc[2 * k2 + 1]);
                        }
                    }
                }
            }
        }
    }
    if (!live) return;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) Y[(int64_t)row * K + k] = s;
    }
}

// K > 1 right-hand sides: each warp computes RPW rows, so one shared-memory read of X serves
// RPW rows (the K = 8 apply was bound by re-reading X for every row: 321 us vs 25 us for K = 1)
template <int K, int RPW>
__global__ void __launch_bounds__(DENSE_THREADS) k_dense_apply_multi(int m, int ld, const double* __restrict__ B,
                                                                     const double* __restrict__ X,
                                                                     double* __restrict__ Y) {
    constexpr int CR = 4096 / K;
    __shared__ __align__(16) double xs[CR * K];
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row0 = (blockIdx.x * DENSE_ROWS_PER_CTA + warp) * RPW;
    double acc[RPW][K];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int k = 0; k < K; ++k) acc[r][k] = 0.0;
    pdl_wait();
    for (int c0 = 0; c0 < ld; c0 += CR) {
        const int cn = min(CR, ld - c0);
        if (c0 > 0) __syncthreads();
        for (int t = threadIdx.x; t < cn * K; t += DENSE_THREADS) {
            const int i = c0 + t / K;
            xs[t] = i < m ? X[(int64_t)c0 * K + t] : 0.0;
        }
        __syncthreads();
        for (int c = 2 * lane; c < cn; c += 64) {
            double2 v[RPW];
#pragma unroll
            for (int r = 0; r < RPW; ++r)
                v[r] = (row0 + r < m) ? ld_stream_f64x2(B + (int64_t)(row0 + r) * ld + c0 + c) : make_double2(0.0, 0.0);
#pragma unroll
            for (int k2 = 0; k2 < K / 2; ++k2) {
                const double2 a2 = *reinterpret_cast<const double2*>(xs + c * K + 2 * k2);
                const double2 b2 = *reinterpret_cast<const double2*>(xs + (c + 1) * K + 2 * k2);
#pragma unroll
                for (int r = 0; r < RPW; ++r) {
                    acc[r][2 * k2] = fma(v[r].x, a2.x, acc[r][2 * k2]);
                    acc[r][2 * k2 + 1] = fma(v[r].x, a2.y, acc[r][2 * k2 + 1]);
                    acc[r][2 * k2] = fma(v[r].y, b2.x, acc[r][2 * k2]);
                    acc[r][2 * k2 + 1] = fma(v[r].y, b2.y, acc[r][2 * k2 + 1]);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        if (row0 + r >= m) break;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = acc[r][k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) Y[(int64_t)(row0 + r) * K + k] = s;
        }
    }
}

// Split over the columns (the reduction dimension) for K > 1: CTA (x, y) computes rows
// [32 x, 32 x + 32) over the column slice y of S (width cs, a multiple of 64) and writes the
// partial sums P[y][row][k]; k_dense_sum adds the S partials in order y = 0..S-1
// (deterministic).  Without the split the K = 8 apply ran 128 CTAs with ~16 KB of B in flight
// per SM: latency-bound at ~1.3 TB/s (109 us for 134 MB).
template <int K, int RPW>
__global__ void __launch_bounds__(DENSE_THREADS) k_dense_apply_split(int m, int ld, int cs,
                                                                     const double* __restrict__ B,
                                                                     const double* __restrict__ X,
                                                                     double* __restrict__ P) {
    constexpr int CR = 4096 / K;
    __shared__ __align__(16) double xs[CR * K];
    pdl_trigger();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row0 = (blockIdx.x * DENSE_ROWS_PER_CTA + warp) * RPW;
    const int cb = blockIdx.y * cs, ce = min(ld, cb + cs);
    double acc[RPW][K];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int k = 0; k < K; ++k) acc[r][k] = 0.0;
    pdl_wait();
    for (int c0 = cb; c0 < ce; c0 += CR) {
        const int cn = min(CR, ce - c0);
        if (c0 > cb) __syncthreads();
        for (int t = threadIdx.x; t < cn * K; t += DENSE_THREADS) {
            const int i = c0 + t / K;
            xs[t] = i < m ? X[(int64_t)c0 * K + t] : 0.0;
        }
        __syncthreads();
        for (int c = 2 * lane; c < cn; c += 64) {
            double2 v[RPW];
#pragma unroll
            for (int r = 0; r < RPW; ++r)
                v[r] = (row0 + r < m) ? ld_stream_f64x2(B + (int64_t)(row0 + r) * ld + c0 + c) : make_double2(0.0, 0.0);
#pragma unroll
            for (int k2 = 0; k2 < K / 2; ++k2) {
                const double2 a2 = *reinterpret_cast<const double2*>(xs + c * K + 2 * k2);
                const double2 b2 = *reinterpret_cast<const double2*>(xs + (c + 1) * K + 2 * k2);
#pragma unroll
                for (int r = 0; r < RPW; ++r) {
                    acc[r][2 * k2] = fma(v[r].x, a2.x, acc[r][2 * k2]);
                    acc[r][2 * k2 + 1] = fma(v[r].x, a2.y, acc[r][2 * k2 + 1]);
                    acc[r][2 * k2] = fma(v[r].y, b2.x, acc[r][2 * k2]);
                    acc[r][2 * k2 + 1] = fma(v[r].y, b2.y, acc[r][2 * k2 + 1]);
                }
            }
        }
    }
    double* Pq = P + (int64_t)blockIdx.y * m * K;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        if (row0 + r >= m) break;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = acc[r][k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) Pq[(int64_t)(row0 + r) * K + k] = s;
        }
    }
}
// Y[t] = sum_{y < S} P[y][t], t < m K (fixed order)
__global__ void k_dense_sum(int64_t mk, int S, const double* __restrict__ P, double* __restrict__ Y) {
    pdl_trigger();
    pdl_wait();
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < mk; t += (int64_t)gridDim.x * blockDim.x) {
        double s = P[t];
        for (int y = 1; y < S; ++y) s += P[(int64_t)y * mk + t];
        Y[t] = s;
    }
}

// e_J (n rows) <- unit vector e_i (setup of B_J, one column per replay)
__global__ void k_unit(int n, int i, double* __restrict__ f) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) f[r] = r == i ? 1.0 : 0.0;
}

// B[r][c] = T[c][r] for r, c < m (T column-major results of the unit replays, leading dim m);
// B has leading dimension ld with zero padding columns m..ld-1
__global__ void k_transpose_pad(int m, int ld, const double* __restrict__ T, double* __restrict__ B) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int c = by + yy, r = bx + threadIdx.x;
        tile[yy][threadIdx.x] = (c < m && r < m) ? T[(int64_t)c * m + r] : 0.0;
    }
    __syncthreads();
    for (int yy = threadIdx.y; yy < 32; yy += blockDim.y) {
        const int r = bx + yy, c = by + threadIdx.x;
        if (r < m && c < ld) B[(int64_t)r * ld + c] = tile[threadIdx.x][yy];
    }
}

}  // namespace mgm
