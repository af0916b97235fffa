// Solve-phase kernels of libmgm (sm_100a, fp64).  All are HBM/latency bound sparse
// gathers: no tensor cores.  Data layout:
//   * L_j, R_j: SELL-32 -- rows in lib order (colour-major, Morton within a colour), slices
//     of 32 consecutive rows stored slot-major (entry k of row r at sptr[r/32] + 32k + r%32),
//     diagonal in slot 0 for L_j, padding = (own row, 0.0).
//   * P_j: ELL, width m, slot-major [m][n_j].
//   * vectors: fp64, lib order; Poisson mode appends the multiplier lambda at index n_j.
//
// Programmatic dependent launch (PDL): inside the V-cycle graph every kernel is launched with
// programmatic stream serialisation.  Each kernel first calls pdl_trigger() so its successor
// can be scheduled, loads the immutable operator data it needs (prologue), then pdl_wait()s
// for its predecessor before reading any vector or writing anything.  Launched without the
// attribute, both instructions are no-ops.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace mgm {

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// L2 prefetch pacing ("L2 prefetch pacing").  Inside the V-cycle graph a
// kernel is handed the operator regions (matrix values, columns, right-hand side block) of
// the NEXT kernel(s) of the schedule; at start every CTA issues bulk L2 prefetches for its
// share of those bytes.  Operator data is immutable during the solve, so the prefetch needs
// no ordering: the HBM streams colour c+1's matrix block while colour c gathers and
// updates out of L2, instead of each small colour kernel paying its own HBM ramp.
// Regions are 16-byte aligned with sizes that are multiples of 16 (the host rounds).
struct PfRegion {
    const char* p;
    int64_t bytes;
};
struct PfList {
    const PfRegion* r;  // device table
    int n;
    int late;  // 1: issue after the kernel's own prologue loads (experiment, MGM_PF_LATE)
};
__device__ __forceinline__ void l2_prefetch_share(const PfList& pf) {
    if (pf.n <= 0 || threadIdx.x != 0) return;
    const int64_t G = gridDim.x, b = blockIdx.x;
    for (int i = 0; i < pf.n; ++i) {
        const PfRegion R = pf.r[i];
        const int64_t lo = (R.bytes * b / G) & ~(int64_t)127;
        const int64_t hi = (b + 1 == G) ? R.bytes : ((R.bytes * (b + 1) / G) & ~(int64_t)127);
        for (int64_t o = lo; o < hi; o += 32768) {
            const int64_t len = hi - o < 32768 ? hi - o : 32768;
            const uint32_t sz = (uint32_t)((len + 15) & ~(int64_t)15);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(R.p + o), "r"(sz) : "memory");
        }
    }
}

// Streaming loads for matrix data (read once per sweep): non-coherent path, no L1
// allocation, L2 evict_first so that the streamed upper levels do not evict the small
// bottom levels (bottom_kernel.cuh loads those with evict_last).  Not volatile, so the
// compiler may batch them ahead of the gathers.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_stream_f64(const double* p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy_evict_first()));
    return v;
}
__device__ __forceinline__ int ld_stream_i32(const int* p) {
    int v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_first()));
    return v;
}

// A chunk of one SELL-32 row held in registers: slots k0, k0+TPR, ..., k0+(CH-1)*TPR.
template <int TPR, int CH>
struct RowFrag {
    int c[CH];
    double a[CH];
    __device__ __forceinline__ void load(const double* __restrict__ v, const int* __restrict__ cc, int w, int k0) {
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int k = k0 + q * TPR;
            c[q] = (k < w) ? ld_stream_i32(cc + 32 * k) : -1;
            a[q] = (k < w) ? ld_stream_f64(v + 32 * k) : 0.0;
        }
    }
    __device__ __forceinline__ double dot(const double* x, double acc) const {
#pragma unroll
        for (int q = 0; q < CH; ++q)
            if (c[q] >= 0) acc = fma(a[q], x[c[q]], acc);
        return acc;
    }
    // the same with L2-coherent gathers (ld.global.cg; values written earlier in this kernel)
    __device__ __forceinline__ double dot_cg(const double* x, double acc) const {
#pragma unroll
        for (int q = 0; q < CH; ++q)
            if (c[q] >= 0) acc = fma(a[q], __ldcg(x + c[q]), acc);
        return acc;
    }
};

template <int TPR>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = TPR >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One colour of a Gauss-Seidel sweep (Poisson variant P:348-352):
//   u_i += (f_i - sum_j a_ij u_j [- c_i lambda]) / a_ii  over rows [r0, r1) of one colour.
// TPR threads per row; threads aligned to 32-row slices.
// ZG (first forward sweep from a zero guess, shifted problems): the later-colour values are
// still 0, so only the first slw[slice] slots of each row (diagonal + earlier-colour
// columns, pack_sell's order) are read and u_i (= 0) is not: u_i = (f_i - sum_lower) / a_ii,
// with the row's own earlier-colour count nlow[r] masking the slots a longer row of the same
// slice needs (they hold this row's later-colour entries).  Skipping the zero products
// leaves the remaining terms' order unchanged.
template <bool POISSON, int TPR, int CH, bool ZG = false>
__global__ void __launch_bounds__(256) k_gs_colour(int r0, int r1, int Wu, const int64_t* __restrict__ sptr,
                                                   const int* __restrict__ scol,
                                                   const double* __restrict__ sval,
                                                   const double* __restrict__ f, double* u,
                                                   const double* __restrict__ c, int n, PfList pf,
                                                   const int* __restrict__ slw, const uint8_t* __restrict__ nlow,
                                                   double* __restrict__ dlt) {
    pdl_trigger();
    if (!pf.late) l2_prefetch_share(pf);
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = (r0 & ~31) + g / TPR;
    const int part = g % TPR;
    const bool live = (r >= r0 && r < r1);
    RowFrag<TPR, CH> fr;
    int w = 0;
    int64_t base = 0;
    double d = 1.0;
    if (live) {
        if (Wu > 0) {  // every slice has width Wu (level 0): the slice offset needs no load
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
        // ZG: only this row's own diagonal + earlier-colour slots are fetched (the slice's
        // wider rows' later slots would be masked anyway; in situ the ZG kernels read 1.6x
        // their algorithmic bytes when the whole slice width was fetched)
        fr.load(sval + base, scol + base, ZG ? lim : w, part);
        if (ZG) {
#pragma unroll
            for (int q = 0; q < CH; ++q)  // the diagonal (u_i not yet written, term 0) and later colours
                if (part + q * TPR == 0 || part + q * TPR >= lim) fr.c[q] = -1;
            w = lim;  // (the tail loop below)
        }
        d = ld_stream_f64(sval + base);
    } else {
        fr.load(sval, scol, 0, 0);
    }
    if (pf.late) l2_prefetch_share(pf);
    pdl_wait();
    // epilogue operands issued together with the gathers (one memory round trip)
    double fr_v = 0.0, ur = 0.0, cl = 0.0;
    if (live && part == 0) {
        fr_v = f[r];
        if (!ZG) ur = u[r];
        if (POISSON) cl = c[r] * u[n];
    }
    double acc = fr.dot(u, 0.0);
    for (int k0 = part + TPR * CH; k0 < w; k0 += TPR * CH) {
        fr.load(sval + base, scol + base, w, k0);
        acc = fr.dot(u, acc);
    }
    acc = group_sum<TPR>(acc);
    if (live && part == 0) {
        double res = fr_v - acc;
        if (POISSON) res -= cl;
        const double dl = res / d;
        u[r] = ur + dl;
        if (dlt) dlt[r] = dl;  // the sweep's increment (the residual identity of k_sell_spmv MODE 3)
    }
}

// y = L x  (MODE 0),  y = f - L x  (MODE 1) on the rows [r0, r1).
// MODE 2: the residual right after a forward Gauss-Seidel sweep from a ZERO guess,
// y = f - L u = -sum_{later colours} a_ij u_j: the sweep made every row's residual zero when
// it updated the row (f_i = a_ii u_i + sum_{earlier colours} a_ij u_j), and only the later
// colours changed since.  Reads the later-colour slots of pack_sell's [diag | earlier |
// later] rows (from sluw[slice] = 1 + the slice's smallest earlier count, masked below
// 1 + nlow[r]); equal to f - L u up to rounding.  Poisson: border term
// c_i * x[nl] (nl = the level's row count; the multiplier sits after the rows).
// MODE 3: A u right after a forward Gauss-Seidel sweep that added the increments d = x to u:
// the sweep left every row's residual zero when it updated the row (with the earlier colours'
// new and the later colours' old values), so (A u)_i = f_i + sum_{later colours} a_ij d_j --
// the later-colour slots only, as MODE 2 (equal to A u up to rounding).
// Restriction fused with colour 0 of the next level's presmooth from zero (MODE 0): for the
// coarse rows r < c0_end (lib order: colour 0 first) also u[r] = f[r] / a_rr -- exactly what
// the zero-guess colour kernel computes for colour 0 (no earlier colours to gather).
struct C0Fuse {
    double* u;
    const int64_t* sptr;
    const double* sval;
    int c0_end;
};

template <int MODE, bool POISSON, int TPR, int CH>
__global__ void __launch_bounds__(256) k_sell_spmv(int r0, int r1, int nl, const int64_t* __restrict__ sptr,
                                                   const int* __restrict__ scol,
                                                   const double* __restrict__ sval,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ f,
                                                   double* __restrict__ y,
                                                   const double* __restrict__ c, PfList pf,
                                                   const int* __restrict__ sluw = nullptr,
                                                   const uint8_t* __restrict__ nlow = nullptr,
                                                   const int* __restrict__ yperm = nullptr,
                                                   C0Fuse c0 = C0Fuse{nullptr, nullptr, nullptr, 0}) {
    pdl_trigger();
    l2_prefetch_share(pf);
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = (r0 & ~31) + g / TPR;
    const int part = g % TPR;
    const bool live = r >= r0 && r < r1;
    RowFrag<TPR, CH> fr;
    int w = 0, k1 = part, lim = 0, yr = r;
    int64_t base = 0;
    if (live) {
        if (yperm) yr = yperm[r];  // output position (the residual in Morton order for the restriction)
        const int64_t s0 = sptr[r >> 5];
        w = (int)((sptr[(r >> 5) + 1] - s0) >> 5);
        base = s0 + (r & 31);
        if (MODE >= 2) {  // later-colour slots only: from the slice's first one, masked per row
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
    double acc = fr.dot(x, 0.0);
    for (int k0 = k1 + TPR * CH; k0 < w; k0 += TPR * CH) {
        fr.load(sval + base, scol + base, w, k0);
        if (MODE >= 2) {
#pragma unroll
            for (int q = 0; q < CH; ++q)
                if (k0 + q * TPR < lim) fr.c[q] = -1;
        }
        acc = fr.dot(x, acc);
    }
    acc = group_sum<TPR>(acc);
    if (live && part == 0) {
        if (POISSON) acc += c[r] * x[nl];
        y[yr] = (MODE == 0) ? acc : (MODE == 1) ? f[r] - acc : (MODE == 2) ? -acc : f[r] + acc;
        if (MODE == 0 && c0.u && r < c0.c0_end) c0.u[r] = 0.0 + (acc - 0.0) / c0.sval[c0.sptr[r >> 5] + (r & 31)];
    }
}

// Fused residual + restriction (Alg. 3 lines 5 and 8, P:392 / P:395; north_star item 4):
//   phase 1  t = f - L_j u  (MODE 1) or -(later-colour part of L_j) u after a zero-guess
//            sweep (MODE 2), every fine row, written once;
//   grid-wide barrier (cooperative launch: every CTA is resident);
//   phase 2  r_{j+1} = R_j t, every coarse row, t gathered from L2 (ld.global.cg), plus
//            colour 0 of level j+1's presmooth from zero when c0.u (C0Fuse).
// One launch instead of two: no second kernel ramp and no PDL hand-off between them; t stays
// in L2 between the phases.  Each fine / coarse row is summed exactly as k_sell_spmv MODE 1/2 /
// MODE 0 sum it (same slots, same threads per row, same order), so the result is bitwise the
// unfused pair's.  Grid-stride over rows with a warp-uniform pass count (group_sum shuffles).
struct ResRestrict {
    int n;                      // fine rows
    const int64_t* sptr;
    const int* scol;
    const double* sval;
    const double* u;
    const double* f;
    double* t;
    const int* sluw;            // MODE 2
    const uint8_t* nlow;        // MODE 2
    const int* yperm;           // t written at yperm[r] (Morton order) if non-null
    int nc;                     // coarse rows
    const int64_t* rptr;
    const int* rcol;
    const double* rval;
    double* y;
    C0Fuse c0;
};

template <int MODE, int TPRL, int TPRR, int CH>
__global__ void __launch_bounds__(256) k_res_restrict(ResRestrict a) {
    const int T = gridDim.x * blockDim.x;
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    // ---- phase 1: fine rows (TPRL threads per row)
    {
        const int per_pass = T / TPRL, part = g % TPRL;
        const int npass = (a.n + per_pass - 1) / per_pass;
        for (int ps = 0; ps < npass; ++ps) {
            const int r = ps * per_pass + g / TPRL;
            const bool live = r < a.n;
            RowFrag<TPRL, CH> fr;
            int w = 0, k1 = part, lim = 0, yr = r;
            int64_t base = 0;
            if (live) {
                if (a.yperm) yr = a.yperm[r];
                const int64_t s0 = a.sptr[r >> 5];
                w = (int)((a.sptr[(r >> 5) + 1] - s0) >> 5);
                base = s0 + (r & 31);
                if (MODE == 2) {
                    k1 = a.sluw[r >> 5] + part;
                    lim = 1 + (int)a.nlow[r];
                }
                fr.load(a.sval + base, a.scol + base, w, k1);
            } else {
                fr.load(a.sval, a.scol, 0, 0);
            }
            if (MODE == 2) {
#pragma unroll
                for (int q = 0; q < CH; ++q)
                    if (k1 + q * TPRL < lim) fr.c[q] = -1;
            }
            if (ps == 0) pdl_wait();  // (the first row's operator chunk was loaded before the wait)
            double acc = fr.dot(a.u, 0.0);
            for (int k0 = k1 + TPRL * CH; k0 < w; k0 += TPRL * CH) {
                fr.load(a.sval + base, a.scol + base, w, k0);
                if (MODE == 2) {
#pragma unroll
                    for (int q = 0; q < CH; ++q)
                        if (k0 + q * TPRL < lim) fr.c[q] = -1;
                }
                acc = fr.dot(a.u, acc);
            }
            acc = group_sum<TPRL>(acc);
            if (live && part == 0) a.t[yr] = (MODE == 1) ? a.f[r] - acc : -acc;
        }
        if (npass == 0) pdl_wait();
    }
    __threadfence();
    cooperative_groups::this_grid().sync();
    pdl_trigger();  // (after the barrier: the successor cannot take the SMs of CTAs not yet resident)
    // ---- phase 2: coarse rows (TPRR threads per row)
    {
        const int per_pass = T / TPRR, part = g % TPRR;
        const int npass = (a.nc + per_pass - 1) / per_pass;
        for (int ps = 0; ps < npass; ++ps) {
            const int r = ps * per_pass + g / TPRR;
            const bool live = r < a.nc;
            RowFrag<TPRR, CH> fr;
            int w = 0;
            int64_t base = 0;
            if (live) {
                const int64_t s0 = a.rptr[r >> 5];
                w = (int)((a.rptr[(r >> 5) + 1] - s0) >> 5);
                base = s0 + (r & 31);
                fr.load(a.rval + base, a.rcol + base, w, part);
            } else {
                fr.load(a.rval, a.rcol, 0, 0);
            }
            double acc = fr.dot_cg(a.t, 0.0);
            for (int k0 = part + TPRR * CH; k0 < w; k0 += TPRR * CH) {
                fr.load(a.rval + base, a.rcol + base, w, k0);
                acc = fr.dot_cg(a.t, acc);
            }
            acc = group_sum<TPRR>(acc);
            if (live && part == 0) {
                a.y[r] = acc;
                if (a.c0.u && r < a.c0.c0_end)
                    a.c0.u[r] = 0.0 + (acc - 0.0) / a.c0.sval[a.c0.sptr[r >> 5] + (r & 31)];
            }
        }
    }
}

// e[r] += sum_k P[k][r] * ec[Pcol[k][r]] on the rows [r0, r1) of a level with n rows
// (interpolate + correct); Poisson: the multiplier e[n] += ec[nc] is added by
// the thread of row n when r1 == n.
template <bool POISSON, int M>
__global__ void __launch_bounds__(256) k_interp_correct(int r0, int r1, int n, int m, const int* __restrict__ pcol,
                                                        const double* __restrict__ pval,
                                                        const double* __restrict__ ec,
                                                        double* __restrict__ e, int nc, PfList pf) {
    pdl_trigger();
    l2_prefetch_share(pf);
    const int r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
    int cidx[M];
    double a[M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
        const bool ok = r < r1 && k < m;
        cidx[k] = ok ? ld_stream_i32(pcol + (int64_t)k * n + r) : -1;
        a[k] = ok ? ld_stream_f64(pval + (int64_t)k * n + r) : 0.0;
    }
    pdl_wait();
    if (r >= r1) {
        if (POISSON && r == n && r1 == n) e[n] += ec[nc];
        return;
    }
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k)
        if (cidx[k] >= 0) acc = fma(a[k], ec[cidx[k]], acc);
    e[r] += acc;
}

// y[r] = sum_k P[k][r] * x[...]  (plain interpolation, test hook)
template <bool POISSON>
__global__ void k_interp(int n, int m, const int* __restrict__ pcol, const double* __restrict__ pval,
                         const double* __restrict__ x, double* __restrict__ y, int nc) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n) return;
    if (r == n) {
        if (POISSON) y[n] = x[nc];
        return;
    }
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc += pval[(int64_t)k * n + r] * x[pcol[(int64_t)k * n + r]];
    y[r] = acc;
}

// Dense coarse solve with the LU factors (column-major) and pivots.  The factors
// are staged in shared memory by the whole CTA (prologue), then one warp solves.
// smem: LU[m*m] (if it fits, else read from global), b[m]
__global__ void __launch_bounds__(256) k_coarse_solve(int m, int lu_in_smem, const double* __restrict__ LU,
                                                      const int* __restrict__ piv,
                                                      const double* __restrict__ rhs,
                                                      double* __restrict__ x) {
    extern __shared__ double sm[];
    pdl_trigger();
    double* b = sm;
    double* L = lu_in_smem ? sm + m : nullptr;
    const double* A = lu_in_smem ? L : LU;
    if (lu_in_smem)
        for (int i = threadIdx.x; i < m * m; i += blockDim.x) L[i] = LU[i];
    pdl_wait();
    for (int i = threadIdx.x; i < m; i += blockDim.x) b[i] = rhs[i];
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    if (lane == 0)
        for (int k = 0; k < m; ++k) {
            int p = piv[k];
            if (p != k) { double t = b[k]; b[k] = b[p]; b[p] = t; }
        }
    __syncwarp();
    for (int k = 0; k < m; ++k) {  // forward, unit lower
        const double xk = b[k];
        const double* col = A + (int64_t)k * m;
        for (int i = k + 1 + lane; i < m; i += 32) b[i] -= col[i] * xk;
        __syncwarp();
    }
    for (int i = m - 1; i >= 0; --i) {  // backward
        const double* col = A + (int64_t)i * m;
        if (lane == 0) b[i] = b[i] / col[i];
        __syncwarp();
        const double xi = b[i];
        for (int r = lane; r < i; r += 32) b[r] -= col[r] * xi;
        __syncwarp();
    }
    for (int i = lane; i < m; i += 32) x[i] = b[i];
}

__global__ void k_fill(int64_t n, double* __restrict__ x, double v, PfList pf) {
    pdl_trigger();
    l2_prefetch_share(pf);
    pdl_wait();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}
__global__ void k_copy1(const double* __restrict__ src, double* __restrict__ dst) {
    pdl_trigger();
    pdl_wait();
    *dst = *src;
}

// out[i] = in[idx[i]]  /  out[idx[i]] = in[i]
__global__ void k_gather(int n, const int* __restrict__ idx, const double* __restrict__ in,
                         double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = in[idx[i]];
}
__global__ void k_scatter(int n, const int* __restrict__ idx, const double* __restrict__ in,
                          double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[idx[i]] = in[i];
}

// ------------------------------- deterministic reductions ------------------------------
constexpr int RED_BLOCKS = 592;   // 4 per SM (measured: GMRES 22.0 -> 21.5 ms vs 2 per SM), fixed so
                                  // reductions are bitwise reproducible
constexpr int RED_THREADS = 256;
constexpr int MD_GROUP = 16;      // vectors per pass of the multi-dot (16: GMRES 21.45 -> 21.3 ms vs 8)

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// partials[b * k1 + j] = sum over block b's chunk of V_j . w   (V_j = V + j*ld)
__global__ void __launch_bounds__(RED_THREADS) k_multidot(int64_t n, const double* __restrict__ V,
                                                          int64_t ld, int k1,
                                                          const double* __restrict__ w,
                                                          double* __restrict__ partials) {
    pdl_trigger();
    pdl_wait();
    __shared__ double red[RED_THREADS / 32][MD_GROUP];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int g = 0; g < k1; g += MD_GROUP) {
        const int gn = min(MD_GROUP, k1 - g);
        double s[MD_GROUP];
#pragma unroll
        for (int q = 0; q < MD_GROUP; ++q) s[q] = 0.0;
        for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
            const double wi = w[i];
#pragma unroll
            for (int q = 0; q < MD_GROUP; ++q)
                if (q < gn) s[q] += V[(int64_t)(g + q) * ld + i] * wi;
        }
#pragma unroll
        for (int q = 0; q < MD_GROUP; ++q) {
            double t = warp_sum(s[q]);
            if (lane == 0) red[warp][q] = t;
        }
        __syncthreads();
        if (threadIdx.x < gn) {
            double t = 0.0;
            for (int ww = 0; ww < RED_THREADS / 32; ++ww) t += red[ww][threadIdx.x];
            partials[(int64_t)blockIdx.x * k1 + g + threadIdx.x] = t;
        }
        __syncthreads();
    }
}

// Last-block finish of a deterministic reduction: every block has written its partials
// (partials[b * k1 + j]); the block that takes the last ticket sums them in block order
// (lanes stride over blocks, then a fixed shuffle tree), so the result is bitwise
// reproducible whichever block finishes last.  out[j] = sum; acc[j] += sum if acc.
__device__ __forceinline__ void finish_partials(const double* partials, int k1, unsigned* ticket, double* out,
                                                double* acc) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int j = warp; j < k1; j += nw) {
        double t = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) t += __ldcg(partials + (int64_t)b * k1 + j);
        t = warp_sum(t);
        if (lane == 0) {
            out[j] = t;
            if (acc) acc[j] += t;
        }
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

// out[j] = V_j . w for j < k1 (V_j = V + j*ld), one launch (block partials + last-block finish)
__global__ void __launch_bounds__(RED_THREADS) k_multidot_fin(int64_t n, const double* __restrict__ V, int64_t ld,
                                                              int k1, const double* __restrict__ w,
                                                              double* __restrict__ partials, unsigned* ticket,
                                                              double* out, double* acc, const int* kdev = nullptr) {
    pdl_trigger();  // (no-ops unless launched with programmatic serialisation: gmres_dev's graph)
    pdl_wait();
    if (kdev) k1 = *kdev + 1;  // device-side GMRES: the Arnoldi step lives in device memory
    __shared__ double red[RED_THREADS / 32][MD_GROUP];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int g = 0; g < k1; g += MD_GROUP) {
        const int gn = min(MD_GROUP, k1 - g);
        double s[MD_GROUP];
#pragma unroll
        for (int q = 0; q < MD_GROUP; ++q) s[q] = 0.0;
        for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
            const double wi = w[i];
#pragma unroll
            for (int q = 0; q < MD_GROUP; ++q)
                if (q < gn) s[q] = fma(V[(int64_t)(g + q) * ld + i], wi, s[q]);
        }
#pragma unroll
        for (int q = 0; q < MD_GROUP; ++q) {
            double t = warp_sum(s[q]);
            if (lane == 0) red[warp][q] = t;
        }
        __syncthreads();
        if (threadIdx.x < gn) {
            double t = 0.0;
            for (int ww = 0; ww < RED_THREADS / 32; ++ww) t += red[ww][threadIdx.x];
            partials[(int64_t)blockIdx.x * k1 + g + threadIdx.x] = t;
        }
        __syncthreads();
    }
    finish_partials(partials, k1, ticket, out, acc);
}

// CGS2's middle two passes in one launch: w -= V h1 (k_multiaxpy's per-row arithmetic), then
// out[j] = V_j . w (k_multidot_fin's block chunks, per-thread order and finish; acc += out), on
// each block's own rows -- no grid-wide dependency between the two, so one kernel.  For k1 <=
// 16 a row's V entries are loaded once into registers and serve both; beyond, the block
// re-reads its chunk for the dots.  Bitwise the unfused pair.
__global__ void __launch_bounds__(RED_THREADS) k_multiaxpy_dot_fin(int64_t n, const double* __restrict__ V, int64_t ld,
                                                                   int k1, const double* __restrict__ h,
                                                                   double* __restrict__ w, double* __restrict__ partials,
                                                                   unsigned* ticket, double* out, double* acc,
                                                                   const int* kdev = nullptr) {
    pdl_trigger();
    pdl_wait();
    if (kdev) k1 = *kdev + 1;
    __shared__ double hs[256];
    __shared__ double red[RED_THREADS / 32][MD_GROUP];
    for (int j = threadIdx.x; j < k1; j += blockDim.x) hs[j] = h[j];
    __syncthreads();
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (k1 <= MD_GROUP) {
        double s[MD_GROUP];
#pragma unroll
        for (int q = 0; q < MD_GROUP; ++q) s[q] = 0.0;
        for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
            double v[MD_GROUP];
#pragma unroll
            for (int q = 0; q < MD_GROUP; ++q) v[q] = (q < k1) ? V[(int64_t)q * ld + i] : 0.0;
            double a = w[i];
#pragma unroll
            for (int q = 0; q < MD_GROUP; ++q)
                if (q < k1) a -= v[q] * hs[q];
            w[i] = a;
#pragma unroll
            for (int q = 0; q < MD_GROUP; ++q)
                if (q < k1) s[q] = fma(v[q], a, s[q]);
        }
#pragma unroll
        for (int q = 0; q < MD_GROUP; ++q) {
            const double t = warp_sum(s[q]);
            if (lane == 0) red[warp][q] = t;
        }
        __syncthreads();
        if (threadIdx.x < k1) {
            double t = 0.0;
            for (int ww = 0; ww < RED_THREADS / 32; ++ww) t += red[ww][threadIdx.x];
            partials[(int64_t)blockIdx.x * k1 + threadIdx.x] = t;
        }
    } else {
        for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
            double a = w[i];
            for (int j = 0; j < k1; ++j) a -= V[(int64_t)j * ld + i] * hs[j];
            w[i] = a;
        }
        for (int g = 0; g < k1; g += MD_GROUP) {  // (each thread re-reads only the rows it wrote)
            const int gn = min(MD_GROUP, k1 - g);
            double s[MD_GROUP];
#pragma unroll
            for (int q = 0; q < MD_GROUP; ++q) s[q] = 0.0;
            for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
                const double wi = w[i];
#pragma unroll
                for (int q = 0; q < MD_GROUP; ++q)
                    if (q < gn) s[q] = fma(V[(int64_t)(g + q) * ld + i], wi, s[q]);
            }
#pragma unroll
            for (int q = 0; q < MD_GROUP; ++q) {
                const double t = warp_sum(s[q]);
                if (lane == 0) red[warp][q] = t;
            }
            __syncthreads();
            if (threadIdx.x < gn) {
                double t = 0.0;
                for (int ww = 0; ww < RED_THREADS / 32; ++ww) t += red[ww][threadIdx.x];
                partials[(int64_t)blockIdx.x * k1 + g + threadIdx.x] = t;
            }
            __syncthreads();
        }
    }
    finish_partials(partials, k1, ticket, out, acc);
}

// w[i] -= sum_j V_j[i] h[j]; nrm2[0] = ||w||^2 (block partials + last-block finish)
__global__ void __launch_bounds__(RED_THREADS) k_multiaxpy_norm(int64_t n, const double* __restrict__ V, int64_t ld,
                                                                int k1, const double* __restrict__ h,
                                                                double* __restrict__ w, double* __restrict__ partials,
                                                                unsigned* ticket, double* nrm2, const int* kdev = nullptr) {
    pdl_trigger();
    pdl_wait();
    if (kdev) k1 = *kdev + 1;
    __shared__ double hs[256];
    __shared__ double red[RED_THREADS / 32];
    for (int j = threadIdx.x; j < k1; j += blockDim.x) hs[j] = h[j];
    __syncthreads();
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
    double s = 0.0;
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
        double a = w[i];
        for (int j = 0; j < k1; ++j) a -= V[(int64_t)j * ld + i] * hs[j];
        w[i] = a;
        s = fma(a, a, s);
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int ww = 0; ww < RED_THREADS / 32; ++ww) t += red[ww];
        partials[blockIdx.x] = t;
    }
    finish_partials(partials, 1, ticket, nrm2, nullptr);
}

// w[i] -= sum_j V_j[i] * h[j]
__global__ void __launch_bounds__(256) k_multiaxpy(int64_t n, const double* __restrict__ V,
                                                   int64_t ld, int k1, const double* __restrict__ h,
                                                   double* __restrict__ w, const int* kdev = nullptr) {
    pdl_trigger();
    pdl_wait();
    if (kdev) k1 = *kdev + 1;
    __shared__ double hs[256];
    for (int j = threadIdx.x; j < k1; j += blockDim.x) hs[j] = h[j];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = w[i];
        for (int j = 0; j < k1; ++j) acc -= V[(int64_t)j * ld + i] * hs[j];
        w[i] = acc;
    }
}

// y[i] = sum_j V_j[i] * h[j]
__global__ void __launch_bounds__(256) k_lincomb(int64_t n, const double* __restrict__ V, int64_t ld,
                                                 int k1, const double* __restrict__ h,
                                                 double* __restrict__ y) {
    __shared__ double hs[256];
    for (int j = threadIdx.x; j < k1; j += blockDim.x) hs[j] = h[j];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < k1; ++j) acc += V[(int64_t)j * ld + i] * hs[j];
        y[i] = acc;
    }
}

// Device-side GMRES (mgm.cu gmres_dev): one CUDA graph per restart cycle whose WHILE node
// runs Arnoldi steps until the device Givens kernel clears the condition.  State:
// gi = {k, its, stop, maxit}; gd = {bnorm, tol, H[(m+1) x m] row-major, cs[m], sn[m],
// g[m+1], hist[...]}.
struct GmresDev {
    int* gi;
    double* gd;
    int m;
    int hist_cap;
};
__device__ __forceinline__ double* gmd_H(const GmresDev& G) { return G.gd + 2; }
__device__ __forceinline__ double* gmd_cs(const GmresDev& G) { return G.gd + 2 + (G.m + 1) * G.m; }
__device__ __forceinline__ double* gmd_sn(const GmresDev& G) { return gmd_cs(G) + G.m; }
__device__ __forceinline__ double* gmd_g(const GmresDev& G) { return gmd_sn(G) + G.m; }
__device__ __forceinline__ double* gmd_hist(const GmresDev& G) { return gmd_g(G) + G.m + 1; }

// dst = V_k (k = gi[0]): the Arnoldi vector to precondition.  With c0.u: also colour 0 of the
// level-0 presmooth from the zero guess (u = f / a_rr for rows < c0_end; C0Fuse), which the
// zero-guess V-cycle graph then skips.
__global__ void k_copy_col(int64_t n, const double* __restrict__ V, int64_t ld, const int* __restrict__ kdev,
                           double* __restrict__ dst, C0Fuse c0) {
    pdl_trigger();
    pdl_wait();
    const double* src = kdev ? V + (int64_t)(*kdev) * ld : V;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = src[i];
        dst[i] = v;
        if (c0.u && i < c0.c0_end) c0.u[i] = 0.0 + (v - 0.0) / c0.sval[c0.sptr[i >> 5] + (i & 31)];
    }
}
// V_{k+1} = w / sqrt(*nrm2)
__global__ void k_scale_col(int64_t n, const double* __restrict__ w, const double* __restrict__ nrm2, double* V,
                            int64_t ld, const int* __restrict__ kdev) {
    pdl_trigger();
    pdl_wait();
    const double inv = 1.0 / sqrt(*nrm2);
    double* dst = V + (int64_t)(*kdev + 1) * ld;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = w[i] * inv;
}
// Z[:, k] = z (k = *kdev): the device GMRES keeps z_k = M v_k, so the restart-cycle update is
// x += Z y instead of x += M (V y) (M is linear: one V-cycle less per restart cycle)
__global__ void k_store_col(int64_t n, const double* __restrict__ z, double* Z, int64_t ld, const int* __restrict__ kdev) {
    pdl_trigger();
    pdl_wait();
    double* dst = Z + (int64_t)(*kdev) * ld;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = z[i];
}
// One Givens step of the Hessenberg least-squares problem (same operations as gmres_lib's
// host loop), the relative residual history, and the loop condition.
__global__ void k_gmres_givens(GmresDev G, const double* __restrict__ h, const double* __restrict__ nrm2,
                               cudaGraphConditionalHandle cond) {
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int m = G.m;
    const int k = G.gi[0], k1 = k + 1;
    double* H = gmd_H(G);
    double* cs = gmd_cs(G);
    double* sn = gmd_sn(G);
    double* g = gmd_g(G);
    for (int i = 0; i < k1; ++i) H[i * m + k] = h[i];
    const double hk1 = sqrt(*nrm2);
    H[k1 * m + k] = hk1;
    for (int i = 0; i < k; ++i) {
        const double t = cs[i] * H[i * m + k] + sn[i] * H[(i + 1) * m + k];
        H[(i + 1) * m + k] = -sn[i] * H[i * m + k] + cs[i] * H[(i + 1) * m + k];
        H[i * m + k] = t;
    }
    const double den = hypot(H[k * m + k], hk1);
    cs[k] = H[k * m + k] / den;
    sn[k] = hk1 / den;
    H[k * m + k] = den;
    H[k1 * m + k] = 0.0;
    g[k1] = -sn[k] * g[k];
    g[k] = cs[k] * g[k];
    const double rel = fabs(g[k1]) / G.gd[0];
    const int its = G.gi[1] + 1;
    if (its - 1 < G.hist_cap) gmd_hist(G)[its - 1] = rel;
    int stop = 0;  // 1: converged / maxit / happy breakdown, 2: non-finite, 3: restart
    if (!isfinite(rel)) stop = 2;
    else if (rel <= G.gd[1] || its >= G.gi[3] || hk1 == 0.0) stop = 1;
    else if (k1 == m) stop = 3;
    G.gi[0] = k1;
    G.gi[1] = its;
    G.gi[2] = stop;
    cudaGraphSetConditional(cond, stop == 0 ? 1u : 0u);
}

// dst = src / sqrt(*nrm2)
__global__ void k_scale_by_invnorm(int64_t n, const double* __restrict__ src,
                                   const double* __restrict__ nrm2, double* __restrict__ dst) {
    const double inv = 1.0 / sqrt(*nrm2);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i] * inv;
}
// dst = a*x + b*y
__global__ void k_axpby(int64_t n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = a * x[i] + b * y[i];
}
// BiCGSTAB direction update p = r + beta (p - omega v)
__global__ void k_bicg_p(int64_t n, const double* __restrict__ r, const double* __restrict__ v, double* p,
                         double beta, double omega) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = r[i] + beta * (p[i] - omega * v[i]);
}
// x += a y + b z
__global__ void k_axpbypz(int64_t n, double* x, double a, const double* __restrict__ y, double b,
                          const double* __restrict__ z) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = x[i] + a * y[i] + b * z[i];
}
// h[j] += h2[j]
__global__ void k_vadd(int k1, double* __restrict__ h, const double* __restrict__ h2) {
    for (int j = threadIdx.x; j < k1; j += blockDim.x) h[j] += h2[j];
}
// y[n] = fs*f[n] + sign*s[0]  (border row of the Poisson system from an all-reduced dot s)
__global__ void k_border_set(const double* __restrict__ s, double fs, const double* __restrict__ f, int n,
                             double sign, double* __restrict__ y) {
    if (threadIdx.x == 0) y[n] = (f ? fs * f[n] : 0.0) + sign * s[0];
}
// y[n] = f[n]*fs - sum   (border row of the Poisson system), single block finish
__global__ void k_border_finish(const double* __restrict__ partials, int nblk, double fs,
                                const double* __restrict__ f, int n, double sign,
                                double* __restrict__ y) {
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int b = 0; b < nblk; ++b) t += partials[b];
        y[n] = (f ? fs * f[n] : 0.0) + sign * t;
    }
}

}  // namespace mgm
