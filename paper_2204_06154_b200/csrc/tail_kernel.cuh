// The bottom of the V-cycle in ONE kernel: levels J..p-1 of Alg. 3 run by a
// single thread-block cluster (up to 16 CTAs on one GPC), with a cluster barrier
// (barrier.cluster arrive.release / wait.acquire) between dependent phases instead of a
// kernel boundary.  On these small levels a kernel launch per colour costs far more than
// the colour's work; a cluster barrier costs ~0.2 us.
//
// Semantics (identical to the per-kernel path): given r^J in lv[J].f, compute e^J in lv[J].u:
//   for j = J..p-2: e_j = 0; nu1 colour sweeps; t_j = r_j - L_j e_j; r_{j+1} = R_j t_j
//   e_{p-1} = L_{p-1}^{-1} r_{p-1}
//   for j = p-2..J: e_j += P_j e_{j+1}; nu2 colour sweeps
// Poisson mode: multipliers travel at index n_j; border dot products are reduced
// deterministically (fixed per-CTA partials, summed in rank order).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "solve_kernels.cuh"

namespace mgm {

namespace cg = cooperative_groups;

constexpr int TAIL_MAX_LEVELS = 16;
constexpr int TAIL_MAX_COLOURS = 128;

struct TailLevel {
    int n, ncol, tpr, rtpr, pm, nnext;
    const int64_t* sptr;
    const int* scol;
    const double* sval;
    const int* pcol;
    const double* pval;
    const int64_t* rptr;
    const int* rcol;
    const double* rval;
    double *u, *f, *t;
    const double* c;
    int coff[TAIL_MAX_COLOURS + 1];
};

struct TailParams {
    int J, p, nu1, nu2, pre_b, post_b, poisson, nc, lu_smem;
    const double* lu;
    const int* piv;
    double* partials;  // >= cluster size doubles
    TailLevel lv[TAIL_MAX_LEVELS];
};

// rows [r0, r1) of a SELL matrix: y[r] = (MODE 0) dot | (MODE 1) f - dot | (MODE 2) GS update
template <int MODE, int TPR>
__device__ __forceinline__ void tail_rows(int r0, int r1, const int64_t* __restrict__ sptr,
                                          const int* __restrict__ scol, const double* __restrict__ sval,
                                          const double* x, const double* f, double* y,
                                          const double* c, double lam, bool poisson, int tid, int nthr) {
    const int rb = r0 & ~31;
    const int total = (r1 - rb) * TPR;
    for (int base = 0; base < total; base += nthr) {
        const int g = base + tid;
        const int r = rb + g / TPR;
        const int part = g % TPR;
        const bool live = g < total && r >= r0 && r < r1;
        double acc = 0.0, d = 1.0;
        if (live) {
            const int64_t s0 = sptr[r >> 5];
            const int w = (int)((sptr[(r >> 5) + 1] - s0) >> 5);
            const int64_t b = s0 + (r & 31);
            RowFrag<TPR, 16> fr;
            for (int k0 = part; k0 < w; k0 += TPR * 16) {
                fr.load(sval + b, scol + b, w, k0);
                acc = fr.dot(x, acc);
            }
            if (MODE == 2) d = ld_stream_f64(sval + b);
        }
        acc = group_sum<TPR>(acc);
        if (live && part == 0) {
            if (MODE == 0) {
                y[r] = acc;
            } else if (MODE == 1) {
                if (poisson) acc += c[r] * lam;
                y[r] = f[r] - acc;
            } else {
                double res = f[r] - acc;
                if (poisson) res -= c[r] * lam;
                y[r] += res / d;
            }
        }
    }
}

template <int MODE>
__device__ __forceinline__ void tail_rows_t(int tpr, int r0, int r1, const int64_t* sptr, const int* scol,
                                            const double* sval, const double* x, const double* f, double* y,
                                            const double* c, double lam, bool poisson, int tid, int nthr) {
    if (tpr == 1) tail_rows<MODE, 1>(r0, r1, sptr, scol, sval, x, f, y, c, lam, poisson, tid, nthr);
    else if (tpr == 2) tail_rows<MODE, 2>(r0, r1, sptr, scol, sval, x, f, y, c, lam, poisson, tid, nthr);
    else tail_rows<MODE, 4>(r0, r1, sptr, scol, sval, x, f, y, c, lam, poisson, tid, nthr);
}

// deterministic cluster-wide sum of v (same value returned to all threads)
__device__ double tail_cluster_sum(double v, double* partials, double* red_sm, cg::cluster_group& cl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red_sm[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < nw; ++i) s += red_sm[i];
        partials[cl.block_rank()] = s;
    }
    cl.sync();
    double tot = 0.0;
    for (unsigned i = 0; i < cl.num_blocks(); ++i) tot += partials[i];
    cl.sync();  // partials may be reused after every CTA has read them
    return tot;
}

__device__ void tail_sweep(const TailParams& P, const TailLevel& L, bool backward, int tid, int nthr,
                           cg::cluster_group& cl) {
    for (int q = 0; q < L.ncol; ++q) {
        const int c = backward ? L.ncol - 1 - q : q;
        const double lam = P.poisson ? L.u[L.n] : 0.0;
        tail_rows_t<2>(L.tpr, L.coff[c], L.coff[c + 1], L.sptr, L.scol, L.sval, L.u, L.f, L.u, L.c, lam,
                       P.poisson != 0, tid, nthr);
        cl.sync();
    }
}

__global__ void __launch_bounds__(512, 1) k_vcycle_tail(const __grid_constant__ TailParams P) {
    extern __shared__ double tsm[];
    __shared__ double red_sm[32];
    cg::cluster_group cl = cg::this_cluster();
    const int nthr = (int)(cl.num_blocks() * blockDim.x);
    const int tid = (int)(cl.block_rank() * blockDim.x + threadIdx.x);
    const bool poisson = P.poisson != 0;
    // stage the coarse LU factors in CTA 0's shared memory (immutable: before the wait)
    double* luS = tsm;
    double* bS = tsm + (P.lu_smem ? (size_t)P.nc * P.nc : 0);
    if (cl.block_rank() == 0 && P.lu_smem)
        for (int i = threadIdx.x; i < P.nc * P.nc; i += blockDim.x) luS[i] = P.lu[i];
    pdl_trigger();
    pdl_wait();
    cl.sync();
    // ---- down: levels J .. p-2
    for (int j = P.J; j + 1 < P.p; ++j) {
        const TailLevel& L = P.lv[j - P.J];
        const int vn = L.n + (poisson ? 1 : 0);
        for (int i = tid; i < vn; i += nthr) L.u[i] = 0.0;
        cl.sync();
        for (int s = 0; s < P.nu1; ++s) tail_sweep(P, L, P.pre_b != 0, tid, nthr, cl);
        // residual t = f - L u (- c lam)
        const double lam = poisson ? L.u[L.n] : 0.0;
        tail_rows_t<1>(L.tpr, 0, L.n, L.sptr, L.scol, L.sval, L.u, L.f, L.t, L.c, lam, poisson, tid, nthr);
        if (poisson) {
            double s = 0.0;
            for (int i = tid; i < L.n; i += nthr) s += L.c[i] * L.u[i];
            const double tot = tail_cluster_sum(s, P.partials, red_sm, cl);
            if (tid == 0) L.t[L.n] = L.f[L.n] - tot;
        }
        cl.sync();
        // restrict r_{j+1} = R_j t
        const TailLevel& Ln = P.lv[j + 1 - P.J];
        tail_rows_t<0>(L.rtpr, 0, Ln.n, L.rptr, L.rcol, L.rval, L.t, nullptr, Ln.f, nullptr, 0.0, false, tid, nthr);
        if (poisson && tid == 0) Ln.f[Ln.n] = L.t[L.n];
        cl.sync();
    }
    // ---- coarsest: dense LU solve by warp 0 of CTA 0
    {
        const TailLevel& C = P.lv[P.p - 1 - P.J];
        if (cl.block_rank() == 0 && threadIdx.x < 32) {
            const int m = P.nc, lane = threadIdx.x;
            const double* A = P.lu_smem ? luS : P.lu;
            for (int i = lane; i < m; i += 32) bS[i] = C.f[i];
            __syncwarp();
            if (lane == 0)
                for (int k = 0; k < m; ++k) {
                    const int pk = P.piv[k];
                    if (pk != k) { double t = bS[k]; bS[k] = bS[pk]; bS[pk] = t; }
                }
            __syncwarp();
            for (int k = 0; k < m; ++k) {
                const double xk = bS[k];
                const double* col = A + (int64_t)k * m;
                for (int i = k + 1 + lane; i < m; i += 32) bS[i] -= col[i] * xk;
                __syncwarp();
            }
            for (int i = m - 1; i >= 0; --i) {
                const double* col = A + (int64_t)i * m;
                if (lane == 0) bS[i] = bS[i] / col[i];
                __syncwarp();
                const double xi = bS[i];
                for (int r = lane; r < i; r += 32) bS[r] -= col[r] * xi;
                __syncwarp();
            }
            for (int i = lane; i < m; i += 32) C.u[i] = bS[i];
        }
        cl.sync();
    }
    // ---- up: levels p-2 .. J
    for (int j = P.p - 2; j >= P.J; --j) {
        const TailLevel& L = P.lv[j - P.J];
        const TailLevel& Ln = P.lv[j + 1 - P.J];
        for (int r = tid; r < L.n; r += nthr) {
            double acc = 0.0;
            for (int k = 0; k < L.pm; ++k)
                acc = fma(L.pval[(int64_t)k * L.n + r], Ln.u[L.pcol[(int64_t)k * L.n + r]], acc);
            L.u[r] += acc;
        }
        if (poisson && tid == 0) L.u[L.n] += Ln.u[Ln.n];
        cl.sync();
        for (int s = 0; s < P.nu2; ++s) tail_sweep(P, L, P.post_b != 0, tid, nthr, cl);
    }
}

}  // namespace mgm
