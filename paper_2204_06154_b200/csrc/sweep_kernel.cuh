// One Gauss-Seidel sweep (all colours) of one level in ONE persistent kernel, with
// point-to-point dependencies between CTAs instead of a kernel boundary per colour.
//
// The multicolour sweep (north_star item 2; O12) updates the rows of colour
// 0, 1, ..., C-1 in turn.  A row of colour c reads its neighbours' u: the NEW values of
// colours < c and the OLD values of colours > c.  Rows are owned by CTAs in Morton blocks
// (CTA b owns the Morton ranks [b n / B, (b+1) n / B); lib order is colour-major with
// Morton order inside a colour, so CTA b's rows of colour c are one contiguous range).
// Each CTA publishes a progress counter (steps completed); before step s it waits until
// every NEIGHBOUR CTA (owner of a column of one of its rows, symmetrised) has completed
// s steps.  That gives exactly the colour-by-colour semantics:
//   * colours < c of neighbours are done (progress >= s);
//   * colours > c of neighbours are not yet updated: a neighbour cannot start step s+1
//     before this CTA has completed step s (the relation is symmetric).
// So the result is bitwise identical to one kernel per colour (same per-row arithmetic),
// while a CTA waits only for its few neighbours (~1 L2 round trip) instead of a grid-wide
// kernel boundary, and fast regions run ahead of slow ones.
//
// Counters are monotonic across launches (every launch adds nsweep * C to every CTA's
// counter), so no reset is needed: a CTA reads its own counter as the launch base.
// Requires all B CTAs to be co-resident (B <= occupancy * #SMs, checked at setup); the
// kernel neither triggers nor waits on programmatic dependents.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "solve_kernels.cuh"

namespace mgm {

constexpr int SW_THREADS = 256;
__device__ int g_sweep_timeout = 0;  // set if a neighbour wait ever gave up (never expected)
constexpr int SW_PROG_STRIDE = 32;  // counters on separate 128-byte lines

struct SweepParams {
    int n, ncol, nsweep, backward;
    const int64_t* sptr;
    const int* scol;
    const double* sval;
    const double* f;
    double* u;
    const int* cstart;   // [ncol][B + 1]: CTA b's rows of colour c = [cstart[c][b], cstart[c][b+1])
    const int* nbr_ptr;  // [B + 1]
    const int* nbr;      // neighbour CTAs
    unsigned* prog;      // [B * SW_PROG_STRIDE]
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int TPR, int CH>
__device__ __forceinline__ void sweep_frag_load(RowFrag<TPR, CH>& fr, const SweepParams& P, int r, bool live,
                                                int part, int& w, int64_t& base, double& d) {
    w = 0;
    base = 0;
    d = 1.0;
    if (live) {
        const int64_t s0 = P.sptr[r >> 5];
        w = (int)((P.sptr[(r >> 5) + 1] - s0) >> 5);
        base = s0 + (r & 31);
        fr.load(P.sval + base, P.scol + base, w, part);
        d = ld_stream_f64(P.sval + base);
    } else {
        fr.load(P.sval, P.scol, 0, 0);
    }
}

template <int TPR, int CH>
__global__ void __launch_bounds__(SW_THREADS) k_gs_sweep(const SweepParams P) {
    const int b = blockIdx.x, B = gridDim.x;
    const int tid = threadIdx.x;
    const int part = tid % TPR;
    const int groups = SW_THREADS / TPR;
    unsigned* myprog = P.prog + (size_t)b * SW_PROG_STRIDE;
    const unsigned base0 = *(volatile unsigned*)myprog;  // only this CTA writes it
    const int nb0 = P.nbr_ptr[b], nb1 = P.nbr_ptr[b + 1];
    const int steps = P.nsweep * P.ncol;
    auto colour = [&](int s) {
        const int c = s % P.ncol;
        return P.backward ? P.ncol - 1 - c : c;
    };
    // prefetch step 0
    int c = colour(0);
    int r0 = P.cstart[c * (B + 1) + b], r1 = P.cstart[c * (B + 1) + b + 1];
    RowFrag<TPR, CH> fr;
    int w;
    int64_t base;
    double d;
    sweep_frag_load(fr, P, r0 + tid / TPR, r0 + tid / TPR < r1, part, w, base, d);
    for (int s = 0; s < steps; ++s) {
        // wait until every neighbour has completed s steps (warp 0 polls, one lane per neighbour)
        if (s > 0 && tid < 32) {
            const unsigned target = base0 + (unsigned)s;
            for (int k = nb0 + tid; k < nb1; k += 32) {
                const unsigned* q = P.prog + (size_t)P.nbr[k] * SW_PROG_STRIDE;
                // bounded spin: a broken co-residency assumption must not hang the GPU
                for (long long spin = 0; (int)(ld_acquire_u32(q) - target) < 0; ++spin)
                    if (spin > (1ll << 26)) {
                        g_sweep_timeout = 1;
                        break;
                    }
            }
        }
        __syncthreads();
        // rows [r0, r1) of colour c: u_i += (f_i - sum_j a_ij u_j) / a_ii  (same arithmetic as k_gs_colour)
        for (int rb = r0; rb < r1; rb += groups) {
            const int r = rb + tid / TPR;
            const bool live = r < r1;
            if (rb != r0) sweep_frag_load(fr, P, r, live, part, w, base, d);
            double fr_v = 0.0, ur = 0.0;
            if (live && part == 0) {
                fr_v = P.f[r];
                ur = __ldcg(P.u + r);
            }
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < CH; ++q)
                if (fr.c[q] >= 0) acc = fma(fr.a[q], __ldcg(P.u + fr.c[q]), acc);
            for (int k0 = part + TPR * CH; k0 < w; k0 += TPR * CH) {
                fr.load(P.sval + base, P.scol + base, w, k0);
#pragma unroll
                for (int q = 0; q < CH; ++q)
                    if (fr.c[q] >= 0) acc = fma(fr.a[q], __ldcg(P.u + fr.c[q]), acc);
            }
            acc = group_sum<TPR>(acc);
            if (live && part == 0) P.u[r] = ur + (fr_v - acc) / d;
        }
        // prefetch the operator rows of step s+1 (immutable), then publish step s
        if (s + 1 < steps) {
            c = colour(s + 1);
            r0 = P.cstart[c * (B + 1) + b];
            r1 = P.cstart[c * (B + 1) + b + 1];
            sweep_frag_load(fr, P, r0 + tid / TPR, r0 + tid / TPR < r1, part, w, base, d);
        }
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release_u32(myprog, base0 + (unsigned)s + 1);
        }
    }
}

}  // namespace mgm
