// One multicolour Gauss-Seidel sweep of one level in ONE persistent launch, ordered by
// point-to-point progress counters between CTAs instead of one kernel boundary per colour.
//
// The multicolour sweep (P:285-291 Gauss-Seidel smoothing; north_star item 2; O12)
// updates the rows of colour 0, 1, ..., C-1 in turn: a row of colour c reads the NEW values of
// its neighbours of colours < c and the OLD values of colours > c.  Any schedule that, for
// every stored entry a_ij with colour(j) < colour(i), updates j before i reads it, and, for
// colour(j) > colour(i), lets i read u_j before j is updated, computes exactly the same
// numbers.  Here CTA b owns the rows whose Morton index lies in [b n / B, (b+1) n / B); the
// lib order is colour-major with Morton order inside a colour, so CTA b's rows of colour c
// are one contiguous range cst[c][b] .. cst[c][b+1].  Each CTA publishes how many colour
// steps it has finished; before step s it waits until every NEIGHBOUR CTA (owner of a column
// of one of its rows, symmetrised) has finished s steps:
//   * colours < c of the neighbours are final;
//   * colours > c of the neighbours are untouched: a neighbour cannot start step s+1 before
//     this CTA has finished step s (the relation is symmetric).
// Per-row arithmetic is k_gs_colour's (same slots, same threads per row, same order), so the
// sweep is bitwise the per-colour-kernel sweep.
//
// What a colour step costs on the critical path: the publish (one release store after the
// CTA barrier), the neighbours' acquire poll, the u gathers from L2 and the row update.  The
// operator rows of step s+1 are loaded into registers right AFTER the publish of step s (so
// the release fence never waits for them) and the L2 is asked to stream the operator bytes
// of step s+1+pf_dist (bulk prefetch, no registers, no ordering): the HBM stream runs ahead
// of the colour front instead of each per-colour kernel paying its own ramp and tail.
//
// Counters are monotonic across launches (every launch adds its step count to every CTA's
// counter; all CTAs run all steps), so no reset is needed: a CTA reads its own counter as the
// launch's base.  All B CTAs must be co-resident: the host launches with the cooperative
// attribute (the launch fails rather than deadlocks if they cannot be).  A wait that never
// completes (impossible unless co-residency is broken) traps after a bounded spin: the
// context reports a CUDA error instead of hanging the GPU.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "solve_kernels.cuh"

namespace mgm {

constexpr int FLOW_THREADS = 256;
constexpr int FLOW_PROG_STRIDE = 32;  // one counter per 128-byte line

struct FlowSweep {
    int n;         // rows of the level (Poisson: the multiplier u[n] follows them)
    int ncol;      // colours
    int s0;        // first step (1 when colour 0 was already set by the restriction)
    int backward;  // colour order C-1 .. 0
    int Wu;        // > 0: every SELL slice has this width
    int pf_dist;   // L2 prefetch distance in steps (0: none)
    const int64_t* sptr;
    const int* scol;
    const double* sval;
    const double* f;
    double* u;
    const double* c;      // Poisson border vector
    const int* cst;       // [ncol][B + 1]
    const int* nbr_ptr;   // [B + 1]
    const int* nbr;       // neighbour CTAs
    unsigned* prog;       // [B * FLOW_PROG_STRIDE]
    const int* slw;       // ZG tables (pack_sell)
    const uint8_t* nlow;
};

__device__ __forceinline__ unsigned flow_ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void flow_st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Operator state of the row a thread group works on (k_gs_colour's prologue).
template <bool ZG, int TPR, int CH>
struct FlowRow {
    RowFrag<TPR, CH> fr;
    int w = 0;
    int64_t base = 0;
    double d = 1.0;
    __device__ __forceinline__ void load(const FlowSweep& P, int r, bool live, int part) {
        w = 0;
        base = 0;
        d = 1.0;
        if (!live) {
            fr.load(P.sval, P.scol, 0, 0);
            return;
        }
        if (P.Wu > 0) {
            w = P.Wu;
            base = (int64_t)(r >> 5) * 32 * P.Wu + (r & 31);
        } else {
            const int64_t s0 = P.sptr[r >> 5];
            w = (int)((P.sptr[(r >> 5) + 1] - s0) >> 5);
            base = s0 + (r & 31);
        }
        int lim = 0;
        if (ZG) {
            w = P.slw[r >> 5];
            lim = 1 + (int)P.nlow[r];
        }
        fr.load(P.sval + base, P.scol + base, ZG ? lim : w, part);
        if (ZG) {
#pragma unroll
            for (int q = 0; q < CH; ++q)
                if (part + q * TPR == 0 || part + q * TPR >= lim) fr.c[q] = -1;
            w = lim;
        }
        d = ld_stream_f64(P.sval + base);
    }
};

// L2 bulk prefetch of the operator bytes (values + columns) of CTA b's rows of colour c.
__device__ __forceinline__ void flow_prefetch(const FlowSweep& P, int c, int b, int B) {
    const int r0 = P.cst[c * (B + 1) + b], r1 = P.cst[c * (B + 1) + b + 1];
    if (r1 <= r0) return;
    const int64_t lo = P.Wu > 0 ? (int64_t)(r0 >> 5) * 32 * P.Wu : P.sptr[r0 >> 5];
    const int64_t hi = P.Wu > 0 ? (int64_t)(((r1 - 1) >> 5) + 1) * 32 * P.Wu : P.sptr[((r1 - 1) >> 5) + 1];
    const char* pv = (const char*)(P.sval + lo);
    const char* pc = (const char*)(P.scol + lo);
    const int64_t bv = (hi - lo) * 8, bc = (hi - lo) * 4;  // multiples of 256 / 128 B (32-row slices)
    for (int64_t o = 0; o < bv; o += 32768) {
        const uint32_t sz = (uint32_t)(bv - o < 32768 ? bv - o : 32768);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pv + o), "r"(sz) : "memory");
    }
    for (int64_t o = 0; o < bc; o += 32768) {
        const uint32_t sz = (uint32_t)(bc - o < 32768 ? bc - o : 32768);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pc + o), "r"(sz) : "memory");
    }
}

template <bool POISSON, int TPR, int CH, bool ZG>
__global__ void __launch_bounds__(FLOW_THREADS) k_gs_flow(const FlowSweep P) {
    pdl_trigger();
    const int b = blockIdx.x, B = gridDim.x, tid = threadIdx.x;
    const int part = tid % TPR, slot = tid / TPR;
    constexpr int G = FLOW_THREADS / TPR;  // rows per pass
    const int nsteps = P.ncol;
    auto colour = [&](int s) { return P.backward ? P.ncol - 1 - s : s; };
    int s = P.s0;
    int c = colour(s);
    int r0 = P.cst[c * (B + 1) + b], r1 = P.cst[c * (B + 1) + b + 1];
    FlowRow<ZG, TPR, CH> row;
    row.load(P, r0 + slot, r0 + slot < r1, part);
    if (tid == 0)
        for (int q = 1; q <= P.pf_dist && s + q < nsteps; ++q) flow_prefetch(P, colour(s + q), b, B);
    const int nb0 = P.nbr_ptr[b], nb1 = P.nbr_ptr[b + 1];
    pdl_wait();
    unsigned* myprog = P.prog + (size_t)b * FLOW_PROG_STRIDE;
    const unsigned base0 = *(volatile unsigned*)myprog;  // only this CTA writes it
    for (; s < nsteps; ++s) {
        if (s > P.s0) {
            if (tid < 32) {
                const unsigned target = base0 + (unsigned)(s - P.s0);
                for (int k = nb0 + tid; k < nb1; k += 32) {
                    const unsigned* q = P.prog + (size_t)P.nbr[k] * FLOW_PROG_STRIDE;
                    for (int spin = 0; (int)(flow_ld_acquire(q) - target) < 0; ++spin)
                        if (spin > (1 << 24)) __trap();
                }
            }
            __syncthreads();
        }
        // rows [r0, r1) of colour c: u_i += (f_i - sum_j a_ij u_j [- c_i lambda]) / a_ii
        for (int rb = r0; rb < r1; rb += G) {
            const int r = rb + slot;
            const bool live = r < r1;
            if (rb != r0) row.load(P, r, live, part);
            double fr_v = 0.0, ur = 0.0, cl = 0.0;
            if (live && part == 0) {
                fr_v = P.f[r];
                if (!ZG) ur = __ldcg(P.u + r);
                if (POISSON) cl = P.c[r] * __ldcg(P.u + P.n);
            }
            double acc = row.fr.dot_cg(P.u, 0.0);
            for (int k0 = part + TPR * CH; k0 < row.w; k0 += TPR * CH) {
                row.fr.load(P.sval + row.base, P.scol + row.base, row.w, k0);
                acc = row.fr.dot_cg(P.u, acc);
            }
            acc = group_sum<TPR>(acc);
            if (live && part == 0) {
                double res = fr_v - acc;
                if (POISSON) res -= cl;
                P.u[r] = ur + res / row.d;
            }
        }
        __syncthreads();
        if (tid == 0) flow_st_release(myprog, base0 + (unsigned)(s - P.s0) + 1);
        if (s + 1 < nsteps) {  // operator rows of the next step (immutable: no ordering needed)
            c = colour(s + 1);
            r0 = P.cst[c * (B + 1) + b];
            r1 = P.cst[c * (B + 1) + b + 1];
            row.load(P, r0 + slot, r0 + slot < r1, part);
            if (tid == 0 && P.pf_dist > 0 && s + 1 + P.pf_dist < nsteps) flow_prefetch(P, colour(s + 1 + P.pf_dist), b, B);
        }
    }
}

}  // namespace mgm
