// The bottom of the V-cycle in ONE kernel launch: levels J..p-1 of Alg. 3 run
// by a single thread-block cluster (16 CTAs on one GPC, or 8), as a list of "phases"
// separated by barriers instead of kernel boundaries.
//
// Why: below ~10^4 rows a colour of the Gauss-Seidel sweep holds a few hundred rows and a
// kernel boundary (~0.7-1 us with PDL inside a graph, measured: tools/micro/sync_costs.cu)
// plus the kernel's own dependent load chain (~2 us) dwarfs its work.  Here the barrier
// between two colours is barrier.cluster (~0.25 us measured) or, for levels small enough
// for one CTA ("local" phases, run by CTA 0 only), __syncthreads (~0.03 us).
//
// The gathered vectors -- the iterates u_J .. u_p -- are REPLICATED in every CTA's shared
// memory (21.8k doubles = 175 KB for cfg3's levels 3..7): every gather is a local
// ld.shared (~30 cycles instead of an L2 round trip of ~300-600 cycles with a 32-byte sector
// per 8-byte value), and every update is stored into all C copies with st.shared::cluster
// (fire-and-forget; the barrier's release orders them).  The right-hand sides f_j and the
// residuals t_j stay in HBM/L2: f_j[row] is read once per row (prefetched with the
// operator row when the previous phase did not write it), t_j is written by the residual
// phase and gathered only by the restriction.  u_J is stored back to HBM at the end for
// the per-kernel up-path.  Each thread prefetches the immutable operator row of its NEXT
// phase (values, columns, 1/a_rr) into registers between the barrier's arrive and wait.
//
// Operators (built by setup_bottom): row-major ELL in global memory, row r at
// val[r*W .. r*W+W), padded with (own first column, 0.0), L_j with its diagonal first; so
// the address of a thread's entries is known without a row-pointer load.  Loads carry an
// L2 evict_last policy (the upper levels stream with evict_first).  GS phases multiply by a
// stored 1/a_rr instead of dividing (the same update up to one rounding).
//
// A phase applies one operator to the rows [r0, r1) with one of these epilogues
// (acc = sum_k val_k x[col_k]; x is a replicated shared vector or, for the restriction and
// the coarsest solve, a global one):
//   BP_ZERO  y[r] = 0 (own copy, all rows)                 (e_J = 0, Alg. 3 line 7)
//   BP_GS    y[r] = x[r] + (f[r] - acc) * dinv[r]          (one colour; y = x = u_j)
//   BP_RES   t[r] = f[r] - acc                             (t_j = r_j - L_j e_j; global)
//   BP_MVZ   f'[r] = acc (global), z[r] = 0                (r_{j+1} = R_j t_j, e_{j+1} = 0)
//   BP_ADD   y[r] += acc                                   (e_j += P_j e_{j+1})
//   BP_MV    y[r] = acc                                    (coarsest: e_p = L_p^{-1} r_p)
//   BP_STORE g[r] = y[r]                                   (e_J back to HBM)
//   BP_LOAD  y[r] = x[r] (own copy, all rows)              (after a grid-wide coarse solve)
// Synchronisation between phases:
//   * local -> local: __syncthreads (CTA 0 only);
//   * DATA-SYNCHRONISED phases (mb >= 0: GS / ADD / MV of a cluster level whose output is a
//     replicated vector): every row value is sent to every CTA with st.async, which signals
//     the receiver's mbarrier (complete_tx, 8 bytes); a CTA proceeds once its mbarrier has
//     received the phase's 8*rows bytes.  No release fence and no cluster barrier: the
//     sender does not wait for acknowledgements (MGM_TRACE=2 timeline: the release of
//     barrier.cluster.arrive cost ~1000 cycles per phase).  Two mbarriers alternate
//     (k & 1); each is re-armed for phase k + 2 as soon as phase k completed, which precedes
//     any byte of phase k + 2 (a sender needs this CTA's phase k + 1 values first), so the
//     tx-count never goes negative.  Write-after-read: a sender can write values of phase
//     k + 1 into this CTA's copy only after receiving all of this CTA's phase-k values, and
//     each value is sent after the reads of its row group;
//   * everything else (outputs in global memory, zeroing, local <-> cluster transitions):
//     barrier.cluster arrive.release / wait.acquire.
// Every output element is produced by one thread group with a fixed summation order, so
// the kernel is deterministic.  Shifted problems only (the Poisson border terms run on the
// per-kernel path).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "solve_kernels.cuh"

namespace mgm {

enum : int { BP_ZERO = 0, BP_GS = 1, BP_RES = 2, BP_MVZ = 3, BP_ADD = 4, BP_MV = 5, BP_STORE = 6, BP_LOAD = 7 };
constexpr int BOT_THREADS = 512;
constexpr int BOT_MAX_PHASES = 1024;
constexpr int BOT_FRAG = 9;  // max operator entries per thread held in registers

struct BPhase {
    int op, local, r0, r1;
    int tpr_log2;  // threads per row = 1 << tpr_log2 (<= 32)
    int W;         // ELL row stride
    int xo;        // shared byte offset of the gathered vector, or -1: global x
    int yo;        // shared byte offset of the output vector (replicated), or -1: global y
    int zo;        // shared byte offset of the vector zeroed by BP_MVZ
    int fpre;      // 1: f may be prefetched with the operator row (not written by the previous phase)
    int mb;        // >= 0: "data-synchronised" phase number k (see below), -1: barrier phase
    int arm;       // bytes every CTA receives in data-synchronised phase k + 2 (0: none)
    const int* col;
    const double* val;
    const double* x;  // global gathered vector (xo < 0)
    double* y;        // global output (yo < 0) / BP_STORE destination
    const double* f;
    const double* dinv;
};

// entries per thread for a given threads-per-row (the host picks tpr so that W <= tpr*CH)
__host__ __device__ constexpr int bot_ch(int tpr) {
    return tpr >= 32 ? 4 : tpr == 16 ? 5 : tpr == 8 ? 9 : tpr == 4 ? 8 : tpr == 2 ? 4 : 8;
}

__device__ __forceinline__ int ld_keep_i32(const int* p, uint64_t pol) {
    int v;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_keep_f64(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void dsm_st_rank(uint32_t local_addr, unsigned rank, double v) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(r), "d"(v) : "memory");
}
// remote store that signals the receiver's mbarrier with 8 transaction bytes
__device__ __forceinline__ void dsm_st_async_rank(uint32_t local_addr, uint32_t local_bar, unsigned rank, double v) {
    uint32_t r, b;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(b) : "r"(local_bar), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(r),
                 "l"(__double_as_longlong(v)), "r"(b)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint32_t bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// wait for the phase of the given parity; a bounded spin (seconds) traps instead of hanging
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned parity) {
    for (long long it = 0;; ++it) {
        uint32_t done;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
        if (it > (1ll << 26)) asm volatile("trap;");
    }
}
// fine-grained phase timeline (MGM_TRACE=2, diagnostics): SM clock after the named value
__device__ __forceinline__ long long clk_after(double v) {
    long long t;
    asm volatile("{ .reg .f64 d; mov.f64 d, %1; mov.u64 %0, %%clock64; }" : "=l"(t) : "d"(v));
    return t;
}
__device__ __forceinline__ long long clk_after_i(int v) {
    long long t;
    asm volatile("{ .reg .s32 q; mov.s32 q, %1; mov.u64 %0, %%clock64; }" : "=l"(t) : "r"(v));
    return t;
}

// The operator entries of one thread's first row of a phase, held in registers.
struct BFrag {
    int c[BOT_FRAG];
    double a[BOT_FRAG];
    double dinv;  // 1/a_rr (GS phases, lane 0)
    double f;     // f[row] when the phase allows the prefetch (lane 0)
};

template <int TPR>
__device__ __forceinline__ void bfrag_load(BFrag& fr, const BPhase& P, int row, int lane, uint64_t pol) {
    constexpr int CH = bot_ch(TPR);
    const bool live = row < P.r1 && P.op != BP_ZERO && P.op != BP_STORE && P.op != BP_LOAD;  // no operator
    const int64_t base = (int64_t)row * P.W;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const int k = lane + q * TPR;
        const bool ok = live && k < P.W;
        fr.c[q] = ok ? ld_keep_i32(P.col + base + k, pol) : -1;
        fr.a[q] = ok ? ld_keep_f64(P.val + base + k, pol) : 0.0;
    }
    fr.dinv = (live && lane == 0 && P.op == BP_GS) ? ld_keep_f64(P.dinv + row, pol) : 0.0;
    fr.f = (live && lane == 0 && P.fpre && (P.op == BP_GS || P.op == BP_RES)) ? P.f[row] : 0.0;
}

// store v at byte offset off + 8*row of every CTA's copy (lanes of the row group share the
// C stores)
__device__ __forceinline__ void bcast_store(uint32_t sbase, int off, int row, double v, int lane, int tpr, int cs) {
    const uint32_t a = sbase + (uint32_t)off + ((uint32_t)row << 3);
    for (int k = lane; k < cs; k += tpr) dsm_st_rank(a, (unsigned)k, v);
}
__device__ __forceinline__ void bcast_store_async(uint32_t sbase, int off, int row, double v, int lane, int tpr, int cs,
                                                  uint32_t bar) {
    const uint32_t a = sbase + (uint32_t)off + ((uint32_t)row << 3);
    for (int k = lane; k < cs; k += tpr) dsm_st_async_rank(a, bar, (unsigned)k, v);
}

template <int TPR>
__device__ __forceinline__ void bottom_phase(const BPhase& P, BFrag& fr, int g, int nthr, const char* smem,
                                             uint32_t sbase, int cs, uint64_t pol, long long* tr, uint32_t mbar) {
    constexpr int CH = bot_ch(TPR);
    const int lane = g & (TPR - 1);
    const int ngroups = nthr / TPR;
    const int nrows = P.r1 - P.r0;
    const double* xs = reinterpret_cast<const double*>(smem + (P.xo >= 0 ? P.xo : 0));
    const double* ys = reinterpret_cast<const double*>(smem + (P.yo >= 0 ? P.yo : 0));
    for (int base = 0; base < nrows; base += ngroups) {  // uniform trip count across threads
        const int row = P.r0 + base + g / TPR;
        const bool live = row < P.r1;
        if (base != 0) bfrag_load<TPR>(fr, P, row, lane, pol);  // rows after the first (in place:
                                                                // fr is reloaded for the next phase anyway)
        // epilogue operand issued together with the gathers
        double ev = 0.0;
        if (live && lane == 0) {
            if (P.op == BP_GS || P.op == BP_RES) ev = P.fpre && base == 0 ? fr.f : P.f[row];
            else if (P.op == BP_ADD) ev = ys[row];
        }
        double xv[CH];
        if (P.xo >= 0) {
#pragma unroll
            for (int q = 0; q < CH; ++q) xv[q] = fr.c[q] >= 0 ? xs[fr.c[q]] : 0.0;
        } else {
#pragma unroll
            for (int q = 0; q < CH; ++q) xv[q] = fr.c[q] >= 0 ? P.x[fr.c[q]] : 0.0;
        }
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < CH; ++q) acc = fma(fr.a[q], xv[q], acc);
        for (int k = lane + CH * TPR; k < P.W; k += TPR) {  // rows wider than TPR*CH (rare)
            if (!live) break;
            const int c = ld_keep_i32(P.col + (int64_t)row * P.W + k, pol);
            acc = fma(ld_keep_f64(P.val + (int64_t)row * P.W + k, pol), P.xo >= 0 ? xs[c] : P.x[c], acc);
        }
        if (tr && base == 0) tr[1] = clk_after(acc);
#pragma unroll
        for (int o = TPR >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        // every lane of the group holds acc; lane 0 computes the row's value, the group stores
        double out = 0.0;
        if (live && lane == 0) {
            switch (P.op) {
                case BP_GS: out = xv[0] + (ev - acc) * fr.dinv; break;  // xv[0] = x[row] (diagonal first)
                case BP_RES: out = ev - acc; break;
                case BP_ADD: out = ev + acc; break;
                default: out = acc; break;  // BP_MVZ, BP_MV
            }
        }
        out = __shfl_sync(0xffffffffu, out, (int)(threadIdx.x & 31) & ~(TPR - 1));
        if (tr && base == 0) tr[2] = clk_after(out);
        if (live) {
            if (P.yo >= 0) {
                if (P.mb >= 0) bcast_store_async(sbase, P.yo, row, out, lane, TPR, cs, mbar + 8u * (unsigned)(P.mb & 1));
                else bcast_store(sbase, P.yo, row, out, lane, TPR, cs);
            } else if (lane == 0) {
                P.y[row] = out;
            }
            if (P.op == BP_MVZ) bcast_store(sbase, P.zo, row, 0.0, lane, TPR, cs);
        }
        if (tr && base == 0) tr[3] = clock64();
    }
}

// Threads per row: 2, 8 or 32 only (BOT_TPR_MASK; the host picks among these).  Fewer
// specialisations keep the kernel's code smaller -- the phase loop is instruction-latency
// bound and its code does not fit the instruction cache.
constexpr unsigned BOT_TPR_MASK = (1u << 1) | (1u << 3) | (1u << 5);
__device__ __forceinline__ void bfrag_load_any(BFrag& fr, const BPhase& P, int g, uint64_t pol) {
    const int row = P.r0 + (g >> P.tpr_log2);
    const int lane = g & ((1 << P.tpr_log2) - 1);
    switch (P.tpr_log2) {
        case 1: bfrag_load<2>(fr, P, row, lane, pol); break;
        case 3: bfrag_load<8>(fr, P, row, lane, pol); break;
        default: bfrag_load<32>(fr, P, row, lane, pol); break;
    }
}
__device__ __forceinline__ void bottom_phase_any(const BPhase& P, BFrag& fr, int g, int nthr, const char* smem,
                                                 uint32_t sbase, int cs, uint64_t pol, long long* tr,
                                                 uint32_t mbar) {
    switch (P.tpr_log2) {
        case 1: bottom_phase<2>(P, fr, g, nthr, smem, sbase, cs, pol, tr, mbar); break;
        case 3: bottom_phase<8>(P, fr, g, nthr, smem, sbase, cs, pol, tr, mbar); break;
        default: bottom_phase<32>(P, fr, g, nthr, smem, sbase, cs, pol, tr, mbar); break;
    }
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_nctas() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// smem: [phase table (nph x BPhase)][replicated vectors at the offsets in the phases]
// TRACE = false: the production instance, no diagnostics code in the phase loop (the trace
// checks cost instructions in a loop that is instruction-latency bound); TRACE = true runs
// when MGM_TRACE is set at setup.
template <bool TRACE>
__global__ void __launch_bounds__(BOT_THREADS, 1)
    k_vcycle_bottom_t(const BPhase* __restrict__ gphases, int nph, unsigned long long* __restrict__ trace, PfList pf,
                      int arm0, int arm1) {
    extern __shared__ __align__(16) char smem[];
    __shared__ __align__(8) unsigned long long mbars[2];  // data-synchronised phases k & 1
    const uint32_t mbar = (uint32_t)__cvta_generic_to_shared(mbars);
    const BPhase* phases = reinterpret_cast<const BPhase*>(smem);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    pdl_trigger();
    l2_prefetch_share(pf);  // (opt-in L2 prefetch pacing, off by default)
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    {
        const int nw = nph * (int)(sizeof(BPhase) / 8);
        const unsigned long long* src = reinterpret_cast<const unsigned long long*>(gphases);
        unsigned long long* dst = reinterpret_cast<unsigned long long*>(smem);
        for (int i = threadIdx.x; i < nw; i += BOT_THREADS) dst[i] = src[i];
        if (threadIdx.x == 0) {
            mbar_init(mbar, 1);
            mbar_init(mbar + 8, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            if (arm0 > 0) mbar_arm(mbar, (unsigned)arm0);
            if (arm1 > 0) mbar_arm(mbar + 8, (unsigned)arm1);
        }
        __syncthreads();
    }
    const int rank = (int)cluster_rank();
    const int cs = (int)cluster_nctas();
    const int nthr_cl = cs * BOT_THREADS;
    const int g_cl = rank * BOT_THREADS + (int)threadIdx.x;
    // prologue (immutable data only): phase 0's operator rows
    BFrag fr;
    {
        const BPhase& P = phases[0];
        if (!P.local || rank == 0) bfrag_load_any(fr, P, P.local ? (int)threadIdx.x : g_cl, pol);
    }
    pdl_wait();
    cluster_arrive();  // every CTA's shared memory is live before any remote store
    cluster_wait();
    // fine timeline (diagnostics): thread 0 of CTA 0 and of the last CTA, 8 clocks per phase
    long long* ftr = nullptr;
    if (TRACE && trace && trace[BOT_MAX_PHASES - 1] == 2ull && threadIdx.x == 0 && (rank == 0 || rank == cs - 1))
        ftr = reinterpret_cast<long long*>(trace) + BOT_MAX_PHASES + (rank == 0 ? 0 : 8 * BOT_MAX_PHASES);
    for (int q = 0; q < nph; ++q) {
        if (TRACE && trace && rank == 0 && threadIdx.x == 0) trace[q] = gtimer();  // diagnostics (MGM_TRACE)
        long long* tr = TRACE && ftr ? ftr + 8 * q : nullptr;
        if (TRACE && tr) { tr[0] = clock64(); tr[7] = clk_after_i(fr.c[0]); }
        const BPhase P = phases[q];
        if (P.op == BP_ZERO) {  // every CTA zeroes its own copy
            double* y = reinterpret_cast<double*>(smem + P.yo);
            for (int r = P.r0 + threadIdx.x; r < P.r1; r += BOT_THREADS) y[r] = 0.0;
        } else if (P.op == BP_STORE) {  // copy back to HBM, split over the cluster
            const double* y = reinterpret_cast<const double*>(smem + P.yo);
            for (int r = P.r0 + g_cl; r < P.r1; r += nthr_cl) P.y[r] = y[r];
        } else if (P.op == BP_LOAD) {  // every CTA fills its own copy from HBM
            double* y = reinterpret_cast<double*>(smem + P.yo);
            for (int r = P.r0 + threadIdx.x; r < P.r1; r += BOT_THREADS) y[r] = P.x[r];
        } else if (!P.local || rank == 0) {
            bottom_phase_any(P, fr, P.local ? (int)threadIdx.x : g_cl, P.local ? BOT_THREADS : nthr_cl, smem, sbase,
                             cs, pol, tr, mbar);
        }
        if (q + 1 == nph) break;
        const BPhase& N = phases[q + 1];
        const bool part = !P.local || rank == 0;
        const bool npart = !N.local || rank == 0;
        const bool ll = P.local && N.local;  // CTA 0 only; the other CTAs skip local phases
        if (P.mb < 0 && !ll) {
            // zeroing / plain remote stores (generic proxy) before later st.async writes to the
            // same words
            if (P.op == BP_ZERO || P.op == BP_MVZ || P.op == BP_LOAD || P.local)
                asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
            cluster_arrive();
        }
        if (TRACE && tr) tr[4] = clock64();
        // the next phase's operator rows, overlapping the synchronisation (one call site: the
        // loop is instruction-latency bound and its code size matters)
        if (npart) bfrag_load_any(fr, N, N.local ? (int)threadIdx.x : g_cl, pol);
        if (TRACE && tr) tr[5] = clock64();
        if (P.mb >= 0) {  // data-synchronised: wait for this phase's bytes, re-arm for phase mb + 2
            const uint32_t b = mbar + 8u * (unsigned)(P.mb & 1);
            mbar_wait(b, (unsigned)((P.mb >> 1) & 1));
            if (threadIdx.x == 0 && P.arm > 0) mbar_arm(b, (unsigned)P.arm);
        } else if (ll) {
            if (part) __syncthreads();
        } else {
            cluster_wait();
        }
        if (TRACE && tr) tr[6] = clock64();
    }
    cluster_arrive();  // no CTA exits while others may still store into its shared memory
    cluster_wait();
}

// y = A x for a dense row-major m x m A (the explicit coarsest inverse when the coarsest level
// is large, e.g. cfg5's 4096 rows = 134 MB: a grid-wide GEMV between the two halves of the
// bottom instead of the cluster's 16 SMs).  One warp per row, fixed reduction order.
__global__ void __launch_bounds__(128) k_dense_gemv(int m, const double* __restrict__ A, const double* __restrict__ x,
                                                    double* __restrict__ y) {
    pdl_trigger();
    const int row = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    pdl_wait();
    if (row >= m) return;
    const double* a = A + (int64_t)row * m;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    int c = lane;
    for (; c + 96 < m; c += 128) {
        acc0 = fma(a[c], x[c], acc0);
        acc1 = fma(a[c + 32], x[c + 32], acc1);
        acc2 = fma(a[c + 64], x[c + 64], acc2);
        acc3 = fma(a[c + 96], x[c + 96], acc3);
    }
    for (; c < m; c += 32) acc0 = fma(a[c], x[c], acc0);
    double acc = (acc0 + acc1) + (acc2 + acc3);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[row] = acc;
}

// the two instances (the host picks by MGM_TRACE)
inline void* bottom_kernel_ptr(bool trace) {
    return trace ? (void*)k_vcycle_bottom_t<true> : (void*)k_vcycle_bottom_t<false>;
}

}  // namespace mgm
