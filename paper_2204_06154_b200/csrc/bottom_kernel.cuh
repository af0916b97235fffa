// The bottom of the V-cycle in ONE kernel launch: levels J..p-1 of Alg. 3 run
// by a single thread-block cluster (16 CTAs on one GPC, or 8), as a list of "phases"
// separated by barriers instead of kernel boundaries.
//
// Why: on the lower levels a colour of the Gauss-Seidel sweep holds a few hundred rows,
// and a kernel boundary (~0.7-1 us with PDL inside a graph, measured in
// tools/micro/sync_costs.cu) plus the kernel's own chain of dependent global-memory round
// trips (~2 us) dwarfs its work.  The design keeps every step of a phase on chip:
//   * VECTORS (u_j, f_j, t_j of levels J..p-1) live in distributed shared memory: entry r
//     of a cluster-level vector sits in CTA (r mod C) at slot r / C; vectors of the
//     smallest ("local") levels sit whole in CTA 0.  Each CTA computes exactly the rows it
//     owns, so every store is to its own shared memory; gathers are ld.shared (local) or
//     ld.shared::cluster (remote, ~200 cycles).
//   * OPERATORS stream from global memory (L2-resident, evict_last) into a 4-stage shared
//     memory ring by TMA bulk copies (cp.async.bulk + mbarrier complete_tx), issued several
//     tiles ahead by one thread, so that the consumers never wait on a global load: at
//     setup every phase's rows are stored per CTA as one contiguous "chunk" of row records
//     [1/a_rr | W values | W columns | pad to 16 B], in exactly the order the CTA
//     processes them (tools/micro measurements: a register prefetch one phase ahead left
//     ~600-1000 cycles of exposed global latency per phase).
//   * BARRIERS: barrier.cluster between phases (~0.25 us), __syncthreads between two
//     local phases (run by CTA 0 alone) and between the tiles of one phase.
// The first phase loads f_J from global memory (written by the per-kernel restriction of
// level J-1) and zeroes u_J; the last phase stores u_J back for the per-kernel up-path.
//
// A phase applies one operator to its rows with one of these epilogues
// (acc = sum_k val_k x[col_k], summed per thread in k order, then a shuffle tree):
//   BP_LOAD  y[r] = g[r], z[r] = 0                     (f_J from global, e_J = 0: Alg. 3 line 7)
//   BP_GS    y[r] = x[r] + (f[r] - acc) / a_rr         (one colour of the sweep; y = x = u;
//                                                       stored as a multiply by 1/a_rr)
//   BP_RES   y[r] = f[r] - acc                         (t_j = r_j - L_j e_j)
//   BP_MVZ   y[r] = acc, z[r] = 0                      (r_{j+1} = R_j t_j, and e_{j+1} = 0)
//   BP_ADD   y[r] += acc                               (e_j += P_j e_{j+1})
//   BP_MV    y[r] = acc                                (coarsest: e_p = L_p^{-1} r_p, dense rows)
//   BP_STORE g[r] = x[r]                               (e_J back to global)
// Every output element is produced by one thread group with a fixed summation order, so
// the kernel is deterministic.  Shifted problems only (the Poisson border terms run on the
// per-kernel path).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "solve_kernels.cuh"

namespace mgm {

enum : int { BP_LOAD = 0, BP_GS = 1, BP_RES = 2, BP_MVZ = 3, BP_ADD = 4, BP_MV = 5, BP_STORE = 6 };
constexpr int BOT_THREADS = 512;
constexpr int BOT_MAX_PHASES = 1024;
constexpr int BOT_STAGES = 4;
constexpr int BOT_STAGE_BYTES = 24 * 1024;  // default ring stage (MGM_BOT_STAGE overrides)

// Vectors in distributed shared memory: byte offset of the slice (same in every CTA) and
// distribution shift s: entry r is in CTA (r & (2^s - 1)) at slot r >> s (s = 0: CTA 0).
// Rows of a phase: local phases (CTA 0) take r0 + i; distributed phases give CTA k the
// rows r = k (mod C) of [r0, r1) in ascending order.
struct BPhase {
    int op, local, r0, r1;
    int tpr_log2;  // threads per row = 1 << tpr_log2 (<= 32)
    int W;         // entries per row record
    int rb;        // row record bytes (multiple of 16)
    int tile_rows; // rows per ring stage
    int xo, xs;    // gathered vector
    int yo, ys;    // output vector (f and z have the same distribution)
    int fo, zo;
    double* g;     // global vector of BP_LOAD / BP_STORE
};

// Per-CTA chunk of a phase in the operator byte stream.
struct BChunk {
    unsigned long long off;  // byte offset of the first row record
    int nrows;
    int pad;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t dsm_addr(uint32_t sbase, int off, int s, int c) {
    const uint32_t local = sbase + (uint32_t)off + ((uint32_t)(c >> s) << 3);
    const uint32_t cta = (uint32_t)c & ((1u << s) - 1u);
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(cta));
    return r;
}
__device__ __forceinline__ double dsm_ld(uint32_t a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void dsm_st(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const void* src, unsigned bytes, uint32_t bar, uint64_t pol) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after generic reads of the stage
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// ---------------------------------------------------------------- consumer: one tile
// Warps 0..14 compute (BOT_CONSUMERS threads); warp 15 issues the TMA tile copies.
constexpr int BOT_CONSUMERS = BOT_THREADS - 32;

template <int TPR>
__device__ __forceinline__ void consume_tile(const BPhase& P, const char* tile, int nr, int i0, int rank,
                                             int cs_log2, char* smem, uint32_t sbase) {
    const int lane = (int)threadIdx.x & (TPR - 1);
    constexpr int groups = BOT_CONSUMERS / TPR;
    const bool xloc = P.xs == 0 && rank == 0;  // gathered vector whole in this CTA's shared memory
    const double* xl = reinterpret_cast<const double*>(smem + P.xo);
    for (int b = 0; b < nr; b += groups) {  // uniform trip count within the CTA
        const int it = b + (int)threadIdx.x / TPR;
        const bool live = it < nr;
        const char* rec = tile + (size_t)(live ? it : 0) * P.rb;
        const double* vals = reinterpret_cast<const double*>(rec + 8);
        const int* cols = reinterpret_cast<const int*>(rec + 8 + 8 * P.W);
        const int i = i0 + it;  // row index within this CTA's chunk
        const int row = P.local ? P.r0 + i : P.r0 + ((rank - P.r0) & ((1 << cs_log2) - 1)) + (i << cs_log2);
        const int slot = row >> P.ys;
        double ev = 0.0;
        if (live && lane == 0) {
            if (P.op == BP_GS || P.op == BP_RES) ev = reinterpret_cast<const double*>(smem + P.fo)[slot];
            else if (P.op == BP_ADD) ev = reinterpret_cast<const double*>(smem + P.yo)[slot];
        }
        double acc = 0.0, x0 = 0.0;
        const int W = live ? P.W : 0;
        for (int k0 = lane; k0 < W; k0 += 4 * TPR) {  // 4 independent gathers in flight per thread
            int c[4];
            double v[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = k0 + u * TPR;
                c[u] = k < W ? cols[k] : -1;
                v[u] = k < W ? vals[k] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                xv[u] = c[u] < 0 ? 0.0 : (xloc ? xl[c[u]] : dsm_ld(dsm_addr(sbase, P.xo, P.xs, c[u])));
            if (k0 == lane) x0 = xv[0];
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = fma(v[u], xv[u], acc);
        }
#pragma unroll
        for (int o = TPR >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (live && lane == 0) {
            double out;
            switch (P.op) {
                case BP_GS: out = x0 + (ev - acc) * *reinterpret_cast<const double*>(rec); break;  // x0 = x[row]
                case BP_RES: out = ev - acc; break;
                case BP_ADD: out = ev + acc; break;
                default: out = acc; break;  // BP_MVZ, BP_MV
            }
            reinterpret_cast<double*>(smem + P.yo)[slot] = out;
            if (P.op == BP_MVZ) reinterpret_cast<double*>(smem + P.zo)[slot] = 0.0;
        }
    }
}

__device__ __forceinline__ void consume_tile_any(const BPhase& P, const char* tile, int nr, int i0, int rank,
                                                 int cs_log2, char* smem, uint32_t sbase) {
    switch (P.tpr_log2) {
        case 0: consume_tile<1>(P, tile, nr, i0, rank, cs_log2, smem, sbase); break;
        case 1: consume_tile<2>(P, tile, nr, i0, rank, cs_log2, smem, sbase); break;
        case 2: consume_tile<4>(P, tile, nr, i0, rank, cs_log2, smem, sbase); break;
        case 3: consume_tile<8>(P, tile, nr, i0, rank, cs_log2, smem, sbase); break;
        case 4: consume_tile<16>(P, tile, nr, i0, rank, cs_log2, smem, sbase); break;
        default: consume_tile<32>(P, tile, nr, i0, rank, cs_log2, smem, sbase); break;
    }
}

// rows of an operator-free phase (BP_LOAD / BP_STORE) owned by this CTA
__device__ __forceinline__ void copy_phase(const BPhase& P, int rank, int cs_log2, char* smem) {
    const int cm = (1 << cs_log2) - 1;
    const int start = P.local ? P.r0 : P.r0 + ((rank - P.r0) & cm);
    const int stride = P.local ? 1 : 1 << cs_log2;
    const int s = P.op == BP_LOAD ? P.ys : P.xs;
    for (int row = start + (int)threadIdx.x * stride; row < P.r1; row += BOT_THREADS * stride) {  // all 16 warps
        if (P.op == BP_LOAD) {
            reinterpret_cast<double*>(smem + P.yo)[row >> s] = P.g[row];
            reinterpret_cast<double*>(smem + P.zo)[row >> s] = 0.0;
        } else {
            P.g[row] = reinterpret_cast<const double*>(smem + P.xo)[row >> s];
        }
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Per-CTA tile list entry (host-built, in consumption order).
struct BTile {
    unsigned long long off;  // byte offset in the operator stream
    unsigned bytes;
    unsigned pad;
};

// smem: [phase table][per-CTA chunk table][tile list][mbarriers][ring][vectors]
// (offsets: tiles_off, ring_off = bars + 64; vector offsets in the phase table are absolute).
// Launch: one cluster of C CTAs.
__global__ void __launch_bounds__(BOT_THREADS, 1)
    k_vcycle_bottom(const BPhase* __restrict__ gphases, const BChunk* __restrict__ gchunks,
                    const BTile* __restrict__ gtiles, const int* __restrict__ gntiles, const char* __restrict__ ops,
                    int nph, int cs_log2, int tiles_off, int ring_off, int stage_bytes,
                    unsigned long long* __restrict__ trace) {
    extern __shared__ __align__(128) char smem[];
    BPhase* phases = reinterpret_cast<BPhase*>(smem);
    BChunk* chunks = reinterpret_cast<BChunk*>(smem + nph * sizeof(BPhase));
    BTile* tiles = reinterpret_cast<BTile*>(smem + tiles_off);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t bars = sbase + ring_off - 64;
    const uint32_t ring = sbase + ring_off;
    const int rank = (int)cluster_rank();
    const int cs = 1 << cs_log2;
    const bool producer = threadIdx.x == BOT_CONSUMERS;  // lane 0 of warp 15
    pdl_trigger();
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const int ntiles = gntiles[rank];
    {  // stage the (immutable) phase table, this CTA's chunk column and tile list
        const int nw = nph * (int)(sizeof(BPhase) / 8);
        const unsigned long long* src = reinterpret_cast<const unsigned long long*>(gphases);
        unsigned long long* dst = reinterpret_cast<unsigned long long*>(smem);
        for (int i = threadIdx.x; i < nw; i += BOT_THREADS) dst[i] = src[i];
        for (int q = threadIdx.x; q < nph; q += BOT_THREADS) chunks[q] = gchunks[(size_t)q * cs + rank];
        const BTile* mt = gtiles + (size_t)rank * gntiles[cs];  // gntiles[cs] = row stride of the tile table
        for (int t = threadIdx.x; t < ntiles; t += BOT_THREADS) tiles[t] = mt[t];
        if (threadIdx.x == 0) {
            for (int s = 0; s < BOT_STAGES; ++s) mbar_init(bars + 8 * s, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    int issued = 0;
    auto issue = [&](int upto) {  // producer: issue tiles [issued, min(upto, ntiles))
        for (; issued < upto && issued < ntiles; ++issued) {
            const int stage = issued % BOT_STAGES;
            const BTile T = tiles[issued];
            mbar_expect_tx(bars + 8 * stage, T.bytes);
            tma_load(ring + stage * stage_bytes, ops + T.off, T.bytes, bars + 8 * stage, pol);
        }
    };
    if (producer) issue(BOT_STAGES - 1);  // operators are immutable: stream before the dependency wait
    pdl_wait();
    cluster_arrive();  // every CTA's shared memory is live before any remote access
    cluster_wait();
    int consumed = 0;
    for (int q = 0; q < nph; ++q) {
        const BPhase P = phases[q];  // registers
        if (trace && rank == 0 && threadIdx.x == 0) trace[q] = gtimer();  // diagnostics (MGM_TRACE)
        // diagnostics: clock64 of thread 0 of CTA 0 (phase start, first tile ready, phase end)
        unsigned long long* st = (trace && rank == 0 && threadIdx.x == 0) ? trace + BOT_MAX_PHASES + 4 * q : nullptr;
        if (st) { st[0] = clock64(); st[1] = st[0]; }
        const bool part = !P.local || rank == 0;
        if (part) {
            if (P.op == BP_LOAD || P.op == BP_STORE) {
                copy_phase(P, rank, cs_log2, smem);
            } else {
                const int nrows = chunks[q].nrows;
                for (int i0 = 0; i0 < nrows; i0 += P.tile_rows) {
                    if (i0 > 0) __syncthreads();  // the previous tile's stage may be refilled
                    const int stage = consumed % BOT_STAGES;
                    if (producer) issue(consumed + BOT_STAGES);
                    if (threadIdx.x < BOT_CONSUMERS) {
                        mbar_wait(bars + 8 * stage, (unsigned)(consumed / BOT_STAGES) & 1u);
                        if (st && i0 == 0) st[1] = clock64();
                        consume_tile_any(P, smem + ring_off + stage * stage_bytes, min(P.tile_rows, nrows - i0),
                                         i0, rank, cs_log2, smem, sbase);
                    }
                    ++consumed;
                }
            }
        }
        if (st) st[2] = clock64();
        if (q + 1 == nph) break;
        if (P.local && phases[q + 1].local) {  // CTA 0 only; the other CTAs skip local phases
            if (part) __syncthreads();
        } else {
            cluster_arrive();
            cluster_wait();
        }
        if (st) st[3] = clock64();
    }
    cluster_arrive();  // no CTA exits while others may still access its shared memory
    cluster_wait();
}

}  // namespace mgm
