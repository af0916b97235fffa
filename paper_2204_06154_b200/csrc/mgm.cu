// libmgm: context, setup orchestration (Alg. 2), V-cycle (Alg. 3)
// captured as a CUDA graph, right-preconditioned GMRES, standalone MGM
// and the C ABI declared in include/mgm.h.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mgm.h"
#include "mgm_internal.h"
#include "solve_kernels.cuh"
#include "bottom_kernel.cuh"
#include "batch_kernels.cuh"
#include "dense_bottom.cuh"

using namespace mgm;

// ---------------------------------------------------------------------------------------
// NCCL, loaded at run time (dlopen "libnccl.so.2": inside a PyTorch process this resolves
// to the NCCL torch already loaded), so libmgm has no link-time NCCL dependency.
// ---------------------------------------------------------------------------------------
namespace {
struct NcclApi {
    bool tried = false, ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) =
        nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    if (!api.tried) {
        api.tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
            api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
            api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
            api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
            api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
            api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
            api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
            api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.AllReduce &&
                     api.GroupStart && api.GroupEnd && api.GetErrorString && api.Send && api.Recv;
        }
    }
    return api;
}
// cuSOLVER (dense LU of the coarsest operator at setup), loaded at run time like NCCL.
struct CusolverApi {
    bool tried = false, ok = false;
    cusolverStatus_t (*Create)(cusolverDnHandle_t*) = nullptr;
    cusolverStatus_t (*Destroy)(cusolverDnHandle_t) = nullptr;
    cusolverStatus_t (*SetStream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
    cusolverStatus_t (*GetrfBuf)(cusolverDnHandle_t, int, int, double*, int, int*) = nullptr;
    cusolverStatus_t (*Getrf)(cusolverDnHandle_t, int, int, double*, int, double*, int*, int*) = nullptr;
    cusolverStatus_t (*Getrs)(cusolverDnHandle_t, cublasOperation_t, int, int, const double*, int, const int*,
                              double*, int, int*) = nullptr;
};
CusolverApi& cusolver() {
    static CusolverApi api;
    if (!api.tried) {
        api.tried = true;
        void* h = dlopen("libcusolver.so.11", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libcusolver.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.Create = (decltype(api.Create))dlsym(h, "cusolverDnCreate");
            api.Destroy = (decltype(api.Destroy))dlsym(h, "cusolverDnDestroy");
            api.SetStream = (decltype(api.SetStream))dlsym(h, "cusolverDnSetStream");
            api.GetrfBuf = (decltype(api.GetrfBuf))dlsym(h, "cusolverDnDgetrf_bufferSize");
            api.Getrf = (decltype(api.Getrf))dlsym(h, "cusolverDnDgetrf");
            api.Getrs = (decltype(api.Getrs))dlsym(h, "cusolverDnDgetrs");
            api.ok = api.Create && api.Destroy && api.SetStream && api.GetrfBuf && api.Getrf && api.Getrs;
        }
    }
    return api;
}
}  // namespace

// ---------------------------------------------------------------------------------------
// Transport of the distributed solve: grouped halo
// send/receive of ghost values, sum-allreduce of Krylov scalars, all-gather of the first
// replicated level.  NcclTransport: one process per GPU (ncclSend/ncclRecv in a group,
// ncclAllReduce, ncclBroadcast per root), capturable in the V-cycle's CUDA graph.
// FakeTransport: R ranks on ONE GPU inside one process, each driven by its own host thread
// (test hook, mgm_fake_group_create): the same collective calls, implemented with device
// copies between the ranks' buffers ordered by CUDA events and a host barrier -- the
// distributed code path itself is unchanged.  Eager only (not capturable).
// ---------------------------------------------------------------------------------------
namespace mgm {
struct Xfer {
    int peer;
    const double* send;
    i64 ns;
    double* recv;
    i64 nr;
};
struct Transport {
    int rank = 0, nranks = 1;
    virtual ~Transport() {}
    virtual bool exchange(const std::vector<Xfer>& x, cudaStream_t st) = 0;
    virtual bool allreduce_sum(double* buf, i64 n, cudaStream_t st) = 0;
    // out[off[q] .. off[q+1]) <- rank q's `mine` (n = off[rank+1] - off[rank] on this rank)
    virtual bool allgatherv(const double* mine, double* out, const std::vector<i64>& off, cudaStream_t st) = 0;
    virtual bool capturable() const = 0;
};

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    bool exchange(const std::vector<Xfer>& x, cudaStream_t st) override {
        if (x.empty()) return true;
        bool ok = nccl().GroupStart() == ncclSuccess;
        for (const Xfer& e : x) {
            if (e.ns > 0) ok &= nccl().Send(e.send, (size_t)e.ns, ncclFloat64, e.peer, comm, st) == ncclSuccess;
            if (e.nr > 0) ok &= nccl().Recv(e.recv, (size_t)e.nr, ncclFloat64, e.peer, comm, st) == ncclSuccess;
        }
        ok &= nccl().GroupEnd() == ncclSuccess;
        return ok;
    }
    bool allreduce_sum(double* buf, i64 n, cudaStream_t st) override {
        return nccl().AllReduce(buf, buf, (size_t)n, ncclFloat64, ncclSum, comm, st) == ncclSuccess;
    }
    bool allgatherv(const double* mine, double* out, const std::vector<i64>& off, cudaStream_t st) override {
        bool ok = nccl().GroupStart() == ncclSuccess;
        for (int q = 0; q < nranks; ++q) {
            const i64 c = off[q + 1] - off[q];
            if (c > 0)
                ok &= nccl().Broadcast(q == rank ? mine : out + off[q], out + off[q], (size_t)c, ncclFloat64, q, comm,
                                       st) == ncclSuccess;
        }
        ok &= nccl().GroupEnd() == ncclSuccess;
        return ok;
    }
    bool capturable() const override { return true; }
    ~NcclTransport() override {
        if (comm) nccl().CommDestroy(comm);
    }
};

// in-process group of R fake ranks (one host thread each, same GPU)
struct FakeGroup {
    int R = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    // posted by each rank for the current collective
    std::vector<std::vector<Xfer>> posted;   // [rank] its sends (peer, ptr, count)
    std::vector<cudaEvent_t> ready, done;    // [rank]
    std::vector<const double*> gather_src;   // [rank]
    std::vector<double*> reduce_buf;         // [rank]
    std::vector<std::vector<double*>> bases; // [rank] the u / t pointers of its distributed levels (peer stores)
    explicit FakeGroup(int r) : R(r), posted(r), ready(r), done(r), gather_src(r), reduce_buf(r), bases(r) {
        for (int q = 0; q < R; ++q) {
            cudaEventCreateWithFlags(&ready[q], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming);
        }
    }
    ~FakeGroup() {
        for (int q = 0; q < R; ++q) {
            cudaEventDestroy(ready[q]);
            cudaEventDestroy(done[q]);
        }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = generation;
        if (++arrived == R) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != g; });
        }
    }
};

__global__ void k_sum_ranks(i64 n, int R, double* const* bufs, double* out) {
    for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < R; ++q) s += bufs[q][i];
        out[i] = s;
    }
}

struct FakeTransport : Transport {
    FakeGroup* g = nullptr;
    double* scratch = nullptr;  // this rank's copy for the allreduce
    i64 scratch_n = 0;
    double** d_bufs = nullptr;  // device table of the ranks' scratch pointers
    // every rank posts, then waits for the others' data to be ready and copies what it receives;
    // then waits until every rank has consumed its sends (so the send buffers may be reused)
    bool exchange(const std::vector<Xfer>& x, cudaStream_t st) override {
        g->posted[rank] = x;
        cudaEventRecord(g->ready[rank], st);
        g->barrier();
        for (const Xfer& e : x) {
            if (e.nr <= 0) continue;
            const Xfer* s = nullptr;
            for (const Xfer& f : g->posted[e.peer])
                if (f.peer == rank) s = &f;
            if (!s || s->ns != e.nr) return false;
            cudaStreamWaitEvent(st, g->ready[e.peer], 0);
            cudaMemcpyAsync(e.recv, s->send, sizeof(double) * e.nr, cudaMemcpyDeviceToDevice, st);
        }
        cudaEventRecord(g->done[rank], st);
        g->barrier();
        for (const Xfer& e : x)
            if (e.ns > 0) cudaStreamWaitEvent(st, g->done[e.peer], 0);
        g->barrier();  // (events re-recorded by the next collective only after everyone waited)
        return true;
    }
    bool allreduce_sum(double* buf, i64 n, cudaStream_t st) override {
        if (n > scratch_n) {
            if (scratch) dev_free(scratch);
            if (dev_malloc((void**)&scratch, sizeof(double) * (size_t)n) != cudaSuccess) return false;
            scratch_n = n;
        }
        if (!d_bufs && dev_malloc((void**)&d_bufs, sizeof(double*) * (size_t)nranks) != cudaSuccess) return false;
        cudaMemcpyAsync(scratch, buf, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
        g->reduce_buf[rank] = scratch;
        cudaEventRecord(g->ready[rank], st);
        g->barrier();
        for (int q = 0; q < nranks; ++q) cudaStreamWaitEvent(st, g->ready[q], 0);
        cudaMemcpyAsync(d_bufs, g->reduce_buf.data(), sizeof(double*) * nranks, cudaMemcpyHostToDevice, st);
        k_sum_ranks<<<(unsigned)std::min<i64>(1024, (n + 255) / 256), 256, 0, st>>>(n, nranks, d_bufs, buf);
        cudaEventRecord(g->done[rank], st);
        cudaStreamSynchronize(st);  // (d_bufs is pageable-host sourced; keep the host table alive)
        g->barrier();
        for (int q = 0; q < nranks; ++q) cudaStreamWaitEvent(st, g->done[q], 0);
        g->barrier();
        return true;
    }
    bool allgatherv(const double* mine, double* out, const std::vector<i64>& off, cudaStream_t st) override {
        g->gather_src[rank] = mine;
        cudaEventRecord(g->ready[rank], st);
        g->barrier();
        for (int q = 0; q < nranks; ++q) {
            const i64 c = off[q + 1] - off[q];
            if (c <= 0) continue;
            cudaStreamWaitEvent(st, g->ready[q], 0);
            cudaMemcpyAsync(out + off[q], g->gather_src[q], sizeof(double) * c, cudaMemcpyDeviceToDevice, st);
        }
        cudaEventRecord(g->done[rank], st);
        g->barrier();
        for (int q = 0; q < nranks; ++q) cudaStreamWaitEvent(st, g->done[q], 0);
        g->barrier();
        return true;
    }
    bool capturable() const override { return false; }
    // run f(stream) on every rank after all ranks' earlier work and before their later work
    // (the fake-rank stand-in for the peer-store flags)
    template <class F>
    bool ordered(F f, cudaStream_t st) {
        cudaEventRecord(g->ready[rank], st);
        g->barrier();
        for (int q = 0; q < nranks; ++q) cudaStreamWaitEvent(st, g->ready[q], 0);
        f(st);
        cudaEventRecord(g->done[rank], st);
        g->barrier();
        for (int q = 0; q < nranks; ++q) cudaStreamWaitEvent(st, g->done[q], 0);
        g->barrier();
        return true;
    }
    ~FakeTransport() override {
        if (scratch) dev_free(scratch);
        if (d_bufs) dev_free(d_bufs);
    }
};
}  // namespace mgm

namespace {

thread_local std::string g_setup_error;
thread_local int64_t g_setup_index = -1;

struct Level {
    i64 n = 0;
    int ncol = 0;
    std::vector<i64> coff;  // colour offsets (lib order)
    // operator L_j (SELL-32)
    i64* sptr = nullptr;
    i32* scol = nullptr;
    double* sval = nullptr;
    i64 sell_stored = 0, nnz = 0;
    std::vector<i64> h_sptr, h_rptr;  // host copies of the slice offsets (L2 prefetch regions)
    i32* slw = nullptr;                 // per slice: slots read by a sweep from a zero guess (pack_sell)
    uint8_t* nlow = nullptr;            // per row: its earlier-colour entries (slots 1..nlow)
    i32* sluw = nullptr;                // per slice: first later-colour slot of its rows (min 1 + nlow)
    i32* l2m = nullptr;                 // lib row -> Morton index (residual written in Morton order)
    i32* rcol_m = nullptr;              // R_j columns as fine Morton indices (same values / layout as rcol)
    std::vector<i64> lower_per_colour;  // per colour: stored entries such a sweep reads (diag + earlier colours)
    int tpr = 1, rtpr = 1;  // threads per row for L_j (colour sweeps) and R_j kernels
    int stpr = 1;           // threads per row for full-level SpMV / residual on L_j
    int gs_block = 256;     // threads per block of the colour kernels
    int uniform_w = 0;      // > 0: every SELL slice has this width
    // interpolation P_j (ELL width pm, slot-major) and restriction R_j (SELL-32, next level rows)
    int pm = 0;
    i32* pcol = nullptr;
    double* pval = nullptr;
    i64 p_nnz = 0;
    i64* rptr = nullptr;
    i32* rcol = nullptr;
    double* rval = nullptr;
    i64 r_stored = 0;
    // vectors
    double* u = nullptr;
    double* f = nullptr;
    double* t = nullptr;
    double* c = nullptr;  // Poisson border
    // host copies (export / test hooks)
    std::vector<i64> ids;        // original point index per lib row
    HostCSR L_lib, P_lib;        // lib order
    std::vector<i32> colour_lib;
    std::vector<double> c_lib;
    std::vector<i64> lib2mor;  // Morton index of each lib row
    // ---- distributed level (mgm_dist_attach): this rank's rows only.
    // Vectors u, t: [owned rows (n) | multiplier (Poisson) | ghosts (nghost)]; f: [owned | mult].
    bool dist = false;
    i64 nghost = 0, gbase = 0;           // ghost slot g lives at index gbase + g
    std::vector<int> peers;              // PartTables
    std::vector<i64> send_off, recv_off, send_coff, recv_coff;
    i32* d_send_idx = nullptr;           // owned row of each send entry
    i64* d_srange = nullptr;             // [ncol + 1][npeers][2] send ranges: all (key 0), colour c (key c + 1)
    // peer-store halos (MGM_P2P=1): the slot each send entry lands in, in the peer's vector
    std::vector<i64> h_rslot;
    i64* d_rslot = nullptr;
    double* peer_u[16] = {};             // the peers' u / t of this level (mapped peer memory)
    double* peer_t[16] = {};
    double* d_sendbuf = nullptr;
    std::vector<int> tpr_col;            // threads per row of each colour (the undistributed launch's)
    std::vector<i64> gcoff;              // the undistributed level's colour offsets
    // on the last distributed level: my coarse rows of the first replicated level are restricted
    // into d_stage_mine, all-gathered into d_stage_all, then permuted (d_stage_perm) into lib order
    i64 nstage = 0;
    std::vector<i64> stage_off;
    double* d_stage_mine = nullptr;
    double* d_stage_all = nullptr;
    i32* d_stage_perm = nullptr;
};

struct KernelTimer {
    bool on = false;
    std::vector<cudaEvent_t> ev;  // pairs
    int used = 0;
    double total_ms = 0.0;
    i64 launches = 0;
    double bytes = 0.0;
};

}  // namespace

struct mgm_ctx {
    mgm_allocator alloc{};  // device allocator (mgm_setup; alloc == NULL: cudaMalloc)
    mgm_stencil_params sp{};
    mgm_level_params lp{};
    i64 N = 0;
    int p = 0;
    bool poisson = false;
    int device = 0;
    int nthreads = 1;
    std::vector<Level> lv;
    // coarsest dense LU
    int nc = 0;
    double* lu = nullptr;
    double* ainv = nullptr;  // explicit inverse of the coarsest operator (batched solves), row-major
    i32* piv = nullptr;
    // level-0 permutation (lib row -> original index)
    i32* d_lib2orig = nullptr;
    // fine weights (export)
    // fine-level weights and stencils in Morton order, exported in original order on demand
    std::vector<double> w_mor;
    std::vector<i32> sten_mor;
    std::vector<i64> perm0;
    int ns0 = 0;
    // streams / graph
    cudaStream_t st = nullptr;
    cudaGraphExec_t vgraph = nullptr;
    cudaGraphExec_t vgraph0 = nullptr;  // the same V-cycle from a zero guess on level 0 (Krylov preconditioner)
    bool vc_zero_guess = false;         // set while enqueueing vgraph0
    bool no_zg = false;                 // MGM_NO_ZG: no zero-guess sweeps (comparison)
    bool no_c0_fuse = false;            // MGM_NO_C0_FUSE: colour 0 not fused into the restriction
    i64 morton_t_min = (i64)1 << 62;    // levels with at least this many rows write the residual in
                                        // Morton order (MGM_MORTON_T_MIN; off: no gain measured at
                                        // cfg3 or cfg5)
    i64 upper_res_min = 131072;         // levels with at least this many rows use the later-colour
                                        // residual after a zero-guess sweep (MGM_UPPER_RES_MIN)
    bool pdl = false;  // set while enqueueing the V-cycle (PDL launches)
    // bottom of the V-cycle (levels botJ..p-1) in one thread-block-cluster kernel
    // (bottom_kernel.cuh); botJ < 0 = off
    // stage trace (MGM_TRACE=1 at setup): %globaltimer stamps between V-cycle stages
    unsigned long long* d_trace = nullptr;
    int ntrace = 0;
    std::vector<std::string> trace_labels;
    int botJ = -1;
    // bottom of the V-cycle as one dense operator B_J (dense_bottom.cuh); denseJ < 0 = off
    int denseJ = -1;
    int dense_m = 0, dense_ld = 0;
    double* dB = nullptr;
    double* d_dlt = nullptr;    // increments of the GMRES graph's last level-0 postsmooth (MODE 3)
    double* bpart = nullptr;    // block partials of the batched multi-dot [RED_BLOCKS][(restart + 1) 8]
    double* bdlt = nullptr;     // K-wide increments of the batched zero-guess graph's last postsmooth
    int bdlt_k = 0;
    double* bdlt_out = nullptr;  // set while capturing that graph
    bool bgraph_zg_dlt[9] = {};
    bool bgraph_dlt[9] = {};
    double* dlt_out = nullptr;  // set while enqueueing that graph's V-cycle
    double* d_dlt_pre = nullptr;    // increments of the general V-cycle's last level-0 presmooth
    double* dlt_pre_out = nullptr;  // set while enqueueing the general V-cycle graph
    bool vgraph_dlt = false;    // the general V-cycle graph writes d_dlt (standalone residual)
    bool vgraph0_dlt = false;   // ... and the zero-guess one (A M v)
    bool last_vc_dlt = false;   // the last run_vcycle left its increments in d_dlt
    double* dP = nullptr;  // partial sums of the column-split multi-RHS dense apply [S][m][8]
    int bot_cluster = 16;
    size_t bot_smem = 0;
    int nphases = 0;
    int bot_arm0 = 0, bot_arm1 = 0;  // bytes of the first two data-synchronised phases
    int bot_arm0b = 0, bot_arm1b = 0;  // ... of the second launch when split
    int bot_split = 0;                 // > 0: phases of the first launch; the coarse solve is a GEMV
    const double* bot_ainv = nullptr;  // the coarsest inverse (row-major) for that GEMV
    BPhase* d_phases = nullptr;
    std::vector<void*> bot_mem;
    i64 vcycle_kernels = 0;
    // batched (multi-RHS) V-cycles: per level interleaved [n_j][bK] buffers, graph per K
    int bK = 0;
    std::vector<double*> bu, bf, bt;
    cudaGraphExec_t bgraph[9] = {};
    cudaGraphExec_t bgraph_zg[9] = {};  // from a zero level-0 guess (batched GMRES)
    double* bres = nullptr;  // residual (n x K)
    // batched GMRES: basis (restart + 1) x n x K, w, x, b (n x K); dots (device) + pinned mirror
    double *bV = nullptr, *bw = nullptr, *bx = nullptr, *bb = nullptr, *bdh = nullptr, *bhh = nullptr;
    int bgK = 0;
    // multi-GPU (mgm_dist_attach / mgm_dist_attach_fake): levels 0..D-1 partitioned by Morton row
    // blocks, D..p-1 replicated
    int rank = 0, nranks = 1;
    Transport* tp = nullptr;
    int D = 0;
    // peer-store halos (MGM_P2P=1 at attach): pushes into the peers' ghost slots + flags
    bool p2p = false;
    unsigned long long* p2p_flags = nullptr;   // [nranks] written by the peers (IPC-exported)
    unsigned long long* p2p_sent = nullptr;    // [nranks] my pushes to each peer
    unsigned long long* p2p_expect = nullptr;  // [nranks] pushes I have waited for, per peer
    unsigned long long* peer_flags[64] = {};   // peer r's flag array (mapped), indexed by rank
    unsigned* p2p_ticket = nullptr;
    std::vector<void*> ipc_opened;
    std::vector<i64> local_ids;  // original ids of my level-0 rows, in my I/O (Morton) order
    // GMRES workspace
    int restart = 50;
    i64 ld = 0;
    double* V = nullptr;
    double* Z = nullptr;  // device GMRES: z_k = M v_k of the current restart cycle (restart x ld)
    double* bZ = nullptr;  // batched GMRES: the same, K-wide (restart x N x K)
    double* w = nullptr;
    double* xs = nullptr;    // solution accumulator (lib order)
    double* b = nullptr;     // rhs (lib order)
    bool warm = false;       // xs holds an initial guess x0 on entry of the solver (mgm_solve x0)
    double* partials = nullptr;
    unsigned* tickets = nullptr;  // last-block counters of the fused reductions (reset by the finisher)
    double* dh = nullptr;    // device scratch: h1[128], h2[128], nrm2, misc
    // device-side GMRES (gmres_dev): Arnoldi loop as a CUDA-graph WHILE node
    cudaGraphExec_t ggraph = nullptr;
    int* g_i = nullptr;       // {k, its, stop, maxit}
    double* g_d = nullptr;    // {bnorm, tol, H, cs, sn, g, hist}
    double* g_h = nullptr;    // pinned mirror of g_d
    int* g_hi = nullptr;      // pinned mirror of g_i
    int g_hist_cap = 4096;
    double* hh = nullptr;    // pinned host mirror
    // timing
    KernelTimer timer[4];
    double setup_ms = 0.0;
    // errors
    std::string err;
    int64_t err_index = -1;
};

// ---------------------------------------------------------------------------------------
// Device allocations through the ctx's allocator (mgm_setup's mgm_allocator; NULL = the CUDA
// runtime).  Thread-local: every ABI entry point installs its ctx's allocator (AllocScope).
// ---------------------------------------------------------------------------------------
static thread_local const mgm_allocator* g_alloc = nullptr;
cudaError_t mgm::dev_malloc(void** p, size_t bytes) {
    if (g_alloc && g_alloc->alloc) {
        *p = g_alloc->alloc(bytes, g_alloc->user);
        return *p ? cudaSuccess : cudaErrorMemoryAllocation;
    }
    return cudaMalloc(p, bytes);
}
// Setup defers cudaFree to its end: cudaFree synchronises the whole device, which would
// stall the setup's concurrent threads (Galerkin stream, colouring) on each other's work.
struct DeferFree {
    std::mutex mu;
    std::vector<void*> ptrs;
    ~DeferFree() {
        for (void* q : ptrs) cudaFree(q);
    }
};
static thread_local DeferFree* g_defer = nullptr;
struct DeferScope {
    DeferFree* prev;
    explicit DeferScope(DeferFree* d) : prev(g_defer) { g_defer = d; }
    ~DeferScope() { g_defer = prev; }
};
void mgm::dev_free(void* p) {
    if (!p) return;
    if (g_defer && !(g_alloc && g_alloc->alloc)) {
        std::lock_guard<std::mutex> lk(g_defer->mu);
        g_defer->ptrs.push_back(p);
        return;
    }
    if (g_alloc && g_alloc->alloc) {
        if (g_alloc->release) g_alloc->release(p, g_alloc->user);
        return;
    }
    cudaFree(p);
}
struct AllocScope {
    const mgm_allocator* prev;
    explicit AllocScope(const mgm_ctx* ctx) : prev(g_alloc) { g_alloc = ctx ? &ctx->alloc : nullptr; }
    ~AllocScope() { g_alloc = prev; }
};

#define CK(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                 \
            return e_ == cudaErrorMemoryAllocation ? MGM_ERR_OOM : MGM_ERR_CUDA;           \
        }                                                                                  \
    } while (0)

template <class T>
static cudaError_t dalloc(T** p, i64 count) {
    return dev_malloc((void**)p, sizeof(T) * (size_t)std::max<i64>(count, 1));
}

static unsigned blocks_for(i64 n, int threads) { return (unsigned)std::max<i64>(1, (n + threads - 1) / threads); }

// Allow a kernel the device's opt-in maximum of dynamic shared memory (process-wide).
static void set_max_dyn_smem(const void* kern) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) optin -= (int)fa.sharedSizeBytes;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
}

// First failed launch since the last check (a failed launch inside stream capture only
// surfaces at cudaStreamEndCapture; this names it).
static thread_local std::string g_launch_err;
static void note_launch(cudaError_t e, unsigned grid, unsigned block, size_t smem) {
    if (e != cudaSuccess && g_launch_err.empty())
        g_launch_err = std::string(cudaGetErrorString(e)) + " (grid " + std::to_string(grid) + ", block " +
                       std::to_string(block) + ", smem " + std::to_string(smem) + ")";
}

// Kernel launch with optional programmatic dependent launch (PDL, see solve_kernels.cuh).
static bool g_use_pdl = std::getenv("MGM_NO_PDL") == nullptr;
// dry enqueue pass (L2 prefetch target recording): nothing is launched or recorded
static thread_local bool g_dry = false;
// set by every communication call (halo, all-gather, allreduce): the kernel launched next waits
// for it fully (no programmatic dependency on a communication node)
static thread_local bool g_after_comm = false;
template <typename... KArgs, typename... Args>
static void launch(bool pdl, void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                   Args... args) {
    if (g_dry) return;
    if (g_after_comm) {
        pdl = false;
        g_after_comm = false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl && g_use_pdl) ? 1 : 0;
    note_launch(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), grid, block, smem);
}

// ---------------------------------------------------------------------------------------
// Setup (Alg. 2)
// ---------------------------------------------------------------------------------------
namespace {

// Pack a Morton-order CSR into lib-order SELL-32 (diagonal first for square operators).
// With a colouring (colour_lib: GS colour of each lib row), the stored row order is
// [diagonal | earlier-colour columns | later-colour columns], each group in ascending Morton
// column, and slw[s] = 1 + the largest earlier-colour count of slice s: a Gauss-Seidel sweep
// from a zero guess reads only those first slw slots (the later-colour values are still 0).
// lib_csr keeps the plain order (diagonal first, ascending column).
// host vectors whose resize() leaves new elements uninitialised (every element is written
// afterwards): no sequential zero fill of the large packed arrays
template <class T>
struct NoInit : std::allocator<T> {
    template <class U>
    struct rebind { using other = NoInit<U>; };
    NoInit() = default;
    template <class U>
    NoInit(const NoInit<U>&) noexcept {}
    template <class U>
    void construct(U* p) noexcept { ::new ((void*)p) U; }
    template <class U, class... Args>
    void construct(U* p, Args&&... a) { ::new ((void*)p) U(std::forward<Args>(a)...); }
};
template <class T>
using hvec = std::vector<T, NoInit<T>>;

static int host_threads() { return std::max(1, std::min(64, (int)std::thread::hardware_concurrency())); }

void pack_sell(const HostCSR& A, const std::vector<i64>& row_lib2mor, const std::vector<i32>& col_mor2lib,
               bool diag_first, std::vector<i64>& sptr, hvec<i32>& scol, hvec<double>& sval,
               HostCSR* lib_csr, const std::vector<i32>* colour_lib = nullptr, std::vector<i32>* slw = nullptr,
               std::vector<i64>* lower_per_colour = nullptr, std::vector<uint8_t>* nlow_row = nullptr,
               std::vector<i32>* sluw = nullptr) {
    // slices are independent once sptr is known: both passes run on threads over slices
    const i64 n = (i64)row_lib2mor.size();
    const i64 ns = (n + 31) / 32;
    const int nt = ns >= 2048 ? host_threads() : 1;
    auto par = [&](auto&& f) {  // f(t, s0, s1) over slice ranges
        if (nt <= 1) { f(0, (i64)0, ns); return; }
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t) th.emplace_back([&, t] { f(t, ns * t / nt, ns * (t + 1) / nt); });
        for (auto& x : th) x.join();
    };
    auto rlen = [&](i64 r) { return A.ptr[row_lib2mor[r] + 1] - A.ptr[row_lib2mor[r]]; };
    sptr.assign(ns + 1, 0);
    par([&](int, i64 s0, i64 s1) {
        for (i64 s = s0; s < s1; ++s) {
            i64 w = 0;
            for (i64 r = s * 32; r < std::min(n, s * 32 + 32); ++r) w = std::max(w, rlen(r));
            sptr[s + 1] = 32 * std::max<i64>(w, 1);
        }
    });
    for (i64 s = 0; s < ns; ++s) sptr[s + 1] += sptr[s];
    scol.resize(sptr[ns]);
    sval.resize(sptr[ns]);
    if (lib_csr) {
        lib_csr->nrows = n;
        lib_csr->ncols = (i64)col_mor2lib.size();
        lib_csr->ptr.assign(n + 1, 0);
        for (i64 r = 0; r < n; ++r) lib_csr->ptr[r + 1] = lib_csr->ptr[r] + rlen(r);
        lib_csr->col.resize(lib_csr->ptr[n]);
        lib_csr->val.resize(lib_csr->ptr[n]);
    }
    if (slw) slw->assign(ns, 1);
    if (nlow_row) nlow_row->assign(n, 0);
    if (sluw) sluw->assign(ns, 1 << 30);
    i32 nc = 0;
    if (lower_per_colour && colour_lib) {
        for (i32 c : *colour_lib) nc = std::max(nc, c + 1);
        lower_per_colour->assign(nc, 0);
    }
    std::vector<std::vector<i64>> lpc(nt, std::vector<i64>(nc, 0));
    par([&](int t, i64 s0, i64 s1) {
        std::vector<std::pair<i32, double>> row, srow;
        for (i64 r = s0 * 32; r < std::min(n, s1 * 32); ++r) {
            i64 mr = row_lib2mor[r];
            row.clear();
            if (diag_first)
                for (i64 q = A.ptr[mr]; q < A.ptr[mr + 1]; ++q)
                    if (A.col[q] == (i32)mr) row.push_back({A.col[q], A.val[q]});
            for (i64 q = A.ptr[mr]; q < A.ptr[mr + 1]; ++q)
                if (!diag_first || A.col[q] != (i32)mr) row.push_back({A.col[q], A.val[q]});
            i64 s = r / 32, lane = r % 32;
            i64 w = (sptr[s + 1] - sptr[s]) / 32;
            srow = row;
            if (colour_lib && diag_first && !row.empty()) {  // [diag | earlier colours | later colours]
                const i32 cr = (*colour_lib)[r];
                i64 o = 1;
                for (size_t k = 1; k < row.size(); ++k)
                    if ((*colour_lib)[col_mor2lib[row[k].first]] < cr) srow[o++] = row[k];
                const i64 nlow = o - 1;
                for (size_t k = 1; k < row.size(); ++k)
                    if ((*colour_lib)[col_mor2lib[row[k].first]] >= cr) srow[o++] = row[k];
                if (slw) (*slw)[s] = std::max<i32>((*slw)[s], (i32)(1 + nlow));
                if (nlow_row) (*nlow_row)[r] = (uint8_t)std::min<i64>(nlow, 255);
                if (sluw) (*sluw)[s] = std::min<i32>((*sluw)[s], (i32)(1 + nlow));
                if (lower_per_colour) lpc[t][cr] += 1 + nlow;
            }
            for (i64 k = 0; k < w; ++k) {
                i64 o = sptr[s] + 32 * k + lane;
                if (k < (i64)srow.size()) {
                    scol[o] = col_mor2lib[srow[k].first];
                    sval[o] = srow[k].second;
                } else {
                    scol[o] = diag_first ? (i32)r : (row.empty() ? 0 : col_mor2lib[row[0].first]);
                    sval[o] = 0.0;
                }
            }
            if (lib_csr) {
                i64 o = lib_csr->ptr[r];
                for (auto& e : row) {
                    lib_csr->col[o] = col_mor2lib[e.first];
                    lib_csr->val[o++] = e.second;
                }
            }
        }
    });
    if (lower_per_colour && colour_lib)
        for (int t = 0; t < nt; ++t)
            for (i32 c = 0; c < nc; ++c) (*lower_per_colour)[c] += lpc[t][c];
    // padded slice rows beyond n point at row 0
    for (i64 r = n; r < ns * 32; ++r) {
        i64 s = r / 32, lane = r % 32;
        for (i64 k = 0; k < (sptr[s + 1] - sptr[s]) / 32; ++k) {
            scol[sptr[s] + 32 * k + lane] = 0;
            sval[sptr[s] + 32 * k + lane] = 0.0;
        }
    }
}

template <class T, class A>
mgm_status upload(mgm_ctx* ctx, T** dst, const std::vector<T, A>& src) {
    CK(dalloc(dst, (i64)src.size()));
    if (!src.empty()) CK(cudaMemcpyAsync(*dst, src.data(), sizeof(T) * src.size(), cudaMemcpyHostToDevice, ctx->st));
    return MGM_OK;
}

mgm_status fail(mgm_ctx* ctx, mgm_status s, const std::string& msg, int64_t idx) {
    ctx->err = msg;
    ctx->err_index = idx;
    return s;
}

// Build the phase list of the one-kernel bottom of the V-cycle (bottom_kernel.cuh) for the
// levels J..p-1, J = the first level >= 1 with N_J <= MGM_BOT_MAX (default 16384; 0 = off).
// Levels with N_j <= MGM_BOT_LOCAL (default 1024) run on CTA 0 alone with __syncthreads.
// Shifted problems only.  Operators are re-packed as lib-order CSR (int32) with the
// diagonal first, row-contiguous so that a thread group reads a row coalesced.
template <class T>
static T* bot_upload(mgm_ctx* ctx, const std::vector<T>& v, bool& ok) {
    T* d = nullptr;
    if (dev_malloc((void**)&d, sizeof(T) * std::max<size_t>(1, v.size())) != cudaSuccess) { ok = false; return nullptr; }
    ctx->bot_mem.push_back(d);
    if (!v.empty() && cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess) ok = false;
    return d;
}

void setup_bottom(mgm_ctx* ctx, const std::vector<double>& LU, const std::vector<i32>& piv) {
    ctx->botJ = -1;
    // measured best split (profiles/r01_notes.md, session 3): the bottom starts at the first
    // level with <= 4096 rows (cfg3: V-cycle 1270 -> 1165 us, cfg2: 1430 -> 1273 us against
    // 16384 -- per-kernel colour steps of a 16k-row level beat its cluster phases now), and only
    // levels <= 64 rows run on CTA 0 alone.  If that would leave only the coarsest level in the
    // bottom (large coarsest, e.g. cfg5's 4096), the bottom starts at <= 16384 rows instead.
    i64 bmax = 4096, blocal = 64;
    const bool bmax_env = std::getenv("MGM_BOT_MAX") != nullptr;
    if (const char* e = std::getenv("MGM_BOT_MAX")) bmax = std::atoll(e);
    if (const char* e = std::getenv("MGM_BOT_LOCAL")) blocal = std::atoll(e);
    if (!bmax_env) {
        int first = -1;
        for (int j = 1; j < ctx->p; ++j)
            if (ctx->lv[j].n <= bmax) { first = j; break; }
        if (first < 0 || first == ctx->p - 1) bmax = 16384;
    }
    if (ctx->poisson || bmax <= 0 || ctx->p < 2) return;
    const int p = ctx->p;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // first level J >= 1 with N_J <= bmax whose phase table + replicated iterates fit
    int J = -1;
    size_t table = 0;
    for (int j = 1; j < p; ++j) {
        if (ctx->lv[j].n > bmax) continue;
        i64 nph = 3 + 2 * (p - j) + 2, vb = 0;  // (+ the STORE / LOAD phases of a split bottom)
        for (int q = j; q < p; ++q) {
            vb += ctx->lv[q].n * (i64)sizeof(double);
            if (q + 1 < p) nph += (i64)(ctx->lp.nu1 + ctx->lp.nu2) * ctx->lv[q].ncol + 3;
        }
        const size_t tb = (size_t)nph * sizeof(BPhase);
        if (nph <= BOT_MAX_PHASES && (tb + 15) / 16 * 16 + (size_t)vb + 1024 <= (size_t)optin) {
            J = j;
            table = (tb + 15) / 16 * 16;
            break;
        }
    }
    if (J < 0) return;
    for (bool tr : {false, true}) {
        cudaFuncSetAttribute(bottom_kernel_ptr(tr), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        set_max_dyn_smem(bottom_kernel_ptr(tr));
    }
    // cluster size: 16 (non-portable) if the device can co-schedule it, else 8
    size_t smem = table;
    std::vector<int> ou(p, -1);
    for (int j = J; j < p; ++j) {
        ou[j] = (int)smem;
        smem += (size_t)ctx->lv[j].n * sizeof(double);
    }
    int cs = 0;
    std::vector<int> sizes = {16, 8};
    if (const char* e = std::getenv("MGM_BOT_CS")) sizes = {std::atoi(e)};  // tuning experiment
    for (int c : sizes) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c);
        cfg.blockDim = dim3(BOT_THREADS);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, bottom_kernel_ptr(false), &cfg) == cudaSuccess && ncl > 0) { cs = c; break; }
        cudaGetLastError();
    }
    if (!cs) return;
    bool ok = true;
    // row-major ELL copy of a lib-order CSR (diagonal first for L, as stored in L_lib)
    struct Ell { const int* col = nullptr; const double* val = nullptr; int W = 0; };
    auto make_ell = [&](const HostCSR& A) {
        Ell E;
        i64 W = 1;
        for (i64 r = 0; r < A.nrows; ++r) W = std::max(W, A.ptr[r + 1] - A.ptr[r]);
        std::vector<int> c((size_t)A.nrows * W);
        std::vector<double> v((size_t)A.nrows * W, 0.0);
        for (i64 r = 0; r < A.nrows; ++r) {
            const i64 a0 = A.ptr[r], len = A.ptr[r + 1] - a0;
            for (i64 k = 0; k < W; ++k) {
                c[(size_t)r * W + k] = k < len ? A.col[a0 + k] : (len > 0 ? A.col[a0] : 0);
                v[(size_t)r * W + k] = k < len ? A.val[a0 + k] : 0.0;
            }
        }
        E.col = bot_upload(ctx, c, ok);
        E.val = bot_upload(ctx, v, ok);
        E.W = (int)W;
        return E;
    };
    std::vector<Ell> EL(p), EP(p), ER(p);
    std::vector<const double*> dinv(p, nullptr);
    for (int j = J; j + 1 < p; ++j) {
        Level& L = ctx->lv[j];
        EL[j] = make_ell(L.L_lib);
        EP[j] = make_ell(L.P_lib);
        ER[j] = make_ell(transpose(L.P_lib));  // R_j = P_j^T, rows = coarse lib order
        std::vector<double> di(L.n);
        for (i64 r = 0; r < L.n; ++r) di[r] = 1.0 / L.L_lib.val[L.L_lib.ptr[r]];
        dinv[j] = bot_upload(ctx, di, ok);
    }
    // coarsest: explicit inverse from the LU factors (same solution up to rounding, O13)
    const int m = ctx->nc;
    Ell EC;
    {
        std::vector<double> Ainv;
        dense_inverse(LU, piv, m, Ainv, ctx->nthreads);
        std::vector<int> ccol((size_t)m * m);
        for (int r = 0; r < m; ++r)
            for (int c = 0; c < m; ++c) ccol[(size_t)r * m + c] = c;
        EC.col = bot_upload(ctx, ccol, ok);
        EC.val = bot_upload(ctx, Ainv, ok);
        EC.W = m;
    }
    if (!ok) return;
    const int nthr_cl = cs * BOT_THREADS;
    std::vector<BPhase> ph;
    auto is_local = [&](int j) { return ctx->lv[j].n <= blocal; };
    // op on rows [r0, r1); x: smem offset xo (>= 0) or global xg; y: smem offset yo or global yg
    auto add = [&](int op, bool local, i64 r0, i64 r1, const Ell* E, int xo, const double* xg, int yo, double* yg,
                   const double* f, int zo, const double* di) {
        if (r1 <= r0) return;
        BPhase P{};
        P.op = op;
        P.local = local ? 1 : 0;
        P.r0 = (int)r0;
        P.r1 = (int)r1;
        P.W = E ? std::max(E->W, 1) : 1;
        P.xo = xo; P.yo = yo; P.zo = zo;
        P.x = xg; P.y = yg; P.f = f; P.dinv = di;
        P.col = E ? E->col : nullptr;
        P.val = E ? E->val : nullptr;
        // f may ride with the operator prefetch unless the previous phase wrote it (the
        // restriction writes f_{j+1}; a GS or residual phase after a GS phase of the
        // same level reads an f that is already final)
        P.fpre = (!ph.empty() && ph.back().op == BP_GS && ph.back().f == f && (op == BP_GS || op == BP_RES)) ? 1 : 0;
        const i64 nthr = local ? BOT_THREADS : nthr_cl;
        int best = -1;
        if (op == BP_ZERO || op == BP_STORE) {
            best = 0;
        } else {
            int smallest_valid = -1;
            int lgmax = 5;  // tuning experiment: MGM_BOT_TPR_MAX caps threads per row
            if (const char* e = std::getenv("MGM_BOT_TPR_MAX")) lgmax = std::max(0, std::min(5, (int)std::log2(std::atoi(e))));
            for (int lg = lgmax; lg >= 0; --lg) {  // largest tpr that covers W and fits one pass
                if (!(BOT_TPR_MASK >> lg & 1u)) continue;  // compiled specialisations only
                const int tpr = 1 << lg;
                if (bot_ch(tpr) * tpr < P.W) continue;
                smallest_valid = lg;
                if (best < 0 && (r1 - r0) * tpr <= nthr) best = lg;
            }
            if (best < 0) best = smallest_valid >= 0 ? smallest_valid : 5;
        }
        if (op == BP_ZERO || op == BP_STORE) best = 5;  // (no operator; any compiled value)
        P.tpr_log2 = best;
        P.mb = -1;
        P.arm = 0;
        ph.push_back(P);
    };
    const bool pre_b = ctx->lp.smoother == 1, post_b = ctx->lp.smoother == 1 || ctx->lp.smoother == 2;
    auto sweep = [&](int j, bool backward) {
        Level& L = ctx->lv[j];
        for (int q = 0; q < L.ncol; ++q) {
            const int c = backward ? L.ncol - 1 - q : q;
            add(BP_GS, is_local(j), L.coff[c], L.coff[c + 1], &EL[j], ou[j], nullptr, ou[j], nullptr, L.f, -1, dinv[j]);
        }
    };
    add(BP_ZERO, false, 0, ctx->lv[J].n, nullptr, -1, nullptr, ou[J], nullptr, nullptr, -1, nullptr);  // u_J = 0
    for (int j = J; j + 1 < p; ++j) {  // Alg. 3 lines 6-9 (and 4-5 for j = J)
        Level& L = ctx->lv[j];
        Level& Ln = ctx->lv[j + 1];
        for (int s2 = 0; s2 < ctx->lp.nu1; ++s2) sweep(j, pre_b);
        add(BP_RES, is_local(j), 0, L.n, &EL[j], ou[j], nullptr, -1, L.t, L.f, -1, nullptr);
        add(BP_MVZ, is_local(j), 0, Ln.n, &ER[j], -1, L.t, -1, Ln.f, nullptr, ou[j + 1], nullptr);
    }
    // a large coarsest level (cfg5: 4096 rows, a 134 MB dense inverse) is solved by a
    // grid-wide GEMV between two launches of the bottom kernel: the first stores the
    // iterates e_J..e_{p-2} to HBM, the second loads them (and e_p) back
    i64 gemv_min = 1024;
    if (const char* e = std::getenv("MGM_BOT_GEMV_MIN")) gemv_min = std::atoll(e);
    const bool split = m >= gemv_min && J < p - 1;
    size_t qa = 0;  // phases of the first launch
    if (split) {
        for (int j = J; j + 1 < p; ++j)
            add(BP_STORE, false, 0, ctx->lv[j].n, nullptr, -1, nullptr, ou[j], ctx->lv[j].u, nullptr, -1, nullptr);
        qa = ph.size();
        add(BP_LOAD, false, 0, m, nullptr, -1, ctx->lv[p - 1].u, ou[p - 1], nullptr, nullptr, -1, nullptr);
        for (int j = J; j + 1 < p; ++j)
            add(BP_LOAD, false, 0, ctx->lv[j].n, nullptr, -1, ctx->lv[j].u, ou[j], nullptr, nullptr, -1, nullptr);
    } else {  // line 10
        Level& C = ctx->lv[p - 1];
        add(BP_MV, is_local(p - 1), 0, m, &EC, -1, C.f, ou[p - 1], nullptr, nullptr, -1, nullptr);
    }
    for (int j = p - 2; j >= J; --j) {  // lines 11-14
        Level& L = ctx->lv[j];
        add(BP_ADD, is_local(j), 0, L.n, &EP[j], ou[j + 1], nullptr, ou[j], nullptr, nullptr, -1, nullptr);
        for (int s2 = 0; s2 < ctx->lp.nu2; ++s2) sweep(j, post_b);
    }
    add(BP_STORE, false, 0, ctx->lv[J].n, nullptr, -1, nullptr, ou[J], ctx->lv[J].u, nullptr, -1, nullptr);
    // data-synchronised phases (bottom_kernel.cuh): cluster GS / ADD / MV phases whose output
    // is a replicated vector; every CTA receives 8 bytes per row of such a phase
    // (numbered per launch: each launch initialises its own mbarriers)
    // (opt-in, MGM_BOT_MBAR=1: the phase-ahead arming assumes every CTA sends rows in every
    // data-synchronised phase, which a small colour spread over 16 CTAs can violate -- ADVICE r01;
    // the cluster bottom is only the fallback of the dense bottom now, so it runs the always-safe
    // barrier.cluster phases by default)
    const bool mbar_on = std::getenv("MGM_BOT_MBAR") != nullptr && std::atoi(std::getenv("MGM_BOT_MBAR")) == 1;
    auto number = [&](size_t q0, size_t q1, int& arm0, int& arm1) {
        std::vector<int> mbq;
        for (size_t q = q0; q + 1 < q1; ++q) {
            BPhase& P = ph[q];
            if (mbar_on && !P.local && P.yo >= 0 && (P.op == BP_GS || P.op == BP_ADD || P.op == BP_MV)) {
                P.mb = (int)mbq.size();
                mbq.push_back((int)q);
            }
        }
        auto mbytes = [&](size_t k) { return 8 * (ph[(size_t)mbq[k]].r1 - ph[(size_t)mbq[k]].r0); };
        for (size_t k = 0; k + 2 < mbq.size(); ++k) ph[(size_t)mbq[k]].arm = mbytes(k + 2);
        arm0 = mbq.size() > 0 ? mbytes(0) : 0;
        arm1 = mbq.size() > 1 ? mbytes(1) : 0;
    };
    if (split) {
        number(0, qa, ctx->bot_arm0, ctx->bot_arm1);
        number(qa, ph.size(), ctx->bot_arm0b, ctx->bot_arm1b);
    } else {
        number(0, ph.size(), ctx->bot_arm0, ctx->bot_arm1);
    }
    ctx->bot_split = split ? (int)qa : 0;
    ctx->bot_ainv = split ? EC.val : nullptr;
    if ((int)ph.size() * sizeof(BPhase) > table) return;
    ctx->d_phases = bot_upload(ctx, ph, ok);
    if (!ok) return;
    ctx->nphases = (int)ph.size();
    ctx->bot_cluster = cs;
    ctx->bot_smem = smem;
    ctx->botJ = J;
}

// Level J of the dense bottom (dense_bottom.cuh): the first level j >= 1 with
// N_j (+1 Poisson) <= MGM_DENSE_MAX (default 4096: B_J = 134 MB, one HBM-bound apply per
// V-cycle instead of the latency-bound colour steps of levels J..p-1); -1 = off.
// column slices of the multi-RHS dense apply (MGM_DENSE_SPLIT; 1 = one kernel, no partials)
static int g_dense_split = std::getenv("MGM_DENSE_SPLIT") ? std::max(1, std::atoi(std::getenv("MGM_DENSE_SPLIT"))) : 4;
int dense_level(const mgm_ctx* ctx) {
    i64 dmax = 4096;
    if (const char* e = std::getenv("MGM_DENSE_MAX")) dmax = std::atoll(e);
    const i64 pad = ctx->poisson ? 1 : 0;
    for (int j = 1; j < ctx->p; ++j)
        if (ctx->lv[j].n + pad <= dmax) return j;
    return -1;
}

// Setup phase timer (MGM_SETUP_TIMING=1 prints host wall time per phase to stderr).
struct SetupTimer {
    bool on = std::getenv("MGM_SETUP_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what, int level = -1) {
        if (!on) return;
        auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[mgm setup] %-22s L%-2d %9.1f ms\n", what, level,
                     std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

// Coarsest LU on the device (cuSOLVER): A row-major on the host -> ctx->lu (column-major
// factors, unit L below the diagonal), ctx->piv (0-based row swaps, as dense_lu_colmajor),
// and with want_inv the explicit inverse ctx->ainv (row-major) from getrs on A^T X = I
// (X = A^-T column-major = A^-1 row-major).  *bad = the first pivot column with
// |u_kk| <= 1e-14 max|a_ij| (dense_lu_colmajor's singularity test), else -1.
__global__ void k_identity(int m, double* X) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (int64_t)m * m;
         t += (int64_t)gridDim.x * blockDim.x)
        X[t] = (t / m == t % m) ? 1.0 : 0.0;
}
__global__ void k_piv0(int m, const int* __restrict__ ipiv1, int* __restrict__ piv0) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) piv0[k] = ipiv1[k] - 1;
}
mgm_status device_lu(mgm_ctx* ctx, const std::vector<double>& A, int m, bool want_inv, i64* bad) {
    cudaStream_t st = ctx->st;
    CusolverApi& cs = cusolver();
    double amax = 0.0;
    for (double v : A) amax = std::max(amax, std::fabs(v));
    std::vector<double> Ac((size_t)m * m);  // column-major copy
    {
        auto cols = [&](i64 a, i64 b) {
            for (i64 j = a; j < b; ++j)
                for (int i = 0; i < m; ++i) Ac[(size_t)j * m + i] = A[(size_t)i * m + j];
        };
        const int nt = m >= 512 ? host_threads() : 1;
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(cols, (i64)m * t / nt, (i64)m * (t + 1) / nt);
        cols(0, (i64)m / nt);
        for (auto& x : th) x.join();
    }
    if (mgm_status s = upload(ctx, &ctx->lu, Ac)) return s;
    cusolverDnHandle_t h = nullptr;
    if (cs.Create(&h) != CUSOLVER_STATUS_SUCCESS) {
        ctx->err = "cusolverDnCreate failed";
        return MGM_ERR_CUDA;
    }
    struct HDel { CusolverApi& cs; cusolverDnHandle_t h; ~HDel() { cs.Destroy(h); } } hdel_{cs, h};
    cs.SetStream(h, st);
    int lwork = 0;
    if (cs.GetrfBuf(h, m, m, ctx->lu, m, &lwork) != CUSOLVER_STATUS_SUCCESS) {
        ctx->err = "cusolverDnDgetrf_bufferSize failed";
        return MGM_ERR_CUDA;
    }
    double* work = nullptr;
    int *ipiv = nullptr, *info = nullptr;
    CK(dalloc(&work, std::max(lwork, 1)));
    CK(dalloc(&ipiv, m));
    CK(dalloc(&info, 1));
    struct WDel { double* w; int* a; int* b; ~WDel() { dev_free(w); dev_free(a); dev_free(b); } } wdel_{work, ipiv, info};
    if (cs.Getrf(h, m, m, ctx->lu, m, work, ipiv, info) != CUSOLVER_STATUS_SUCCESS) {
        ctx->err = "cusolverDnDgetrf failed";
        return MGM_ERR_CUDA;
    }
    std::vector<double> dg(m);
    CK(cudaMemcpy2DAsync(dg.data(), sizeof(double), ctx->lu, sizeof(double) * (m + 1), sizeof(double), m,
                         cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *bad = -1;
    for (int k = 0; k < m; ++k)
        if (!(std::fabs(dg[k]) > 1e-14 * amax)) {
            *bad = k;
            return MGM_OK;
        }
    CK(dalloc(&ctx->piv, m));
    k_piv0<<<blocks_for(m, 256), 256, 0, st>>>(m, ipiv, ctx->piv);
    if (want_inv) {
        CK(dalloc(&ctx->ainv, (i64)m * m));
        k_identity<<<1184, 256, 0, st>>>(m, ctx->ainv);
        if (cs.Getrs(h, CUBLAS_OP_T, m, m, ctx->lu, m, ipiv, ctx->ainv, m, info) != CUSOLVER_STATUS_SUCCESS) {
            ctx->err = "cusolverDnDgetrs failed";
            return MGM_ERR_CUDA;
        }
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    return MGM_OK;
}

mgm_status do_setup(mgm_ctx* ctx, const double* points, const double* normals, i64 N) {
    DeferFree deferred;  // (destroyed last: after every setup thread has been joined)
    DeferScope defer_(&deferred);
    SetupTimer tm;
    const auto& sp = ctx->sp;
    const auto& lp = ctx->lp;
    cudaStream_t st = ctx->st;
    int nth = ctx->nthreads;
    // ---- input checks
    for (i64 i = 0; i < 3 * N; ++i)
        if (!std::isfinite(points[i]) || !std::isfinite(normals[i])) return fail(ctx, MGM_ERR_INPUT, "non-finite input", i / 3);
    // ---- Alg. 2 lines 2-3: order (Morton, O1)
    std::vector<i64> perm;
    if (!morton_order(points, N, perm)) return fail(ctx, MGM_ERR_INPUT, "degenerate point cloud", -1);
    std::vector<double> X(3 * N), NR(3 * N);
    for (i64 k = 0; k < N; ++k)
        for (int a = 0; a < 3; ++a) {
            X[3 * k + a] = points[3 * perm[k] + a];
            NR[3 * k + a] = normals[3 * perm[k] + a];
        }
    // duplicates (the nearest-other distances are level 0's WSE input too)
    // (on the GPU after the upload below unless MGM_HOST_WSE=1 or N < 3)
    const bool use_host_wse = std::getenv("MGM_HOST_WSE") && std::atoi(std::getenv("MGM_HOST_WSE")) != 0;
    std::vector<double> nn2_0;
    if (use_host_wse || N < 3) {
        i64 dup = nearest_other(X.data(), N, nn2_0, nth);
        if (dup >= 0) return fail(ctx, MGM_ERR_INPUT, "duplicate points", perm[dup]);
    }
    tm.mark("morton+duplicates");
    // ---- level count (Alg. 2 line 4)
    int p = lp.num_levels;
    if (p <= 0) {
        p = (int)std::floor(std::log((double)N / lp.n_min) / std::log((double)lp.coarsen_factor)) + 1;
        p = std::max(p, 1);
    }
    {
        i64 n = N;
        for (int j = 1; j < p; ++j) {
            n /= lp.coarsen_factor;
            if (n < 2 || n < lp.interp_m) return fail(ctx, MGM_ERR_ARG, "too many levels for the point count", j);
        }
    }
    ctx->p = p;
    // ---- fine stencils and weights on the GPU
    const int ns = sp.stencil_n;
    double *dX = nullptr, *dN = nullptr, *dW = nullptr, *drho = nullptr;
    i32* dS = nullptr;
    i64* dfail = nullptr;
    CK(dalloc(&dX, 3 * N));
    CK(dalloc(&dS, N * ns));
    CK(cudaMemcpyAsync(dX, X.data(), sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    if (nn2_0.empty()) {
        int e2 = 0;
        i64 dup = nearest_other_device(X.data(), dX, N, nn2_0, st, &e2);
        if (e2 || dup >= 0) {
            dev_free(dX);
            dev_free(dS);
            if (e2) return fail(ctx, MGM_ERR_CUDA, "nearest-other kernels", -1);
            return fail(ctx, MGM_ERR_INPUT, "duplicate points", perm[dup]);
        }
        tm.mark("duplicates (GPU)");
    }
    std::vector<i32> sten((size_t)N * ns);
    if (knn_device(X.data(), dX, N, dX, N, ns, dS, st) == 0) {  // O2 stencils on the GPU
        CK(cudaMemcpyAsync(sten.data(), dS, sizeof(i32) * N * ns, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    } else {  // (k > 64)
        cudaGetLastError();
        knn_grid(X.data(), N, X.data(), N, ns, sten, nth);
        CK(cudaMemcpyAsync(dS, sten.data(), sizeof(i32) * N * ns, cudaMemcpyHostToDevice, st));
    }
    tm.mark("fine kNN");
    HostCSR pat0;  // pattern of L_1: row i's columns are its stencil
    pat0.nrows = pat0.ncols = N;
    pat0.ptr.resize(N + 1);
    for (i64 i = 0; i <= N; ++i) pat0.ptr[i] = i * ns;
    pat0.col = sten;
    std::vector<HostCSR> Lm(p), Pm(p);
    // colourings (O11) run on background threads, each started as soon as its level's
    // pattern is final (L_1's is the stencil lists, right after the kNN; L_{j+1}'s after its
    // Galerkin product), so they overlap the rest of the setup; joined before the lib orders
    // are built (and on every early return).  A colouring reads only the pattern.
    std::vector<std::vector<i32>> colour_mor(p);
    std::vector<int> ncol_j(p, 0);
    // ... and each thread then builds its level's lib order and packs L_j's SELL arrays
    // (host), once L_j's values are final (level 0: after the assembly below)
    struct LevelPack {
        bool done = false;
        std::vector<i64> coff, lib2mor;
        std::vector<i32> mor2lib, colour_lib;
        std::vector<i64> sptr, lower_per_colour;
        hvec<i32> scol;
        hvec<double> sval;
        std::vector<i32> slw, sluw;
        std::vector<uint8_t> nlow;
        HostCSR L_lib;
    };
    std::vector<LevelPack> pk(p);
    struct Gate {  // opened when L_1's values are assembled; aborted on an early return
        std::mutex mu;
        std::condition_variable cv;
        bool open = false, abort = false;
        void set(bool ab) {
            {
                std::lock_guard<std::mutex> lk(mu);
                (ab ? abort : open) = true;
            }
            cv.notify_all();
        }
        bool wait() {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return open || abort; });
            return open;
        }
    } l0_values;
    struct Joiner {
        Gate* g;
        std::vector<std::thread> th;
        ~Joiner() {
            g->set(true);
            join();
        }
        void join() {
            for (auto& t : th)
                if (t.joinable()) t.join();
        }
    } colour_th{&l0_values, {}};
    int setup_dev = 0;
    cudaGetDevice(&setup_dev);
    auto start_colouring = [&](int j, const HostCSR* A) {
        if (j + 1 >= p) return;
        colour_th.th.emplace_back([&, j, A] {
            const int nc = greedy_colouring(*A, colour_mor[j], colour_passes(), setup_dev);
            ncol_j[j] = nc;
            LevelPack& q = pk[j];
            const std::vector<i32>& cm = colour_mor[j];
            const i64 n = A->nrows;
            q.coff.assign(nc + 1, 0);  // lib order: colours ascending, Morton order within
            for (i64 i = 0; i < n; ++i) q.coff[cm[i] + 1]++;
            for (int c = 0; c < nc; ++c) q.coff[c + 1] += q.coff[c];
            q.lib2mor.resize(n);
            q.mor2lib.resize(n);
            std::vector<i64> fillp(q.coff.begin(), q.coff.end() - 1);
            for (i64 i = 0; i < n; ++i) q.lib2mor[fillp[cm[i]]++] = i;
            for (i64 r = 0; r < n; ++r) q.mor2lib[q.lib2mor[r]] = (i32)r;
            q.colour_lib.resize(n);
            for (i64 r = 0; r < n; ++r) q.colour_lib[r] = cm[q.lib2mor[r]];
            if (j == 0 && !l0_values.wait()) return;
            const bool coloured = nc > 0;
            pack_sell(Lm[j], q.lib2mor, q.mor2lib, true, q.sptr, q.scol, q.sval, &q.L_lib,
                      coloured ? &q.colour_lib : nullptr, coloured ? &q.slw : nullptr,
                      coloured ? &q.lower_per_colour : nullptr, coloured ? &q.nlow : nullptr,
                      coloured ? &q.sluw : nullptr);
            q.done = true;
        });
    };
    start_colouring(0, &pat0);
    CK(dalloc(&dN, 3 * N));
    CK(dalloc(&dW, N * ns));
    CK(dalloc(&dfail, 1));
    CK(cudaMemcpyAsync(dN, NR.data(), sizeof(double) * 3 * N, cudaMemcpyHostToDevice, st));
    i64 none = INT64_MAX;
    CK(cudaMemcpyAsync(dfail, &none, sizeof(i64), cudaMemcpyHostToDevice, st));
    int rc;
    if (sp.method == 0) {
        rc = launch_rbffd_weights(dX, dN, dS, N, ns, sp.poly_degree, sp.phs_k, dW, dfail, st);
    } else {
        CK(dalloc(&drho, N));
        rc = launch_stencil_radius(dX, dN, dS, N, ns, drho, st);
        if (!rc) rc = launch_gfd_weights(dX, dN, dS, N, ns, sp.poly_degree, sp.gfd_alpha, drho, dW, dfail, st);
    }
    if (rc) return fail(ctx, MGM_ERR_CUDA, std::string("weight kernel: ") + cudaGetErrorString((cudaError_t)rc), -1);
    std::vector<double> W((size_t)N * ns);
    i64 hfail = 0;
    CK(cudaMemcpyAsync(W.data(), dW, sizeof(double) * N * ns, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&hfail, dfail, sizeof(i64), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    dev_free(dW);
    dev_free(dS);
    dev_free(dN);
    if (drho) dev_free(drho);
    if (hfail != INT64_MAX)
        return fail(ctx, MGM_ERR_UNISOLVENT, sp.method == 0 ? "RBF-FD stencil not unisolvent" : "GFD stencil rank deficient",
                    perm[hfail]);
    tm.mark("fine weights (GPU)");
    // export copy of weights in original order
    // ---- L_1, Morton order CSR with ascending columns
    {
        HostCSR& A = Lm[0];
        A.nrows = A.ncols = N;
        A.ptr.resize(N + 1);
        A.col.resize((size_t)N * ns);
        A.val.resize((size_t)N * ns);
        std::vector<std::thread> th;  // rows are independent: threads over row ranges
        const int nt = std::max(1, std::min(nth, (int)(N / 65536) + 1));
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                std::vector<int> ord(ns);
                for (i64 i = N * t / nt; i < N * (t + 1) / nt; ++i) {
                    A.ptr[i] = i * ns;
                    for (int j = 0; j < ns; ++j) ord[j] = j;
                    std::sort(ord.begin(), ord.end(), [&](int a, int b) { return sten[i * ns + a] < sten[i * ns + b]; });
                    for (int j = 0; j < ns; ++j) {
                        int q = ord[j];
                        double wv = W[i * ns + q];
                        double v;
                        if (sp.problem == 0) v = (q == 0) ? 1.0 - sp.mu * wv : -(sp.mu * wv);
                        else v = wv;
                        A.col[i * ns + j] = sten[i * ns + q];
                        A.val[i * ns + j] = v;
                    }
                }
            });
        for (auto& t : th) t.join();
        A.ptr[N] = N * ns;
    }
    l0_values.set(false);
    ctx->w_mor = std::move(W);
    ctx->sten_mor = std::move(sten);
    ctx->perm0 = perm;
    ctx->ns0 = ns;
    tm.mark("assemble L1");
    // ---- level loop (Alg. 2 lines 5-12)
    std::vector<std::vector<double>> Xl(p);
    std::vector<std::vector<i64>> idsl(p);
    Xl[0] = X;
    idsl[0] = perm;
    double* dXf = dX;
    // Galerkin products on their own thread and stream, pipelined against the point
    // hierarchy: RAP_j needs L_j (the previous product) and P_j (this loop), while WSE and the
    // transfers of the next levels need only the points.
    struct RapPipe {
        std::mutex mu;
        std::condition_variable cv;
        int ready = -1;  // highest j whose P_j is final
        bool abort = false;
        mgm_status status = MGM_OK;
        std::string err;
        i64 err_j = -1;
        std::thread th;
        void publish(int j) {
            {
                std::lock_guard<std::mutex> lk(mu);
                ready = j;
            }
            cv.notify_all();
        }
        void stop() {
            {
                std::lock_guard<std::mutex> lk(mu);
                abort = true;
            }
            cv.notify_all();
            if (th.joinable()) th.join();
        }
        ~RapPipe() { stop(); }
    } rap;
    rap.th = std::thread([&] {
        AllocScope as_(ctx);
        DeferScope defer_(&deferred);
        cudaStream_t rs = nullptr;
        if (cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking) != cudaSuccess) {
            rap.status = MGM_ERR_CUDA;
            rap.err = "cannot create the Galerkin stream";
            return;
        }
        SetupTimer rtm;
        for (int j = 0; j + 1 < p; ++j) {
            {
                std::unique_lock<std::mutex> lk(rap.mu);
                rap.cv.wait(lk, [&] { return rap.ready >= j || rap.abort; });
                if (rap.ready < j) break;
            }
            rtm.t0 = std::chrono::steady_clock::now();
            const HostCSR& P = Pm[j];
            HostCSR R = transpose(P);  // P:370, exact
            // Galerkin L_{j+1} = R (L P) on the GPU
            DevCSR dL, dP, dR, dLP, dC;
            auto release = [&] {
                free_dev_csr(dL);
                free_dev_csr(dP);
                free_dev_csr(dR);
                free_dev_csr(dLP);
                free_dev_csr(dC);
            };
            std::string e1;
            mgm_status st_ = MGM_OK;
            if (upload_csr(Lm[j], dL, rs) || upload_csr(P, dP, rs) || upload_csr(R, dR, rs)) {
                st_ = MGM_ERR_OOM;
                e1 = "upload for SpGEMM";
            } else if (spgemm_device(dL, dP, dLP, rs, e1)) {
                st_ = MGM_ERR_CUDA;
                e1 = "SpGEMM L*P: " + e1;
            } else if (spgemm_device(dR, dLP, dC, rs, e1)) {
                st_ = MGM_ERR_CUDA;
                e1 = "SpGEMM R*(LP): " + e1;
            } else if (download_csr(dC, Lm[j + 1], rs)) {
                st_ = MGM_ERR_CUDA;
                e1 = "download Galerkin";
            }
            release();
            if (st_ != MGM_OK) {
                rap.status = st_;
                rap.err = e1;
                rap.err_j = j;
                break;
            }
            start_colouring(j + 1, &Lm[j + 1]);
            rtm.mark("Galerkin RAP", j);
        }
        cudaStreamSynchronize(rs);
        cudaStreamDestroy(rs);
    });
    for (int j = 0; j + 1 < p; ++j) {
        i64 nf = (i64)Xl[j].size() / 3, ncs = nf / lp.coarsen_factor;
        // WSE: rounds of local maxima on the GPU (wse_device; MGM_HOST_WSE=1: the
        // host's threaded rounds -- the same survivors)
        std::vector<double> nn2;
        if (j == 0) {
            nn2.swap(nn2_0);
        } else if (use_host_wse || nf < 3) {
            nearest_other(Xl[j].data(), nf, nn2, nth);
        } else {
            int e2 = 0;
            nearest_other_device(Xl[j].data(), dXf, nf, nn2, st, &e2);  // (coarse points: distinct)
            if (e2) return fail(ctx, MGM_ERR_CUDA, "nearest-other kernels", -1);
        }
        std::vector<i64> keep;
        if (use_host_wse) {
            wse_eliminate(Xl[j].data(), nf, ncs, nn2, keep, nth);
        } else {
            rc = wse_device(dXf, Xl[j].data(), nf, ncs, nn2, keep, st);
            if (rc) return fail(ctx, MGM_ERR_CUDA, "WSE kernels", -1);
        }
        if ((i64)keep.size() != ncs) return fail(ctx, MGM_ERR_INPUT, "WSE: no non-degenerate elimination radius", -1);
        tm.mark("WSE", j);
        Xl[j + 1].resize(3 * ncs);
        idsl[j + 1].resize(ncs);
        for (i64 k = 0; k < ncs; ++k) {
            for (int a = 0; a < 3; ++a) Xl[j + 1][3 * k + a] = Xl[j][3 * keep[k] + a];
            idsl[j + 1][k] = idsl[j][keep[k]];
        }
        // interpolation stencils (m nearest coarse points, O2) and weights on the GPU
        const int m = lp.interp_m;
        double *dXc = nullptr, *dPw = nullptr;
        i32 *dI = nullptr, *dcnt = nullptr;
        CK(dalloc(&dXc, 3 * ncs));
        CK(dalloc(&dPw, nf * m));
        CK(dalloc(&dI, nf * m));
        CK(dalloc(&dcnt, nf));
        CK(cudaMemcpyAsync(dXc, Xl[j + 1].data(), sizeof(double) * 3 * ncs, cudaMemcpyHostToDevice, st));
        std::vector<i32> ist((size_t)nf * m);
        if (knn_device(Xl[j + 1].data(), dXc, ncs, dXf, nf, m, dI, st) == 0) {
            CK(cudaMemcpyAsync(ist.data(), dI, sizeof(i32) * nf * m, cudaMemcpyDeviceToHost, st));
        } else {  // (m > 64)
            cudaGetLastError();
            knn_grid(Xl[j + 1].data(), ncs, Xl[j].data(), nf, m, ist, nth);
            CK(cudaMemcpyAsync(dI, ist.data(), sizeof(i32) * nf * m, cudaMemcpyHostToDevice, st));
        }
        tm.mark("interp kNN", j);
        CK(cudaMemcpyAsync(dfail, &none, sizeof(i64), cudaMemcpyHostToDevice, st));
        rc = launch_interp_weights(dXf, nf, dXc, dI, m, dPw, dcnt, dfail, st);
        if (rc) return fail(ctx, MGM_ERR_CUDA, "interp kernel", -1);
        std::vector<double> Pw((size_t)nf * m);
        std::vector<i32> pc(nf);
        CK(cudaMemcpyAsync(Pw.data(), dPw, sizeof(double) * nf * m, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(pc.data(), dcnt, sizeof(i32) * nf, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&hfail, dfail, sizeof(i64), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        dev_free(dPw);
        dev_free(dI);
        dev_free(dcnt);
        dev_free(dXf);
        dXf = dXc;
        if (hfail != INT64_MAX) return fail(ctx, MGM_ERR_SINGULAR, "singular transfer system", idsl[j][hfail]);
        HostCSR& P = Pm[j];
        P.nrows = nf;
        P.ncols = ncs;
        P.ptr.assign(nf + 1, 0);
        for (i64 i = 0; i < nf; ++i) P.ptr[i + 1] = P.ptr[i] + pc[i];
        P.col.resize(P.ptr[nf]);
        P.val.resize(P.ptr[nf]);
        {  // rows sorted by column, independent: threads over rows
            auto rows = [&](i64 r0, i64 r1) {
                std::vector<int> ord(m);
                for (i64 i = r0; i < r1; ++i) {
                    int c = pc[i];
                    for (int t = 0; t < c; ++t) ord[t] = t;
                    std::sort(ord.begin(), ord.begin() + c, [&](int a, int b) { return ist[i * m + a] < ist[i * m + b]; });
                    for (int t = 0; t < c; ++t) {
                        P.col[P.ptr[i] + t] = ist[i * m + ord[t]];
                        P.val[P.ptr[i] + t] = Pw[i * m + ord[t]];
                    }
                }
            };
            const int nt = nf >= 65536 ? host_threads() : 1;
            std::vector<std::thread> th;
            for (int t = 1; t < nt; ++t) th.emplace_back(rows, nf * t / nt, nf * (t + 1) / nt);
            rows(0, nf / nt);
            for (auto& x : th) x.join();
        }
        tm.mark("interp weights", j);
        rap.publish(j);
    }
    rap.stop();
    if (rap.status != MGM_OK) return fail(ctx, rap.status, rap.err, rap.err_j);
    tm.mark("Galerkin pipeline wait");
    dev_free(dXf);
    dev_free(dfail);
    // ---- colouring (O11) and lib orders
    ctx->lv.assign(p, Level());
    std::vector<std::vector<i64>> lib2mor(p);
    std::vector<std::vector<i32>> mor2lib(p);
    colour_th.join();
    for (int j = 0; j + 1 < p; ++j) {
        if (!pk[j].done) return fail(ctx, MGM_ERR_ARG, "colouring thread did not finish", j);
        ctx->lv[j].ncol = ncol_j[j];
    }
    for (int j = 0; j < p; ++j) {
        Level& L = ctx->lv[j];
        i64 n = Lm[j].nrows;
        L.n = n;
        if (j + 1 < p) {
            L.coff = std::move(pk[j].coff);
            lib2mor[j] = std::move(pk[j].lib2mor);
            mor2lib[j] = std::move(pk[j].mor2lib);
            L.colour_lib = std::move(pk[j].colour_lib);
        } else {
            L.ncol = 0;
            colour_mor[j].assign(n, 0);
            lib2mor[j].resize(n);
            mor2lib[j].resize(n);
            for (i64 i = 0; i < n; ++i) lib2mor[j][i] = i;
            for (i64 r = 0; r < n; ++r) mor2lib[j][lib2mor[j][r]] = (i32)r;
            L.colour_lib.assign(n, 0);
        }
        L.lib2mor = lib2mor[j];
        L.ids.resize(n);
        for (i64 r = 0; r < n; ++r) L.ids[r] = idsl[j][lib2mor[j][r]];
    }
    tm.mark("colouring");
    // ---- pack solve-phase layout
    mgm_status s;
    for (int j = 0; j < p; ++j) {
        Level& L = ctx->lv[j];
        i64 n = L.n;
        L.nnz = Lm[j].nnz();
        std::vector<i64> sptr;
        hvec<i32> scol;
        hvec<double> sval;
        std::vector<i32> slw, sluw;
        std::vector<uint8_t> nlow;
        bool coloured = L.ncol > 0 && j + 1 < p;
        if (j + 1 < p) {  // packed by the level's colouring thread
            LevelPack& q = pk[j];
            sptr = std::move(q.sptr);
            scol = std::move(q.scol);
            sval = std::move(q.sval);
            slw = std::move(q.slw);
            sluw = std::move(q.sluw);
            nlow = std::move(q.nlow);
            L.L_lib = std::move(q.L_lib);
            L.lower_per_colour = std::move(q.lower_per_colour);
        } else {
            pack_sell(Lm[j], lib2mor[j], mor2lib[j], true, sptr, scol, sval, &L.L_lib);
        }
        for (i64 r = 0; r < n && coloured; ++r)
            if (nlow[(size_t)r] == 255) coloured = false;  // (no zero-guess sweeps for such rows)
        if (coloured && ((s = upload(ctx, &L.slw, slw)) || (s = upload(ctx, &L.nlow, nlow)) ||
                         (s = upload(ctx, &L.sluw, sluw))))
            return s;
        L.sell_stored = (i64)sval.size();
        {
            double wavg = (double)L.sell_stored / (double)std::max<i64>(1, (n + 31) / 32 * 32);
            // threads per row: colour sweeps (short kernels) want more threads per row, the
            // full-level SpMV / residual fewer (measured, profiles/r01_notes.md)
            L.tpr = wavg <= 12 ? 1 : (wavg <= 40 ? 2 : 4);
            // small colours: more threads per row (shorter per-thread chains; L2 of cfg3:
            // 112.8 -> 87.6 us per sweep with 8 instead of 4)
            if (L.ncol > 0 && (double)n / L.ncol * L.tpr < 16384.0 && L.tpr < 8) L.tpr *= 2;
            L.stpr = 1;
            {
                const i64 ns = (n + 31) / 32;
                bool uni = ns > 0;
                for (i64 q = 0; q < ns && uni; ++q) uni = sptr[q + 1] - sptr[q] == sptr[1] - sptr[0];
                L.uniform_w = uni ? (int)((sptr[1] - sptr[0]) / 32) : 0;
            }
            // colours with fewer threads than one 256-thread block per SM run 64-thread blocks
            // (cfg3 L1+L2: -19 us per V-cycle, profiles/r01_notes.md)
            {
                int b = 64;
                if (const char* e = std::getenv("MGM_GS_BLOCK_SMALL")) b = std::atoi(e);
                if ((b == 64 || b == 128 || b == 256) && L.ncol > 0 && (double)n / L.ncol * L.tpr < 148.0 * 256)
                    L.gs_block = b;
                if (const char* e = std::getenv("MGM_GS_BLOCK_L0"))
                    if (j == 0) L.gs_block = std::atoi(e);
            }
            if (const char* e = std::getenv(j == 0 ? "MGM_L0_TPR" : "MGM_LJ_TPR")) {  // tuning experiments
                const int t = std::atoi(e);
                if (t == 1 || t == 2 || t == 4 || t == 8) L.tpr = t;
            }
            if (const char* e = std::getenv(j == 0 ? "MGM_L0_STPR" : "MGM_LJ_STPR")) {
                const int t = std::atoi(e);
                if (t == 1 || t == 2 || t == 4 || t == 8) L.stpr = t;
            }
        }
        if ((s = upload(ctx, &L.sptr, sptr)) || (s = upload(ctx, &L.scol, scol)) || (s = upload(ctx, &L.sval, sval))) return s;
        L.h_sptr = sptr;
        tm.mark("pack L (SELL)", j);
        if (j + 1 < p) {
            const HostCSR& P = Pm[j];
            const int m = lp.interp_m;
            L.pm = m;
            L.p_nnz = P.nnz();
            std::vector<i32> pcol((size_t)m * n);
            std::vector<double> pval((size_t)m * n, 0.0);
            L.P_lib.nrows = n;
            L.P_lib.ncols = Lm[j + 1].nrows;
            L.P_lib.ptr.assign(n + 1, 0);
            for (i64 r = 0; r < n; ++r)
                L.P_lib.ptr[r + 1] = L.P_lib.ptr[r] + P.ptr[lib2mor[j][r] + 1] - P.ptr[lib2mor[j][r]];
            L.P_lib.col.resize(L.P_lib.ptr[n]);
            L.P_lib.val.resize(L.P_lib.ptr[n]);
            auto prow = [&](i64 r0, i64 r1) {
                for (i64 r = r0; r < r1; ++r) {
                    i64 mr = lib2mor[j][r];
                    i64 a = P.ptr[mr], cnt = P.ptr[mr + 1] - a;
                    for (int k = 0; k < m; ++k) {
                        if (k < cnt) {
                            pcol[(size_t)k * n + r] = mor2lib[j + 1][P.col[a + k]];
                            pval[(size_t)k * n + r] = P.val[a + k];
                        } else {
                            pcol[(size_t)k * n + r] = mor2lib[j + 1][P.col[a]];
                            pval[(size_t)k * n + r] = 0.0;
                        }
                    }
                    for (i64 k = 0; k < cnt; ++k) {
                        L.P_lib.col[L.P_lib.ptr[r] + k] = mor2lib[j + 1][P.col[a + k]];
                        L.P_lib.val[L.P_lib.ptr[r] + k] = P.val[a + k];
                    }
                }
            };
            {
                const int nt = n >= 65536 ? host_threads() : 1;
                std::vector<std::thread> th;
                for (int t = 1; t < nt; ++t) th.emplace_back(prow, n * t / nt, n * (t + 1) / nt);
                prow(0, nt > 1 ? n / nt : n);
                for (auto& x : th) x.join();
            }
            if ((s = upload(ctx, &L.pcol, pcol)) || (s = upload(ctx, &L.pval, pval))) return s;
            tm.mark("pack P", j);
            HostCSR R = transpose(P);
            std::vector<i64> rptr;
            hvec<i32> rcol;
            hvec<double> rval;
            pack_sell(R, lib2mor[j + 1], mor2lib[j], false, rptr, rcol, rval, nullptr);
            L.r_stored = (i64)rval.size();
            {  // the same R with Morton columns (same entry order, so the same sums)
                std::vector<i32> ident(n), l2m(n);
                for (i64 r = 0; r < n; ++r) ident[(size_t)r] = (i32)r;
                for (i64 r = 0; r < n; ++r) l2m[(size_t)r] = (i32)lib2mor[j][(size_t)r];
                std::vector<i64> rptr2;
                hvec<i32> rcol2;
                hvec<double> rval2;
                pack_sell(R, lib2mor[j + 1], ident, false, rptr2, rcol2, rval2, nullptr);
                if ((s = upload(ctx, &L.rcol_m, rcol2)) || (s = upload(ctx, &L.l2m, l2m))) return s;
            }
            {
                i64 nn = Lm[j + 1].nrows;
                double wavg = (double)L.r_stored / (double)std::max<i64>(1, (nn + 31) / 32 * 32);
                L.rtpr = wavg <= 12 ? 1 : (wavg <= 40 ? 2 : 4);
                if (const char* e = std::getenv("MGM_RTPR")) {  // tuning experiment
                    const int t = std::atoi(e);
                    if (t == 1 || t == 2 || t == 4 || t == 8) L.rtpr = t;
                }
            }
            L.h_rptr = rptr;
            if ((s = upload(ctx, &L.rptr, rptr)) || (s = upload(ctx, &L.rcol, rcol)) || (s = upload(ctx, &L.rval, rval)))
                return s;
            tm.mark("pack R", j);
        }
        i64 vn = n + (ctx->poisson ? 1 : 0);
        CK(dalloc(&L.u, vn));
        CK(dalloc(&L.f, vn));
        CK(dalloc(&L.t, vn));
        CK(cudaMemsetAsync(L.u, 0, sizeof(double) * vn, st));
        CK(cudaMemsetAsync(L.f, 0, sizeof(double) * vn, st));
        CK(cudaMemsetAsync(L.t, 0, sizeof(double) * vn, st));
    }
    tm.mark("pack vectors");
    // ---- Poisson border vectors c_{j+1} = P_j^T c_j, Morton order then lib
    if (ctx->poisson) {
        std::vector<double> cm(N, 1.0);
        for (int j = 0; j < p; ++j) {
            Level& L = ctx->lv[j];
            L.c_lib.resize(L.n);
            for (i64 r = 0; r < L.n; ++r) L.c_lib[r] = cm[lib2mor[j][r]];
            if ((s = upload(ctx, &L.c, L.c_lib))) return s;
            if (j + 1 < p) {
                HostCSR R = transpose(Pm[j]);
                std::vector<double> cn(R.nrows, 0.0);
                for (i64 a = 0; a < R.nrows; ++a) {
                    double acc = 0.0;
                    for (i64 t = R.ptr[a]; t < R.ptr[a + 1]; ++t) acc = acc + R.val[t] * cm[R.col[t]];
                    cn[a] = acc;
                }
                cm.swap(cn);
            }
        }
    }
    // ---- coarsest dense LU (Alg. 2 line 13; O13)
    {
        Level& L = ctx->lv[p - 1];
        int n = (int)L.n;
        int m = n + (ctx->poisson ? 1 : 0);
        if (m > 8192) return fail(ctx, MGM_ERR_ARG, "coarsest level too large for the dense solve", m);
        std::vector<double> A((size_t)m * m, 0.0);
        const HostCSR& C = Lm[p - 1];  // lib order == Morton order on the coarsest level
        for (int i = 0; i < n; ++i)
            for (i64 t = C.ptr[i]; t < C.ptr[i + 1]; ++t) A[(size_t)i * m + C.col[t]] += C.val[t];
        if (ctx->poisson)
            for (int i = 0; i < n; ++i) {
                A[(size_t)i * m + n] = L.c_lib[i];
                A[(size_t)n * m + i] = L.c_lib[i];
            }
        std::vector<double> LU;
        std::vector<i32> piv;
        tm.mark("border vectors");
        ctx->nc = m;
        // large coarsest levels (MGM_DEVICE_LU_MIN, default 1024 rows): LU with partial
        // pivoting and the explicit inverse on the GPU (cuSOLVER getrf / getrs; same pivot rule
        // -- the first row of largest magnitude -- the sums in another order, O13)
        const i64 dlu_min = std::getenv("MGM_DEVICE_LU_MIN") ? std::atoll(std::getenv("MGM_DEVICE_LU_MIN")) : 1024;
        if (m >= dlu_min && cusolver().ok) {
            i64 bad = -1;
            if ((s = device_lu(ctx, A, m, m <= 4096, &bad))) return s;
            tm.mark("coarse LU (device)", p - 1);
            if (bad >= 0) return fail(ctx, MGM_ERR_SINGULAR, "singular coarsest operator", bad);
            ctx->denseJ = dense_level(ctx);
            if (ctx->denseJ < 0) {  // the cluster bottom takes host factors
                LU.resize((size_t)m * m);
                piv.resize(m);
                CK(cudaMemcpy(LU.data(), ctx->lu, sizeof(double) * LU.size(), cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(piv.data(), ctx->piv, sizeof(i32) * m, cudaMemcpyDeviceToHost));
                setup_bottom(ctx, LU, piv);
            }
        } else {
            i64 bad = dense_lu_colmajor(A, m, LU, piv);
            tm.mark("coarse LU", p - 1);
            if (bad >= 0) return fail(ctx, MGM_ERR_SINGULAR, "singular coarsest operator", bad);
            if ((s = upload(ctx, &ctx->lu, LU)) || (s = upload(ctx, &ctx->piv, piv))) return s;
            CK(cudaStreamSynchronize(st));
            ctx->denseJ = dense_level(ctx);
            if (ctx->denseJ < 0) setup_bottom(ctx, LU, piv);  // (the dense bottom replaces it)
            tm.mark("bottom kernel setup", p - 1);
            if (m <= 4096) {  // explicit inverse for the batched coarse solve (same solution up to rounding, O13)
                std::vector<double> Ainv;
                dense_inverse(LU, piv, m, Ainv, nth);
                if ((s = upload(ctx, &ctx->ainv, Ainv))) return s;
                tm.mark("coarse inverse", p - 1);
            }
        }
        cudaGetLastError();
    }
    // ---- level-0 permutation
    {
        std::vector<i32> l2o(N);
        for (i64 r = 0; r < N; ++r) l2o[r] = (i32)ctx->lv[0].ids[r];
        if ((s = upload(ctx, &ctx->d_lib2orig, l2o))) return s;
    }
    if (std::getenv("MGM_TRACE")) {
        CK(dalloc(&ctx->d_trace, 256 + 17 * BOT_MAX_PHASES));
        // MGM_TRACE=2: the bottom kernel also records its fine per-phase clock timeline
        const unsigned long long mode = std::atoi(std::getenv("MGM_TRACE")) == 2 ? 2ull : 0ull;
        CK(cudaMemcpy(ctx->d_trace + 256 + BOT_MAX_PHASES - 1, &mode, 8, cudaMemcpyHostToDevice));
    }
    if (const char* e = std::getenv("MGM_L2_PERSIST"))  // experiment: persisting-L2 carve-out (bytes)
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)std::atoll(e));
    CK(cudaStreamSynchronize(st));
    return MGM_OK;
}

// ---------------------------------------------------------------------------------------
// Solve-phase enqueue helpers (all on stream `st`)
// ---------------------------------------------------------------------------------------
void timer_begin(mgm_ctx* ctx, int cls, cudaStream_t st) {
    KernelTimer& T = ctx->timer[cls];
    if (!T.on || g_dry) return;
    if (T.used + 2 > (int)T.ev.size()) {
        for (int q = 0; q < 64; ++q) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            T.ev.push_back(e);
        }
    }
    cudaEventRecord(T.ev[T.used], st);
}
void timer_end(mgm_ctx* ctx, int cls, cudaStream_t st, double bytes, int nlaunch = 1) {
    KernelTimer& T = ctx->timer[cls];
    if (!T.on || g_dry) return;
    cudaEventRecord(T.ev[T.used + 1], st);
    T.used += 2;
    T.launches += nlaunch;
    T.bytes += bytes;
}
void timer_collect(mgm_ctx* ctx) {
    for (auto& T : ctx->timer) {
        if (!T.on || T.used == 0) continue;
        for (int q = 0; q < T.used; q += 2) {
            cudaEventSynchronize(T.ev[q + 1]);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, T.ev[q], T.ev[q + 1]);
            T.total_ms += ms;
        }
        T.used = 0;
    }
}

double sweep_colour_bytes(const Level& L, i64 rows) {
    // algorithmic: 12 B per stored nonzero of those rows (approximated by the level mean)
    // + f read + u read/write (8+16 B per row)
    return (double)rows * (12.0 * (double)L.nnz / (double)L.n + 24.0);
}

// kernel variants by threads-per-row (chosen per level from the SELL width)
constexpr int CHUNK = 16;
// increments of the sweep being enqueued (enqueue_sweep with dlt; k_sell_spmv MODE 3)
static thread_local double* g_dlt = nullptr;
template <bool P, int TPR>
void gs_launch_t(bool pdl, int r0, int r1, int span, const Level& L, cudaStream_t st, PfList pf, bool zg) {
    // block size: colours too small to give every SM a 256-thread block use smaller blocks
    // (spreads the gathers over more SMs)
    const int bs = L.gs_block;
    if (zg && !P)
        launch(pdl, k_gs_colour<false, TPR, CHUNK, true>, blocks_for((i64)span * TPR, bs), bs, 0, st, r0, r1,
               L.uniform_w, L.sptr, L.scol, L.sval, L.f, L.u, L.c, (int)L.n, pf, (const int*)L.slw,
               (const uint8_t*)L.nlow, (double*)nullptr);
    else
        launch(pdl, k_gs_colour<P, TPR, CHUNK>, blocks_for((i64)span * TPR, bs), bs, 0, st, r0, r1, L.uniform_w, L.sptr,
               L.scol, L.sval, L.f, L.u, L.c, (int)L.n, pf, (const int*)nullptr, (const uint8_t*)nullptr, g_dlt);
}
// Threads one wave of colour kernels can hold (all SMs, register-limited occupancy).
static i64 gs_wave_threads(int tpr, int block) {
    static i64 cache[4][4] = {};
    const int ti = tpr == 1 ? 0 : tpr == 2 ? 1 : tpr == 4 ? 2 : 3;
    const int bi = block == 64 ? 0 : block == 128 ? 1 : block == 256 ? 2 : 3;
    if (cache[ti][bi]) return cache[ti][bi];
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const void* k = tpr == 1 ? (const void*)k_gs_colour<false, 1, CHUNK>
                  : tpr == 2 ? (const void*)k_gs_colour<false, 2, CHUNK>
                  : tpr == 4 ? (const void*)k_gs_colour<false, 4, CHUNK>
                             : (const void*)k_gs_colour<false, 8, CHUNK>;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, block, 0) != cudaSuccess) {
        cudaGetLastError();
        per = 1;
    }
    return cache[ti][bi] = (i64)per * nsm * block;
}

void launch_gs(bool pdl, bool poisson, int tpr, int r0, int r1, int span, const Level& L, cudaStream_t st,
               PfList pf = {}, bool zg = false) {
    // a colour slightly larger than one wave would run a nearly empty second wave (ncu:
    // "1.04 waves" on the largest level-0 colours): halve the threads per row instead
    while (tpr > 1 && (i64)span * tpr > gs_wave_threads(tpr, L.gs_block) &&
           (i64)span * (tpr / 2) <= gs_wave_threads(tpr / 2, L.gs_block))
        tpr /= 2;
    if (poisson) {
        if (tpr == 1) gs_launch_t<true, 1>(pdl, r0, r1, span, L, st, pf, zg);
        else if (tpr == 2) gs_launch_t<true, 2>(pdl, r0, r1, span, L, st, pf, zg);
        else if (tpr == 4) gs_launch_t<true, 4>(pdl, r0, r1, span, L, st, pf, zg);
        else gs_launch_t<true, 8>(pdl, r0, r1, span, L, st, pf, zg);
    } else {
        if (tpr == 1) gs_launch_t<false, 1>(pdl, r0, r1, span, L, st, pf, zg);
        else if (tpr == 2) gs_launch_t<false, 2>(pdl, r0, r1, span, L, st, pf, zg);
        else if (tpr == 4) gs_launch_t<false, 4>(pdl, r0, r1, span, L, st, pf, zg);
        else gs_launch_t<false, 8>(pdl, r0, r1, span, L, st, pf, zg);
    }
}
// distributed levels: the threads per row the undistributed colour launch used (L.tpr_col), so
// every row is summed by the same threads in the same order
void launch_gs_fixed(bool pdl, bool poisson, int tpr, int r0, int r1, int span, const Level& L, cudaStream_t st,
                     bool zg) {
    const PfList pf{nullptr, 0, 0};
    if (poisson) {
        if (tpr == 1) gs_launch_t<true, 1>(pdl, r0, r1, span, L, st, pf, zg);
        else if (tpr == 2) gs_launch_t<true, 2>(pdl, r0, r1, span, L, st, pf, zg);
        else if (tpr == 4) gs_launch_t<true, 4>(pdl, r0, r1, span, L, st, pf, zg);
        else gs_launch_t<true, 8>(pdl, r0, r1, span, L, st, pf, zg);
    } else {
        if (tpr == 1) gs_launch_t<false, 1>(pdl, r0, r1, span, L, st, pf, zg);
        else if (tpr == 2) gs_launch_t<false, 2>(pdl, r0, r1, span, L, st, pf, zg);
        else if (tpr == 4) gs_launch_t<false, 4>(pdl, r0, r1, span, L, st, pf, zg);
        else gs_launch_t<false, 8>(pdl, r0, r1, span, L, st, pf, zg);
    }
}
// the threads per row launch_gs picks for a colour of `span` rows
static int gs_tpr_for(int tpr, i64 span, int block) {
    while (tpr > 1 && span * tpr > gs_wave_threads(tpr, block) && span * (tpr / 2) <= gs_wave_threads(tpr / 2, block))
        tpr /= 2;
    return tpr;
}

// (MODE 2 reads the level's later-colour slot tables g_sluw / g_nlow, set by enqueue_residual)
static thread_local const int* g_sluw = nullptr;
static thread_local const uint8_t* g_nlow = nullptr;
static thread_local const int* g_yperm = nullptr;  // residual output permutation (enqueue_residual)
static thread_local C0Fuse g_c0 = C0Fuse{nullptr, nullptr, nullptr, 0};  // restriction + colour 0 (enqueue_restrict)
template <int MODE, bool P, int TPR>
void spmv_launch_t(bool pdl, i64 r0, i64 r1, i64 nl, const i64* sptr, const i32* scol, const double* sval,
                   const double* x, const double* f, double* y, const double* c, cudaStream_t st, PfList pf) {
    launch(pdl, k_sell_spmv<MODE, P, TPR, CHUNK>, blocks_for((r1 - (r0 & ~31)) * TPR, 256), 256, 0, st, (int)r0,
           (int)r1, (int)nl, sptr, scol, sval, x, f, y, c, pf, MODE >= 2 ? g_sluw : (const int*)nullptr,
           MODE >= 2 ? g_nlow : (const uint8_t*)nullptr, MODE != 0 ? g_yperm : (const int*)nullptr,
           MODE == 0 ? g_c0 : C0Fuse{nullptr, nullptr, nullptr, 0});
}
template <int MODE, bool P>
void spmv_launch_p(bool pdl, int tpr, i64 r0, i64 r1, i64 nl, const i64* sptr, const i32* scol, const double* sval,
                   const double* x, const double* f, double* y, const double* c, cudaStream_t st, PfList pf) {
    if (tpr == 1) spmv_launch_t<MODE, P, 1>(pdl, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
    else if (tpr == 2) spmv_launch_t<MODE, P, 2>(pdl, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
    else if (tpr == 4) spmv_launch_t<MODE, P, 4>(pdl, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
    else spmv_launch_t<MODE, P, 8>(pdl, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
}
// rows [r0, r1) of a SELL operator whose level has nl rows
void launch_spmv(bool pdl, int mode, bool poisson, int tpr, i64 r0, i64 r1, i64 nl, const i64* sptr,
                 const i32* scol, const double* sval, const double* x, const double* f, double* y, const double* c,
                 cudaStream_t st, PfList pf = {}) {
    if (r1 <= r0) return;
    if (mode == 2) {  // residual after a zero-guess sweep (shifted problems)
        spmv_launch_p<2, false>(pdl, tpr, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
    } else if (mode == 3) {  // A u after a forward sweep that added x to u (shifted problems)
        spmv_launch_p<3, false>(pdl, tpr, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
    } else if (mode == 0) {
        if (poisson) spmv_launch_p<0, true>(pdl, tpr, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
        else spmv_launch_p<0, false>(pdl, tpr, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
    } else {
        if (poisson) spmv_launch_p<1, true>(pdl, tpr, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
        else spmv_launch_p<1, false>(pdl, tpr, r0, r1, nl, sptr, scol, sval, x, f, y, c, st, pf);
    }
}

// ---------------------------------------------------------------------------------------
// Multi-GPU (mgm_dist_attach): on the distributed
// levels 0..D-1 each rank holds only its Morton block of rows plus ghost copies of the rows
// its operators read (PartTables); every operator application runs on the owned rows with
// the same per-row arithmetic as one GPU, and halos refresh the ghosts:
//   * after each colour of a Gauss-Seidel sweep: that colour's values (one send / receive
//     per peer, received straight into the ghost slots),
//   * after interpolation + correction, before a restriction (t), before an SpMV: all ghosts.
// The last distributed level restricts its share of the first replicated level D; the shares
// are all-gathered; levels D..p-1 (incl. the dense bottom) run redundantly on every rank.
// ---------------------------------------------------------------------------------------
static bool dist_level(const mgm_ctx* ctx, int j) { return ctx->tp && j < ctx->D; }
static bool dist_on(const mgm_ctx* ctx) { return ctx->tp != nullptr; }

// pack the send entries [range[2p], range[2p+1]) of every peer p (chunks CTAs per peer)
__global__ void k_pack(int chunks, const i64* __restrict__ range, const i32* __restrict__ idx,
                       const double* __restrict__ v, double* __restrict__ out) {
    const int p = blockIdx.x / chunks, b = blockIdx.x % chunks;
    const i64 lo = range[2 * p], hi = range[2 * p + 1];
    for (i64 e = lo + (i64)b * blockDim.x + threadIdx.x; e < hi; e += (i64)chunks * blockDim.x) out[e] = v[idx[e]];
}

// Peer-store halos (MGM_P2P=1; SURVEY 8(e) "B200-native mitigations"): instead of pack + NCCL,
// one kernel stores every send entry straight into the peer's ghost slot (mapped peer memory
// over NVLink: cudaIpc), then its last CTA publishes, per peer, the number of pushes it has
// made to that peer (st.release.sys into the peer's flag array); the consumer side runs a
// one-CTA kernel that waits (ld.acquire.sys) until every peer's count reaches the number of
// exchanges it expects from that peer.  Per-pair counters: ranks need not agree on anything
// but the (symmetric) sequence of exchanges between each pair.  In a fake-rank group the
// flags are replaced by the group's event/barrier ordering (no kernel waits on another).
struct PeerPtrs {
    double* p[16];
};
struct P2PSignal {
    unsigned long long* flag[16];  // &peer_flags[me] on each peer
    int rank[16];                  // peer ranks
    unsigned long long* sent;      // [nranks], this rank's push counters
    unsigned* ticket;
    int npeers;
};
__global__ void k_push(int chunks, const i64* __restrict__ range, const i32* __restrict__ idx,
                       const i64* __restrict__ rslot, const double* __restrict__ v, PeerPtrs dst, P2PSignal sig) {
    const int p = blockIdx.x / chunks, b = blockIdx.x % chunks;
    const i64 lo = range[2 * p], hi = range[2 * p + 1];
    double* d = dst.p[p];
    for (i64 e = lo + (i64)b * blockDim.x + threadIdx.x; e < hi; e += (i64)chunks * blockDim.x) d[rslot[e]] = v[idx[e]];
    if (!sig.sent) return;  // (fake ranks: the group orders the pushes)
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(sig.ticket, 1u) == gridDim.x - 1) {
        *sig.ticket = 0u;
        __threadfence_system();
        for (int i = 0; i < sig.npeers; ++i) {
            const unsigned long long s = ++sig.sent[sig.rank[i]];
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(sig.flag[i]), "l"(s) : "memory");
        }
    }
}
__global__ void k_wait_peers(P2PSignal sig, const unsigned long long* flags, unsigned long long* expect) {
    if (threadIdx.x < sig.npeers) {
        const int r = sig.rank[threadIdx.x];
        const unsigned long long e = ++expect[r];
        unsigned long long got;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(got) : "l"(flags + r) : "memory");
            if (got < e) __nanosleep(64);
        } while (got < e);
    }
    __syncthreads();
}

static void exch_p2p(mgm_ctx* ctx, int j, double* v, int c, cudaStream_t st);

// halo of vector v on distributed level j: colour c's owned values (c < 0: every ghost)
static void exch(mgm_ctx* ctx, int j, double* v, int c, cudaStream_t st) {
    if (!dist_level(ctx, j) || g_dry) return;
    Level& L = ctx->lv[j];
    const int np = (int)L.peers.size();
    if (np == 0) return;
    if (ctx->p2p) {
        exch_p2p(ctx, j, v, c, st);
        return;
    }
    const int nc1 = L.ncol + 1;
    std::vector<Xfer> x((size_t)np);
    i64 maxlen = 0;
    for (int i = 0; i < np; ++i) {
        const i64 s0 = c < 0 ? L.send_off[i] : L.send_coff[(size_t)i * nc1 + c];
        const i64 s1 = c < 0 ? L.send_off[i + 1] : L.send_coff[(size_t)i * nc1 + c + 1];
        const i64 r0 = c < 0 ? L.recv_off[i] : L.recv_coff[(size_t)i * nc1 + c];
        const i64 r1 = c < 0 ? L.recv_off[i + 1] : L.recv_coff[(size_t)i * nc1 + c + 1];
        maxlen = std::max(maxlen, s1 - s0);
        x[(size_t)i] = Xfer{L.peers[(size_t)i], L.d_sendbuf + s0, s1 - s0, v + L.gbase + r0, r1 - r0};
    }
    if (maxlen > 0) {
        const int chunks = (int)std::min<i64>(32, (maxlen + 255) / 256);
        launch(false, k_pack, (unsigned)(chunks * np), 256, 0, st, chunks,
               (const i64*)(L.d_srange + (size_t)(c + 1) * 2 * np), (const i32*)L.d_send_idx, (const double*)v,
               L.d_sendbuf);
    }
    if (!ctx->tp->exchange(x, st) && ctx->err.empty()) ctx->err = "halo exchange failed";
    g_after_comm = true;
    ctx->vcycle_kernels += 2;
}

static void exch_p2p(mgm_ctx* ctx, int j, double* v, int c, cudaStream_t st) {
    Level& L = ctx->lv[j];
    const int np = (int)L.peers.size();
    const int nc1 = L.ncol + 1;
    i64 maxlen = 0;
    for (int i = 0; i < np; ++i) {
        const i64 s0 = c < 0 ? L.send_off[i] : L.send_coff[(size_t)i * nc1 + c];
        const i64 s1 = c < 0 ? L.send_off[i + 1] : L.send_coff[(size_t)i * nc1 + c + 1];
        maxlen = std::max(maxlen, s1 - s0);
    }
    const bool is_u = v == L.u;
    PeerPtrs dst{};
    for (int i = 0; i < np; ++i) dst.p[i] = is_u ? L.peer_u[i] : L.peer_t[i];
    P2PSignal sig{};
    sig.npeers = np;
    for (int i = 0; i < np; ++i) {
        sig.rank[i] = L.peers[(size_t)i];
        sig.flag[i] = ctx->peer_flags[L.peers[(size_t)i]] ? ctx->peer_flags[L.peers[(size_t)i]] + ctx->rank : nullptr;
    }
    const int chunks = (int)std::max<i64>(1, std::min<i64>(32, (maxlen + 255) / 256));
    const i64* rng = L.d_srange + (size_t)(c + 1) * 2 * np;
    if (!ctx->tp->capturable()) {  // fake ranks: the group orders the pushes (no flags)
        auto push = [&](cudaStream_t s2) {
            launch(false, k_push, (unsigned)(chunks * np), 256, 0, s2, chunks, rng, (const i32*)L.d_send_idx,
                   (const i64*)L.d_rslot, (const double*)v, dst, P2PSignal{});
        };
        if (!static_cast<FakeTransport*>(ctx->tp)->ordered(push, st) && ctx->err.empty()) ctx->err = "p2p halo failed";
    } else {
        sig.sent = ctx->p2p_sent;
        sig.ticket = ctx->p2p_ticket;
        launch(false, k_push, (unsigned)(chunks * np), 256, 0, st, chunks, rng, (const i32*)L.d_send_idx,
               (const i64*)L.d_rslot, (const double*)v, dst, sig);
        launch(false, k_wait_peers, 1u, 32u, 0, st, sig, (const unsigned long long*)ctx->p2p_flags, ctx->p2p_expect);
    }
    g_after_comm = true;
    ctx->vcycle_kernels += 2;
}

// Krylov / border inner products: rows this rank contributes (the replicated Poisson
// multiplier is counted once, by rank 0)
static i64 dot_rows(const mgm_ctx* ctx) {
    return ctx->lv[0].n + ((ctx->poisson && ctx->rank == 0) ? 1 : 0);
}
// rows of a level-0 vector (owned rows + multiplier; ghosts excluded)
static i64 vec_rows(const mgm_ctx* ctx) { return ctx->lv[0].n + (ctx->poisson ? 1 : 0); }

bool timing_on(const mgm_ctx* ctx);
// zg: first forward sweep from a zero guess (k_gs_colour ZG; shifted problems only)
void enqueue_sweep(mgm_ctx* ctx, int j, bool backward, cudaStream_t st, bool zg = false, bool skip_c0 = false) {
    Level& L = ctx->lv[j];
    zg = zg && !backward && !ctx->poisson && L.slw;
    // timing class 0: CUDA events around the whole level-0 sweep (the colour kernels keep
    // their PDL overlap inside it); launches and algorithmic bytes are summed over colours
    const int tcls = zg ? 3 : 0;  // zero-guess level-0 sweeps are their own timing class
    if (j == 0) timer_begin(ctx, tcls, st);
    double bytes = 0.0;
    int nl = 0;
    for (int q = (skip_c0 && zg) ? 1 : 0; q < L.ncol; ++q) {  // (colour 0 done by the restriction)
        const int c = backward ? L.ncol - 1 - q : q;
        const i64 c0 = L.coff[c], c1 = L.coff[c + 1];
        if (c1 > c0) {
            if (L.dist)  // the undistributed launch's threads per row: same per-row arithmetic
                launch_gs_fixed(ctx->pdl, ctx->poisson, L.tpr_col[(size_t)c], (int)c0, (int)c1,
                                (int)(c1 - (c0 & ~31)), L, st, zg);
            else
                launch_gs(ctx->pdl, ctx->poisson, L.tpr, (int)c0, (int)c1, (int)(c1 - (c0 & ~31)), L, st,
                          PfList{nullptr, 0, 0}, zg);
            // algorithmic bytes; a zero-guess sweep reads its stored entries and f, writes u
            bytes += zg ? (12.0 * (double)L.lower_per_colour[c] + 16.0 * (double)(c1 - c0))
                        : sweep_colour_bytes(L, c1 - c0);
            ++nl;
            ctx->vcycle_kernels++;
        }
        exch(ctx, j, L.u, c, st);  // (collective: every rank calls it, even with no rows of c)
    }
    if (j == 0) timer_end(ctx, tcls, st, bytes, nl);
}

// Poisson border row: y[n] = fs*f[n] + sign * (c . x)  (distributed: + allreduce of c . x)
void enqueue_border_dot(mgm_ctx* ctx, int j, const double* x, const double* f, double fs, double sign, double* y,
                        cudaStream_t st) {
    const Level& L = ctx->lv[j];
    if (dist_level(ctx, j)) {
        double* s = ctx->dh + 600;
        k_multidot_fin<<<RED_BLOCKS, RED_THREADS, 0, st>>>((i64)L.n, (const double*)L.c, (i64)0, 1, x, ctx->partials,
                                                           ctx->tickets, s, (double*)nullptr);
        if (!ctx->tp->allreduce_sum(s, 1, st) && ctx->err.empty()) ctx->err = "allreduce failed";
        g_after_comm = true;
        k_border_set<<<1, 32, 0, st>>>(s, fs, f, (int)L.n, sign, y);
        ctx->vcycle_kernels += 3;
        return;
    }
    launch(ctx->pdl, k_multidot, RED_BLOCKS, RED_THREADS, 0, st, (i64)L.n, (const double*)L.c, (i64)0, 1, x,
           ctx->partials);
    launch(ctx->pdl, k_border_finish, 1, 32, 0, st, (const double*)ctx->partials, (int)RED_BLOCKS, fs, f, (int)L.n,
           sign, y);
    ctx->vcycle_kernels += 2;
}

// y = L x (level j); distributed: x must have its ghosts current (the callers exchange)
void enqueue_spmv(mgm_ctx* ctx, int j, const double* x, double* y, cudaStream_t st) {
    Level& L = ctx->lv[j];
    if (j == 0) timer_begin(ctx, 1, st);
    launch_spmv(ctx->pdl, 0, ctx->poisson, L.stpr, 0, L.n, L.n, L.sptr, L.scol, L.sval, x, nullptr, y, L.c, st);
    if (j == 0) timer_end(ctx, 1, st, 12.0 * L.nnz + 16.0 * L.n);
    if (ctx->poisson) enqueue_border_dot(ctx, j, x, nullptr, 0.0, 1.0, y, st);
}

// t = f - L u (level j), Poisson: t[n] = f[n] - c.u.  after_zg: u is the result of ONE forward
// sweep from a zero guess, so t = -(later-colour part of L) u (k_sell_spmv MODE 2)
// morton_t: write t in the level's Morton order (the restriction then gathers with Morton
// columns, a few sectors per coarse row instead of one per fine entry; not on distributed levels)
void enqueue_residual(mgm_ctx* ctx, int j, const double* f, const double* u, double* t, cudaStream_t st,
                      bool after_zg = false, bool morton_t = false) {
    Level& L = ctx->lv[j];
    g_yperm = (morton_t && L.l2m && !L.dist) ? L.l2m : nullptr;
    struct ResetP { ~ResetP() { g_yperm = nullptr; } } resetp_;
    // (bandwidth-bound levels only: on the small latency-bound levels the extra per-row table
    // loads cost more than the skipped entries save -- cfg3 L2/L3 17 -> 23 us)
    const int mode = (after_zg && L.sluw && !ctx->poisson && !ctx->no_zg && L.n >= ctx->upper_res_min) ? 2 : 1;
    g_sluw = L.sluw;
    g_nlow = L.nlow;
    launch_spmv(ctx->pdl, mode, ctx->poisson, L.stpr, 0, L.n, L.n, L.sptr, L.scol, L.sval, u, f, t, L.c, st);
    ctx->vcycle_kernels++;
    if (ctx->poisson) enqueue_border_dot(ctx, j, u, f, 1.0, -1.0, t, st);
}

// y (next level) = R_j x
// fuse_c0: also set colour 0 of level j+1's presmooth from zero (u = f / a_rr), which the
// following sweep then skips (undistributed, shifted problems)
// Distributed level j: x's ghosts (the fine residual rows the restriction reads) are exchanged
// first; if level j+1 is the first replicated level, this rank's coarse rows go to the staging
// vector, which is all-gathered and permuted into y.
void enqueue_restrict(mgm_ctx* ctx, int j, double* x, double* y, cudaStream_t st, bool morton_x = false,
                      bool fuse_c0 = false) {
    Level& L = ctx->lv[j];
    Level& Ln = ctx->lv[j + 1];
    if (fuse_c0) g_c0 = C0Fuse{Ln.u, Ln.sptr, Ln.sval, (int)Ln.coff[1]};
    struct ResetC0 { ~ResetC0() { g_c0 = C0Fuse{nullptr, nullptr, nullptr, 0}; } } resetc0_;
    const i32* rcol = (morton_x && L.rcol_m && !L.dist) ? L.rcol_m : L.rcol;
    exch(ctx, j, x, -1, st);
    const bool to_stage = L.dist && L.d_stage_all;
    const i64 nrows = to_stage ? L.nstage : Ln.n;
    double* out = to_stage ? L.d_stage_mine : y;
    launch_spmv(ctx->pdl, 0, false, L.rtpr, 0, nrows, nrows, L.rptr, rcol, L.rval, x, nullptr, out, nullptr, st);
    ctx->vcycle_kernels++;
    if (to_stage) {
        if (!ctx->tp->allgatherv(L.d_stage_mine, L.d_stage_all, L.stage_off, st) && ctx->err.empty())
            ctx->err = "all-gather failed";
        g_after_comm = true;
        k_scatter<<<blocks_for(Ln.n, 256), 256, 0, st>>>((int)Ln.n, L.d_stage_perm, L.d_stage_all, y);
        ctx->vcycle_kernels += 2;
    }
    if (ctx->poisson) {
        launch(ctx->pdl, k_copy1, 1, 1, 0, st, (const double*)(x + L.n), y + Ln.n);
        ctx->vcycle_kernels++;
    }
}

// Fused residual + restriction (solve_kernels.cuh k_res_restrict, north_star item 4): one
// cooperative launch, grid = every CTA the kernel can keep resident.  Undistributed shifted
// levels with one thread per residual row and 1/2/4 per restriction row; MGM_NO_FUSE_RR=1
// keeps the two kernels (comparison).
static bool g_no_fuse_rr = std::getenv("MGM_NO_FUSE_RR") != nullptr;
// levels with at least this many rows (MGM_FUSE_RR_MIN): below it the grid barrier and the
// lost PDL overlap cost more than the second kernel (cfg3 L1-L3: 34 / 18 / 15 us unfused vs
// 47 / 25 / 23 fused; L0: 106.5 vs 103.3)
static i64 g_fuse_rr_min = std::getenv("MGM_FUSE_RR_MIN") ? std::atoll(std::getenv("MGM_FUSE_RR_MIN")) : 524288;
bool fused_rr_ok(const mgm_ctx* ctx, int j) {
    const Level& L = ctx->lv[j];
    return !g_no_fuse_rr && L.n >= g_fuse_rr_min && !dist_on(ctx) && !ctx->poisson && L.stpr == 1 &&
           (L.rtpr == 1 || L.rtpr == 2 || L.rtpr == 4) && j + 1 < ctx->p;
}
template <int MODE, int TPRR>
static void launch_rr(mgm_ctx* ctx, const ResRestrict& a, cudaStream_t st) {
    auto kern = k_res_restrict<MODE, 1, TPRR, CHUNK>;
    static int grid = 0;
    if (!grid) {
        int dev = 0, nsm = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0) != cudaSuccess || per < 1) per = 1;
        grid = per * nsm;
    }
    if (g_dry) return;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (ctx->pdl && g_use_pdl) ? 2 : 1;
    note_launch(cudaLaunchKernelEx(&cfg, kern, a), (unsigned)grid, 256, 0);
}
void enqueue_res_restrict(mgm_ctx* ctx, int j, const double* f, const double* u, double* t, double* y,
                          cudaStream_t st, bool after_zg, bool morton_t, bool fuse_c0) {
    Level& L = ctx->lv[j];
    Level& Ln = ctx->lv[j + 1];
    const int mode = (after_zg && L.sluw && !ctx->no_zg && L.n >= ctx->upper_res_min) ? 2 : 1;
    ResRestrict a{};
    a.n = (int)L.n;
    a.sptr = L.sptr;
    a.scol = L.scol;
    a.sval = L.sval;
    a.u = u;
    a.f = f;
    a.t = t;
    a.sluw = L.sluw;
    a.nlow = L.nlow;
    a.yperm = (morton_t && L.l2m) ? L.l2m : nullptr;
    a.nc = (int)Ln.n;
    a.rptr = L.rptr;
    a.rcol = (morton_t && L.rcol_m) ? L.rcol_m : L.rcol;
    a.rval = L.rval;
    a.y = y;
    a.c0 = fuse_c0 ? C0Fuse{Ln.u, Ln.sptr, Ln.sval, (int)Ln.coff[1]} : C0Fuse{nullptr, nullptr, nullptr, 0};
    if (mode == 2) {
        if (L.rtpr == 1) launch_rr<2, 1>(ctx, a, st);
        else if (L.rtpr == 2) launch_rr<2, 2>(ctx, a, st);
        else launch_rr<2, 4>(ctx, a, st);
    } else {
        if (L.rtpr == 1) launch_rr<1, 1>(ctx, a, st);
        else if (L.rtpr == 2) launch_rr<1, 2>(ctx, a, st);
        else launch_rr<1, 4>(ctx, a, st);
    }
    ctx->vcycle_kernels++;
}

// e_j += P_j e_{j+1}; distributed: the ghosts of e_j are refreshed afterwards
void enqueue_interp_correct(mgm_ctx* ctx, int j, const double* ec, double* e, cudaStream_t st) {
    Level& L = ctx->lv[j];
    Level& Ln = ctx->lv[j + 1];
    auto kern = ctx->poisson ? (L.pm <= 8 ? k_interp_correct<true, 8> : k_interp_correct<true, 16>)
                             : (L.pm <= 8 ? k_interp_correct<false, 8> : k_interp_correct<false, 16>);
    const i64 extra = ctx->poisson ? 1 : 0;  // multiplier thread
    launch(ctx->pdl, kern, blocks_for(L.n + extra, 256), 256, 0, st, 0, (int)L.n, (int)L.n, L.pm, (const i32*)L.pcol,
           (const double*)L.pval, ec, e, (int)Ln.n, PfList{nullptr, 0, 0});
    ctx->vcycle_kernels++;
    exch(ctx, j, e, -1, st);
}

void enqueue_coarse(mgm_ctx* ctx, const double* r, double* e, cudaStream_t st) {
    const int m = ctx->nc;
    if (m >= 1024 && ctx->ainv) {  // large coarsest: grid-wide GEMV with the explicit inverse (O13)
        launch(ctx->pdl, k_dense_gemv, (unsigned)((m + 3) / 4), 128, 0, st, m, (const double*)ctx->ainv, r, e);
        ctx->vcycle_kernels++;
        return;
    }
    const int in_smem = (size_t)(m + m * m) * sizeof(double) <= 200 * 1024 ? 1 : 0;
    const size_t smem = sizeof(double) * (m + (in_smem ? (size_t)m * m : 0));
    set_max_dyn_smem((const void*)k_coarse_solve);
    launch(ctx->pdl, k_coarse_solve, 1, 256, smem, st, m, in_smem, (const double*)ctx->lu, (const i32*)ctx->piv, r, e);
    ctx->vcycle_kernels++;
}

void enqueue_zero(mgm_ctx* ctx, double* x, i64 n, cudaStream_t st) {
    launch(ctx->pdl, k_fill, blocks_for(n, 256), 256, 0, st, n, x, 0.0, PfList{nullptr, 0, 0});
    ctx->vcycle_kernels++;
}

// Trace stamp: waits for its predecessor (PDL) and records %globaltimer (ns).
__global__ void k_stamp(unsigned long long* slot) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *slot = t;
}
void stamp(mgm_ctx* ctx, const char* label, int level, cudaStream_t st) {
    if (!ctx->d_trace || ctx->ntrace >= 256) return;
    launch(true, k_stamp, 1, 1, 0, st, ctx->d_trace + ctx->ntrace);
    ctx->trace_labels.push_back(std::string(label) + " L" + std::to_string(level));
    ctx->ntrace++;
}

mgm_status ensure_krylov(mgm_ctx* ctx);
// Alg. 3 lines 6-14 for the levels J..p-1 (J >= 1) from e_J = 0, one kernel per colour /
// operator, no zero-guess shortcuts: rhs lv[J].f, result lv[J].u.  Builds the dense bottom.
void enqueue_levels_plain(mgm_ctx* ctx, int J, cudaStream_t st) {
    auto& lv = ctx->lv;
    const int p = ctx->p;
    const int nu1 = ctx->lp.nu1, nu2 = ctx->lp.nu2;
    const bool pre_b = ctx->lp.smoother == 1, post_b = ctx->lp.smoother == 1 || ctx->lp.smoother == 2;
    const i64 pad = ctx->poisson ? 1 : 0;
    if (J == p - 1) {
        enqueue_coarse(ctx, lv[J].f, lv[J].u, st);
        return;
    }
    for (int j = J; j + 1 < p; ++j) {                                    // lines 6-9
        enqueue_zero(ctx, lv[j].u, lv[j].n + pad, st);
        for (int s = 0; s < nu1; ++s) enqueue_sweep(ctx, j, pre_b, st);
        enqueue_residual(ctx, j, lv[j].f, lv[j].u, lv[j].t, st);
        enqueue_restrict(ctx, j, lv[j].t, lv[j + 1].f, st);
    }
    enqueue_coarse(ctx, lv[p - 1].f, lv[p - 1].u, st);                  // line 10
    for (int j = p - 2; j >= J; --j) {                                   // lines 11-14
        enqueue_interp_correct(ctx, j, lv[j + 1].u, lv[j].u, st);
        for (int s = 0; s < nu2; ++s) enqueue_sweep(ctx, j, post_b, st);
    }
}

mgm_status build_dense_columns_b(mgm_ctx* ctx, int J, int mdim, double* T, cudaStream_t st);
// B_J = the matrix of lines 6-14 for levels >= J (dense_bottom.cuh), one column per replay
// of enqueue_levels_plain on a unit vector; on the coarsest level it is L_p^{-1} (the
// explicit inverse, O13).  Row-major, leading dimension padded to 64 with zeros.
mgm_status setup_dense_bottom(mgm_ctx* ctx) {
    const int J = ctx->denseJ;
    if (J < 0) return MGM_OK;
    {
        mgm_status s = ensure_krylov(ctx);  // (reduction scratch of the Poisson border terms)
        if (s) return s;
    }
    cudaStream_t st = ctx->st;
    const i64 pad = ctx->poisson ? 1 : 0;
    const int mdim = (int)(ctx->lv[J].n + pad);
    const int ld = (mdim + 63) / 64 * 64;
    double* T = nullptr;
    CK(dalloc(&ctx->dB, (i64)mdim * ld));
    CK(dalloc(&T, (i64)mdim * mdim));
    struct FreeT { double* t; ~FreeT() { dev_free(t); } } freet_{T};
    if (!ctx->poisson && ctx->bK == 0 && J < ctx->p - 1 && ctx->ainv && !std::getenv("MGM_DENSE_BUILD_SINGLE")) {
        // 8 unit vectors per replay through the batched level kernels (non-Poisson)
        mgm_status s = build_dense_columns_b(ctx, J, mdim, T, st);
        if (s) return s;
        k_transpose_pad<<<dim3((mdim + 31) / 32, ld / 32), dim3(32, 8), 0, st>>>(mdim, ld, T, ctx->dB);
        CK(cudaStreamSynchronize(st));
        CK(cudaGetLastError());
        ctx->dense_m = mdim;
        ctx->dense_ld = ld;
        if (g_dense_split > 1) CK(dalloc(&ctx->dP, (i64)g_dense_split * mdim * 8));
        return MGM_OK;
    }
    cudaGraph_t g = nullptr;
    cudaGraphExec_t gx = nullptr;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    g_launch_err.clear();
    ctx->pdl = true;
    enqueue_levels_plain(ctx, J, st);
    ctx->pdl = false;
    const cudaError_t ce = cudaStreamEndCapture(st, &g);
    if (ce != cudaSuccess || !g_launch_err.empty()) {
        ctx->err = "dense bottom capture failed: " + std::string(cudaGetErrorString(ce)) + "; " + g_launch_err;
        g_launch_err.clear();
        cudaGetLastError();
        return MGM_ERR_CUDA;
    }
    CK(cudaGraphInstantiate(&gx, g, 0));
    cudaGraphDestroy(g);
    Level& L = ctx->lv[J];
    for (int i = 0; i < mdim; ++i) {
        k_unit<<<blocks_for(mdim, 256), 256, 0, st>>>(mdim, i, L.f);
        CK(cudaGraphLaunch(gx, st));
        CK(cudaMemcpyAsync(T + (i64)i * mdim, L.u, sizeof(double) * mdim, cudaMemcpyDeviceToDevice, st));
    }
    k_transpose_pad<<<dim3((mdim + 31) / 32, ld / 32), dim3(32, 8), 0, st>>>(mdim, ld, T, ctx->dB);
    CK(cudaStreamSynchronize(st));
    cudaGraphExecDestroy(gx);
    CK(cudaGetLastError());
    ctx->dense_m = mdim;
    ctx->dense_ld = ld;
    if (g_dense_split > 1) CK(dalloc(&ctx->dP, (i64)g_dense_split * mdim * 8));
    return MGM_OK;
}

// e_J = B_J r_J (the whole bottom of the V-cycle, dense_bottom.cuh); K interleaved columns
void enqueue_dense_bottom(mgm_ctx* ctx, int K, const double* r, double* e, cudaStream_t st) {
    const unsigned grid = blocks_for(ctx->dense_m, DENSE_ROWS_PER_CTA);
    const int mm = ctx->dense_m, ld = ctx->dense_ld;
    const double* B = ctx->dB;
    if (K > 1 && ctx->dP && g_dense_split > 1) {  // column-split apply + ordered sum of the partials
        const int S = g_dense_split;
        const int cs = (int)(((ld + S - 1) / S + 63) / 64 * 64);
        const dim3 g2(blocks_for(mm, 4 * DENSE_ROWS_PER_CTA), (unsigned)((ld + cs - 1) / cs));
        auto go = [&](auto kern) {
            if (g_dry) return;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = g2;
            cfg.blockDim = dim3(DENSE_THREADS);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = g_use_pdl ? 1 : 0;
            note_launch(cudaLaunchKernelEx(&cfg, kern, mm, ld, cs, B, r, ctx->dP), g2.x * g2.y, DENSE_THREADS, 0);
        };
        if (K == 2) go(k_dense_apply_split<2, 4>);
        else if (K == 4) go(k_dense_apply_split<4, 4>);
        else go(k_dense_apply_split<8, 4>);
        launch(true, k_dense_sum, blocks_for((i64)mm * K, 256), 256, 0, st, (int64_t)mm * K, (int)g2.y,
               (const double*)ctx->dP, e);
        ctx->vcycle_kernels += 2;
        return;
    }
    switch (K) {
        case 1: launch(ctx->pdl, k_dense_apply<1>, grid, DENSE_THREADS, 0, st, mm, ld, B, r, e); break;
        case 2: launch(true, k_dense_apply_multi<2, 4>, blocks_for(mm, 4 * DENSE_ROWS_PER_CTA), DENSE_THREADS, 0, st,
                       mm, ld, B, r, e); break;
        case 4: launch(true, k_dense_apply_multi<4, 4>, blocks_for(mm, 4 * DENSE_ROWS_PER_CTA), DENSE_THREADS, 0, st,
                       mm, ld, B, r, e); break;
        default: launch(true, k_dense_apply_multi<8, 4>, blocks_for(mm, 4 * DENSE_ROWS_PER_CTA), DENSE_THREADS, 0, st,
                        mm, ld, B, r, e); break;
    }
    ctx->vcycle_kernels++;
}

bool c0_fused_l0(const mgm_ctx* ctx);
// Alg. 3 on level-0 buffers lv[0].f (rhs) and lv[0].u (guess in, result out), lib order.
void enqueue_vcycle(mgm_ctx* ctx, cudaStream_t st) {
    ctx->ntrace = 0;
    ctx->trace_labels.clear();
    auto& lv = ctx->lv;
    const int p = ctx->p;
    const int nu1 = ctx->lp.nu1, nu2 = ctx->lp.nu2;
    const bool pre_b = ctx->lp.smoother == 1, post_b = ctx->lp.smoother == 1 || ctx->lp.smoother == 2;
    const i64 pad = ctx->poisson ? 1 : 0;
    ctx->vcycle_kernels = 0;
    ctx->pdl = true;
    struct Reset { mgm_ctx* c; ~Reset() { c->pdl = false; } } reset_{ctx};
    if (p == 1) {
        enqueue_coarse(ctx, lv[0].f, lv[0].u, st);
        return;
    }
    // levels >= D run as the dense bottom B_D or in the one-kernel cluster bottom (if
    // enabled), else D = p - 1 (the coarse solve)
    const int D = ctx->denseJ > 0 ? ctx->denseJ : ctx->botJ > 0 ? ctx->botJ : p - 1;
    stamp(ctx, "start", 0, st);
    const bool bottom_only = std::getenv("MGM_DEBUG_BOTTOM_ONLY") && ctx->botJ > 0;  // timing experiment only
    if (!bottom_only) {
    // level 0 from a zero guess (preconditioner applications): the first sweep reads only
    // the diagonal and earlier-colour entries (k_gs_colour ZG)
    for (int s = 0; s < nu1; ++s) {  // line 4 (colour 0 from zero: done with the input copy, c0_fused_l0)
        g_dlt = (s + 1 == nu1) ? ctx->dlt_pre_out : nullptr;  // the last presmooth's increments
        enqueue_sweep(ctx, 0, pre_b, st, s == 0 && ctx->vc_zero_guess, s == 0 && ctx->vc_zero_guess && c0_fused_l0(ctx));
        g_dlt = nullptr;
    }
    stamp(ctx, "presmooth", 0, st);
    // after a forward presmooth with increments d: t = f - L u = -(later-colour part of L) d
    // (MODE 2 on d, as after a zero-guess sweep where d = u)
    const bool res_d = ctx->dlt_pre_out != nullptr;
    const double* ures = res_d ? ctx->dlt_pre_out : lv[0].u;
    const bool res_m2 = res_d || (ctx->vc_zero_guess && nu1 == 1);
    // residual in Morton order for the restriction's gathers (opt-in: cfg3 restrict L0 30.4 ->
    // 26.7 us but residual 80 -> 85 us; cfg5 solve 206.6 vs 205.2 ms without)
    const bool mt0 = !dist_level(ctx, 0) && lv[0].n >= ctx->morton_t_min;
    // levels whose first presmooth colour (from zero) is fused into the restriction before them
    auto zg_level = [&](int j) { return nu1 >= 1 && !pre_b && !ctx->poisson && lv[j].slw && !ctx->no_zg; };
    auto c0_fused = [&](int j) {
        return j < D && zg_level(j) && !dist_level(ctx, j) && !dist_level(ctx, j - 1) && lv[j].ncol > 1 &&
               !ctx->no_c0_fuse;
    };
    if (fused_rr_ok(ctx, 0)) {                                           // lines 5 (+ 8's restriction)
        enqueue_res_restrict(ctx, 0, lv[0].f, ures, lv[0].t, lv[1].f, st, res_m2, mt0, c0_fused(1));
        stamp(ctx, "residual+restrict", 0, st);
    } else {
        enqueue_residual(ctx, 0, lv[0].f, ures, lv[0].t, st, res_m2, mt0);  // line 5
        stamp(ctx, "residual", 0, st);
        enqueue_restrict(ctx, 0, lv[0].t, lv[1].f, st, mt0, c0_fused(1));
        stamp(ctx, "restrict", 0, st);
    }
    for (int j = 1; j < D; ++j) {                                         // lines 6-9
        // e_j = 0 then presmooth; the first forward sweep from the zero guess writes every row
        // and reads only earlier-colour values, so the zero fill is not needed
        const bool zg = zg_level(j);
        if (!zg) enqueue_zero(ctx, lv[j].u, lv[j].n + pad + lv[j].nghost, st);  // (+ ghosts: distributed)
        for (int s = 0; s < nu1; ++s) enqueue_sweep(ctx, j, pre_b, st, s == 0 && zg, s == 0 && c0_fused(j));
        stamp(ctx, "zero+presmooth", j, st);
        const bool mt = !dist_level(ctx, j) && lv[j].n >= ctx->morton_t_min;
        if (fused_rr_ok(ctx, j)) {
            enqueue_res_restrict(ctx, j, lv[j].f, lv[j].u, lv[j].t, lv[j + 1].f, st, zg && nu1 == 1, mt,
                                 c0_fused(j + 1));
        } else {
            enqueue_residual(ctx, j, lv[j].f, lv[j].u, lv[j].t, st, zg && nu1 == 1, mt);
            enqueue_restrict(ctx, j, lv[j].t, lv[j + 1].f, st, mt, c0_fused(j + 1));
        }
        stamp(ctx, "residual+restrict", j, st);
    }
    }
    if (ctx->denseJ > 0) {                                                // lines 6-14 for j >= J
        enqueue_dense_bottom(ctx, 1, lv[D].f, lv[D].u, st);
    } else if (ctx->botJ > 0) {                                           // lines 6-14 for j >= J
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctx->bot_cluster);
        cfg.blockDim = dim3(BOT_THREADS);
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = ctx->bot_cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = g_use_pdl ? 2 : 1;
        cfg.dynamicSmemBytes = ctx->bot_smem;
        const PfList pf{nullptr, 0, 0};
        auto bottom = [&](int q0, int nph, int arm0, int arm1, PfList pfl) {
            if (g_dry) return;
            const BPhase* ph = (const BPhase*)ctx->d_phases + q0;
            note_launch(ctx->d_trace
                            ? cudaLaunchKernelEx(&cfg, k_vcycle_bottom_t<true>, ph, nph, ctx->d_trace + 256, pfl, arm0,
                                                 arm1)
                            : cudaLaunchKernelEx(&cfg, k_vcycle_bottom_t<false>, ph, nph,
                                                 (unsigned long long*)nullptr, pfl, arm0, arm1),
                        ctx->bot_cluster, BOT_THREADS, ctx->bot_smem);
            ctx->vcycle_kernels++;
        };
        if (ctx->bot_split > 0) {  // down half, grid-wide coarse GEMV, up half
            bottom(0, ctx->bot_split, ctx->bot_arm0, ctx->bot_arm1, pf);
            const int m = ctx->nc;
            launch(ctx->pdl, k_dense_gemv, (unsigned)((m + 3) / 4), 128, 0, st, m, ctx->bot_ainv,
                   (const double*)lv[p - 1].f, lv[p - 1].u);
            if (!g_dry) ctx->vcycle_kernels++;
            bottom(ctx->bot_split, ctx->nphases - ctx->bot_split, ctx->bot_arm0b, ctx->bot_arm1b, PfList{nullptr, 0, 0});
        } else {
            bottom(0, ctx->nphases, ctx->bot_arm0, ctx->bot_arm1, pf);
        }
    } else {
        enqueue_coarse(ctx, lv[p - 1].f, lv[p - 1].u, st);                 // line 10
    }
    stamp(ctx, "bottom", D, st);
    if (bottom_only) return;
    for (int j = D - 1; j >= 1; --j) {                                    // lines 11-14
        enqueue_interp_correct(ctx, j, lv[j + 1].u, lv[j].u, st);
        for (int s = 0; s < nu2; ++s) enqueue_sweep(ctx, j, post_b, st);
        stamp(ctx, "interp+postsmooth", j, st);
    }
    enqueue_interp_correct(ctx, 0, lv[1].u, lv[0].u, st);                 // line 15
    stamp(ctx, "interp", 0, st);
    for (int s = 0; s < nu2; ++s) {                                       // line 16
        g_dlt = (s + 1 == nu2) ? ctx->dlt_out : nullptr;  // the last sweep's increments (MODE 3 A z)
        enqueue_sweep(ctx, 0, post_b, st);
        g_dlt = nullptr;
    }
    stamp(ctx, "postsmooth", 0, st);
}

bool timing_on(const mgm_ctx* ctx) { return ctx->timer[0].on || ctx->timer[1].on || ctx->timer[3].on; }

bool zg_capable(const mgm_ctx* ctx);
// The last level-0 postsmooth of the V-cycle writes its increments d (k_gs_colour dlt): after
// that forward sweep the residual is f - A u = -(later-colour part of L_1) d (k_sell_spmv
// MODE 2 on d) and A u = f + (later-colour part) d (MODE 3) -- equal up to rounding, about half
// the operator bytes of a full SpMV.  Shifted, undistributed, forward postsmoothing only.
bool mode3_ok(const mgm_ctx* ctx) {
    const Level& L0 = ctx->lv[0];
    return !ctx->poisson && !dist_on(ctx) && ctx->p >= 2 && ctx->lp.nu2 >= 1 && ctx->lp.smoother == 0 && L0.sluw &&
           L0.nlow && !ctx->no_zg && std::getenv("MGM_NO_MODE3") == nullptr;
}
// the general V-cycle's level-0 residual from the last presmooth's increments (MODE 2 on d)
bool dpre_ok(const mgm_ctx* ctx) {
    const Level& L0 = ctx->lv[0];
    return !ctx->poisson && !dist_on(ctx) && ctx->p >= 2 && ctx->lp.nu1 >= 1 && ctx->lp.smoother != 1 && L0.sluw &&
           L0.nlow && !ctx->no_zg && L0.n >= ctx->upper_res_min && std::getenv("MGM_NO_MODE3") == nullptr;
}
mgm_status build_graph(mgm_ctx* ctx, bool zero_guess = false) {
    cudaGraphExec_t& gx = zero_guess ? ctx->vgraph0 : ctx->vgraph;
    if (gx) return MGM_OK;
    ctx->vc_zero_guess = zero_guess && zg_capable(ctx);
    struct ResetZ {
        mgm_ctx* c;
        ~ResetZ() {
            c->vc_zero_guess = false;
            c->dlt_out = nullptr;
            c->dlt_pre_out = nullptr;
        }
    } resetz_{ctx};
    // both V-cycle graphs leave the last postsmooth's increments in d_dlt (standalone residual;
    // A M v in BiCGSTAB and the host-loop GMRES)
    const bool dl = mode3_ok(ctx);
    if (dl && !ctx->d_dlt) CK(dalloc(&ctx->d_dlt, ctx->lv[0].n));
    ctx->dlt_out = dl ? ctx->d_dlt : nullptr;
    (zero_guess ? ctx->vgraph0_dlt : ctx->vgraph_dlt) = dl;
    // the general V-cycle: the level-0 residual from the last presmooth's increments
    const Level& L0 = ctx->lv[0];
    const bool dpre = !zero_guess && dpre_ok(ctx);
    if (dpre && !ctx->d_dlt_pre) CK(dalloc(&ctx->d_dlt_pre, L0.n));
    ctx->dlt_pre_out = dpre ? ctx->d_dlt_pre : nullptr;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
    g_launch_err.clear();
    enqueue_vcycle(ctx, ctx->st);
    const cudaError_t ce = cudaStreamEndCapture(ctx->st, &g);
    if (ce != cudaSuccess || !g_launch_err.empty()) {
        ctx->err = "V-cycle capture failed: " + std::string(cudaGetErrorString(ce)) + "; first failed launch: " +
                   (g_launch_err.empty() ? std::string("none recorded") : g_launch_err);
        g_launch_err.clear();
        cudaGetLastError();
        return MGM_ERR_CUDA;
    }
    CK(cudaGraphInstantiate(&gx, g, 0));
    cudaGraphDestroy(g);
    return MGM_OK;
}

// run one V-cycle on lv[0].f / lv[0].u
// zero_guess: lv[0].u holds no guess (Krylov preconditioner): the level-0 presmooth starts
// from 0 without reading u (see zg_capable)
bool zg_capable(const mgm_ctx* ctx) {
    return !ctx->no_zg && !ctx->poisson && ctx->lp.nu1 >= 1 && ctx->lp.smoother != 1 && ctx->p > 1 && ctx->lv[0].slw;
}
mgm_status run_vcycle(mgm_ctx* ctx, cudaStream_t st, bool zero_guess = false) {
    zero_guess = zero_guess && zg_capable(ctx);
    ctx->last_vc_dlt = false;
    if (timing_on(ctx) || (ctx->tp && !ctx->tp->capturable())) {  // eager: event timing / fake ranks
        ctx->vc_zero_guess = zero_guess;
        timer_begin(ctx, 2, st);
        enqueue_vcycle(ctx, st);
        ctx->vc_zero_guess = false;
        timer_end(ctx, 2, st, 0.0);
        return MGM_OK;
    }
    mgm_status s = build_graph(ctx, zero_guess);
    if (s) return s;
    timer_begin(ctx, 2, st);
    CK(cudaGraphLaunch(zero_guess ? ctx->vgraph0 : ctx->vgraph, st));
    timer_end(ctx, 2, st, 0.0);
    ctx->last_vc_dlt = zero_guess ? ctx->vgraph0_dlt : ctx->vgraph_dlt;
    return MGM_OK;
}

void enqueue_apply_A(mgm_ctx* ctx, const double* x, double* y, cudaStream_t st);
// y = A u right after run_vcycle on lv[0] (u = lv[0].u): from the last postsmooth's increments
// when the graph recorded them (A u = f + (later-colour part of L_1) d, k_sell_spmv MODE 3),
// else the plain SpMV
void enqueue_apply_A_after_vcycle(mgm_ctx* ctx, double* y, cudaStream_t st) {
    if (!ctx->last_vc_dlt) {
        enqueue_apply_A(ctx, ctx->lv[0].u, y, st);
        return;
    }
    const Level& L0 = ctx->lv[0];
    g_sluw = L0.sluw;
    g_nlow = L0.nlow;
    launch_spmv(false, 3, false, L0.stpr, 0, L0.n, L0.n, L0.sptr, L0.scol, L0.sval, ctx->d_dlt, L0.f, y, L0.c, st);
    g_sluw = nullptr;
    g_nlow = nullptr;
}

mgm_status ensure_krylov(mgm_ctx* ctx) {
    if (ctx->V) return MGM_OK;
    i64 n = ctx->N + (ctx->poisson ? 1 : 0);
    ctx->ld = (n + 31) / 32 * 32;
    CK(dalloc(&ctx->V, ctx->ld * std::max(ctx->restart + 1, 8)));  // >= 8 BiCGSTAB vectors
    CK(dalloc(&ctx->w, ctx->ld));
    CK(dalloc(&ctx->xs, ctx->ld));
    CK(dalloc(&ctx->b, ctx->ld));
    CK(dalloc(&ctx->partials, (i64)RED_BLOCKS * 256));
    CK(dev_malloc((void**)&ctx->tickets, 64 * sizeof(unsigned)));
    CK(cudaMemset(ctx->tickets, 0, 64 * sizeof(unsigned)));
    CK(dalloc(&ctx->dh, 1024));
    CK(cudaMallocHost((void**)&ctx->hh, sizeof(double) * 1024));
    return MGM_OK;
}

// dot over n entries of a and b -> device scalar out
// Krylov inner products: on nranks > 1 each rank reduces its own row piece (deterministic
// in-kernel finish) and the pieces are summed with ncclAllReduce (identical on every rank).
void enqueue_multidot(mgm_ctx* ctx, i64 n, const double* V, i64 ld, int k1, const double* w, double* out,
                      double* acc, cudaStream_t st) {
    if (!dist_on(ctx)) {
        k_multidot_fin<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, V, ld, k1, w, ctx->partials, ctx->tickets, out, acc);
        return;
    }
    // distributed: this rank's rows (deterministic in-kernel finish), then a sum-allreduce
    k_multidot_fin<<<RED_BLOCKS, RED_THREADS, 0, st>>>(dot_rows(ctx), V, ld, k1, w, ctx->partials, ctx->tickets, out,
                                                       nullptr);
    if (!ctx->tp->allreduce_sum(out, k1, st) && ctx->err.empty()) ctx->err = "allreduce failed";
    if (acc) k_vadd<<<1, 128, 0, st>>>(k1, acc, out);
}
void enqueue_dot(mgm_ctx* ctx, i64 n, const double* a, const double* b, double* out, cudaStream_t st) {
    enqueue_multidot(ctx, n, a, 0, 1, b, out, nullptr, st);
}

// A x on level 0 (bordered in Poisson mode), n-vector incl. multiplier.  Distributed: x is
// copied into the ghosted scratch lv[0].t (unless it is lv[0].u, which has ghost slots) and
// its ghosts are refreshed before the SpMV.
void enqueue_apply_A(mgm_ctx* ctx, const double* x, double* y, cudaStream_t st) {
    if (!dist_on(ctx)) {
        enqueue_spmv(ctx, 0, x, y, st);
        return;
    }
    Level& L0 = ctx->lv[0];
    double* xg = L0.u;
    if (x != L0.u) {
        xg = L0.t;
        cudaMemcpyAsync(xg, x, sizeof(double) * vec_rows(ctx), cudaMemcpyDeviceToDevice, st);
    }
    exch(ctx, 0, xg, -1, st);
    enqueue_spmv(ctx, 0, xg, y, st);
}

// z = M(v): one V-cycle from zero, result left in lv[0].u
// colour 0 of the level-0 presmooth from the zero guess done while copying the input (the
// zero-guess V-cycle graph then starts at colour 1)
bool c0_fused_l0(const mgm_ctx* ctx) {
    return zg_capable(ctx) && !dist_level(ctx, 0) && ctx->lv[0].ncol > 1 && !ctx->no_c0_fuse;
}
C0Fuse c0_l0(mgm_ctx* ctx) {
    return c0_fused_l0(ctx) ? C0Fuse{ctx->lv[0].u, ctx->lv[0].sptr, ctx->lv[0].sval, (int)ctx->lv[0].coff[1]}
                            : C0Fuse{nullptr, nullptr, nullptr, 0};
}
mgm_status enqueue_precond(mgm_ctx* ctx, const double* v, cudaStream_t st) {
    const i64 n = vec_rows(ctx);
    if (c0_fused_l0(ctx))
        k_copy_col<<<RED_BLOCKS, 256, 0, st>>>(n, v, 0, (const int*)nullptr, ctx->lv[0].f, c0_l0(ctx));
    else
        CK(cudaMemcpyAsync(ctx->lv[0].f, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    if (!zg_capable(ctx))  // (ghost slots too: the first sweep reads them)
        CK(cudaMemsetAsync(ctx->lv[0].u, 0, sizeof(double) * (n + ctx->lv[0].nghost), st));
    return run_vcycle(ctx, st, true);  // M v from the zero guess
}

// Right-preconditioned GMRES(restart) with CGS2 orthogonalisation (equal to MGS in exact
// arithmetic; O15), Givens rotations on the host.  b, x in lib order (x = 0 on entry).
// GMRES keeps Z = M V (MGM_GMRES_NO_Z=1: x += M (V y) at the end of a restart cycle)
static bool gmres_keep_z() { return std::getenv("MGM_GMRES_NO_Z") == nullptr; }
mgm_status gmres_lib(mgm_ctx* ctx, double tol, int maxit, mgm_report* rep, cudaStream_t st) {
    const i64 n = vec_rows(ctx);
    const int m = ctx->restart;
    const i64 ld = ctx->ld;
    if (gmres_keep_z() && !ctx->Z) CK(dalloc(&ctx->Z, (i64)m * ld));
    double* V = ctx->V;
    double* w = ctx->w;
    double* h1 = ctx->dh;
    double* h2 = ctx->dh + 256;
    double* nr = ctx->dh + 512;
    mgm_status s;
    if (!ctx->warm) CK(cudaMemsetAsync(ctx->xs, 0, sizeof(double) * n, st));
    enqueue_dot(ctx, n, ctx->b, ctx->b, nr, st);
    CK(cudaMemcpyAsync(ctx->hh, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const double bnorm = std::sqrt(ctx->hh[0]);
    int its = 0, hist_n = 0;
    bool converged = false;
    if (bnorm == 0.0) {  // x = 0 solves A x = 0 (whatever x0)
        CK(cudaMemsetAsync(ctx->xs, 0, sizeof(double) * n, st));
        if (rep) { rep->iterations = 0; rep->converged = 1; rep->final_rel_residual = 0.0; }
        return MGM_OK;
    }
    std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), y(m);
    bool first = !ctx->warm;  // r0 = b - A x0 (x0 = 0: r0 = b, no SpMV)
    while (true) {
        // r = b - A x ; beta
        if (first) {
            CK(cudaMemcpyAsync(w, ctx->b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        } else {
            enqueue_apply_A(ctx, ctx->xs, w, st);
            k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->b, -1.0, w, w);
        }
        first = false;
        enqueue_dot(ctx, n, w, w, nr, st);
        CK(cudaMemcpyAsync(ctx->hh, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double beta = std::sqrt(ctx->hh[0]);
        if (beta / bnorm <= tol || its >= maxit) {
            converged = beta / bnorm <= tol;
            break;
        }
        k_scale_by_invnorm<<<RED_BLOCKS, 256, 0, st>>>(n, w, nr, V);
        std::fill(H.begin(), H.end(), 0.0);
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = beta;
        int kdone = 0;
        bool stop = false;
        for (int k = 0; k < m; ++k) {
            if ((s = enqueue_precond(ctx, V + (i64)k * ld, st))) return s;
            if (ctx->Z)  // z_k = M v_k (x += Z y at the end of the cycle)
                CK(cudaMemcpyAsync(ctx->Z + (i64)k * ld, ctx->lv[0].u, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            enqueue_apply_A_after_vcycle(ctx, w, st);
            ++its;
            const int k1 = k + 1;
            // CGS2: h = V^T w; w -= V h; h2 = V^T w; w -= V h2; h += h2
            // CGS2 in 5 launches: h1 = V^T w; w -= V h1; h2 = V^T w (h1 += h2); w -= V h2 with
            // ||w||^2; v_{k+1} = w / ||w||.  Reductions finish in the last block (deterministic).
            enqueue_multidot(ctx, n, V, ld, k1, w, h1, nullptr, st);
            if (!dist_on(ctx)) {  // w -= V h1 and h2 = V^T w (h1 += h2) in one pass over V
                k_multiaxpy_dot_fin<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, V, ld, k1, h1, w, ctx->partials,
                                                                        ctx->tickets, h2, h1);
            } else {
                k_multiaxpy<<<RED_BLOCKS * 2, 256, 0, st>>>(n, V, ld, k1, h1, w);
                enqueue_multidot(ctx, n, V, ld, k1, w, h2, h1, st);
            }
            if (!dist_on(ctx)) {
                k_multiaxpy_norm<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, V, ld, k1, h2, w, ctx->partials, ctx->tickets,
                                                                     nr);
            } else {  // local update, distributed norm
                k_multiaxpy<<<RED_BLOCKS * 2, 256, 0, st>>>(n, V, ld, k1, h2, w);
                enqueue_dot(ctx, n, w, w, nr, st);
            }
            k_scale_by_invnorm<<<RED_BLOCKS, 256, 0, st>>>(n, w, nr, V + (i64)k1 * ld);
            CK(cudaMemcpyAsync(ctx->hh, h1, sizeof(double) * k1, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(ctx->hh + 512, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (timing_on(ctx)) timer_collect(ctx);
            for (int i = 0; i < k1; ++i) H[(size_t)i * m + k] = ctx->hh[i];
            double hk1 = std::sqrt(ctx->hh[512]);
            H[(size_t)k1 * m + k] = hk1;
            for (int i = 0; i < k; ++i) {
                double t = cs[i] * H[(size_t)i * m + k] + sn[i] * H[(size_t)(i + 1) * m + k];
                H[(size_t)(i + 1) * m + k] = -sn[i] * H[(size_t)i * m + k] + cs[i] * H[(size_t)(i + 1) * m + k];
                H[(size_t)i * m + k] = t;
            }
            double den = std::hypot(H[(size_t)k * m + k], hk1);
            cs[k] = H[(size_t)k * m + k] / den;
            sn[k] = hk1 / den;
            H[(size_t)k * m + k] = den;
            H[(size_t)k1 * m + k] = 0.0;
            g[k1] = -sn[k] * g[k];
            g[k] = cs[k] * g[k];
            double rel = std::fabs(g[k1]) / bnorm;
            if (rep && rep->history && hist_n < rep->history_cap) rep->history[hist_n++] = rel;
            kdone = k1;
            if (!std::isfinite(rel)) return fail(ctx, MGM_ERR_BREAKDOWN, "non-finite GMRES residual", its);
            if (rel <= tol || its >= maxit || hk1 == 0.0) {
                stop = true;
                break;
            }
        }
        for (int i = kdone - 1; i >= 0; --i) {
            double sacc = g[i];
            for (int j2 = i + 1; j2 < kdone; ++j2) sacc -= H[(size_t)i * m + j2] * y[j2];
            y[i] = sacc / H[(size_t)i * m + i];
        }
        CK(cudaMemcpyAsync(h1, y.data(), sizeof(double) * kdone, cudaMemcpyHostToDevice, st));
        if (ctx->Z) {  // x += Z y
            k_lincomb<<<RED_BLOCKS * 2, 256, 0, st>>>(n, ctx->Z, ld, kdone, h1, w);
            k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->xs, 1.0, w, ctx->xs);
        } else {       // x += M (V y)
            k_lincomb<<<RED_BLOCKS * 2, 256, 0, st>>>(n, V, ld, kdone, h1, w);
            if ((s = enqueue_precond(ctx, w, st))) return s;
            k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->xs, 1.0, ctx->lv[0].u, ctx->xs);
        }
        if (stop) {
            converged = std::fabs(g[kdone]) / bnorm <= tol;
            break;
        }
    }
    // true residual
    enqueue_apply_A(ctx, ctx->xs, w, st);
    k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->b, -1.0, w, w);
    enqueue_dot(ctx, n, w, w, nr, st);
    CK(cudaMemcpyAsync(ctx->hh, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (ctx->poisson) CK(cudaMemcpyAsync(ctx->hh + 1, ctx->xs + ctx->lv[0].n, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (rep) {
        rep->iterations = its;
        rep->converged = converged ? 1 : 0;
        rep->final_rel_residual = std::sqrt(ctx->hh[0]) / bnorm;
        rep->lambda = ctx->poisson ? ctx->hh[1] : 0.0;
    }
    return MGM_OK;
}

// ---------------------------------------------------------------------------------------
// Device-side GMRES: the Arnoldi steps of a restart cycle run as ONE graph launch, a WHILE
// conditional node whose body is [V_k -> f_0, V-cycle from the zero guess, SpMV, CGS2 (5
// kernels), V_{k+1} = w/||w||, Givens step] and whose condition the Givens kernel sets on the
// device (solve_kernels.cuh k_gmres_givens).  The host synchronises once per restart cycle
// instead of once per iteration.  Same arithmetic as gmres_lib (which remains the path for
// Poisson problems, multi-GPU, kernel timing, restart > 128 and MGM_HOST_GMRES).
// ---------------------------------------------------------------------------------------
static size_t gmres_dev_doubles(const mgm_ctx* ctx) {
    const size_t m = (size_t)ctx->restart;
    return 2 + (m + 1) * m + 2 * m + (m + 1) + (size_t)ctx->g_hist_cap;
}
static bool gmres_dev_ok(const mgm_ctx* ctx) {
    return !ctx->poisson && !dist_on(ctx) && !timing_on(ctx) && ctx->restart <= 128 && ctx->p >= 1 &&
           std::getenv("MGM_HOST_GMRES") == nullptr;
}
static mgm_status build_gmres_graph(mgm_ctx* ctx) {
    if (ctx->ggraph) return MGM_OK;
    const i64 n = ctx->N;
    const int m = ctx->restart;
    const i64 ld = ctx->ld;
    cudaStream_t st = ctx->st;
    if (!ctx->g_i) {
        CK(dalloc(&ctx->g_i, 8));
        CK(dalloc(&ctx->g_d, (i64)gmres_dev_doubles(ctx)));
        CK(cudaMallocHost((void**)&ctx->g_h, sizeof(double) * gmres_dev_doubles(ctx)));
        CK(cudaMallocHost((void**)&ctx->g_hi, sizeof(int) * 8));
    }
    // w = A z from the last level-0 postsmooth's increments (below); its buffer is allocated
    // before the capture
    const Level& L0 = ctx->lv[0];
    const bool mode3 = mode3_ok(ctx);
    if (mode3 && !ctx->d_dlt) CK(dalloc(&ctx->d_dlt, n));
    if (gmres_keep_z() && !ctx->Z) CK(dalloc(&ctx->Z, (i64)m * ctx->ld));
    GmresDev G{ctx->g_i, ctx->g_d, m, ctx->g_hist_cap};
    double* V = ctx->V;
    double* w = ctx->w;
    double* h1 = ctx->dh;
    double* h2 = ctx->dh + 256;
    double* nr = ctx->dh + 512;
    const int* kdev = ctx->g_i;
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    struct GDel { cudaGraph_t g; ~GDel() { cudaGraphDestroy(g); } } gdel_{g};
    cudaGraphConditionalHandle cond;
    CK(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CK(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    g_launch_err.clear();
    // every node with programmatic serialisation (PDL): each kernel waits for its predecessor
    // with griddepcontrol.wait, and its launch overlaps the predecessor's tail
    launch(true, k_copy_col, RED_BLOCKS, 256, 0, st, n, (const double*)V, ld, kdev, ctx->lv[0].f,
           c0_l0(ctx));  // f_0 = V_k (and colour 0 of the presmooth)
    const bool zg = zg_capable(ctx);
    if (!zg) cudaMemsetAsync(ctx->lv[0].u, 0, sizeof(double) * n, st);
    ctx->vc_zero_guess = zg;
    // w = A z from the last level-0 postsmooth's increments d: A z = V_k + (later-colour part
    // of L_1) d (k_sell_spmv MODE 3) -- half the operator bytes of the plain SpMV
    ctx->dlt_out = mode3 ? ctx->d_dlt : nullptr;
    enqueue_vcycle(ctx, st);                                              // u = M V_k
    ctx->dlt_out = nullptr;
    ctx->vc_zero_guess = false;
    ctx->pdl = true;
    if (ctx->Z)                                                           // Z_k = M V_k
        launch(true, k_store_col, RED_BLOCKS, 256, 0, st, n, (const double*)ctx->lv[0].u, ctx->Z, ld, kdev);
    if (mode3) {                                                          // w = A M V_k
        g_sluw = L0.sluw;
        g_nlow = L0.nlow;
        launch_spmv(true, 3, false, L0.stpr, 0, L0.n, L0.n, L0.sptr, L0.scol, L0.sval, ctx->d_dlt, L0.f, w, L0.c, st);
        g_sluw = nullptr;
        g_nlow = nullptr;
    } else {
        enqueue_apply_A(ctx, ctx->lv[0].u, w, st);
    }
    ctx->pdl = false;
    // CGS2: h1 = V^T w; w -= V h1; h2 = V^T w (h1 += h2); w -= V h2, ||w||^2
    launch(true, k_multidot_fin, RED_BLOCKS, RED_THREADS, 0, st, n, (const double*)V, ld, 0, (const double*)w,
           ctx->partials, ctx->tickets, h1, (double*)nullptr, kdev);
    launch(true, k_multiaxpy_dot_fin, RED_BLOCKS, RED_THREADS, 0, st, n, (const double*)V, ld, 0, (const double*)h1, w,
           ctx->partials, ctx->tickets, h2, h1, kdev);
    launch(true, k_multiaxpy_norm, RED_BLOCKS, RED_THREADS, 0, st, n, (const double*)V, ld, 0, (const double*)h2, w,
           ctx->partials, ctx->tickets, nr, kdev);
    launch(true, k_scale_col, RED_BLOCKS, 256, 0, st, n, (const double*)w, (const double*)nr, V, ld, kdev);  // V_{k+1}
    launch(true, k_gmres_givens, 1, 32, 0, st, G, (const double*)h1, (const double*)nr, cond);
    cudaGraph_t cap = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &cap);
    if (ce != cudaSuccess || !g_launch_err.empty()) {
        ctx->err = "GMRES graph capture failed: " + std::string(cudaGetErrorString(ce)) + "; first failed launch: " +
                   (g_launch_err.empty() ? std::string("none recorded") : g_launch_err);
        g_launch_err.clear();
        cudaGetLastError();
        return MGM_ERR_CUDA;
    }
    CK(cudaGraphInstantiate(&ctx->ggraph, g, 0));
    return MGM_OK;
}

mgm_status gmres_dev(mgm_ctx* ctx, double tol, int maxit, mgm_report* rep, cudaStream_t st) {
    const i64 n = ctx->N;
    const int m = ctx->restart;
    const i64 ld = ctx->ld;
    double* V = ctx->V;
    double* w = ctx->w;
    double* h1 = ctx->dh;
    double* nr = ctx->dh + 512;
    mgm_status s;
    if ((s = build_gmres_graph(ctx))) return s;
    if (!ctx->warm) CK(cudaMemsetAsync(ctx->xs, 0, sizeof(double) * n, st));
    enqueue_dot(ctx, n, ctx->b, ctx->b, nr, st);
    CK(cudaMemcpyAsync(ctx->hh, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const double bnorm = std::sqrt(ctx->hh[0]);
    int its = 0, hist_n = 0;
    bool converged = false;
    if (bnorm == 0.0) {  // x = 0 solves A x = 0 (whatever x0)
        CK(cudaMemsetAsync(ctx->xs, 0, sizeof(double) * n, st));
        if (rep) { rep->iterations = 0; rep->converged = 1; rep->final_rel_residual = 0.0; }
        return MGM_OK;
    }
    const size_t nd = gmres_dev_doubles(ctx);
    double* gh = ctx->g_h;
    double* Hh = gh + 2;
    double* gg = Hh + (size_t)(m + 1) * m + 2 * (size_t)m;
    double* hist = gg + (m + 1);
    std::vector<double> y(m);
    bool first = !ctx->warm;  // r0 = b - A x0 (x0 = 0: r0 = b, no SpMV; ||r0||^2 is still in nr)
    while (true) {
        double beta = bnorm;
        if (first) {  // r = b - A x ; beta
            CK(cudaMemcpyAsync(w, ctx->b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        } else {
            enqueue_apply_A(ctx, ctx->xs, w, st);
            k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->b, -1.0, w, w);
            enqueue_dot(ctx, n, w, w, nr, st);
            CK(cudaMemcpyAsync(ctx->hh, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            beta = std::sqrt(ctx->hh[0]);
        }
        first = false;
        if (beta / bnorm <= tol || its >= maxit) {
            converged = beta / bnorm <= tol;
            break;
        }
        k_scale_by_invnorm<<<RED_BLOCKS, 256, 0, st>>>(n, w, nr, V);
        // cycle state: k = 0, its, stop = 0, maxit; bnorm, tol; H = cs = sn = 0; g = beta e_1
        std::fill(gh, gh + nd - ctx->g_hist_cap, 0.0);
        gh[0] = bnorm;
        gh[1] = tol;
        gg[0] = beta;
        ctx->g_hi[0] = 0;
        ctx->g_hi[1] = its;
        ctx->g_hi[2] = 0;
        ctx->g_hi[3] = maxit;
        CK(cudaMemcpyAsync(ctx->g_d, gh, sizeof(double) * (nd - ctx->g_hist_cap), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(ctx->g_i, ctx->g_hi, sizeof(int) * 4, cudaMemcpyHostToDevice, st));
        CK(cudaGraphLaunch(ctx->ggraph, st));
        CK(cudaMemcpyAsync(ctx->g_hi, ctx->g_i, sizeof(int) * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(gh, ctx->g_d, sizeof(double) * nd, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const int kdone = ctx->g_hi[0];
        const int its0 = its;
        its = ctx->g_hi[1];
        const int stop = ctx->g_hi[2];
        for (int q = its0; q < its && q < ctx->g_hist_cap; ++q)
            if (rep && rep->history && hist_n < rep->history_cap) rep->history[hist_n++] = hist[q];
        if (stop == 2) return fail(ctx, MGM_ERR_BREAKDOWN, "non-finite GMRES residual", its);
        for (int i = kdone - 1; i >= 0; --i) {
            double sacc = gg[i];
            for (int j2 = i + 1; j2 < kdone; ++j2) sacc -= Hh[(size_t)i * m + j2] * y[j2];
            y[i] = sacc / Hh[(size_t)i * m + i];
        }
        CK(cudaMemcpyAsync(h1, y.data(), sizeof(double) * kdone, cudaMemcpyHostToDevice, st));
        if (ctx->Z) {  // x += Z y (z_j = M v_j kept by the graph)
            k_lincomb<<<RED_BLOCKS * 2, 256, 0, st>>>(n, ctx->Z, ld, kdone, h1, w);
            k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->xs, 1.0, w, ctx->xs);
        } else {       // x += M (V y)
            k_lincomb<<<RED_BLOCKS * 2, 256, 0, st>>>(n, V, ld, kdone, h1, w);
            if ((s = enqueue_precond(ctx, w, st))) return s;
            k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->xs, 1.0, ctx->lv[0].u, ctx->xs);
        }
        if (stop == 1) {
            converged = std::fabs(gg[kdone]) / bnorm <= tol;
            break;
        }
    }
    // true residual
    enqueue_apply_A(ctx, ctx->xs, w, st);
    k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->b, -1.0, w, w);
    enqueue_dot(ctx, n, w, w, nr, st);
    CK(cudaMemcpyAsync(ctx->hh, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (rep) {
        rep->iterations = its;
        rep->converged = converged ? 1 : 0;
        rep->final_rel_residual = std::sqrt(ctx->hh[0]) / bnorm;
        rep->lambda = 0.0;
    }
    return MGM_OK;
}

// Right-preconditioned BiCGSTAB (oracle.bicgstab, O18): Saad's
// Alg. 7.7 on A M with x = M z; two V-cycles (preconditioner applications, counted as the
// iterations) and two SpMVs per step; the relative residual after each half step.  b, x
// in lib order (x = 0 on entry).  Workspace columns of V: r_hat, r, p, v, p_hat, s, t
// (r_hat/r and s/t adjacent so that one multi-dot gives two inner products).
mgm_status bicgstab_lib(mgm_ctx* ctx, double tol, int maxit, mgm_report* rep, cudaStream_t st) {
    const i64 n = vec_rows(ctx);
    const i64 ld = ctx->ld;
    double* rh = ctx->V;
    double* r = ctx->V + ld;
    double* p = ctx->V + 2 * ld;
    double* v = ctx->V + 3 * ld;
    double* ph = ctx->V + 4 * ld;
    double* sv = ctx->V + 5 * ld;
    double* t = ctx->V + 6 * ld;
    double* dd = ctx->dh + 512;  // device scalars
    double* hh = ctx->hh;
    const unsigned nb = RED_BLOCKS, nt = 256;
    mgm_status s;
    auto fetch = [&](int k) -> mgm_status {
        CK(cudaMemcpyAsync(hh, dd, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return MGM_OK;
    };
    if (!ctx->warm) CK(cudaMemsetAsync(ctx->xs, 0, sizeof(double) * n, st));
    enqueue_dot(ctx, n, ctx->b, ctx->b, dd, st);
    if ((s = fetch(1))) return s;
    const double bnorm = std::sqrt(hh[0]);
    int its = 0, hist_n = 0, restarts = 0;
    bool converged = false;
    if (bnorm == 0.0) {  // x = 0 solves A x = 0 (whatever x0)
        CK(cudaMemsetAsync(ctx->xs, 0, sizeof(double) * n, st));
        if (rep) { rep->iterations = 0; rep->converged = 1; rep->final_rel_residual = 0.0; rep->lambda = 0.0; }
        return MGM_OK;
    }
    auto record = [&](double rel) {
        if (rep && rep->history && hist_n < rep->history_cap) rep->history[hist_n++] = rel;
    };
    if (ctx->warm) {  // r = b - A x0
        enqueue_apply_A(ctx, ctx->xs, r, st);
        k_axpby<<<nb, nt, 0, st>>>(n, 1.0, ctx->b, -1.0, r, r);
    } else {
        CK(cudaMemcpyAsync(r, ctx->b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));  // r = b - A 0
    }
    while (true) {
        CK(cudaMemcpyAsync(rh, r, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemsetAsync(p, 0, sizeof(double) * n, st));
        CK(cudaMemsetAsync(v, 0, sizeof(double) * n, st));
        double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
        enqueue_dot(ctx, n, rh, r, dd, st);
        if ((s = fetch(1))) return s;
        double rho = hh[0];
        bool broke = false;
        while (its < maxit) {
            if (std::fabs(rho) < 1e-30 * bnorm * bnorm) { broke = true; break; }
            const double beta = (rho / rho_prev) * (alpha / omega);
            k_bicg_p<<<nb, nt, 0, st>>>(n, r, v, p, beta, omega);
            if ((s = enqueue_precond(ctx, p, st))) return s;  // p_hat = M p
            ++its;
            CK(cudaMemcpyAsync(ph, ctx->lv[0].u, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            enqueue_apply_A_after_vcycle(ctx, v, st);
            enqueue_dot(ctx, n, rh, v, dd, st);
            if ((s = fetch(1))) return s;
            alpha = rho / hh[0];
            k_axpby<<<nb, nt, 0, st>>>(n, 1.0, r, -alpha, v, sv);  // s = r - alpha v
            enqueue_dot(ctx, n, sv, sv, dd, st);
            if ((s = fetch(1))) return s;
            const double rel_s = std::sqrt(hh[0]) / bnorm;
            record(rel_s);
            if (!std::isfinite(rel_s)) return fail(ctx, MGM_ERR_BREAKDOWN, "non-finite BiCGSTAB residual", its);
            if (rel_s <= tol) {
                k_axpby<<<nb, nt, 0, st>>>(n, 1.0, ctx->xs, alpha, ph, ctx->xs);
                converged = true;
                break;
            }
            if ((s = enqueue_precond(ctx, sv, st))) return s;  // s_hat = M s (in lv[0].u)
            ++its;
            enqueue_apply_A_after_vcycle(ctx, t, st);
            enqueue_multidot(ctx, n, sv, ld, 2, t, dd, nullptr, st);  // (s, t), (t, t)
            if ((s = fetch(2))) return s;
            omega = hh[1] > 0.0 ? hh[0] / hh[1] : 0.0;
            k_axpbypz<<<nb, nt, 0, st>>>(n, ctx->xs, alpha, ph, omega, ctx->lv[0].u);
            k_axpby<<<nb, nt, 0, st>>>(n, 1.0, sv, -omega, t, r);  // r = s - omega t
            enqueue_multidot(ctx, n, rh, ld, 2, r, dd, nullptr, st);  // (r_hat, r), (r, r)
            if ((s = fetch(2))) return s;
            const double rel = std::sqrt(hh[1]) / bnorm;
            record(rel);
            if (timing_on(ctx)) timer_collect(ctx);
            if (rel <= tol) { converged = true; break; }
            if (std::fabs(omega) < 1e-30) { broke = true; break; }
            rho_prev = rho;
            rho = hh[0];
        }
        if (converged || its >= maxit || !broke || restarts >= 1) break;
        ++restarts;  // breakdown: restart once from the current iterate (r is current)
    }
    // true residual
    enqueue_apply_A(ctx, ctx->xs, ctx->w, st);
    k_axpby<<<nb, nt, 0, st>>>(n, 1.0, ctx->b, -1.0, ctx->w, ctx->w);
    enqueue_dot(ctx, n, ctx->w, ctx->w, dd, st);
    CK(cudaMemcpyAsync(hh, dd, sizeof(double), cudaMemcpyDeviceToHost, st));
    if (ctx->poisson) CK(cudaMemcpyAsync(hh + 1, ctx->xs + ctx->lv[0].n, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (rep) {
        rep->iterations = its;
        rep->converged = converged ? 1 : 0;
        rep->final_rel_residual = std::sqrt(hh[0]) / bnorm;
        rep->lambda = ctx->poisson ? hh[1] : 0.0;
    }
    return MGM_OK;
}

// Standalone MGM: u <- V-cycle(f, u) from u = 0 until ||f - A u|| / ||f|| <= tol.
// ---------------------------------------------------------------------------------------
// Batched (multi-RHS) V-cycle and standalone MGM: K right-hand sides in
// one pass over every operator; vectors interleaved [row][K] in lib order; the small levels
// run the per-kernel path (the one-kernel bottom holds a single right-hand side).
// ---------------------------------------------------------------------------------------
// threads per row cap of the batched colour kernels (MGM_BATCH_TPR_CAP; experiment)
static int g_batch_tpr_cap = std::getenv("MGM_BATCH_TPR_CAP") ? std::max(1, std::atoi(std::getenv("MGM_BATCH_TPR_CAP"))) : 8;
// batched levels with at least this many rows write the residual in Morton order
// (MGM_BATCH_MORTON_T_MIN; off by default: cfg3 K = 8 residual+restrict L0 437 vs 413 us)
static i64 g_batch_morton_min = std::getenv("MGM_BATCH_MORTON_T_MIN") ? std::atoll(std::getenv("MGM_BATCH_MORTON_T_MIN"))
                                                                      : (i64)1 << 62;
template <int K>
static i64 gs_wave_threads_bs(int tpr, int block) {
    static i64 cache[4][4] = {};
    const int ti = tpr == 1 ? 0 : tpr == 2 ? 1 : tpr == 4 ? 2 : 3;
    const int bi = block == 64 ? 0 : block == 128 ? 1 : block == 256 ? 2 : 3;
    if (cache[ti][bi]) return cache[ti][bi];
    int dev = 0, nsm = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const void* k = tpr == 1 ? (const void*)k_gs_colour_bs<1, CHUNK, K>
                  : tpr == 2 ? (const void*)k_gs_colour_bs<2, CHUNK, K>
                  : tpr == 4 ? (const void*)k_gs_colour_bs<4, CHUNK, K>
                             : (const void*)k_gs_colour_bs<8, CHUNK, K>;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, block, 0) != cudaSuccess) {
        cudaGetLastError();
        per = 1;
    }
    return cache[ti][bi] = (i64)per * nsm * block;
}
// 8-slot register chunks in the batched kernels (fewer registers, more CTAs per SM) on the
// bandwidth-bound levels; 16-slot chunks (fewer dependent operator loads) on the small K = 8
// levels.  Measured at cfg3 (traced V-cycle, tools/batch_trace.py): K = 8 L0 presmooth 457 ->
// 364 us, residual+restrict 414 -> 381, postsmooth 514 -> 420, but L3 postsmooth 78 -> 102;
// K = 4 every level gains.  MGM_BATCH_CH8=0/1 forces either.
static int g_batch_ch8_env = std::getenv("MGM_BATCH_CH8") ? std::atoi(std::getenv("MGM_BATCH_CH8")) : -1;
static bool batch_ch8(int K, i64 n) { return g_batch_ch8_env >= 0 ? g_batch_ch8_env != 0 : (K == 4 || n >= 131072); }
// increments of the batched sweep being enqueued (the batched GMRES's A z, MODE 3)
static thread_local double* g_bdlt = nullptr;
// K right-hand sides (K even): TPR * K/2 threads per row (batch_kernels.cuh)
template <int K>
static void b_gs(mgm_ctx* ctx, const Level& L, int j, int r0, int r1, cudaStream_t st, bool zg = false) {
    const int span = r1 - (r0 & ~31);
    const int bs = L.gs_block;
    auto go = [&](auto kern, int t) {
        launch(true, kern, blocks_for((i64)span * t * (K / 2), bs), bs, 0, st, r0, r1, L.uniform_w,
               (const i64*)L.sptr, (const i32*)L.scol, (const double*)L.sval, (const double*)ctx->bf[j], ctx->bu[j],
               (const i32*)L.slw, (const uint8_t*)L.nlow, zg ? (double*)nullptr : g_bdlt);
    };
    // a colour just above one (register-limited) wave: halve the threads per row (cf. launch_gs)
    int t = std::min(L.tpr, std::min(g_batch_tpr_cap, 64 / K));
    while (t > 1 && (i64)span * t * (K / 2) > gs_wave_threads_bs<K>(t, bs) &&
           (i64)span * (t / 2) * (K / 2) <= gs_wave_threads_bs<K>(t / 2, bs))
        t /= 2;
    if constexpr (K >= 4) {
        if (batch_ch8(K, L.n)) {
            if (zg) {
                if (t == 1) go(k_gs_colour_bs<1, 8, K, true>, 1);
                else if (t == 2) go(k_gs_colour_bs<2, 8, K, true>, 2);
                else if (t == 4) go(k_gs_colour_bs<4, 8, K, true>, 4);
                else go(k_gs_colour_bs<8, 8, K, true>, 8);
            } else {
                if (t == 1) go(k_gs_colour_bs<1, 8, K>, 1);
                else if (t == 2) go(k_gs_colour_bs<2, 8, K>, 2);
                else if (t == 4) go(k_gs_colour_bs<4, 8, K>, 4);
                else go(k_gs_colour_bs<8, 8, K>, 8);
            }
            return;
        }
    }
    if (zg) {
        if (t == 1) go(k_gs_colour_bs<1, CHUNK, K, true>, 1);
        else if (t == 2) go(k_gs_colour_bs<2, CHUNK, K, true>, 2);
        else if (t == 4) go(k_gs_colour_bs<4, CHUNK, K, true>, 4);
        else go(k_gs_colour_bs<8, CHUNK, K, true>, 8);
    } else {
        if (t == 1) go(k_gs_colour_bs<1, CHUNK, K>, 1);
        else if (t == 2) go(k_gs_colour_bs<2, CHUNK, K>, 2);
        else if (t == 4) go(k_gs_colour_bs<4, CHUNK, K>, 4);
        else go(k_gs_colour_bs<8, CHUNK, K>, 8);
    }
}
template <int MODE, int K>
static void b_spmv(int tpr, i64 r1, const i64* sptr, const i32* scol, const double* sval, const double* x,
                   const double* f, double* y, cudaStream_t st, const i32* sluw = nullptr,
                   const uint8_t* nlow = nullptr, const i32* yperm = nullptr) {
    auto go = [&](auto kern, int t) {
        launch(true, kern, blocks_for(r1 * t * (K / 2), 256), 256, 0, st, 0, (int)r1, sptr, scol, sval, x, f, y, sluw,
               nlow, yperm);
    };
    tpr = std::min(tpr, 64 / K);
    if constexpr (K >= 4) {
        if (batch_ch8(K, r1)) {
            if (tpr == 1) go(k_sell_spmv_bs<MODE, 1, 8, K>, 1);
            else if (tpr == 2) go(k_sell_spmv_bs<MODE, 2, 8, K>, 2);
            else if (tpr == 4) go(k_sell_spmv_bs<MODE, 4, 8, K>, 4);
            else go(k_sell_spmv_bs<MODE, 8, 8, K>, 8);
            return;
        }
    }
    if (tpr == 1) go(k_sell_spmv_bs<MODE, 1, CHUNK, K>, 1);
    else if (tpr == 2) go(k_sell_spmv_bs<MODE, 2, CHUNK, K>, 2);
    else if (tpr == 4) go(k_sell_spmv_bs<MODE, 4, CHUNK, K>, 4);
    else go(k_sell_spmv_bs<MODE, 8, CHUNK, K>, 8);
}
template <int K>
static void b_interp(const Level& L, const double* ec, double* e, cudaStream_t st) {
    auto kern = L.pm <= 8 ? k_interp_correct_bs<8, K> : k_interp_correct_bs<16, K>;
    launch(true, kern, blocks_for(L.n * (K / 2), 256), 256, 0, st, (int)L.n, L.pm, (const i32*)L.pcol,
           (const double*)L.pval, ec, e);
}
template <int K>
static void enqueue_vcycle_b(mgm_ctx* ctx, cudaStream_t st, bool zero0) {
    auto& lv = ctx->lv;
    const int p = ctx->p;
    ctx->ntrace = 0;
    ctx->trace_labels.clear();
    const int nu1 = ctx->lp.nu1, nu2 = ctx->lp.nu2;
    const bool pre_b = ctx->lp.smoother == 1, post_b = ctx->lp.smoother == 1 || ctx->lp.smoother == 2;
    auto sweep = [&](int j, bool backward, bool zg = false) {
        const Level& L = lv[j];
        for (int q = 0; q < L.ncol; ++q) {
            const int c = backward ? L.ncol - 1 - q : q;
            if (L.coff[c + 1] > L.coff[c]) b_gs<K>(ctx, L, j, (int)L.coff[c], (int)L.coff[c + 1], st, zg);
        }
    };
    // the first presmooth of a coarse level starts from zero: zero-guess colour kernels
    auto zg_ok = [&](int j) { return !pre_b && !ctx->poisson && lv[j].slw && lv[j].nlow && !ctx->no_zg; };
    auto coarse = [&]() {
        const int m = ctx->nc;
        launch(true, k_dense_mv_b<K>, blocks_for((i64)m * K, 256), 256, 0, st, m, (const double*)ctx->ainv,
               (const double*)ctx->bf[p - 1], ctx->bu[p - 1]);
    };
    if (p == 1) { coarse(); return; }
    // levels >= D: the dense bottom B_D applied to the K columns at once (dense_bottom.cuh)
    const int D = ctx->denseJ > 0 ? ctx->denseJ : p - 1;
    stamp(ctx, "start", 0, st);
    for (int s = 0; s < nu1; ++s) sweep(0, pre_b, zero0 && s == 0 && zg_ok(0));   // line 4
    stamp(ctx, "presmooth", 0, st);
    for (int j = 0; j < D; ++j) {                                                   // lines 5-9
        const Level& L = lv[j];
        if (j > 0) {
            cudaMemsetAsync(ctx->bu[j], 0, sizeof(double) * L.n * K, st);
            for (int s = 0; s < nu1; ++s) sweep(j, pre_b, s == 0 && zg_ok(j));
        }
        if (j > 0) stamp(ctx, "zero+presmooth", j, st);
        // after exactly one presmooth from the zero guess: the later-colour residual (MODE 2);
        // the residual in Morton order for the restriction's Morton columns (split kernels)
        const bool after_zg = nu1 == 1 && zg_ok(j) && (j > 0 || zero0);
        const bool m2 = after_zg && L.sluw && L.n >= ctx->upper_res_min;
        const bool mt = L.l2m && L.rcol_m && L.n >= g_batch_morton_min;
        if (m2)
            b_spmv<2, K>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bu[j], ctx->bf[j], ctx->bt[j], st, L.sluw, L.nlow,
                         mt ? L.l2m : nullptr);
        else
            b_spmv<1, K>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bu[j], ctx->bf[j], ctx->bt[j], st, nullptr, nullptr,
                         mt ? L.l2m : nullptr);
        b_spmv<0, K>(L.rtpr, lv[j + 1].n, L.rptr, mt ? L.rcol_m : L.rcol, L.rval, ctx->bt[j], nullptr, ctx->bf[j + 1],
                     st);
        stamp(ctx, "residual+restrict", j, st);
    }
    if (ctx->denseJ > 0) enqueue_dense_bottom(ctx, K, ctx->bf[D], ctx->bu[D], st);
    else coarse();                                                                   // line 10
    stamp(ctx, "bottom", D, st);
    for (int j = D - 1; j >= 0; --j) {                                              // lines 11-16
        const Level& L = lv[j];
        b_interp<K>(L, ctx->bu[j + 1], ctx->bu[j], st);
        for (int s = 0; s < nu2; ++s) {
            g_bdlt = (j == 0 && s + 1 == nu2) ? ctx->bdlt_out : nullptr;  // last level-0 postsmooth: increments
            sweep(j, post_b);
            g_bdlt = nullptr;
        }
        stamp(ctx, "interp+postsmooth", j, st);
    }
}
static void enqueue_vcycle_bk(mgm_ctx* ctx, int K, cudaStream_t st, bool zero0) {
    switch (K) {
        case 2: enqueue_vcycle_b<2>(ctx, st, zero0); break;
        case 4: enqueue_vcycle_b<4>(ctx, st, zero0); break;
        default: enqueue_vcycle_b<8>(ctx, st, zero0); break;
    }
}
// Alg. 3 lines 6-14 for the levels J..p-1 from e_J = 0 on K interleaved columns (the batched
// kernels of enqueue_vcycle_b): the dense bottom's build, K unit vectors per replay.
template <int K>
static void enqueue_levels_plain_b(mgm_ctx* ctx, int J, cudaStream_t st) {
    auto& lv = ctx->lv;
    const int p = ctx->p;
    const int nu1 = ctx->lp.nu1, nu2 = ctx->lp.nu2;
    const bool pre_b = ctx->lp.smoother == 1, post_b = ctx->lp.smoother == 1 || ctx->lp.smoother == 2;
    auto sweep = [&](int j, bool backward) {
        const Level& L = lv[j];
        for (int q = 0; q < L.ncol; ++q) {
            const int c = backward ? L.ncol - 1 - q : q;
            if (L.coff[c + 1] > L.coff[c]) b_gs<K>(ctx, L, j, (int)L.coff[c], (int)L.coff[c + 1], st);
        }
    };
    auto coarse = [&]() {
        const int m = ctx->nc;
        launch(true, k_dense_mv_b<K>, blocks_for((i64)m * K, 256), 256, 0, st, m, (const double*)ctx->ainv,
               (const double*)ctx->bf[p - 1], ctx->bu[p - 1]);
    };
    for (int j = J; j + 1 < p; ++j) {                                               // lines 6-9
        const Level& L = lv[j];
        cudaMemsetAsync(ctx->bu[j], 0, sizeof(double) * L.n * K, st);
        for (int s = 0; s < nu1; ++s) sweep(j, pre_b);
        b_spmv<1, K>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bu[j], ctx->bf[j], ctx->bt[j], st);
        b_spmv<0, K>(L.rtpr, lv[j + 1].n, L.rptr, L.rcol, L.rval, ctx->bt[j], nullptr, ctx->bf[j + 1], st);
    }
    coarse();                                                                        // line 10
    for (int j = p - 2; j >= J; --j) {                                              // lines 11-14
        const Level& L = lv[j];
        b_interp<K>(L, ctx->bu[j + 1], ctx->bu[j], st);
        for (int s = 0; s < nu2; ++s) sweep(j, post_b);
    }
}
template <int K>
__global__ void k_unit_b(int n, int i0, double* __restrict__ f) {  // f[r][c] = (r == i0 + c)
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n * K; q += gridDim.x * blockDim.x)
        f[q] = q / K == i0 + q % K ? 1.0 : 0.0;
}
template <int K>
__global__ void k_take_b(int n, int i0, const double* __restrict__ u, double* __restrict__ T) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n * K; q += gridDim.x * blockDim.x) {
        const int r = q / K, c = q % K;
        if (i0 + c < n) T[(i64)(i0 + c) * n + r] = u[q];
    }
}
mgm_status build_dense_columns_b(mgm_ctx* ctx, int J, int mdim, double* T, cudaStream_t st) {
    // S independent buffer sets, each with its own captured graph, replayed on S streams
    // (the small levels' kernels are latency-bound: the replays overlap)
    constexpr int K = 8, S = 4;
    const int p = ctx->p;
    if (ctx->bK != 0 || J >= p - 1 || !ctx->ainv) return MGM_ERR_ARG;
    struct Set {
        std::vector<double*> bu, bf, bt;
        cudaGraphExec_t gx = nullptr;
        cudaStream_t s = nullptr;
    };
    std::vector<Set> sets(S);
    struct Release {
        mgm_ctx* c;
        std::vector<Set>& v;
        ~Release() {
            for (auto& q : v) {
                for (auto* w : {&q.bu, &q.bf, &q.bt})
                    for (double* ptr : *w) dev_free(ptr);
                if (q.gx) cudaGraphExecDestroy(q.gx);
                if (q.s) cudaStreamDestroy(q.s);
            }
            c->bu.clear();
            c->bf.clear();
            c->bt.clear();
        }
    } release_{ctx, sets};
    for (auto& q : sets) {
        q.bu.assign(p, nullptr);
        q.bf.assign(p, nullptr);
        q.bt.assign(p, nullptr);
        for (int j = J; j < p; ++j) {
            CK(dalloc(&q.bu[j], ctx->lv[j].n * K));
            CK(dalloc(&q.bf[j], ctx->lv[j].n * K));
            CK(dalloc(&q.bt[j], ctx->lv[j].n * K));
        }
        CK(cudaStreamCreateWithFlags(&q.s, cudaStreamNonBlocking));
        ctx->bu = q.bu;
        ctx->bf = q.bf;
        ctx->bt = q.bt;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        g_launch_err.clear();
        enqueue_levels_plain_b<K>(ctx, J, st);
        const cudaError_t ce = cudaStreamEndCapture(st, &g);
        if (ce != cudaSuccess || !g_launch_err.empty()) {
            ctx->err = "dense bottom capture failed: " + std::string(cudaGetErrorString(ce)) + "; " + g_launch_err;
            g_launch_err.clear();
            cudaGetLastError();
            return MGM_ERR_CUDA;
        }
        CK(cudaGraphInstantiate(&q.gx, g, 0));
        cudaGraphDestroy(g);
    }
    CK(cudaStreamSynchronize(st));  // (T allocated and zero state before the side streams)
    for (int i0 = 0, b = 0; i0 < mdim; i0 += K, b = (b + 1) % S) {
        Set& q = sets[b];
        k_unit_b<K><<<blocks_for((i64)mdim * K, 256), 256, 0, q.s>>>(mdim, i0, q.bf[J]);
        CK(cudaGraphLaunch(q.gx, q.s));
        k_take_b<K><<<blocks_for((i64)mdim * K, 256), 256, 0, q.s>>>(mdim, i0, q.bu[J], T);
    }
    for (auto& q : sets) CK(cudaStreamSynchronize(q.s));
    return MGM_OK;
}

static mgm_status ensure_batch(mgm_ctx* ctx, int K) {
    if (ctx->bK >= K) return MGM_OK;
    for (auto* q : {&ctx->bu, &ctx->bf, &ctx->bt})
        for (double* ptr : *q) dev_free(ptr);
    ctx->bu.assign(ctx->p, nullptr);
    ctx->bf.assign(ctx->p, nullptr);
    ctx->bt.assign(ctx->p, nullptr);
    for (int j = 0; j < ctx->p; ++j) {
        CK(dalloc(&ctx->bu[j], ctx->lv[j].n * K));
        CK(dalloc(&ctx->bf[j], ctx->lv[j].n * K));
        CK(dalloc(&ctx->bt[j], ctx->lv[j].n * K));
    }
    if (ctx->bres) dev_free(ctx->bres);
    CK(dalloc(&ctx->bres, ctx->N * K));
    for (auto& gx : ctx->bgraph)
        if (gx) { cudaGraphExecDestroy(gx); gx = nullptr; }
    for (auto& gx : ctx->bgraph_zg)
        if (gx) { cudaGraphExecDestroy(gx); gx = nullptr; }
    ctx->bK = K;
    return MGM_OK;
}
// zero0: the level-0 guess is zero (Krylov preconditioning): zero-guess first presmooth
static mgm_status run_vcycle_b(mgm_ctx* ctx, int K, cudaStream_t st, bool zero0 = false) {
    cudaGraphExec_t& gx = zero0 ? ctx->bgraph_zg[K] : ctx->bgraph[K];
    if (!gx) {
        // both batched graphs leave their last postsmooth's increments in bdlt (the batched GMRES's
        // A z, the batched standalone residual)
        const bool dl = mode3_ok(ctx);
        if (dl && ctx->bdlt_k < K) {
            if (ctx->bdlt) dev_free(ctx->bdlt);
            ctx->bdlt = nullptr;
            CK(dalloc(&ctx->bdlt, ctx->N * K));
            ctx->bdlt_k = K;
        }
        ctx->bdlt_out = dl ? ctx->bdlt : nullptr;
        (zero0 ? ctx->bgraph_zg_dlt : ctx->bgraph_dlt)[K] = dl;
        struct ResetB { mgm_ctx* c; ~ResetB() { c->bdlt_out = nullptr; } } resetb_{ctx};
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(ctx->st, cudaStreamCaptureModeThreadLocal));
        g_launch_err.clear();
        enqueue_vcycle_bk(ctx, K, ctx->st, zero0);
        const cudaError_t ce = cudaStreamEndCapture(ctx->st, &g);
        if (ce != cudaSuccess || !g_launch_err.empty()) {
            ctx->err = "batched V-cycle capture failed: " + std::string(cudaGetErrorString(ce)) + "; " + g_launch_err;
            g_launch_err.clear();
            cudaGetLastError();
            return MGM_ERR_CUDA;
        }
        CK(cudaGraphInstantiate(&gx, g, 0));
        cudaGraphDestroy(g);
    }
    CK(cudaGraphLaunch(gx, st));
    return MGM_OK;
}
static void enqueue_bdot(mgm_ctx* ctx, int K, i64 n, const double* a, const double* b, double* out, cudaStream_t st) {
    switch (K) {
        case 2: k_bdot_fin<2><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, a, b, ctx->partials, ctx->tickets, out); break;
        case 4: k_bdot_fin<4><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, a, b, ctx->partials, ctx->tickets, out); break;
        default: k_bdot_fin<8><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, a, b, ctx->partials, ctx->tickets, out); break;
    }
}
// out[j K + k] = V_j[:, k] . w[:, k] for j < k1, one launch (k_bmultidot_fin; partials in bpart)
static void enqueue_bmultidot(mgm_ctx* ctx, int K, i64 n, const double* V, i64 stride, int k1, const double* w,
                              double* out, cudaStream_t st) {
    switch (K) {
        case 2: k_bmultidot_fin<2, 8><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, V, stride, k1, w, ctx->bpart, ctx->tickets,
                                                                           out); break;
        case 4: k_bmultidot_fin<4, 4><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, V, stride, k1, w, ctx->bpart, ctx->tickets,
                                                                           out); break;
        default: k_bmultidot_fin<8, 2><<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, V, stride, k1, w, ctx->bpart, ctx->tickets,
                                                                            out); break;
    }
}
static void enqueue_res_b(mgm_ctx* ctx, int K, cudaStream_t st) {  // bres = bf0 - L_1 bu0
    const Level& L = ctx->lv[0];
    if (ctx->bgraph_dlt[K]) {  // after the general batched V-cycle: -(later-colour part of L_1) d
        switch (K) {
            case 2: b_spmv<2, 2>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bdlt, nullptr, ctx->bres, st, L.sluw, L.nlow); break;
            case 4: b_spmv<2, 4>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bdlt, nullptr, ctx->bres, st, L.sluw, L.nlow); break;
            default: b_spmv<2, 8>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bdlt, nullptr, ctx->bres, st, L.sluw, L.nlow); break;
        }
        return;
    }
    switch (K) {
        case 2: b_spmv<1, 2>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bu[0], ctx->bf[0], ctx->bres, st); break;
        case 4: b_spmv<1, 4>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bu[0], ctx->bf[0], ctx->bres, st); break;
        default: b_spmv<1, 8>(L.stpr, L.n, L.sptr, L.scol, L.sval, ctx->bu[0], ctx->bf[0], ctx->bres, st); break;
    }
}

mgm_status standalone_lib(mgm_ctx* ctx, double tol, int maxit, mgm_report* rep, cudaStream_t st) {
    const i64 n = vec_rows(ctx);
    double* nr = ctx->dh + 512;
    mgm_status s;
    enqueue_dot(ctx, n, ctx->b, ctx->b, nr, st);
    CK(cudaMemcpyAsync(ctx->hh, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const double fn = std::sqrt(ctx->hh[0]);
    if (ctx->warm && fn != 0.0)  // u starts at x0 (the applications' warm start)
        CK(cudaMemcpyAsync(ctx->lv[0].u, ctx->xs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    else
        CK(cudaMemsetAsync(ctx->lv[0].u, 0, sizeof(double) * (n + ctx->lv[0].nghost), st));
    exch(ctx, 0, ctx->lv[0].u, -1, st);  // (distributed: the first sweep reads the ghosts of x0)
    CK(cudaMemsetAsync(ctx->xs, 0, sizeof(double) * n, st));
    if (fn == 0.0) {
        if (rep) { rep->iterations = 0; rep->converged = 1; rep->final_rel_residual = 0.0; }
        return MGM_OK;
    }
    CK(cudaMemcpyAsync(ctx->lv[0].f, ctx->b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    int it = 0, hist_n = 0;
    double rel = 1.0;
    bool conv = false;
    // the residual from the last postsmooth's increments when the V-cycle graph records them
    const bool from_dlt = !timing_on(ctx) && mode3_ok(ctx);
    while (it < maxit) {
        if ((s = run_vcycle(ctx, st))) return s;
        ++it;
        if (from_dlt && ctx->last_vc_dlt) {  // r = f - A u = -(later-colour part of L_1) d
            const Level& L0 = ctx->lv[0];
            g_sluw = L0.sluw;
            g_nlow = L0.nlow;
            launch_spmv(false, 2, false, L0.stpr, 0, L0.n, L0.n, L0.sptr, L0.scol, L0.sval, ctx->d_dlt, nullptr, ctx->w,
                        L0.c, st);
            g_sluw = nullptr;
            g_nlow = nullptr;
        } else {
            enqueue_apply_A(ctx, ctx->lv[0].u, ctx->w, st);
            k_axpby<<<RED_BLOCKS, 256, 0, st>>>(n, 1.0, ctx->b, -1.0, ctx->w, ctx->w);
        }
        enqueue_dot(ctx, n, ctx->w, ctx->w, nr, st);
        CK(cudaMemcpyAsync(ctx->hh, nr, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (timing_on(ctx)) timer_collect(ctx);
        rel = std::sqrt(ctx->hh[0]) / fn;
        if (rep && rep->history && hist_n < rep->history_cap) rep->history[hist_n++] = rel;
        if (rel <= tol) { conv = true; break; }
        if (!std::isfinite(rel)) break;
    }
    CK(cudaMemcpyAsync(ctx->xs, ctx->lv[0].u, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    if (ctx->poisson) {
        CK(cudaMemcpyAsync(ctx->hh + 1, ctx->xs + ctx->lv[0].n, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    if (rep) {
        rep->iterations = it;
        rep->converged = conv ? 1 : 0;
        rep->final_rel_residual = rel;
        rep->lambda = ctx->poisson ? ctx->hh[1] : 0.0;
    }
    return MGM_OK;
}

mgm_status check_ctx(mgm_ctx* ctx) {
    if (!ctx || ctx->lv.empty()) return MGM_ERR_ARG;
    cudaSetDevice(ctx->device);
    return MGM_OK;
}

}  // namespace

// ---------------------------------------------------------------------------------------
// Partition of the hierarchy (mgm_dist_attach): levels 0..D-1 become this rank's Morton
// block + ghosts (PartTables, host_setup.cpp partition_level), built from the undistributed
// structures every rank holds after the (deterministic, replicated) setup; the
// undistributed device arrays of those levels are freed.  Every local operator row keeps
// the undistributed row's entries in the same order, and each colour launch keeps its
// threads per row, so the distributed V-cycle computes every row with the same arithmetic.
// ---------------------------------------------------------------------------------------
namespace {

template <class T>
std::vector<T> download(const T* d, i64 n) {
    std::vector<T> h((size_t)std::max<i64>(n, 0));
    if (n > 0) cudaMemcpy(h.data(), d, sizeof(T) * (size_t)n, cudaMemcpyDeviceToHost);
    return h;
}

// first level of the replicated bottom: the dense bottom, the cluster bottom, or the coarsest
int bottom_level(const mgm_ctx* ctx) {
    return ctx->denseJ > 0 ? ctx->denseJ : ctx->botJ > 0 ? ctx->botJ : ctx->p - 1;
}

// distributed levels: 0 .. D-1 with at least MGM_DIST_MIN_ROWS (default 16384) rows per rank
// (below that a level is cheaper redundant than exchanged), never the bottom
int choose_D(const mgm_ctx* ctx, int nranks) {
    const int top = bottom_level(ctx);
    i64 min_rows = 16384;
    if (const char* e = std::getenv("MGM_DIST_MIN_ROWS")) min_rows = std::max<i64>(1, std::atoll(e));
    int D = 1;
    while (D < top && ctx->lv[D].n / nranks >= min_rows) ++D;
    if (const char* e = std::getenv("MGM_DIST_LEVELS")) D = std::max(1, std::min(top, std::atoi(e)));
    return D;
}

void free_level_device(Level& L) {
    for (void* ptr : {(void*)L.sptr, (void*)L.scol, (void*)L.sval, (void*)L.pcol, (void*)L.pval, (void*)L.rptr,
                      (void*)L.rcol, (void*)L.rval, (void*)L.u, (void*)L.f, (void*)L.t, (void*)L.c, (void*)L.slw,
                      (void*)L.nlow, (void*)L.sluw, (void*)L.l2m, (void*)L.rcol_m, (void*)L.d_send_idx,
                      (void*)L.d_sendbuf, (void*)L.d_srange, (void*)L.d_stage_mine, (void*)L.d_stage_all,
                      (void*)L.d_stage_perm, (void*)L.d_rslot})
        if (ptr) dev_free(ptr);
}

}  // namespace

mgm_status dist_partition(mgm_ctx* ctx) {
    const int P = ctx->nranks, q = ctx->rank;
    if (ctx->p < 2) {
        ctx->err = "multi-GPU solve needs at least two levels";
        return MGM_ERR_ARG;
    }
    const int D = choose_D(ctx, P);
    const i64 N = ctx->N;
    const i64 pad = ctx->poisson ? 1 : 0;
    cudaStream_t st = ctx->st;
    auto& lv = ctx->lv;
    // ---- owners: rank r owns the level-0 Morton indices [floor(rN/P), floor((r+1)N/P)); a
    // coarse point keeps the owner of its level-0 point (coarse sets inherit the order)
    std::vector<i64> mstart(P + 1);
    for (int r = 0; r <= P; ++r) mstart[(size_t)r] = (i64)((__int128)r * N / P);
    auto owner_of_m = [&](i64 m) {
        return (int)(std::upper_bound(mstart.begin(), mstart.end(), m) - mstart.begin()) - 1;
    };
    std::vector<i64> mor0((size_t)N);
    for (i64 r = 0; r < N; ++r) mor0[(size_t)lv[0].ids[(size_t)r]] = lv[0].lib2mor[(size_t)r];
    std::vector<std::vector<int>> owner((size_t)D + 1);
    for (int j = 0; j <= D; ++j) {
        owner[(size_t)j].resize((size_t)lv[j].n);
        for (i64 r = 0; r < lv[j].n; ++r) owner[(size_t)j][(size_t)r] = owner_of_m(mor0[(size_t)lv[j].ids[(size_t)r]]);
    }
    // ---- partition tables (this rank's) of the distributed levels
    std::vector<PartTables> T((size_t)D);
    std::vector<std::vector<i64>> rslot((size_t)D);
    for (int j = 0; j < D; ++j) {
        std::vector<PartTables> all;
        partition_level(lv[j].L_lib, owner[(size_t)j], lv[j].colour_lib, lv[j].ncol, &lv[j].P_lib, &owner[(size_t)j + 1],
                        j > 0 ? &lv[j - 1].P_lib : nullptr, j > 0 ? &owner[(size_t)j - 1] : nullptr, P, all);
        {  // peer-store slots: where each of my send entries lands in the peer's vector
            const PartTables& Tq = all[(size_t)q];
            auto& rs = rslot[(size_t)j];
            rs.assign(Tq.send_rows.size(), 0);
            for (size_t i = 0; i < Tq.peers.size(); ++i) {
                const PartTables& Tp = all[(size_t)Tq.peers[i]];
                const size_t k = (size_t)(std::find(Tp.peers.begin(), Tp.peers.end(), q) - Tp.peers.begin());
                const i64 base = (i64)Tp.rows.size() + pad + Tp.recv_off[k];
                for (i64 e = Tq.send_off[i]; e < Tq.send_off[i + 1]; ++e) rs[(size_t)e] = base + (e - Tq.send_off[i]);
            }
        }
        T[(size_t)j] = std::move(all[(size_t)q]);
    }
    // global row -> local column index (owned: 0..n-1; ghost g: n + pad + g), per level
    std::vector<std::vector<i64>> cmap((size_t)D);
    for (int j = 0; j < D; ++j) {
        auto& c = cmap[(size_t)j];
        c.assign((size_t)lv[j].n, -1);
        const i64 nl = (i64)T[(size_t)j].rows.size();
        for (i64 k = 0; k < nl; ++k) c[(size_t)T[(size_t)j].rows[(size_t)k]] = k;
        for (size_t g = 0; g < T[(size_t)j].ghosts.size(); ++g) c[(size_t)T[(size_t)j].ghosts[g]] = nl + pad + (i64)g;
    }
    mgm_status s;
    std::vector<Level> loc((size_t)D);
    for (int j = 0; j < D; ++j) {
        const Level& G = lv[j];
        const PartTables& Tj = T[(size_t)j];
        Level& L = loc[(size_t)j];
        const i64 nl = (i64)Tj.rows.size();
        const auto& cm = cmap[(size_t)j];
        auto col_of = [&](i64 g) -> i32 {
            const i64 v = cm[(size_t)g];
            return (i32)(v >= 0 ? v : 0);  // (every column read is owned or a ghost by construction)
        };
        L.dist = true;
        L.n = nl;
        L.ncol = G.ncol;
        L.nghost = (i64)Tj.ghosts.size();
        L.gbase = nl + pad;
        L.tpr = G.tpr;
        L.rtpr = G.rtpr;
        L.stpr = G.stpr;
        L.gs_block = G.gs_block;
        L.pm = G.pm;
        L.gcoff = G.coff;
        L.coff.assign((size_t)G.ncol + 1, 0);
        for (i64 r : Tj.rows) L.coff[(size_t)G.colour_lib[(size_t)r] + 1]++;
        for (int c = 0; c < G.ncol; ++c) L.coff[(size_t)c + 1] += L.coff[(size_t)c];
        L.tpr_col.resize((size_t)G.ncol);
        for (int c = 0; c < G.ncol; ++c)
            L.tpr_col[(size_t)c] =
                gs_tpr_for(G.tpr, G.coff[(size_t)c + 1] - (G.coff[(size_t)c] & ~(i64)31), G.gs_block);
        L.ids.resize((size_t)nl);
        L.colour_lib.resize((size_t)nl);
        for (i64 k = 0; k < nl; ++k) {
            L.ids[(size_t)k] = G.ids[(size_t)Tj.rows[(size_t)k]];
            L.colour_lib[(size_t)k] = G.colour_lib[(size_t)Tj.rows[(size_t)k]];
        }
        // -- L_j: the undistributed SELL rows (pack_sell order), columns remapped
        {
            const auto gcol = download(G.scol, G.sell_stored);
            const auto gval = download(G.sval, G.sell_stored);
            const std::vector<uint8_t> gnlow = G.nlow ? download(G.nlow, G.n) : std::vector<uint8_t>();
            const i64 ns = (nl + 31) / 32;
            std::vector<i64> sptr((size_t)ns + 1, 0);
            auto rlen = [&](i64 k) { const i64 r = Tj.rows[(size_t)k]; return G.L_lib.ptr[(size_t)r + 1] - G.L_lib.ptr[(size_t)r]; };
            for (i64 sl = 0; sl < ns; ++sl) {
                i64 w = 1;
                for (i64 k = sl * 32; k < std::min(nl, sl * 32 + 32); ++k) w = std::max(w, rlen(k));
                sptr[(size_t)sl + 1] = sptr[(size_t)sl] + 32 * w;
            }
            std::vector<i32> scol((size_t)sptr[(size_t)ns], 0);
            std::vector<double> sval((size_t)sptr[(size_t)ns], 0.0);
            std::vector<i32> slw, sluw;
            std::vector<uint8_t> nlow;
            if (G.nlow) {
                slw.assign((size_t)ns, 1);
                sluw.assign((size_t)ns, 1 << 30);
                nlow.assign((size_t)nl, 0);
                L.lower_per_colour.assign((size_t)G.ncol, 0);
            }
            for (i64 k = 0; k < nl; ++k) {
                const i64 r = Tj.rows[(size_t)k], gs = r >> 5, gl = r & 31;
                const i64 sl = k >> 5, lane = k & 31, w = (sptr[(size_t)sl + 1] - sptr[(size_t)sl]) / 32;
                const i64 len = rlen(k);
                for (i64 e = 0; e < w; ++e) {
                    const i64 o = sptr[(size_t)sl] + 32 * e + lane;
                    if (e < len) {
                        const i64 go = G.h_sptr[(size_t)gs] + 32 * e + gl;
                        scol[(size_t)o] = col_of(gcol[(size_t)go]);
                        sval[(size_t)o] = gval[(size_t)go];
                    } else {
                        scol[(size_t)o] = (i32)k;
                        sval[(size_t)o] = 0.0;
                    }
                }
                if (G.nlow) {
                    const int nlw = gnlow[(size_t)r];
                    nlow[(size_t)k] = (uint8_t)nlw;
                    slw[(size_t)sl] = std::max<i32>(slw[(size_t)sl], 1 + nlw);
                    sluw[(size_t)sl] = std::min<i32>(sluw[(size_t)sl], 1 + nlw);
                    L.lower_per_colour[(size_t)L.colour_lib[(size_t)k]] += 1 + nlw;
                }
            }
            L.nnz = 0;
            for (i64 k = 0; k < nl; ++k) L.nnz += rlen(k);
            L.sell_stored = sptr[(size_t)ns];
            bool uni = ns > 0;
            for (i64 sl = 0; sl < ns && uni; ++sl) uni = sptr[(size_t)sl + 1] - sptr[(size_t)sl] == sptr[1] - sptr[0];
            L.uniform_w = uni ? (int)((sptr[1] - sptr[0]) / 32) : 0;
            L.h_sptr = sptr;
            if ((s = upload(ctx, &L.sptr, sptr)) || (s = upload(ctx, &L.scol, scol)) || (s = upload(ctx, &L.sval, sval)))
                return s;
            if (G.nlow && ((s = upload(ctx, &L.slw, slw)) || (s = upload(ctx, &L.nlow, nlow)) ||
                           (s = upload(ctx, &L.sluw, sluw))))
                return s;
        }
        // -- P_j (ELL [pm][n], fine rows = my rows) and R_j (SELL, my coarse rows)
        const bool next_dist = j + 1 < D;
        const Level& Gn = lv[j + 1];
        auto ccol_of = [&](i64 g) -> i32 {
            if (!next_dist) return (i32)g;  // replicated coarse level: global lib index
            const i64 v = cmap[(size_t)j + 1][(size_t)g];
            return (i32)(v >= 0 ? v : 0);
        };
        {
            const int pm = G.pm;
            std::vector<i32> pcol((size_t)pm * nl);
            std::vector<double> pval((size_t)pm * nl, 0.0);
            i64 pnnz = 0;
            for (i64 k = 0; k < nl; ++k) {
                const i64 r = Tj.rows[(size_t)k];
                const i64 a = G.P_lib.ptr[(size_t)r], cnt = G.P_lib.ptr[(size_t)r + 1] - a;
                pnnz += cnt;
                for (int e = 0; e < pm; ++e) {
                    pcol[(size_t)e * nl + k] = ccol_of(G.P_lib.col[(size_t)(a + (e < cnt ? e : 0))]);
                    pval[(size_t)e * nl + k] = e < cnt ? G.P_lib.val[(size_t)(a + e)] : 0.0;
                }
            }
            L.p_nnz = pnnz;
            if ((s = upload(ctx, &L.pcol, pcol)) || (s = upload(ctx, &L.pval, pval))) return s;
        }
        {
            // my coarse rows: owned rows of level j+1 (ascending lib index)
            std::vector<i64> crow;
            if (next_dist) crow = T[(size_t)j + 1].rows;
            else
                for (i64 c = 0; c < Gn.n; ++c)
                    if (owner[(size_t)j + 1][(size_t)c] == q) crow.push_back(c);
            std::vector<i64> rcnt((size_t)Gn.n, 0);
            for (i32 c : G.P_lib.col) rcnt[(size_t)c]++;
            const auto grcol = download(G.rcol, G.r_stored);
            const auto grval = download(G.rval, G.r_stored);
            const i64 nc = (i64)crow.size(), ns = (nc + 31) / 32;
            std::vector<i64> rptr((size_t)ns + 1, 0);
            for (i64 sl = 0; sl < ns; ++sl) {
                i64 w = 1;
                for (i64 k = sl * 32; k < std::min(nc, sl * 32 + 32); ++k) w = std::max(w, rcnt[(size_t)crow[(size_t)k]]);
                rptr[(size_t)sl + 1] = rptr[(size_t)sl] + 32 * w;
            }
            std::vector<i32> rcol((size_t)rptr[(size_t)ns], 0);
            std::vector<double> rval((size_t)rptr[(size_t)ns], 0.0);
            for (i64 k = 0; k < nc; ++k) {
                const i64 c = crow[(size_t)k], gs = c >> 5, gl = c & 31;
                const i64 sl = k >> 5, lane = k & 31, w = (rptr[(size_t)sl + 1] - rptr[(size_t)sl]) / 32;
                const i64 len = rcnt[(size_t)c];
                i32 first = 0;
                for (i64 e = 0; e < w; ++e) {
                    const i64 o = rptr[(size_t)sl] + 32 * e + lane;
                    if (e < len) {
                        const i64 go = G.h_rptr[(size_t)gs] + 32 * e + gl;
                        rcol[(size_t)o] = col_of(grcol[(size_t)go]);
                        rval[(size_t)o] = grval[(size_t)go];
                        if (e == 0) first = rcol[(size_t)o];
                    } else {
                        rcol[(size_t)o] = first;
                        rval[(size_t)o] = 0.0;
                    }
                }
            }
            L.r_stored = rptr[(size_t)ns];
            L.h_rptr = rptr;
            if ((s = upload(ctx, &L.rptr, rptr)) || (s = upload(ctx, &L.rcol, rcol)) || (s = upload(ctx, &L.rval, rval)))
                return s;
            if (!next_dist) {  // all-gather of the first replicated level
                L.nstage = nc;
                L.stage_off.assign((size_t)P + 1, 0);
                for (i64 c = 0; c < Gn.n; ++c) L.stage_off[(size_t)owner[(size_t)j + 1][(size_t)c] + 1]++;
                for (int r = 0; r < P; ++r) L.stage_off[(size_t)r + 1] += L.stage_off[(size_t)r];
                std::vector<i32> perm((size_t)Gn.n);
                std::vector<i64> fill(L.stage_off.begin(), L.stage_off.end() - 1);
                for (i64 c = 0; c < Gn.n; ++c) perm[(size_t)fill[(size_t)owner[(size_t)j + 1][(size_t)c]]++] = (i32)c;
                if ((s = upload(ctx, &L.d_stage_perm, perm))) return s;
                CK(dalloc(&L.d_stage_mine, std::max<i64>(nc, 1)));
                CK(dalloc(&L.d_stage_all, Gn.n));
            }
        }
        // -- Poisson border, vectors
        if (ctx->poisson) {
            L.c_lib.resize((size_t)nl);
            for (i64 k = 0; k < nl; ++k) L.c_lib[(size_t)k] = G.c_lib[(size_t)Tj.rows[(size_t)k]];
            if ((s = upload(ctx, &L.c, L.c_lib))) return s;
        }
        const i64 vn = nl + pad + L.nghost;
        CK(dalloc(&L.u, vn));
        CK(dalloc(&L.f, vn));
        CK(dalloc(&L.t, vn));
        CK(cudaMemsetAsync(L.u, 0, sizeof(double) * vn, st));
        CK(cudaMemsetAsync(L.f, 0, sizeof(double) * vn, st));
        CK(cudaMemsetAsync(L.t, 0, sizeof(double) * vn, st));
        // -- halo tables
        L.peers = Tj.peers;
        L.h_rslot = rslot[(size_t)j];
        L.send_off = Tj.send_off;
        L.recv_off = Tj.recv_off;
        L.send_coff = Tj.send_coff;
        L.recv_coff = Tj.recv_coff;
        {
            std::vector<i32> sidx(Tj.send_rows.size());
            for (size_t e = 0; e < sidx.size(); ++e) sidx[e] = (i32)cm[(size_t)Tj.send_rows[e]];
            if ((s = upload(ctx, &L.d_send_idx, sidx))) return s;
            CK(dalloc(&L.d_sendbuf, (i64)std::max<size_t>(1, sidx.size())));
            const size_t np = L.peers.size(), nc1 = (size_t)G.ncol + 1;
            std::vector<i64> rng(nc1 * np * 2);
            for (size_t i = 0; i < np; ++i) {
                rng[2 * i] = L.send_off[i];
                rng[2 * i + 1] = L.send_off[i + 1];
                for (size_t c = 0; c + 1 < nc1; ++c) {
                    rng[(c + 1) * np * 2 + 2 * i] = L.send_coff[i * nc1 + c];
                    rng[(c + 1) * np * 2 + 2 * i + 1] = L.send_coff[i * nc1 + c + 1];
                }
            }
            if ((s = upload(ctx, &L.d_srange, rng))) return s;
        }
    }
    // ---- level-0 I/O order: my level-0 points in Morton order
    {
        const PartTables& T0 = T[0];
        const i64 nl = (i64)T0.rows.size(), m0 = mstart[(size_t)q];
        ctx->local_ids.assign((size_t)nl, -1);
        std::vector<i32> l2io((size_t)nl);
        for (i64 k = 0; k < nl; ++k) {
            const i64 r = T0.rows[(size_t)k];
            const i64 io = lv[0].lib2mor[(size_t)r] - m0;
            l2io[(size_t)k] = (i32)io;
            ctx->local_ids[(size_t)io] = lv[0].ids[(size_t)r];
        }
        dev_free(ctx->d_lib2orig);
        ctx->d_lib2orig = nullptr;
        if ((s = upload(ctx, &ctx->d_lib2orig, l2io))) return s;
    }
    CK(cudaStreamSynchronize(st));
    for (int j = 0; j < D; ++j) {
        free_level_device(lv[j]);
        lv[j] = std::move(loc[(size_t)j]);
    }
    ctx->D = D;
    for (cudaGraphExec_t* gx : {&ctx->vgraph, &ctx->vgraph0, &ctx->ggraph})  // re-capture with the halos
        if (*gx) {
            cudaGraphExecDestroy(*gx);
            *gx = nullptr;
        }
    return MGM_OK;
}

// Peer-store halos (MGM_P2P=1 at attach): slot tables on the device, counters, and the peers'
// u / t / flag pointers -- opened with cudaIpcOpenMemHandle (handles all-gathered over NCCL),
// or taken from the group table for fake ranks.
mgm_status p2p_setup(mgm_ctx* ctx) {
    const int P = ctx->nranks, q = ctx->rank;
    const bool fake = !ctx->tp->capturable();
    if (!fake && ctx->alloc.alloc) {
        ctx->err = "peer-store halos need cudaMalloc memory (no allocator hook)";
        return MGM_ERR_ARG;
    }
    if (P > 64) return MGM_ERR_ARG;
    for (int j = 0; j < ctx->D; ++j)
        if (ctx->lv[j].peers.size() > 16) {
            ctx->err = "peer-store halos: more than 16 peers on a level";
            return MGM_ERR_ARG;
        }
    mgm_status s;
    CK(dalloc(&ctx->p2p_flags, P));
    CK(dalloc(&ctx->p2p_sent, P));
    CK(dalloc(&ctx->p2p_expect, P));
    CK(dalloc(&ctx->p2p_ticket, 1));
    CK(cudaMemset(ctx->p2p_flags, 0, sizeof(unsigned long long) * P));
    CK(cudaMemset(ctx->p2p_sent, 0, sizeof(unsigned long long) * P));
    CK(cudaMemset(ctx->p2p_expect, 0, sizeof(unsigned long long) * P));
    CK(cudaMemset(ctx->p2p_ticket, 0, sizeof(unsigned)));
    for (int j = 0; j < ctx->D; ++j)
        if ((s = upload(ctx, &ctx->lv[j].d_rslot, ctx->lv[j].h_rslot))) return s;
    // my pointers: u, t of every distributed level, then the flag array
    std::vector<void*> mine;
    for (int j = 0; j < ctx->D; ++j) {
        mine.push_back(ctx->lv[j].u);
        mine.push_back(ctx->lv[j].t);
    }
    mine.push_back(ctx->p2p_flags);
    const size_t nptr = mine.size();
    std::vector<std::vector<void*>> theirs((size_t)P, std::vector<void*>(nptr, nullptr));
    if (fake) {
        auto* ft = static_cast<FakeTransport*>(ctx->tp);
        std::vector<double*> b;
        for (void* x : mine) b.push_back((double*)x);
        ft->g->bases[(size_t)q] = b;
        ft->g->barrier();
        for (int r = 0; r < P; ++r)
            for (size_t k = 0; k < nptr; ++k) theirs[(size_t)r][k] = ft->g->bases[(size_t)r][k];
        ft->g->barrier();
    } else {
        if (!nccl().AllGather) return MGM_ERR_NCCL;
        const size_t hb = sizeof(cudaIpcMemHandle_t);
        std::vector<char> h(nptr * hb);
        for (size_t k = 0; k < nptr; ++k) CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t*)(h.data() + k * hb), mine[k]));
        char *d_mine = nullptr, *d_all = nullptr;
        CK(cudaMalloc((void**)&d_mine, h.size()));
        CK(cudaMalloc((void**)&d_all, h.size() * P));
        CK(cudaMemcpy(d_mine, h.data(), h.size(), cudaMemcpyHostToDevice));
        auto* nt = static_cast<NcclTransport*>(ctx->tp);
        if (nccl().AllGather(d_mine, d_all, h.size(), ncclChar, nt->comm, ctx->st) != ncclSuccess) return MGM_ERR_NCCL;
        std::vector<char> all(h.size() * P);
        CK(cudaStreamSynchronize(ctx->st));
        CK(cudaMemcpy(all.data(), d_all, all.size(), cudaMemcpyDeviceToHost));
        cudaFree(d_mine);
        cudaFree(d_all);
        for (int r = 0; r < P; ++r) {
            if (r == q) continue;
            for (size_t k = 0; k < nptr; ++k) {
                cudaIpcMemHandle_t hh;
                std::memcpy(&hh, all.data() + (size_t)r * h.size() + k * hb, hb);
                void* ptr = nullptr;
                CK(cudaIpcOpenMemHandle(&ptr, hh, cudaIpcMemLazyEnablePeerAccess));
                ctx->ipc_opened.push_back(ptr);
                theirs[(size_t)r][k] = ptr;
            }
        }
    }
    for (int j = 0; j < ctx->D; ++j) {
        Level& L = ctx->lv[j];
        for (size_t i = 0; i < L.peers.size(); ++i) {
            L.peer_u[i] = (double*)theirs[(size_t)L.peers[i]][2 * (size_t)j];
            L.peer_t[i] = (double*)theirs[(size_t)L.peers[i]][2 * (size_t)j + 1];
        }
    }
    for (int r = 0; r < P; ++r)
        ctx->peer_flags[r] = r == q ? nullptr : (unsigned long long*)theirs[(size_t)r][nptr - 1];
    ctx->p2p = true;
    CK(cudaDeviceSynchronize());
    return MGM_OK;
}

// =======================================================================================
// C ABI
// =======================================================================================
extern "C" {

mgm_status mgm_setup(const double* points, const double* normals, int64_t n_points,
                     const mgm_stencil_params* stencil, const mgm_level_params* levels,
                     const mgm_allocator* allocator, void* cuda_stream, mgm_ctx** out) {
    g_setup_error.clear();
    g_setup_index = -1;
    if (out) *out = nullptr;
    if (!points || !normals || !stencil || !levels || !out || n_points < 2) {
        g_setup_error = "invalid argument";
        return MGM_ERR_ARG;
    }
    const mgm_stencil_params& sp = *stencil;
    const mgm_level_params& lp = *levels;
    if (sp.method < 0 || sp.method > 1 || sp.poly_degree < 0 || sp.poly_degree > 8 || sp.stencil_n < 2 ||
        sp.stencil_n > 96 || sp.stencil_n > n_points || (sp.method == 0 && (sp.phs_k < 1 || sp.phs_k > 8)) ||
        sp.problem < 0 || sp.problem > 1 || (sp.problem == 0 && !(sp.mu > 0)) || lp.interp_m < 1 ||
        lp.interp_m > 16 || lp.nu1 < 0 || lp.nu2 < 0 || lp.coarsen_factor < 2 || lp.restart < 1 ||
        lp.restart > 128 || lp.smoother < 0 || lp.smoother > 2 || (lp.num_levels <= 0 && lp.n_min < 1) ||
        n_points > INT32_MAX / 2) {
        g_setup_error = "invalid stencil or level parameters";
        return MGM_ERR_ARG;
    }
    if (sp.method == 1 && sp.stencil_n < (sp.poly_degree + 1) * (sp.poly_degree + 2) / 2) {
        g_setup_error = "GFD stencil smaller than the polynomial space";
        return MGM_ERR_ARG;
    }
    auto t0 = std::chrono::steady_clock::now();
    if (allocator && allocator->alloc && !allocator->release) {
        g_setup_error = "allocator without a release function";
        return MGM_ERR_ARG;
    }
    mgm_ctx* ctx = new mgm_ctx();
    if (allocator) ctx->alloc = *allocator;
    AllocScope as_(ctx);
    ctx->sp = sp;
    ctx->lp = lp;
    ctx->N = n_points;
    ctx->poisson = sp.problem == 1;
    ctx->restart = lp.restart;
    ctx->nthreads = std::max(1, std::min(64, (int)std::thread::hardware_concurrency()));
    if (std::getenv("MGM_NO_ZG")) ctx->no_zg = true;
    if (std::getenv("MGM_NO_C0_FUSE")) ctx->no_c0_fuse = true;
    if (const char* e = std::getenv("MGM_UPPER_RES_MIN")) ctx->upper_res_min = std::atoll(e);
    if (const char* e = std::getenv("MGM_MORTON_T_MIN")) ctx->morton_t_min = std::atoll(e);
    cudaGetDevice(&ctx->device);
    (void)cuda_stream;
    if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess) {
        g_setup_error = "cannot create CUDA stream (no device?)";
        delete ctx;
        return MGM_ERR_CUDA;
    }
    mgm_status s = do_setup(ctx, points, normals, n_points);
    if (s == MGM_OK) {
        SetupTimer tm;
        s = setup_dense_bottom(ctx);
        tm.mark("dense bottom B_J", ctx->denseJ);
    }
    ctx->setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (s != MGM_OK) {
        g_setup_error = ctx->err;
        g_setup_index = ctx->err_index;
        ctx->lv.clear();
        *out = ctx;
        return s;
    }
    *out = ctx;
    return MGM_OK;
}

// batch width used for K right-hand sides: 2, 4 or 8 (extra columns are zero)
static int batch_width(int K) { return K <= 2 ? 2 : K <= 4 ? 4 : 8; }
static mgm_status batch_check(mgm_ctx* ctx, int K) {
    mgm_status s = check_ctx(ctx);
    if (s) return s;
    if (K < 1 || K > 8 || ctx->poisson || !ctx->ainv || dist_on(ctx)) {
        ctx->err = "batched solves: 1 <= K <= 8, shifted problem, coarsest level <= 4096 rows, one GPU";
        return MGM_ERR_ARG;
    }
    if ((s = ensure_krylov(ctx))) return s;
    return ensure_batch(ctx, batch_width(K));
}

mgm_status mgm_vcycle_batch(mgm_ctx* ctx, int K, const double* f_dev, double* u_dev, void* cuda_stream) {
    AllocScope as_(ctx);
    if (K == 1) return mgm_vcycle(ctx, f_dev, u_dev, cuda_stream);
    mgm_status s = batch_check(ctx, K);
    if (s) return s;
    if (!f_dev || !u_dev) return MGM_ERR_ARG;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const i64 N = ctx->N;
    const int KK = batch_width(K);
    k_gather_b<<<blocks_for(N * KK, 256), 256, 0, st>>>((int)N, K, KK, ctx->d_lib2orig, f_dev, ctx->bf[0]);
    k_gather_b<<<blocks_for(N * KK, 256), 256, 0, st>>>((int)N, K, KK, ctx->d_lib2orig, u_dev, ctx->bu[0]);
    if ((s = run_vcycle_b(ctx, KK, st))) return s;
    k_scatter_b<<<blocks_for(N * KK, 256), 256, 0, st>>>((int)N, K, KK, ctx->d_lib2orig, ctx->bu[0], u_dev);
    CK(cudaGetLastError());
    return MGM_OK;
}

}  // extern "C"

// K independent right-preconditioned GMRES(restart) processes (CGS2, as gmres_lib) sharing
// every operator pass: one batched V-cycle (from zero) and one batched SpMV per Arnoldi step
// for all K columns; Givens rotations per column on the host.  A column that met tol (or
// broke down) is frozen: its further basis vectors are zero and its update uses the steps it
// took, so each column follows its own single-RHS iteration.  bf[0] holds b, x -> bx.
template <int K>
static mgm_status gmres_batch(mgm_ctx* ctx, int Kreal, double tol, int maxit, mgm_report* reports, cudaStream_t st) {
    const i64 N = ctx->N;
    const int m = ctx->restart;
    const Level& L0 = ctx->lv[0];
    if (ctx->bgK < K) {
        for (double** q : {&ctx->bV, &ctx->bw, &ctx->bx, &ctx->bb, &ctx->bdh, &ctx->bpart, &ctx->bZ})
            if (*q) { dev_free(*q); *q = nullptr; }
        if (ctx->bhh) { cudaFreeHost(ctx->bhh); ctx->bhh = nullptr; }
        CK(dalloc(&ctx->bV, (i64)(m + 1) * N * K));
        if (gmres_keep_z()) CK(dalloc(&ctx->bZ, (i64)m * N * K));
        CK(dalloc(&ctx->bpart, (i64)RED_BLOCKS * (m + 1) * K));
        CK(dalloc(&ctx->bw, N * K));
        CK(dalloc(&ctx->bx, N * K));
        CK(dalloc(&ctx->bb, N * K));
        CK(dalloc(&ctx->bdh, (i64)(2 * (m + 1) + 4) * K));
        CK(cudaMallocHost((void**)&ctx->bhh, sizeof(double) * (3 * (m + 1) + 4) * K));
        ctx->bgK = K;
    }
    const i64 nk = N * K;
    const unsigned nb = blocks_for(nk, 256);
    double *V = ctx->bV, *w = ctx->bw, *x = ctx->bx, *b = ctx->bb;
    double *h1 = ctx->bdh, *h2 = ctx->bdh + (i64)(m + 1) * K, *nr = ctx->bdh + (i64)2 * (m + 1) * K;
    double* coef = nr + K;  // (K scale factors; reused for the y coefficients below: m * K)
    double* hh = ctx->bhh;
    mgm_status s;
    CK(cudaMemcpyAsync(b, ctx->bf[0], sizeof(double) * nk, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(x, 0, sizeof(double) * nk, st));
    enqueue_bdot(ctx, K, N, b, b, nr, st);
    CK(cudaMemcpyAsync(hh, nr, sizeof(double) * K, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<double> bnorm(K), H((size_t)K * (m + 1) * m), cs((size_t)K * m), sn((size_t)K * m),
        g((size_t)K * (m + 1)), y((size_t)m * K), sc(K), rel(K, 0.0);
    std::vector<int> its(K, 0), kdone(K, 0), hist(K, 0);
    std::vector<char> conv(K, 0), active(K, 0);
    for (int c = 0; c < K; ++c) {
        bnorm[c] = std::sqrt(hh[c]);
        if (c >= Kreal || bnorm[c] == 0.0) conv[c] = 1;  // (padding columns are zero)
    }
    auto Hc = [&](int c, int i, int k) -> double& { return H[((size_t)c * (m + 1) + i) * m + k]; };
    // pinned mirror: h1 | h2 | norms (read back), then two upload areas: y (m K) and K scalars
    // (each area is rewritten only after a stream synchronisation or in the other area)
    double* up_y = hh + (size_t)(2 * (m + 1) + 1) * K;
    double* up_k = up_y + (size_t)(m + 1) * K;
    auto upload_coef = [&](const std::vector<double>& v, double* dst) -> mgm_status {
        double* src = v.size() > (size_t)K ? up_y : up_k;
        std::copy(v.begin(), v.end(), src);
        CK(cudaMemcpyAsync(dst, src, sizeof(double) * v.size(), cudaMemcpyHostToDevice, st));
        return MGM_OK;
    };
    bool first = true;
    int cycles_its = 0;  // Arnoldi steps taken (shared by all columns)
    while (true) {
        // r = b - A x ; beta per column
        if (first)
            CK(cudaMemcpyAsync(w, b, sizeof(double) * nk, cudaMemcpyDeviceToDevice, st));
        else
            b_spmv<1, K>(L0.stpr, N, L0.sptr, L0.scol, L0.sval, x, b, w, st);
        first = false;
        enqueue_bdot(ctx, K, N, w, w, nr, st);
        CK(cudaMemcpyAsync(hh, nr, sizeof(double) * K, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        bool any = false;
        for (int c = 0; c < K; ++c) {
            const double beta = std::sqrt(hh[c]);
            active[c] = !conv[c] && its[c] < maxit && !(beta / bnorm[c] <= tol);
            if (!conv[c] && beta / bnorm[c] <= tol) conv[c] = 1;
            sc[c] = active[c] ? 1.0 / beta : 0.0;
            std::fill(g.begin() + (size_t)c * (m + 1), g.begin() + (size_t)(c + 1) * (m + 1), 0.0);
            g[(size_t)c * (m + 1)] = beta;
            kdone[c] = 0;
            any = any || active[c];
        }
        if (!any) break;
        std::fill(H.begin(), H.end(), 0.0);
        if ((s = upload_coef(sc, coef))) return s;
        launch(false, k_bscale<K>, nb, 256, 0, st, N, (const double*)w, (const double*)coef, V);
        for (int k = 0; k < m; ++k) {
            // z = M^{-1} v_k (batched V-cycle from zero), w = A z
            CK(cudaMemcpyAsync(ctx->bf[0], V + (i64)k * nk, sizeof(double) * nk, cudaMemcpyDeviceToDevice, st));
            if ((s = run_vcycle_b(ctx, K, st, true))) return s;
            if (ctx->bZ)
                CK(cudaMemcpyAsync(ctx->bZ + (i64)k * nk, ctx->bu[0], sizeof(double) * nk, cudaMemcpyDeviceToDevice, st));
            if (ctx->bgraph_zg_dlt[K])  // A z = v_k + (later-colour part of L_1) d (MODE 3)
                b_spmv<3, K>(L0.stpr, N, L0.sptr, L0.scol, L0.sval, ctx->bdlt, ctx->bf[0], w, st, L0.sluw, L0.nlow);
            else
                b_spmv<0, K>(L0.stpr, N, L0.sptr, L0.scol, L0.sval, ctx->bu[0], nullptr, w, st);
            ++cycles_its;
            const int k1 = k + 1;
            // CGS2 per column: h1 = V^T w; w -= V h1; h2 = V^T w; w -= V h2; h = h1 + h2
            enqueue_bmultidot(ctx, K, N, V, nk, k1, w, h1, st);
            launch(false, k_blincomb<K>, nb, 256, 0, st, N, k1, (const double*)V, nk, (const double*)h1, -1.0, 1, w);
            enqueue_bmultidot(ctx, K, N, V, nk, k1, w, h2, st);
            launch(false, k_blincomb<K>, nb, 256, 0, st, N, k1, (const double*)V, nk, (const double*)h2, -1.0, 1, w);
            enqueue_bdot(ctx, K, N, w, w, nr, st);
            CK(cudaMemcpyAsync(hh, h1, sizeof(double) * k1 * K, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(hh + (m + 1) * K, h2, sizeof(double) * k1 * K, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(hh + 2 * (m + 1) * K, nr, sizeof(double) * K, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            bool still = false;
            for (int c = 0; c < K; ++c) {
                if (!active[c]) {
                    sc[c] = 0.0;
                    continue;
                }
                for (int i = 0; i < k1; ++i) Hc(c, i, k) = hh[(size_t)i * K + c] + hh[(size_t)(m + 1) * K + (size_t)i * K + c];
                const double hk1 = std::sqrt(hh[(size_t)2 * (m + 1) * K + c]);
                Hc(c, k1, k) = hk1;
                double* csc = cs.data() + (size_t)c * m;
                double* snc = sn.data() + (size_t)c * m;
                double* gc = g.data() + (size_t)c * (m + 1);
                for (int i = 0; i < k; ++i) {
                    const double t = csc[i] * Hc(c, i, k) + snc[i] * Hc(c, i + 1, k);
                    Hc(c, i + 1, k) = -snc[i] * Hc(c, i, k) + csc[i] * Hc(c, i + 1, k);
                    Hc(c, i, k) = t;
                }
                const double den = std::hypot(Hc(c, k, k), hk1);
                csc[k] = Hc(c, k, k) / den;
                snc[k] = hk1 / den;
                Hc(c, k, k) = den;
                Hc(c, k1, k) = 0.0;
                gc[k1] = -snc[k] * gc[k];
                gc[k] = csc[k] * gc[k];
                rel[c] = std::fabs(gc[k1]) / bnorm[c];
                ++its[c];
                kdone[c] = k1;
                if (reports && reports[c].history && hist[c] < reports[c].history_cap) reports[c].history[hist[c]++] = rel[c];
                if (!std::isfinite(rel[c])) return fail(ctx, MGM_ERR_BREAKDOWN, "non-finite GMRES residual", c);
                if (rel[c] <= tol || its[c] >= maxit || hk1 == 0.0) {
                    active[c] = 0;  // frozen: further basis vectors of this column are zero
                    if (rel[c] <= tol) conv[c] = 1;
                    sc[c] = 0.0;
                } else {
                    sc[c] = 1.0 / hk1;
                    still = true;
                }
            }
            if (!still || k1 == m) break;
            if ((s = upload_coef(sc, coef))) return s;
            launch(false, k_bscale<K>, nb, 256, 0, st, N, (const double*)w, (const double*)coef, V + (i64)k1 * nk);
        }
        // x += M^{-1} V y per column (y = 0 beyond the column's own steps)
        int kmax = 0;
        std::fill(y.begin(), y.end(), 0.0);
        for (int c = 0; c < K; ++c) {
            const int kd = kdone[c];
            kmax = std::max(kmax, kd);
            std::vector<double> yc(kd);
            for (int i = kd - 1; i >= 0; --i) {
                double sacc = g[(size_t)c * (m + 1) + i];
                for (int j2 = i + 1; j2 < kd; ++j2) sacc -= Hc(c, i, j2) * yc[j2];
                yc[i] = sacc / Hc(c, i, i);
            }
            for (int i = 0; i < kd; ++i) y[(size_t)i * K + c] = yc[i];
        }
        if (kmax > 0) {
            std::vector<double> yv(y.begin(), y.begin() + (size_t)kmax * K);
            if ((s = upload_coef(yv, h1))) return s;
            if (ctx->bZ) {  // x += Z y (z_j = M v_j kept per step)
                launch(false, k_blincomb<K>, nb, 256, 0, st, N, kmax, (const double*)ctx->bZ, nk, (const double*)h1,
                       1.0, 1, x);
            } else {
                launch(false, k_blincomb<K>, nb, 256, 0, st, N, kmax, (const double*)V, nk, (const double*)h1, 1.0, 0,
                       ctx->bf[0]);
                if ((s = run_vcycle_b(ctx, K, st, true))) return s;
                std::vector<double> one(K, 1.0);
                if ((s = upload_coef(one, coef))) return s;
                launch(false, k_blincomb<K>, nb, 256, 0, st, N, 1, (const double*)ctx->bu[0], nk, (const double*)coef,
                       1.0, 1, x);
            }
        }
        bool left = false;
        for (int c = 0; c < K; ++c) left = left || (!conv[c] && its[c] < maxit);
        if (!left) break;
    }
    // true residuals
    b_spmv<1, K>(L0.stpr, N, L0.sptr, L0.scol, L0.sval, x, b, w, st);
    enqueue_bdot(ctx, K, N, w, w, nr, st);
    CK(cudaMemcpyAsync(hh, nr, sizeof(double) * K, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (reports)
        for (int c = 0; c < Kreal; ++c) {
            reports[c].iterations = its[c];
            reports[c].converged = conv[c];
            reports[c].final_rel_residual = bnorm[c] > 0.0 ? std::sqrt(hh[c]) / bnorm[c] : 0.0;
            reports[c].lambda = 0.0;
        }
    (void)cycles_its;
    return MGM_OK;
}

extern "C" {

mgm_status mgm_solve_batch(mgm_ctx* ctx, int K, const double* rhs_dev, double* x_dev, double tol, int maxit,
                           int krylov, mgm_report* reports, void* cuda_stream) {
    AllocScope as_(ctx);
    if (krylov != 0 && krylov != 1) return MGM_ERR_ARG;
    if (K == 1) return mgm_solve(ctx, rhs_dev, nullptr, x_dev, tol, maxit, krylov, reports, cuda_stream);
    mgm_status s = batch_check(ctx, K);
    if (s) return s;
    if (!rhs_dev || !x_dev || !(tol >= 0) || maxit < 0) return MGM_ERR_ARG;
    if (krylov == 1) {
        cudaStream_t st = (cudaStream_t)cuda_stream;
        const i64 N = ctx->N;
        const int KK = batch_width(K);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, st);
        k_gather_b<<<blocks_for(N * KK, 256), 256, 0, st>>>((int)N, K, KK, ctx->d_lib2orig, rhs_dev, ctx->bf[0]);
        s = KK == 2 ? gmres_batch<2>(ctx, K, tol, maxit, reports, st)
          : KK == 4 ? gmres_batch<4>(ctx, K, tol, maxit, reports, st)
                    : gmres_batch<8>(ctx, K, tol, maxit, reports, st);
        if (s) return s;
        k_scatter_b<<<blocks_for(N * KK, 256), 256, 0, st>>>((int)N, K, KK, ctx->d_lib2orig, ctx->bx, x_dev);
        cudaEventRecord(e1, st);
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (reports)
            for (int k = 0; k < K; ++k) {
                reports[k].solve_ms = ms;
                reports[k].setup_ms = ctx->setup_ms;
            }
        CK(cudaGetLastError());
        return MGM_OK;
    }
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const i64 N = ctx->N;
    const int KK = batch_width(K);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    k_gather_b<<<blocks_for(N * KK, 256), 256, 0, st>>>((int)N, K, KK, ctx->d_lib2orig, rhs_dev, ctx->bf[0]);
    CK(cudaMemsetAsync(ctx->bu[0], 0, sizeof(double) * N * KK, st));
    double* dd = ctx->dh + 512;
    enqueue_bdot(ctx, KK, N, ctx->bf[0], ctx->bf[0], dd, st);
    CK(cudaMemcpyAsync(ctx->hh, dd, sizeof(double) * KK, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::vector<double> fn(KK), rel(KK, 1.0);
    std::vector<int> its(KK, 0), hist(KK, 0);
    std::vector<char> conv(KK, 0);
    for (int k = 0; k < KK; ++k) {
        fn[k] = std::sqrt(ctx->hh[k]);
        if (fn[k] == 0.0) { conv[k] = 1; rel[k] = 0.0; }
    }
    int it = 0;
    auto all = [&]() {
        for (int k = 0; k < K; ++k)
            if (!conv[k]) return false;
        return true;
    };
    while (it < maxit && !all()) {
        if ((s = run_vcycle_b(ctx, KK, st))) return s;
        ++it;
        enqueue_res_b(ctx, KK, st);
        enqueue_bdot(ctx, KK, N, ctx->bres, ctx->bres, dd, st);
        CK(cudaMemcpyAsync(ctx->hh, dd, sizeof(double) * KK, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int k = 0; k < K; ++k) {
            if (fn[k] == 0.0) continue;
            rel[k] = std::sqrt(ctx->hh[k]) / fn[k];
            if (reports && reports[k].history && hist[k] < reports[k].history_cap) reports[k].history[hist[k]++] = rel[k];
            if (!conv[k]) {
                its[k] = it;
                if (rel[k] <= tol) conv[k] = 1;
            }
        }
    }
    k_scatter_b<<<blocks_for(N * KK, 256), 256, 0, st>>>((int)N, K, KK, ctx->d_lib2orig, ctx->bu[0], x_dev);
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (reports)
        for (int k = 0; k < K; ++k) {
            reports[k].iterations = its[k];
            reports[k].converged = conv[k];
            reports[k].final_rel_residual = rel[k];
            reports[k].lambda = 0.0;
            reports[k].solve_ms = ms;
            reports[k].setup_ms = ctx->setup_ms;
        }
    CK(cudaGetLastError());
    return MGM_OK;
}

mgm_status mgm_nccl_unique_id(void* id128) {
    if (!id128) return MGM_ERR_ARG;
    if (!nccl().ok) return MGM_ERR_NCCL;
    ncclUniqueId id;
    if (nccl().GetUniqueId(&id) != ncclSuccess) return MGM_ERR_NCCL;
    std::memcpy(id128, &id, sizeof(id));
    return MGM_OK;
}

mgm_status mgm_dist_attach(mgm_ctx* ctx, int rank, int nranks, const void* id128) {
    AllocScope as_(ctx);
    if (!ctx || ctx->lv.empty() || nranks < 1 || rank < 0 || rank >= nranks || !id128) return MGM_ERR_ARG;
    if (ctx->tp) return MGM_ERR_ARG;
    if (!nccl().ok) {
        ctx->err = "libnccl.so.2 not found";
        return MGM_ERR_NCCL;
    }
    cudaSetDevice(ctx->device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    const ncclResult_t r = nccl().CommInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) {
        ctx->err = std::string("ncclCommInitRank: ") + nccl().GetErrorString(r);
        return MGM_ERR_NCCL;
    }
    auto* t = new NcclTransport();
    t->comm = comm;
    t->rank = rank;
    t->nranks = nranks;
    ctx->tp = t;
    ctx->rank = rank;
    ctx->nranks = nranks;
    mgm_status s = dist_partition(ctx);
    if (s == MGM_OK && std::getenv("MGM_P2P") && std::atoi(std::getenv("MGM_P2P")) == 1) s = p2p_setup(ctx);
    return s;
}

mgm_status mgm_fake_group_create(int nranks, void** group) {
    if (nranks < 1 || !group) return MGM_ERR_ARG;
    *group = new FakeGroup(nranks);
    return MGM_OK;
}

mgm_status mgm_fake_group_destroy(void* group) {
    delete static_cast<FakeGroup*>(group);
    return MGM_OK;
}

mgm_status mgm_dist_attach_fake(mgm_ctx* ctx, int rank, void* group) {
    AllocScope as_(ctx);
    auto* g = static_cast<FakeGroup*>(group);
    if (!ctx || ctx->lv.empty() || !g || rank < 0 || rank >= g->R || ctx->tp) return MGM_ERR_ARG;
    cudaSetDevice(ctx->device);
    auto* t = new FakeTransport();
    t->g = g;
    t->rank = rank;
    t->nranks = g->R;
    ctx->tp = t;
    ctx->rank = rank;
    ctx->nranks = g->R;
    mgm_status s = dist_partition(ctx);
    if (s == MGM_OK && std::getenv("MGM_P2P") && std::atoi(std::getenv("MGM_P2P")) == 1) s = p2p_setup(ctx);
    return s;
}

mgm_status mgm_dist_comm_time(mgm_ctx* ctx, int reps, double* halo_ms_per_vcycle, double* allreduce_us,
                              void* cuda_stream) {
    AllocScope as_(ctx);
    mgm_status s = check_ctx(ctx);
    if (s) return s;
    if (!ctx->tp || reps < 1) return MGM_ERR_ARG;
    if ((s = ensure_krylov(ctx))) return s;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    auto schedule = [&]() {  // the halos and the all-gather of one V-cycle, in order, no compute
        for (int j = 0; j < ctx->D; ++j) {
            Level& L = ctx->lv[j];
            for (int s2 = 0; s2 < ctx->lp.nu1; ++s2)
                for (int c = 0; c < L.ncol; ++c) exch(ctx, j, L.u, c, st);
            exch(ctx, j, L.t, -1, st);
            if (L.d_stage_all) ctx->tp->allgatherv(L.d_stage_mine, L.d_stage_all, L.stage_off, st);
        }
        for (int j = ctx->D - 1; j >= 0; --j) {
            Level& L = ctx->lv[j];
            exch(ctx, j, L.u, -1, st);
            for (int s2 = 0; s2 < ctx->lp.nu2; ++s2)
                for (int c = 0; c < L.ncol; ++c) exch(ctx, j, L.u, c, st);
        }
    };
    schedule();  // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) schedule();
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (halo_ms_per_vcycle) *halo_ms_per_vcycle = ms / reps;
    double* buf = ctx->dh + 700;
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) ctx->tp->allreduce_sum(buf, 16, st);
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    if (allreduce_us) *allreduce_us = 1e3 * ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return MGM_OK;
}

mgm_status mgm_local_rows(const mgm_ctx* ctx, int64_t* n_local, int64_t* original_ids) {
    if (!ctx || ctx->lv.empty()) return MGM_ERR_ARG;
    const i64 n = ctx->tp ? (i64)ctx->local_ids.size() : ctx->N;
    if (n_local) *n_local = n;
    if (original_ids)
        for (i64 k = 0; k < n; ++k) original_ids[k] = ctx->tp ? ctx->local_ids[(size_t)k] : k;
    return MGM_OK;
}

mgm_status mgm_dist_info(const mgm_ctx* ctx, int* dist_levels, int64_t* ghosts, int64_t* halo_values_per_vcycle) {
    if (!ctx || ctx->lv.empty()) return MGM_ERR_ARG;
    if (dist_levels) *dist_levels = ctx->tp ? ctx->D : 0;
    i64 g = 0, hv = 0;
    for (int j = 0; j < (ctx->tp ? ctx->D : 0); ++j) {
        const Level& L = ctx->lv[j];
        g += L.nghost;
        // received values per V-cycle: every colour of nu1 + nu2 sweeps once, plus the full
        // halos after interpolation and before the restriction
        hv += (i64)(ctx->lp.nu1 + ctx->lp.nu2) * L.nghost + 2 * L.nghost;
    }
    if (ghosts) *ghosts = g;
    if (halo_values_per_vcycle) *halo_values_per_vcycle = hv;
    return MGM_OK;
}

mgm_status mgm_destroy(mgm_ctx* ctx) {
    AllocScope as_(ctx);
    if (!ctx) return MGM_OK;
    cudaSetDevice(ctx->device);
    if (ctx->st) cudaStreamSynchronize(ctx->st);
    for (auto& L : ctx->lv) free_level_device(L);
    for (void* ptr : {(void*)ctx->lu, (void*)ctx->piv, (void*)ctx->d_lib2orig, (void*)ctx->V, (void*)ctx->w,
                      (void*)ctx->xs, (void*)ctx->b, (void*)ctx->partials, (void*)ctx->dh, (void*)ctx->tickets})
        if (ptr) dev_free(ptr);
    if (ctx->hh) cudaFreeHost(ctx->hh);
    if (ctx->ggraph) cudaGraphExecDestroy(ctx->ggraph);
    if (ctx->g_i) dev_free(ctx->g_i);
    if (ctx->g_d) dev_free(ctx->g_d);
    if (ctx->g_h) cudaFreeHost(ctx->g_h);
    if (ctx->g_hi) cudaFreeHost(ctx->g_hi);
    for (void* q : ctx->bot_mem) dev_free(q);
    if (ctx->d_trace) dev_free(ctx->d_trace);
    if (ctx->vgraph) cudaGraphExecDestroy(ctx->vgraph);
    if (ctx->vgraph0) cudaGraphExecDestroy(ctx->vgraph0);
    for (void* ptr : ctx->ipc_opened) cudaIpcCloseMemHandle(ptr);
    for (void* ptr : {(void*)ctx->p2p_flags, (void*)ctx->p2p_sent, (void*)ctx->p2p_expect, (void*)ctx->p2p_ticket})
        if (ptr) dev_free(ptr);
    delete ctx->tp;
    ctx->tp = nullptr;
    for (auto* q : {&ctx->bu, &ctx->bf, &ctx->bt})
        for (double* ptr : *q) dev_free(ptr);
    for (auto& gx : ctx->bgraph)
        if (gx) cudaGraphExecDestroy(gx);
    for (auto& gx : ctx->bgraph_zg)
        if (gx) cudaGraphExecDestroy(gx);
    if (ctx->bres) dev_free(ctx->bres);
    for (double* ptr : {ctx->bV, ctx->bw, ctx->bx, ctx->bb, ctx->bdh})
        if (ptr) dev_free(ptr);
    if (ctx->bhh) cudaFreeHost(ctx->bhh);
    if (ctx->ainv) dev_free(ctx->ainv);
    if (ctx->dB) dev_free(ctx->dB);
    if (ctx->d_dlt) dev_free(ctx->d_dlt);
    if (ctx->Z) dev_free(ctx->Z);
    if (ctx->bZ) dev_free(ctx->bZ);
    if (ctx->bpart) dev_free(ctx->bpart);
    if (ctx->bdlt) dev_free(ctx->bdlt);
    if (ctx->d_dlt_pre) dev_free(ctx->d_dlt_pre);
    if (ctx->dP) dev_free(ctx->dP);
    for (auto& T : ctx->timer)
        for (auto e : T.ev) cudaEventDestroy(e);
    if (ctx->st) cudaStreamDestroy(ctx->st);
    delete ctx;
    return MGM_OK;
}

const char* mgm_last_error(const mgm_ctx* ctx, int64_t* failing_index) {
    if (!ctx) {
        if (failing_index) *failing_index = g_setup_index;
        return g_setup_error.c_str();
    }
    if (failing_index) *failing_index = ctx->err_index;
    return ctx->err.c_str();
}

mgm_status mgm_vcycle(mgm_ctx* ctx, const double* f_dev, double* u_dev, void* cuda_stream) {
    AllocScope as_(ctx);
    mgm_status s = check_ctx(ctx);
    if (s) return s;
    if (!f_dev || !u_dev) return MGM_ERR_ARG;
    if ((s = ensure_krylov(ctx))) return s;
    cudaStream_t st = (cudaStream_t)cuda_stream;
    const i64 N = ctx->lv[0].n;  // (multi-GPU: this rank's rows, mgm_local_rows order)
    Level& L0 = ctx->lv[0];
    k_gather<<<blocks_for(N, 256), 256, 0, st>>>((int)N, ctx->d_lib2orig, f_dev, L0.f);
    k_gather<<<blocks_for(N, 256), 256, 0, st>>>((int)N, ctx->d_lib2orig, u_dev, L0.u);
    if (ctx->poisson) {
        CK(cudaMemsetAsync(L0.f + N, 0, sizeof(double), st));
        CK(cudaMemsetAsync(L0.u + N, 0, sizeof(double), st));
    }
    exch(ctx, 0, L0.u, -1, st);  // (distributed: the presmooth reads the guess's ghosts)
    if ((s = run_vcycle(ctx, st))) return s;
    k_scatter<<<blocks_for(N, 256), 256, 0, st>>>((int)N, ctx->d_lib2orig, L0.u, u_dev);
    CK(cudaGetLastError());
    if (timing_on(ctx)) {
        CK(cudaStreamSynchronize(st));
        timer_collect(ctx);
    }
    return MGM_OK;
}

static mgm_status solve_impl(mgm_ctx* ctx, const double* rhs, const double* x0, double* x, bool host, double tol,
                             int maxit, int krylov, mgm_report* rep, cudaStream_t st) {
    AllocScope as_(ctx);
    mgm_status s = check_ctx(ctx);
    if (s) return s;
    if (!rhs || !x || !(tol >= 0) || maxit < 0 || krylov < 0 || krylov > 2) return MGM_ERR_ARG;
    if ((s = ensure_krylov(ctx))) return s;
    const i64 N = ctx->lv[0].n;  // (multi-GPU: this rank's rows, mgm_local_rows order)
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    const double* rhs_dev = rhs;
    if (host) {
        CK(cudaMemcpyAsync(ctx->w, rhs, sizeof(double) * N, cudaMemcpyHostToDevice, st));
        rhs_dev = ctx->w;
    }
    k_gather<<<blocks_for(N, 256), 256, 0, st>>>((int)N, ctx->d_lib2orig, rhs_dev, ctx->b);
    if (ctx->poisson) CK(cudaMemsetAsync(ctx->b + N, 0, sizeof(double), st));
    ctx->warm = x0 != nullptr;
    struct ResetW { mgm_ctx* c; ~ResetW() { c->warm = false; } } resetw_{ctx};
    if (x0) {  // x0 -> lib order (xs); Poisson: the multiplier starts at 0
        const double* x0_dev = x0;
        if (host) {  // (x0 may alias x; rhs already sits in w, so x0 goes through lv[0].t)
            CK(cudaMemcpyAsync(ctx->lv[0].t, x0, sizeof(double) * N, cudaMemcpyHostToDevice, st));
            x0_dev = ctx->lv[0].t;
        }
        k_gather<<<blocks_for(N, 256), 256, 0, st>>>((int)N, ctx->d_lib2orig, x0_dev, ctx->xs);
        if (ctx->poisson) CK(cudaMemsetAsync(ctx->xs + N, 0, sizeof(double), st));
    }
    s = krylov == 1 ? (gmres_dev_ok(ctx) ? gmres_dev(ctx, tol, maxit, rep, st) : gmres_lib(ctx, tol, maxit, rep, st))
        : krylov == 2 ? bicgstab_lib(ctx, tol, maxit, rep, st)
                      : standalone_lib(ctx, tol, maxit, rep, st);
    if (s) return s;
    if (host) {
        k_scatter<<<blocks_for(N, 256), 256, 0, st>>>((int)N, ctx->d_lib2orig, ctx->xs, ctx->w);
        CK(cudaMemcpyAsync(x, ctx->w, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
    } else {
        k_scatter<<<blocks_for(N, 256), 256, 0, st>>>((int)N, ctx->d_lib2orig, ctx->xs, x);
    }
    cudaEventRecord(e1, st);
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rep) {
        rep->solve_ms = ms;
        rep->setup_ms = ctx->setup_ms;
    }
    CK(cudaGetLastError());
    return MGM_OK;
}

mgm_status mgm_solve(mgm_ctx* ctx, const double* rhs_dev, const double* x0_dev, double* x_dev, double tol,
                     int maxit, int krylov, mgm_report* report, void* cuda_stream) {
    return solve_impl(ctx, rhs_dev, x0_dev, x_dev, false, tol, maxit, krylov, report, (cudaStream_t)cuda_stream);
}

mgm_status mgm_solve_host(mgm_ctx* ctx, const double* rhs_host, const double* x0_host, double* x_host, double tol,
                          int maxit, int krylov, mgm_report* report, void* cuda_stream) {
    return solve_impl(ctx, rhs_host, x0_host, x_host, true, tol, maxit, krylov, report, (cudaStream_t)cuda_stream);
}

mgm_status mgm_num_levels(const mgm_ctx* ctx, int* p) {
    if (!ctx || ctx->lv.empty() || !p) return MGM_ERR_ARG;
    *p = ctx->p;
    return MGM_OK;
}

mgm_status mgm_level_info(const mgm_ctx* ctx, int level, int64_t* n_rows, int64_t* nnz_L, int64_t* nnz_P,
                          int* n_colours, int64_t* stored_bytes) {
    if (!ctx || ctx->lv.empty() || level < 0 || level >= ctx->p) return MGM_ERR_ARG;
    const Level& L = ctx->lv[level];
    if (n_rows) *n_rows = L.n;
    if (nnz_L) *nnz_L = L.nnz;
    if (nnz_P) *nnz_P = L.p_nnz;
    if (n_colours) *n_colours = L.ncol;
    if (stored_bytes)
        *stored_bytes = 12 * L.sell_stored + 8 * ((L.n + 31) / 32 + 1) + 12 * (i64)L.pm * L.n + 12 * L.r_stored +
                        24 * L.n;
    return MGM_OK;
}

mgm_status mgm_export_level(const mgm_ctx* ctx, int level, int64_t* ids, int64_t* L_ptr, int32_t* L_col,
                            double* L_val, int32_t* colour, int64_t* P_ptr, int32_t* P_col, double* P_val,
                            double* border) {
    if (!ctx || ctx->lv.empty() || level < 0 || level >= ctx->p) return MGM_ERR_ARG;
    const Level& L = ctx->lv[level];
    if (ids) std::copy(L.ids.begin(), L.ids.end(), ids);
    if (L_ptr) std::copy(L.L_lib.ptr.begin(), L.L_lib.ptr.end(), L_ptr);
    if (L_col) std::copy(L.L_lib.col.begin(), L.L_lib.col.end(), L_col);
    if (L_val) std::copy(L.L_lib.val.begin(), L.L_lib.val.end(), L_val);
    if (colour) std::copy(L.colour_lib.begin(), L.colour_lib.end(), colour);
    if (level + 1 < ctx->p) {
        if (P_ptr) std::copy(L.P_lib.ptr.begin(), L.P_lib.ptr.end(), P_ptr);
        if (P_col) std::copy(L.P_lib.col.begin(), L.P_lib.col.end(), P_col);
        if (P_val) std::copy(L.P_lib.val.begin(), L.P_lib.val.end(), P_val);
    }
    if (border) {
        if (!ctx->poisson) return MGM_ERR_ARG;
        std::copy(L.c_lib.begin(), L.c_lib.end(), border);
    }
    return MGM_OK;
}

mgm_status mgm_export_weights(const mgm_ctx* ctx, double* w, int64_t* sten) {
    if (!ctx || ctx->lv.empty()) return MGM_ERR_ARG;
    const i64 N = (i64)ctx->perm0.size(), ns = ctx->ns0;
    const std::vector<i64>& perm = ctx->perm0;
    for (i64 k = 0; k < N; ++k)  // Morton row k is original row perm[k]
        for (i64 j = 0; j < ns; ++j) {
            if (w) w[perm[k] * ns + j] = ctx->w_mor[k * ns + j];
            if (sten) sten[perm[k] * ns + j] = perm[ctx->sten_mor[k * ns + j]];
        }
    return MGM_OK;
}

mgm_status mgm_apply(mgm_ctx* ctx, int level, int op, const double* x, const double* f, double* y,
                     void* cuda_stream) {
    AllocScope as_(ctx);
    mgm_status s = check_ctx(ctx);
    if (s) return s;
    if (level < 0 || level >= ctx->p || !x || !y) return MGM_ERR_ARG;
    if (dist_on(ctx)) {
        ctx->err = "mgm_apply: test hook of the undistributed hierarchy";
        return MGM_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)cuda_stream;
    Level& L = ctx->lv[level];
    const i64 pad = ctx->poisson ? 1 : 0;
    const i64 vn = L.n + pad;
    if ((s = ensure_krylov(ctx))) return s;
    switch (op) {
        case MGM_OP_SPMV:
            enqueue_spmv(ctx, level, x, y, st);
            break;
        case MGM_OP_SWEEP:
            if (!f || level == ctx->p - 1) return MGM_ERR_ARG;
            CK(cudaMemcpyAsync(L.u, x, sizeof(double) * vn, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(L.f, f, sizeof(double) * vn, cudaMemcpyDeviceToDevice, st));
            enqueue_sweep(ctx, level, false, st);
            CK(cudaMemcpyAsync(y, L.u, sizeof(double) * vn, cudaMemcpyDeviceToDevice, st));
            break;
        case MGM_OP_RESIDUAL:
            if (!f) return MGM_ERR_ARG;
            enqueue_residual(ctx, level, f, x, y, st);
            break;
        case MGM_OP_RESTRICT:
            if (level == ctx->p - 1) return MGM_ERR_ARG;
            enqueue_restrict(ctx, level, const_cast<double*>(x), y, st);  // (undistributed: x is only read)
            break;
        case MGM_OP_INTERP: {
            if (level == ctx->p - 1) return MGM_ERR_ARG;
            const Level& Ln = ctx->lv[level + 1];
            if (ctx->poisson)
                k_interp<true><<<blocks_for(L.n + 1, 256), 256, 0, st>>>((int)L.n, L.pm, L.pcol, L.pval, x, y, (int)Ln.n);
            else
                k_interp<false><<<blocks_for(L.n + 1, 256), 256, 0, st>>>((int)L.n, L.pm, L.pcol, L.pval, x, y, (int)Ln.n);
            break;
        }
        case MGM_OP_COARSE:
            enqueue_coarse(ctx, x, y, st);
            break;
        case MGM_OP_SWEEP_ZG: {  // one forward sweep from the zero guess; u starts as NaN (never read)
            if (!f || level == ctx->p - 1) return MGM_ERR_ARG;
            if (!L.slw || ctx->poisson) return MGM_ERR_ARG;
            k_fill<<<blocks_for(vn, 256), 256, 0, st>>>(vn, L.u, std::nan(""), PfList{nullptr, 0, 0});
            CK(cudaMemcpyAsync(L.f, f, sizeof(double) * vn, cudaMemcpyDeviceToDevice, st));
            enqueue_sweep(ctx, level, false, st, true);
            CK(cudaMemcpyAsync(y, L.u, sizeof(double) * vn, cudaMemcpyDeviceToDevice, st));
            break;
        }
        case MGM_OP_PRECOND: {  // y = M x, the Krylov preconditioner (level ignored, level-0 lib order)
            Level& L0 = ctx->lv[0];
            const i64 n0 = L0.n + pad;
            k_fill<<<blocks_for(n0, 256), 256, 0, st>>>(n0, L0.u, zg_capable(ctx) ? std::nan("") : 0.0,
                                                         PfList{nullptr, 0, 0});
            if ((s = enqueue_precond(ctx, x, st))) return s;
            CK(cudaMemcpyAsync(y, L0.u, sizeof(double) * n0, cudaMemcpyDeviceToDevice, st));
            break;
        }
        default:
            return MGM_ERR_ARG;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return MGM_OK;
}

mgm_status mgm_timing_enable(mgm_ctx* ctx, int cls, int enable) {
    if (!ctx || cls < 0 || cls > 3) return MGM_ERR_ARG;
    KernelTimer& T = ctx->timer[cls];
    T.on = enable != 0;
    T.used = 0;
    T.total_ms = 0.0;
    T.launches = 0;
    T.bytes = 0.0;
    return MGM_OK;
}

mgm_status mgm_timing_read(mgm_ctx* ctx, int cls, double* total_ms, int64_t* launches, double* alg_bytes) {
    if (!ctx || cls < 0 || cls > 3) return MGM_ERR_ARG;
    timer_collect(ctx);
    const KernelTimer& T = ctx->timer[cls];
    if (total_ms) *total_ms = T.total_ms;
    if (launches) *launches = T.launches;
    if (alg_bytes) *alg_bytes = T.bytes;
    return MGM_OK;
}

mgm_status mgm_bytes_model(const mgm_ctx* ctx, double* vcycle_bytes, double* spmv_bytes) {
    if (!ctx || ctx->lv.empty()) return MGM_ERR_ARG;
    const int p = ctx->p;
    const double nu = ctx->lp.nu1 + ctx->lp.nu2;
    const double bp = ctx->poisson ? 8.0 : 0.0;
    double B = 0.0;
    for (int j = 0; j + 1 < p; ++j) {
        const Level& L = ctx->lv[j];
        const double n = (double)L.n, z = (double)L.nnz, q = (double)L.p_nnz, nn = (double)ctx->lv[j + 1].n;
        B += nu * (12.0 * z + 24.0 * n + bp * n);                   // sweeps
        if (j >= 1 && zg_capable(ctx)) {  // the first presmooth from e_j = 0 reads diag + earlier colours only
            double low = 0.0;
            for (i64 v : L.lower_per_colour) low += (double)v;
            B -= (12.0 * z + 24.0 * n) - (12.0 * low + 16.0 * n);
            // and with nu1 = 1 the residual reads only the later-colour entries, no f
            if (ctx->lp.nu1 == 1 && L.n >= ctx->upper_res_min)
                B -= (12.0 * z + 16.0 * n) - (12.0 * (z - low) + 8.0 * n);
        }
        B += 12.0 * z + 16.0 * n + 12.0 * q + 8.0 * nn + 16.0 * n + bp * n;  // residual + restrict (unfused)
        B += 12.0 * q + 8.0 * nn + 16.0 * n;                        // interp + correct
        if (j == 0 && dpre_ok(ctx)) {  // the general V-cycle (mgm_vcycle): the residual from the presmooth's
            double low = 0.0;          // increments d (written: +8 n), later-colour entries only
            for (i64 v : L.lower_per_colour) low += (double)v;
            B -= (12.0 * z + 16.0 * n) - (12.0 * (z - low) + 8.0 * n);
            B += 8.0 * n;
        }
        if (j == 0 && mode3_ok(ctx)) B += 8.0 * n;  // the last postsmooth writes its increments
    }
    const double np = (double)ctx->nc;
    B += 8.0 * np * np + 16.0 * np;
    if (vcycle_bytes) *vcycle_bytes = B;
    if (spmv_bytes) *spmv_bytes = 12.0 * ctx->lv[0].nnz + 16.0 * ctx->lv[0].n;
    return MGM_OK;
}

mgm_status mgm_dense_bottom_info(const mgm_ctx* ctx, int* level, int64_t* rows, int64_t* bytes) {
    if (!ctx || ctx->lv.empty()) return MGM_ERR_ARG;
    if (level) *level = ctx->denseJ;
    if (rows) *rows = ctx->denseJ >= 0 ? ctx->dense_m : 0;
    if (bytes) *bytes = ctx->denseJ >= 0 ? (int64_t)8 * ctx->dense_m * ctx->dense_ld : 0;
    return MGM_OK;
}

mgm_status mgm_level_zg_nnz(const mgm_ctx* ctx, int level, int64_t* nnz_zg) {
    if (!ctx || level < 0 || level >= ctx->p || !nnz_zg) return MGM_ERR_ARG;
    i64 s = 0;
    for (i64 v : ctx->lv[level].lower_per_colour) s += v;
    *nnz_zg = zg_capable(ctx) ? s : ctx->lv[level].nnz;
    return MGM_OK;
}

mgm_status mgm_trace_read(const mgm_ctx* ctx, uint64_t* stamps_ns, int cap, int* n, char* labels, int label_cap) {
    if (!ctx || !n) return MGM_ERR_ARG;
    *n = ctx->d_trace ? ctx->ntrace : 0;
    if (*n == 0) return MGM_OK;
    if (cap < *n) return MGM_ERR_ARG;
    if (cudaMemcpy(stamps_ns, ctx->d_trace, sizeof(uint64_t) * *n, cudaMemcpyDeviceToHost) != cudaSuccess)
        return MGM_ERR_CUDA;
    if (labels && label_cap > 0) {
        std::string all;
        for (auto& l : ctx->trace_labels) all += l + "\n";
        std::strncpy(labels, all.c_str(), label_cap - 1);
        labels[label_cap - 1] = 0;
    }
    return MGM_OK;
}

mgm_status mgm_bottom_trace_read(const mgm_ctx* ctx, uint64_t* stamps_ns, int cap, int* n, int32_t* meta) {
    if (!ctx || !n) return MGM_ERR_ARG;
    *n = (ctx->d_trace && ctx->botJ > 0) ? ctx->nphases : 0;
    if (*n == 0) return MGM_OK;
    if (cap < *n) return MGM_ERR_ARG;
    if (cudaMemcpy(stamps_ns, ctx->d_trace + 256, sizeof(uint64_t) * *n, cudaMemcpyDeviceToHost) != cudaSuccess)
        return MGM_ERR_CUDA;
    if (meta) {
        std::vector<BPhase> ph(*n);
        if (cudaMemcpy(ph.data(), ctx->d_phases, sizeof(BPhase) * *n, cudaMemcpyDeviceToHost) != cudaSuccess)
            return MGM_ERR_CUDA;
        for (int q = 0; q < *n; ++q) {
            meta[4 * q] = ph[q].op;
            meta[4 * q + 1] = ph[q].local;
            meta[4 * q + 2] = ph[q].r1 - ph[q].r0;  // rows
            meta[4 * q + 3] = 1 << ph[q].tpr_log2;
        }
    }
    return MGM_OK;
}

mgm_status mgm_bottom_ftrace_read(const mgm_ctx* ctx, int64_t* clk, int cap, int* n) {
    if (!ctx || !n || !clk) return MGM_ERR_ARG;
    *n = (ctx->d_trace && ctx->botJ > 0) ? ctx->nphases : 0;
    if (*n == 0) return MGM_OK;
    if (cap < *n) return MGM_ERR_ARG;
    for (int c = 0; c < 2; ++c)
        if (cudaMemcpy(clk + (size_t)c * 8 * cap, ctx->d_trace + 256 + BOT_MAX_PHASES + (size_t)c * 8 * BOT_MAX_PHASES,
                       sizeof(int64_t) * 8 * (size_t)*n, cudaMemcpyDeviceToHost) != cudaSuccess)
            return MGM_ERR_CUDA;
    return MGM_OK;
}

mgm_status mgm_vcycle_kernel_count(const mgm_ctx* ctx, int64_t* count) {
    if (!ctx || ctx->lv.empty() || !count) return MGM_ERR_ARG;
    if (ctx->vcycle_kernels > 0) { *count = ctx->vcycle_kernels; return MGM_OK; }
    i64 c = 0;
    const int p = ctx->p;
    if (p == 1) { *count = 1; return MGM_OK; }
    for (int j = 0; j + 1 < p; ++j) {
        c += (i64)(ctx->lp.nu1 + ctx->lp.nu2) * ctx->lv[j].ncol;
        c += 2 + 1 + (j > 0 ? 1 : 0);
        if (ctx->poisson) c += 3;
    }
    *count = c + 1;
    return MGM_OK;
}

mgm_status mgm_host_morton(const double* points, int64_t n, int64_t* perm) {
    if (!points || !perm || n < 1) return MGM_ERR_ARG;
    std::vector<i64> p;
    if (!morton_order(points, n, p)) return MGM_ERR_INPUT;
    std::copy(p.begin(), p.end(), perm);
    return MGM_OK;
}

mgm_status mgm_host_knn(const double* points, int64_t n, const double* queries, int64_t nq, int k,
                        int32_t* out) {
    if (!points || !queries || !out || k < 1 || k > n) return MGM_ERR_ARG;
    std::vector<i32> o;
    knn_grid(points, n, queries, nq, k, o, std::max(1, (int)std::thread::hardware_concurrency()));
    std::copy(o.begin(), o.end(), out);
    return MGM_OK;
}

mgm_status mgm_device_knn(const double* points, int64_t n, const double* queries, int64_t nq, int k,
                          int32_t* out) {
    if (!points || !queries || !out || k < 1 || k > n || k > 64 || nq < 0) return MGM_ERR_ARG;
    if (nq == 0) return MGM_OK;
    double *dp = nullptr, *dq = nullptr;
    i32* dout = nullptr;
    struct Free {
        double** a;
        double** b;
        i32** c;
        ~Free() {
            cudaFree(*a);
            cudaFree(*b);
            cudaFree(*c);
        }
    } free_{&dp, &dq, &dout};
    if (cudaMalloc(&dp, sizeof(double) * 3 * n) != cudaSuccess || cudaMalloc(&dq, sizeof(double) * 3 * nq) != cudaSuccess ||
        cudaMalloc(&dout, sizeof(i32) * nq * k) != cudaSuccess)
        return MGM_ERR_CUDA;
    cudaStream_t st = nullptr;
    if (cudaMemcpy(dp, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(dq, queries, sizeof(double) * 3 * nq, cudaMemcpyHostToDevice) != cudaSuccess)
        return MGM_ERR_CUDA;
    if (knn_device(points, dp, n, dq, nq, k, dout, st) != 0) return MGM_ERR_CUDA;
    if (cudaMemcpy(out, dout, sizeof(i32) * nq * k, cudaMemcpyDeviceToHost) != cudaSuccess) return MGM_ERR_CUDA;
    return MGM_OK;
}

mgm_status mgm_host_wse(const double* points, int64_t n, int64_t nt, int64_t* keep) {
    if (!points || !keep || nt < 1 || nt > n) return MGM_ERR_ARG;
    int nth = std::max(1, (int)std::thread::hardware_concurrency());
    std::vector<double> nn2;
    if (nearest_other(points, n, nn2, nth) >= 0) return MGM_ERR_INPUT;
    std::vector<i64> k;
    wse_eliminate(points, n, nt, nn2, k, nth);
    std::copy(k.begin(), k.end(), keep);
    return MGM_OK;
}

mgm_status mgm_device_wse(const double* points, int64_t n, int64_t nt, int64_t* keep) {
    if (!points || !keep || nt < 1 || nt > n) return MGM_ERR_ARG;
    int nth = std::max(1, (int)std::thread::hardware_concurrency());
    std::vector<double> nn2;
    if (nearest_other(points, n, nn2, nth) >= 0) return MGM_ERR_INPUT;
    double* dp = nullptr;
    if (cudaMalloc(&dp, sizeof(double) * 3 * n) != cudaSuccess) return MGM_ERR_CUDA;
    std::vector<i64> k;
    int rc = (int)cudaMemcpy(dp, points, sizeof(double) * 3 * n, cudaMemcpyHostToDevice);
    if (!rc) rc = wse_device(dp, points, n, nt, nn2, k, nullptr);
    cudaFree(dp);
    if (rc) return MGM_ERR_CUDA;
    if ((i64)k.size() != nt) return MGM_ERR_INPUT;
    std::copy(k.begin(), k.end(), keep);
    return MGM_OK;
}

mgm_status mgm_host_partition_level(int64_t n, const int64_t* L_ptr, const int32_t* L_col, const int32_t* colour,
                                    int ncol, const int32_t* owner, int64_t nc, const int64_t* P_ptr,
                                    const int32_t* P_col, const int32_t* owner_c, int64_t nf, const int64_t* Pf_ptr,
                                    const int32_t* Pf_col, const int32_t* owner_f, int nranks, int rank,
                                    int64_t* n_rows, int64_t* rows, int64_t* n_ghosts, int64_t* ghosts, int* n_peers,
                                    int32_t* peers, int64_t* send_rows, int64_t* send_off, int64_t* recv_off,
                                    int64_t* send_coff, int64_t* recv_coff) {
    if (n < 1 || !L_ptr || !L_col || !colour || !owner || ncol < 1 || nranks < 1 || rank < 0 || rank >= nranks)
        return MGM_ERR_ARG;
    auto csr = [](int64_t nr, int64_t ncl, const int64_t* ptr, const int32_t* col) {
        HostCSR A;
        A.nrows = nr;
        A.ncols = ncl;
        A.ptr.assign(ptr, ptr + nr + 1);
        A.col.assign(col, col + ptr[nr]);
        return A;
    };
    const HostCSR L = csr(n, n, L_ptr, L_col);
    HostCSR Pj, Pf;
    std::vector<int> ow(owner, owner + n), owc, owf;
    if (P_ptr && P_col && owner_c) {
        Pj = csr(n, nc, P_ptr, P_col);
        owc.assign(owner_c, owner_c + nc);
    }
    if (Pf_ptr && Pf_col && owner_f) {
        Pf = csr(nf, n, Pf_ptr, Pf_col);
        owf.assign(owner_f, owner_f + nf);
    }
    std::vector<i32> colv(colour, colour + n);
    std::vector<PartTables> all;
    partition_level(L, ow, colv, ncol, owc.empty() ? nullptr : &Pj, owc.empty() ? nullptr : &owc,
                    owf.empty() ? nullptr : &Pf, owf.empty() ? nullptr : &owf, nranks, all);
    const PartTables& T = all[(size_t)rank];
    if (n_rows) *n_rows = (int64_t)T.rows.size();
    if (rows) std::copy(T.rows.begin(), T.rows.end(), rows);
    if (n_ghosts) *n_ghosts = (int64_t)T.ghosts.size();
    if (ghosts) std::copy(T.ghosts.begin(), T.ghosts.end(), ghosts);
    if (n_peers) *n_peers = (int)T.peers.size();
    if (peers) std::copy(T.peers.begin(), T.peers.end(), peers);
    if (send_rows) std::copy(T.send_rows.begin(), T.send_rows.end(), send_rows);
    if (send_off) std::copy(T.send_off.begin(), T.send_off.end(), send_off);
    if (recv_off) std::copy(T.recv_off.begin(), T.recv_off.end(), recv_off);
    if (send_coff) std::copy(T.send_coff.begin(), T.send_coff.end(), send_coff);
    if (recv_coff) std::copy(T.recv_coff.begin(), T.recv_coff.end(), recv_coff);
    return MGM_OK;
}

mgm_status mgm_host_colouring(int64_t n, const int64_t* ptr, const int32_t* col, int32_t* colour,
                              int* n_colours) {
    if (!ptr || !col || !colour || n < 1) return MGM_ERR_ARG;
    HostCSR A;
    A.nrows = A.ncols = n;
    A.ptr.assign(ptr, ptr + n + 1);
    A.col.assign(col, col + ptr[n]);
    std::vector<i32> c;
    int nc = greedy_colouring(A, c, colour_passes());
    std::copy(c.begin(), c.end(), colour);
    if (n_colours) *n_colours = nc;
    return MGM_OK;
}

}  // extern "C"
