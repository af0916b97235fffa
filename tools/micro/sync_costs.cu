// Microbenchmarks of synchronisation costs on B200 (informs the V-cycle kernel design):
//  1. cluster barrier (barrier.cluster.arrive.release + wait.acquire) for cluster sizes 1..16
//  2. software grid barrier (one atomic counter + generation flag) for 148 / 296 CTAs
//  3. per-kernel cost of a chain of dependent tiny kernels in a CUDA graph, with / without PDL
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__global__ void k_cluster_sync(int iters, int* out) {
    cg::cluster_group cl = cg::this_cluster();
    for (int i = 0; i < iters; ++i) cl.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
__global__ void k_block_sync(int iters, int* out) {
    for (int i = 0; i < iters; ++i) __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}

__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned*)gen, 1u);
        } else {
            while (*gen == g) {}
        }
        __threadfence();
    }
    __syncthreads();
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// barrier using a monotone counter: arrive with red.release, wait until counter >= target
__device__ __forceinline__ void grid_barrier2(unsigned* count, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        while (ld_acquire(count) < target) {}
    }
    __syncthreads();
}
__global__ void k_grid_sync(int iters, unsigned* count, unsigned* gen) {
    for (int i = 0; i < iters; ++i) grid_barrier(count, gen, gridDim.x);
}
__global__ void k_grid_sync2(int iters, unsigned* count) {
    for (int i = 0; i < iters; ++i) grid_barrier2(count, (unsigned)(i + 1) * gridDim.x);
}
__global__ void k_empty(int* x) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) x[0]++;
}

int main() {
    int* d;
    unsigned *cnt, *gen;
    cudaMalloc(&d, 64);
    cudaMalloc(&cnt, 64);
    cudaMalloc(&gen, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const int iters = 2000;
    cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int threads : {256, 512, 1024}) {
        k_block_sync<<<1, threads>>>(iters, d);
        cudaEventRecord(e0);
        k_block_sync<<<1, threads>>>(iters, d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("syncthreads  threads=%4d: %.1f ns\n", threads, ms * 1e6 / iters);
        for (int cs : {2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs);
            cfg.blockDim = dim3(threads);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_cluster_sync, iters, d);
            cudaEventRecord(e0);
            cudaError_t err = cudaLaunchKernelEx(&cfg, k_cluster_sync, iters, d);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("cluster.sync cs=%2d threads=%4d: %.1f ns (%s)\n", cs, threads, ms * 1e6 / iters,
                   cudaGetErrorString(err));
        }
    }
    for (int blocks : {148, 296}) {
        for (int threads : {256, 512}) {
            cudaMemset(cnt, 0, 64);
            cudaMemset(gen, 0, 64);
            k_grid_sync<<<blocks, threads>>>(iters, cnt, gen);
            cudaEventRecord(e0);
            k_grid_sync<<<blocks, threads>>>(iters, cnt, gen);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("grid barrier (gen flag) blocks=%d threads=%d: %.1f ns  %s\n", blocks, threads, ms * 1e6 / iters,
                   cudaGetErrorString(cudaGetLastError()));
            cudaMemset(cnt, 0, 64);
            k_grid_sync2<<<blocks, threads>>>(iters, cnt);
            cudaMemset(cnt, 0, 64);
            cudaEventRecord(e0);
            k_grid_sync2<<<blocks, threads>>>(iters, cnt);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("grid barrier (red.release counter) blocks=%d threads=%d: %.1f ns  %s\n", blocks, threads,
                   ms * 1e6 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    // graph of N dependent kernels
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int pdl : {0, 1}) {
        for (int grid : {1, 148, 592}) {
            const int N = 400;
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
            for (int i = 0; i < N; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = st;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl;
                cudaLaunchKernelEx(&cfg, k_empty, d);
            }
            cudaStreamEndCapture(st, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphLaunch(ge, st);
            cudaStreamSynchronize(st);
            cudaEventRecord(e0, st);
            for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, st);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("graph chain pdl=%d grid=%d: %.2f us per kernel\n", pdl, grid, ms * 1e3 / (5 * N));
        }
    }
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
