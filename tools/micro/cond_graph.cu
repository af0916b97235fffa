// Can a CUDA-graph WHILE conditional node hold the solver's step: a chain of PDL kernels,
// a thread-block-cluster kernel with large dynamic smem, memset/memcpy nodes, and a
// device-side decision (cudaGraphSetConditional)?  And what does one iteration cost?
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o cond_graph cond_graph.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_chain(double* a, int i) {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) a[0] += 1.0;
}
__global__ void __cluster_dims__(1, 1, 1) k_dummy() {}
__global__ void k_cluster(double* a) {
    extern __shared__ double sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    sm[threadIdx.x] = threadIdx.x;
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) a[1] += 1.0;
}
__global__ void k_decide(cudaGraphConditionalHandle h, int* iter, int maxit, double* a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int k = ++*iter;
    a[2] = k;
    cudaGraphSetConditional(h, k < maxit ? 1 : 0);
}

static void launch_pdl(cudaStream_t st, void (*kern)(double*, int), double* a, int i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8); cfg.blockDim = dim3(128); cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a, i);
}

int main() {
    cudaStream_t st; CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double* a; CK(cudaMalloc(&a, 1 << 20)); CK(cudaMemset(a, 0, 1 << 20));
    double* b; CK(cudaMalloc(&b, 1 << 20));
    int* iter; CK(cudaMalloc(&iter, 4)); CK(cudaMemset(iter, 0, 4));
    const int NK = 200, MAXIT = 50;
    CK(cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));

    cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CK(cudaGraphAddNode(&cn, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // capture the body
    CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    CK(cudaMemcpyAsync(b, a, 4096, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(b + 1024, 0, 4096, st));
    for (int i = 0; i < NK; ++i) launch_pdl(st, k_chain, a, i);
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16); cfg.blockDim = dim3(512); cfg.stream = st; cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 2;
        CK(cudaLaunchKernelEx(&cfg, k_cluster, a));
    }
    for (int i = 0; i < NK; ++i) launch_pdl(st, k_chain, a, i);
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1); cfg.blockDim = dim3(1); cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k_decide, h, iter, MAXIT, a));
    }
    cudaGraph_t cap;
    CK(cudaStreamEndCapture(st, &cap));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphUpload(ge, st));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaMemsetAsync(iter, 0, 4, st));
        CK(cudaMemsetAsync(a, 0, 64, st));
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double h3[3]; CK(cudaMemcpy(h3, a, 24, cudaMemcpyDeviceToHost));
        printf("while-graph: %d iterations, chain %g (expect %d), cluster %g, %.1f us/iteration (%d kernels each)\n",
               (int)h3[2], h3[0], 2 * NK * MAXIT, h3[1], 1000.0 * ms / MAXIT, 2 * NK + 2);
    }
    // reference: same body as a plain graph launched MAXIT times from the host (no sync)
    cudaGraphExec_t be; CK(cudaGraphInstantiate(&be, body, 0));
    CK(cudaGraphLaunch(be, st)); CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < MAXIT; ++i) CK(cudaGraphLaunch(be, st));
    CK(cudaEventRecord(e1, st)); CK(cudaStreamSynchronize(st));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("host-launched body graphs: %.1f us/iteration\n", 1000.0 * ms / MAXIT);
    // with a sync + D2H read per iteration (the current GMRES pattern)
    double hv;
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < MAXIT; ++i) { CK(cudaGraphLaunch(be, st)); CK(cudaMemcpyAsync(&hv, a, 8, cudaMemcpyDeviceToHost, st)); CK(cudaStreamSynchronize(st)); }
    CK(cudaEventRecord(e1, st)); CK(cudaStreamSynchronize(st));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("host-launched + sync per iteration: %.1f us/iteration\n", 1000.0 * ms / MAXIT);
    printf("OK\n");
    return 0;
}
