// Dependent-load latency on B200: pointer chase with one thread over a buffer of a given
// size (L2-resident vs DRAM), plain ld.global vs ld.global.nc with an L2 evict_last hint,
// and shared / distributed-shared-memory chase.  Prints ns and cycles per load.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

__global__ void chase(const uint32_t* __restrict__ next, int steps, int mode, unsigned long long* out) {
    uint32_t i = 0;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        if (mode == 0) i = next[i];
        else if (mode == 1) asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(i) : "l"(next + i), "l"(pol));
        else asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(i) : "l"(next + i));
    }
    long long t1 = clock64();
    out[0] = (unsigned long long)(t1 - t0);
    out[1] = i;
}

int main() {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    unsigned long long* d_out;
    cudaMalloc(&d_out, 16);
    for (size_t bytes : {(size_t)1 << 20, (size_t)16 << 20, (size_t)64 << 20, (size_t)1 << 30}) {
        size_t n = bytes / 4;
        // random cyclic permutation with stride >= 128 B (one element per 128-B line)
        size_t lines = bytes / 128;
        std::vector<uint32_t> order(lines);
        for (size_t k = 0; k < lines; ++k) order[k] = (uint32_t)k;
        std::mt19937 rng(1);
        std::shuffle(order.begin() + 1, order.end(), rng);
        std::vector<uint32_t> h(n, 0);
        for (size_t k = 0; k < lines; ++k) h[(size_t)order[k] * 32] = order[(k + 1) % lines] * 32;
        uint32_t* d;
        cudaMalloc(&d, bytes);
        cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 3; ++mode) {
            const int steps = 20000;
            chase<<<1, 1>>>(d, steps, mode, d_out);  // warm
            cudaEventRecord(e0);
            chase<<<1, 1>>>(d, steps, mode, d_out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long hc[2];
            cudaMemcpy(hc, d_out, 16, cudaMemcpyDeviceToHost);
            printf("buffer %7zu KB mode %s: %.1f ns/load, %.0f cycles/load\n", bytes >> 10,
                   mode == 0 ? "ld.global     " : mode == 1 ? "ld.nc+evict_last" : "ld.global.cg  ", ms * 1e6 / steps,
                   (double)hc[0] / steps);
        }
        cudaFree(d);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
