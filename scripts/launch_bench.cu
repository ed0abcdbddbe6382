// Microbenchmark: event-measured time vs in-kernel %globaltimer span for
// kernels that write remote (NVLink peer) memory, local memory or nothing.
// Tells how much of a collective's event time is launch + end-of-grid cost.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/launch_bench scripts/launch_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

__device__ __forceinline__ uint64_t gt() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void kern(float4* dst, int per_cta, uint64_t* span, int fence) {
    uint64_t t0 = gt();
    float4 v = make_float4(1, 2, 3, 4);
    for (int j = 0; j < per_cta; ++j) dst[((int64_t)blockIdx.x * per_cta + j) * blockDim.x + threadIdx.x] = v;
    if (fence == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
    if (fence == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    uint64_t t1 = gt();
    if (threadIdx.x == 0) {
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = t1;
    }
}

int main() {
    int n = 0;
    cudaGetDeviceCount(&n);
    float4* peer = nullptr;
    if (n >= 2) {
        cudaSetDevice(1);
        cudaMalloc(&peer, 256 << 20);
    }
    cudaSetDevice(0);
    if (n >= 2) cudaDeviceEnablePeerAccess(1, 0);
    float4* local;
    uint64_t* span;
    cudaMalloc(&local, 256 << 20);
    cudaMalloc(&span, 1 << 20);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int G = 444, T = 256;
    std::vector<uint64_t> h(2 * G);
    const char* fn[] = {"none", "fence.sys", "fence.gpu"};
    for (int tgt = 0; tgt < (n >= 2 ? 2 : 1); ++tgt)
        for (int per : {0, 1, 16})
            for (int f = 0; f < 3; ++f) {
                std::vector<float> ev, sp;
                for (int rep = 0; rep < 20; ++rep) {
                    cudaEventRecord(e0);
                    kern<<<G, T>>>(tgt ? peer : local, per, span, f);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    cudaMemcpy(h.data(), span, 16 * G, cudaMemcpyDeviceToHost);
                    uint64_t lo = ~0ull, hi = 0;
                    for (int b = 0; b < G; ++b) {
                        lo = std::min(lo, h[2 * b]);
                        hi = std::max(hi, h[2 * b + 1]);
                    }
                    if (rep >= 3) {
                        ev.push_back(ms * 1000.f);
                        sp.push_back((hi - lo) / 1000.f);
                    }
                }
                std::sort(ev.begin(), ev.end());
                std::sort(sp.begin(), sp.end());
                printf("%-6s stores/thread=%2d %-9s event %.2f us  span %.2f us  gap %.2f us\n", tgt ? "remote" : "local",
                       per, fn[f], ev[ev.size() / 2], sp[sp.size() / 2], ev[ev.size() / 2] - sp[sp.size() / 2]);
            }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
