// Microbenchmark: PCIe bandwidth of pinned host memory moved by
//   (a) the copy engines (cudaMemcpyAsync H2D, D2H, and both at once on two streams),
//   (b) SM loads/stores (zero-copy, 128-bit, grid-stride),
//   (c) TMA bulk copies (cp.async.bulk global->shared with an mbarrier, and
//       shared->global bulk stores), from a persistent grid,
// each alone and full duplex.  Decides how the host-buffer entry point
// (firecaffe_sgd_step_host) should move its bytes.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/tma_host_bench scripts/tma_host_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int TILE = 16384;  // bytes per bulk copy
constexpr int NST = 4;       // ring stages per CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode bit 0: load host->smem (TMA), bit 1: store smem->host (TMA)
__global__ void __launch_bounds__(128) tma_kernel(const char* src, char* dst, int64_t bytes, int mode, float* sink) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t bar[NST];
    const int64_t ntiles = bytes / TILE;
    const int t = threadIdx.x;
    if (t == 0) {
        for (int s = 0; s < NST; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float acc = 0.f;
    uint32_t phase[NST] = {0};
    // prologue
    int64_t k0 = blockIdx.x;
    if (t == 0 && (mode & 1)) {
        for (int s = 0; s < NST; ++s) {
            const int64_t k = k0 + (int64_t)s * gridDim.x;
            if (k >= ntiles) break;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(TILE));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(smem_u32(smem + s * TILE)), "l"(src + k * TILE), "r"(TILE), "r"(smem_u32(&bar[s])) : "memory");
        }
    }
    int it = 0;
    for (int64_t k = k0; k < ntiles; k += gridDim.x, ++it) {
        const int s = it % NST;
        if (mode & 1) {
            uint32_t done = 0;
            while (!done) {
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(phase[s]));
            }
            phase[s] ^= 1;
            acc += reinterpret_cast<const float*>(smem + s * TILE)[t];
        }
        if (mode & 2) {
            __syncthreads();
            if (t == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             ::"l"(dst + k * TILE), "r"(smem_u32(smem + s * TILE)), "r"(TILE) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NST - 1) : "memory");
            }
        }
        __syncthreads();
        if ((mode & 1) && t == 0) {
            const int64_t kn = k + (int64_t)NST * gridDim.x;
            if (kn < ntiles) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(TILE));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(smem + s * TILE)), "l"(src + kn * TILE), "r"(TILE), "r"(smem_u32(&bar[s])) : "memory");
            }
        }
    }
    if ((mode & 2) && t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (acc == 1234.5f) sink[0] = acc;
}

// SM zero-copy: mode bit0 load from src, bit1 store to dst
__global__ void __launch_bounds__(256) zc_kernel(const float4* src, float4* dst, int64_t n4, int mode, float* sink) {
    float acc = 0.f;
    const float4 z = make_float4(1, 2, 3, 4);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        if (mode & 1) { float4 v = src[i]; acc += v.x; }
        if (mode & 2) dst[i] = z;
    }
    if (acc == 1234.5f) sink[0] = acc;
}

int main() {
    const int64_t bytes = 256ll << 20;
    char *hA, *hB, *dA, *dB;
    float* sink;
    CK(cudaHostAlloc(&hA, bytes, cudaHostAllocMapped));
    CK(cudaHostAlloc(&hB, bytes, cudaHostAllocMapped));
    memset(hA, 1, bytes);
    memset(hB, 2, bytes);
    CK(cudaMalloc(&dA, bytes));
    CK(cudaMalloc(&dB, bytes));
    CK(cudaMalloc(&sink, 64));
    char *hAd, *hBd;
    CK(cudaHostGetDevicePointer((void**)&hAd, hA, 0));
    CK(cudaHostGetDevicePointer((void**)&hBd, hB, 0));
    cudaStream_t s0, s1;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = NST * TILE;
    CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    auto timeit = [&](const char* name, double moved, auto fn) {
        std::vector<float> ms;
        for (int r = 0; r < 7; ++r) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, s0);
            cudaStreamWaitEvent(s1, e0, 0);
            fn();
            cudaEvent_t j;
            cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
            cudaEventRecord(j, s1);
            cudaStreamWaitEvent(s0, j, 0);
            cudaEventRecord(e1, s0);
            cudaEventSynchronize(e1);
            float m = 0;
            cudaEventElapsedTime(&m, e0, e1);
            cudaEventDestroy(j);
            if (r) ms.push_back(m);
        }
        std::sort(ms.begin(), ms.end());
        const float m = ms[ms.size() / 2];
        printf("%-44s %8.3f ms  %7.1f GB/s  (%s)\n", name, m, moved / (m * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    const double B = (double)bytes;
    timeit("CE H2D", B, [&] { cudaMemcpyAsync(dA, hA, bytes, cudaMemcpyHostToDevice, s0); });
    timeit("CE D2H", B, [&] { cudaMemcpyAsync(hB, dB, bytes, cudaMemcpyDeviceToHost, s0); });
    timeit("CE H2D || D2H (2 streams), per direction", B, [&] {
        cudaMemcpyAsync(dA, hA, bytes, cudaMemcpyHostToDevice, s0);
        cudaMemcpyAsync(hB, dB, bytes, cudaMemcpyDeviceToHost, s1);
    });
    for (int g : {sms, 2 * sms, 4 * sms}) {
        char nm[96];
        snprintf(nm, sizeof nm, "SM zc load  grid %d", g);
        timeit(nm, B, [&] { zc_kernel<<<g, 256, 0, s0>>>((const float4*)hAd, nullptr, bytes / 16, 1, sink); });
        snprintf(nm, sizeof nm, "SM zc store grid %d", g);
        timeit(nm, B, [&] { zc_kernel<<<g, 256, 0, s0>>>(nullptr, (float4*)hBd, bytes / 16, 2, sink); });
        snprintf(nm, sizeof nm, "SM zc load+store grid %d, per direction", g);
        timeit(nm, B, [&] { zc_kernel<<<g, 256, 0, s0>>>((const float4*)hAd, (float4*)hBd, bytes / 16, 3, sink); });
    }
    for (int g : {sms, 2 * sms}) {
        char nm[96];
        snprintf(nm, sizeof nm, "TMA load  grid %d (16 KB x %d stages)", g, NST);
        timeit(nm, B, [&] { tma_kernel<<<g, 128, smem, s0>>>(hAd, nullptr, bytes, 1, sink); });
        snprintf(nm, sizeof nm, "TMA store grid %d", g);
        timeit(nm, B, [&] { tma_kernel<<<g, 128, smem, s0>>>(nullptr, hBd, bytes, 2, sink); });
        snprintf(nm, sizeof nm, "TMA load+store grid %d, per direction", g);
        timeit(nm, B, [&] { tma_kernel<<<g, 128, smem, s0>>>(hAd, hBd, bytes, 3, sink); });
    }
    timeit("CE H2D || SM zc store (grid 2x), per direction", B, [&] {
        cudaMemcpyAsync(dA, hA, bytes, cudaMemcpyHostToDevice, s0);
        zc_kernel<<<2 * sms, 256, 0, s1>>>(nullptr, (float4*)hBd, bytes / 16, 2, sink);
    });
    timeit("CE H2D || TMA store, per direction", B, [&] {
        cudaMemcpyAsync(dA, hA, bytes, cudaMemcpyHostToDevice, s0);
        tma_kernel<<<sms, 128, smem, s1>>>(nullptr, hBd, bytes, 2, sink);
    });
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
