// Microbenchmark: cost of sys/gpu-scope fences and release stores on B200,
// with and without outstanding NVLink peer stores.  Needs 2 GPUs with P2P.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fence_bench scripts/fence_bench.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <algorithm>
#include <vector>

__device__ __forceinline__ uint64_t gt() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// mode bits: 1 = remote stores before, 2 = local stores before
// op: 0 fence.acq_rel.sys, 1 fence.acq_rel.gpu, 2 st.release.sys remote flag,
//     3 st.relaxed.sys remote flag, 4 fence.sc.sys, 5 nothing, 6 st.release.gpu local flag
__global__ void kern(float4* remote, float4* local, uint32_t* rflag, uint32_t* lflag, int mode, int op,
                     uint64_t* out) {
    const int t = threadIdx.x, b = blockIdx.x;
    float4 v = make_float4(1, 2, 3, 4);
    if (mode & 1)
        for (int j = 0; j < 4; ++j) remote[(b * 4 + j) * blockDim.x + t] = v;
    if (mode & 2)
        for (int j = 0; j < 4; ++j) local[(b * 4 + j) * blockDim.x + t] = v;
    __syncthreads();
    if (t == 0) {
        uint64_t t0 = gt();
        switch (op) {
            case 0: asm volatile("fence.acq_rel.sys;" ::: "memory"); break;
            case 1: asm volatile("fence.acq_rel.gpu;" ::: "memory"); break;
            case 2: asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(rflag + b), "r"(1u) : "memory"); break;
            case 3: asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(rflag + b), "r"(1u) : "memory"); break;
            case 4: asm volatile("fence.sc.sys;" ::: "memory"); break;
            case 5: break;
            case 6: asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(lflag + b), "r"(1u) : "memory"); break;
        }
        uint64_t t1 = gt();
        out[b] = t1 - t0;
    }
}

// Warp-level variants of the exit stamp: op 0 = lanes 0..7 each st.release.sys
// (one store each), op 1 = lane 0 fence.acq_rel.sys then 8 relaxed stores.
__global__ void kern_warp(float4* remote, uint32_t* rflag, int op, uint64_t* out) {
    const int t = threadIdx.x, b = blockIdx.x;
    float4 v = make_float4(1, 2, 3, 4);
    for (int j = 0; j < 4; ++j) remote[(b * 4 + j) * blockDim.x + t] = v;
    __syncthreads();
    uint64_t t0 = gt();
    if (op == 0) {
        if (t < 8) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(rflag + b * 8 + t), "r"(1u) : "memory");
    } else {
        if (t == 0) {
            asm volatile("fence.acq_rel.sys;" ::: "memory");
            for (int k = 0; k < 8; ++k)
                asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(rflag + b * 8 + k), "r"(1u) : "memory");
        }
    }
    __syncwarp();
    uint64_t t1 = gt();
    if (t == 0) out[b] = t1 - t0;
}

int main() {
    int n = 0;
    cudaGetDeviceCount(&n);
    if (n < 2) { printf("need 2 GPUs\n"); return 1; }
    cudaSetDevice(1);
    float4* peerbuf;
    uint32_t* peerflag;
    cudaMalloc(&peerbuf, 64 << 20);
    cudaMalloc(&peerflag, 1 << 20);
    cudaSetDevice(0);
    cudaDeviceEnablePeerAccess(1, 0);
    float4* localbuf;
    uint32_t* localflag;
    uint64_t* out;
    cudaMalloc(&localbuf, 64 << 20);
    cudaMalloc(&localflag, 1 << 20);
    cudaMalloc(&out, 4096 * 8);
    const char* opn[] = {"fence.acq_rel.sys", "fence.acq_rel.gpu", "st.release.sys(remote)", "st.relaxed.sys(remote)",
                         "fence.sc.sys", "nothing", "st.release.gpu(local)"};
    const char* moden[] = {"no prior stores", "remote stores", "local stores", "both"};
    int G = 148;
    std::vector<uint64_t> h(G);
    for (int mode = 0; mode < 3; ++mode)
        for (int op = 0; op < 7; ++op) {
            std::vector<double> meds;
            for (int rep = 0; rep < 5; ++rep) {
                kern<<<G, 256>>>(peerbuf, localbuf, peerflag, localflag, mode, op, out);
                cudaDeviceSynchronize();
                cudaMemcpy(h.data(), out, G * 8, cudaMemcpyDeviceToHost);
                std::sort(h.begin(), h.end());
                meds.push_back((double)h[G / 2]);
            }
            std::sort(meds.begin(), meds.end());
            printf("%-16s %-24s median %.0f ns (max-CTA of last rep %llu)\n", moden[mode], opn[op], meds[2],
                   (unsigned long long)h[G - 1]);
        }
    for (int op = 0; op < 2; ++op) {
        std::vector<double> meds;
        for (int rep = 0; rep < 5; ++rep) {
            kern_warp<<<G, 256>>>(peerbuf, peerflag, op, out);
            cudaDeviceSynchronize();
            cudaMemcpy(h.data(), out, G * 8, cudaMemcpyDeviceToHost);
            std::sort(h.begin(), h.end());
            meds.push_back((double)h[G / 2]);
        }
        std::sort(meds.begin(), meds.end());
        printf("remote stores    %-40s median %.0f ns\n",
               op == 0 ? "8 lanes x st.release.sys" : "lane 0: fence.sys + 8 relaxed stores", meds[2]);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
