// Microbenchmark: the device-side cost of one kernel launch as bench.py times
// it (a GPU sleep first, so the kernel is already queued when the start event
// is recorded; CUDA events on the stream; median of 200).  Reports event time,
// in-kernel %globaltimer span (first CTA start .. last CTA end) and the gap.
// Variants: empty kernels of several shapes and parameter sizes, a device
// counter read + last-CTA atomic (what the collectives do per call), and
// local / remote (NVLink peer) stores followed by a sys fence.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/gap_bench scripts/gap_bench.cu
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

__global__ void sleep_kernel(uint64_t ns) {
    const uint64_t t0 = gt();
    while (gt() - t0 < ns) {
    }
}

struct Big {
    uint64_t a[120];  // ~1 KB of kernel parameters
};

__global__ void empty_kernel(uint64_t* span) {
    const uint64_t t0 = gt();
    if (threadIdx.x == 0) {
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = gt();
    }
}

__global__ void big_kernel(Big b, uint64_t* span) {
    const uint64_t t0 = gt();
    if (threadIdx.x == 0) {
        span[2 * blockIdx.x] = t0 + (b.a[threadIdx.x & 7] & 0);
        span[2 * blockIdx.x + 1] = gt();
    }
}

// read the call counter at entry, last CTA bumps it at exit (the collectives' epoch)
__global__ void counter_kernel(uint32_t* ctl, uint64_t* span) {
    const uint64_t t0 = gt();
    __shared__ uint32_t e;
    if (threadIdx.x == 0) e = *(volatile uint32_t*)ctl + 1u;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t done = atomicAdd(ctl + 1, 1u) + 1u;
        if (done == gridDim.x) {
            ctl[1] = 0u;
            __threadfence();
            atomicExch(ctl, e);
        }
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = gt();
    }
}

__global__ void store_kernel(float4* dst, int per, int fence, uint64_t* span) {
    const uint64_t t0 = gt();
    const float4 v = make_float4(1, 2, 3, 4);
    for (int j = 0; j < per; ++j) dst[((int64_t)blockIdx.x * per + j) * blockDim.x + threadIdx.x] = v;
    if (fence) asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = gt();
    }
}

// The collectives' rank-level exit, step by step (coll_common.cuh exit_rank):
// every CTA stores `per` float4 per thread (remote or local), orders them with
// a gpu fence (or a sys fence: bit 8) and arrives on a counter; the last CTA
// then does: bit 1 fence.sys, bit 2 a remote relaxed stamp store, bit 4 a
// remote acquire load, bit 16 a LOCAL relaxed stamp store, then resets the
// counter and bumps the epoch.  Which step makes the kernel's completion slow?
__global__ void proto_kernel(float4* dst, int per, int mode, uint32_t* ctl, uint64_t* rflag,
                             uint64_t* lflag, uint64_t* span) {
    const uint64_t t0 = gt();
    const float4 v = make_float4(1, 2, 3, 4);
    for (int j = 0; j < per; ++j) dst[((int64_t)blockIdx.x * per + j) * blockDim.x + threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode & 8) asm volatile("fence.acq_rel.sys;" ::: "memory");
        else __threadfence();
        const uint32_t done = atomicAdd(ctl + 1, 1u) + 1u;
        if (done == gridDim.x) {
            __threadfence();
            if (mode & 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
            if (mode & 2) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(rflag), "l"((uint64_t)t0) : "memory");
            if (mode & 16) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(lflag), "l"((uint64_t)t0) : "memory");
            if (mode & 4) {
                uint64_t x;
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(rflag) : "memory");
                if (x == 1) ctl[3] = 1;
            }
            ctl[1] = 0u;
            __threadfence();
            atomicExch(ctl, ctl[0] + 1);
        }
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = gt();
    }
}

// remote (or local) 128-bit loads, summed so they cannot be dropped, optional fence.sys
__global__ void load_kernel(const float4* src, int per, int fence, uint64_t* span, float* sink) {
    const uint64_t t0 = gt();
    float acc = 0.f;
    for (int j = 0; j < per; ++j) {
        float4 v;
        const float4* p = src + ((int64_t)blockIdx.x * per + j) * blockDim.x + threadIdx.x;
        asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 12345.f) sink[0] = acc;
    if (fence) asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = gt();
    }
}

// remote (or local) bulk loads into shared memory with TMA (cp.async.bulk + mbarrier), 16 KB per
// copy, one copy in flight per CTA at a time, `per` copies per CTA
__global__ void __launch_bounds__(128) tma_load_kernel(const char* src, int per, uint64_t* span, float* sink) {
    extern __shared__ __align__(128) char sm[];
    __shared__ __align__(8) uint64_t bar;
    const uint64_t t0 = gt();
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(sm);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    float acc = 0.f;
    for (int j = 0; j < per; ++j) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(16384));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(d), "l"(src + ((int64_t)blockIdx.x * per + j) * 16384), "r"(16384), "r"(b) : "memory");
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(b), "r"((uint32_t)(j & 1)));
        acc += reinterpret_cast<const float*>(sm)[threadIdx.x];
        __syncthreads();
    }
    if (acc == 12345.f) sink[0] = acc;
    if (threadIdx.x == 0) {
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = gt();
    }
}

int main() {
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    float4* peer = nullptr;
    if (ndev >= 2) {
        cudaSetDevice(1);
        cudaMalloc(&peer, 64 << 20);
    }
    cudaSetDevice(0);
    if (ndev >= 2) cudaDeviceEnablePeerAccess(1, 0);
    float4* local;
    uint64_t* span;
    uint32_t* ctl;
    cudaMalloc(&local, 64 << 20);
    cudaMalloc(&span, 1 << 20);
    cudaMalloc(&ctl, 64);
    cudaMemset(ctl, 0, 64);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    Big big{};
    std::vector<uint64_t> h(2 * 1024);
    auto run = [&](const char* name, int G, int T, int what, int per, int fence, bool remote) {
        std::vector<float> ev, sp;
        for (int rep = 0; rep < 220; ++rep) {
            sleep_kernel<<<1, 32, 0, st>>>(30000);
            cudaEventRecord(e0, st);
            switch (what) {
                case 0: break;  // events only
                case 1: empty_kernel<<<G, T, 0, st>>>(span); break;
                case 2: big_kernel<<<G, T, 0, st>>>(big, span); break;
                case 3: counter_kernel<<<G, T, 0, st>>>(ctl, span); break;
                case 4: store_kernel<<<G, T, 0, st>>>(remote ? peer : local, per, fence, span); break;
                case 7: tma_load_kernel<<<G, 128, 16384, st>>>(remote ? (const char*)peer : (const char*)local, per, span, (float*)local); break;
                case 6: load_kernel<<<G, T, 0, st>>>(remote ? peer : local, per, fence, span, (float*)local); break;
                case 5:
                    proto_kernel<<<G, T, 0, st>>>(remote ? peer : local, per, fence, ctl,
                                                  (uint64_t*)(remote ? peer : local) + (5 << 20),
                                                  (uint64_t*)local + (6 << 20), span);
                    break;
            }
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            uint64_t lo = ~0ull, hi = 0;
            if (what) {
                cudaMemcpy(h.data(), span, 16 * G, cudaMemcpyDeviceToHost);
                for (int b = 0; b < G; ++b) {
                    lo = std::min(lo, h[2 * b]);
                    hi = std::max(hi, h[2 * b + 1]);
                }
            }
            if (rep >= 20) {
                ev.push_back(ms * 1000.f);
                sp.push_back(what ? (hi - lo) / 1000.f : 0.f);
            }
        }
        std::sort(ev.begin(), ev.end());
        std::sort(sp.begin(), sp.end());
        const float e = ev[ev.size() / 2], s = sp[sp.size() / 2];
        printf("%-34s G=%4d T=%4d  event %6.2f us  span %6.2f us  gap %6.2f us  (event p10 %.2f p90 %.2f)\n", name, G,
               T, e, s, e - s, ev[ev.size() / 10], ev[ev.size() * 9 / 10]);
    };
    run("events only", 0, 0, 0, 0, 0, false);
    run("empty", 1, 32, 1, 0, 0, false);
    run("empty", 148, 512, 1, 0, 0, false);
    run("empty", 296, 512, 1, 0, 0, false);
    run("empty 1KB params", 148, 512, 2, 0, 0, false);
    run("counter read + last-CTA atomic", 148, 512, 3, 0, 0, false);
    run("local stores x4", 148, 512, 4, 4, 0, false);
    run("local stores x4 + fence.sys", 148, 512, 4, 4, 1, false);
    if (peer) {
        run("remote stores x1", 148, 512, 4, 1, 0, true);
        run("remote stores x1 + fence.sys", 148, 512, 4, 1, 1, true);
        run("remote stores x16", 148, 512, 4, 16, 0, true);
        run("remote stores x16 + fence.sys", 148, 512, 4, 16, 1, true);
        run("exit: remote x4, gpu fence + ctr", 148, 512, 5, 4, 0, true);
        run("exit: + last fence.sys", 148, 512, 5, 4, 1, true);
        run("exit: + last fence.sys + rstamp", 148, 512, 5, 4, 3, true);
        run("exit: + last fence.sys + racq", 148, 512, 5, 4, 5, true);
        run("exit: + last fence.sys + lstamp", 148, 512, 5, 4, 17, true);
        run("exit: all sys fence + ctr", 148, 512, 5, 4, 8, true);
        run("exit: all sys + last rstamp", 148, 512, 5, 4, 10, true);
        run("exit: local x4, gpu fence + ctr", 148, 512, 5, 4, 0, false);
        run("exit: local + last fence.sys", 148, 512, 5, 4, 1, false);
        run("remote loads x4", 148, 512, 6, 4, 0, true);
        run("remote loads x16", 148, 512, 6, 16, 0, true);
        run("remote loads x16 + fence.sys", 148, 512, 6, 16, 1, true);
        run("local loads x16", 148, 512, 6, 16, 0, false);
        run("remote TMA loads 16 KB x4", 148, 128, 7, 4, 0, true);
        run("remote TMA loads 16 KB x16", 148, 128, 7, 16, 0, true);
        run("local TMA loads 16 KB x16", 148, 128, 7, 16, 0, false);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
