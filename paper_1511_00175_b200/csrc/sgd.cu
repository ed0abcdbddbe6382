// firecaffe_sgd_step kernel: the 1-GPU fused SGD update.
//
// HBM-bound streaming kernel: per parameter it reads grad, w, mom and writes
// w, mom (20 algorithmic bytes).  128-bit accesses, U independent float4 per
// thread per operand in flight (all loads issued before any math), grid sized
// to the SM count x resident CTAs so every SM streams.
#include <cuda_runtime.h>

#include "fc_device.cuh"
#include "fc_launch.h"

namespace fc {

// DB = true: the next grid-stride iteration's loads are issued before the
// current iteration's math and stores (register double buffering), so a
// thread always has loads in flight.
template <int U, bool DB>
__global__ void __launch_bounds__(256) sgd_step_kernel(float4* __restrict__ w4,
                                                       const float4* __restrict__ g4,
                                                       float4* __restrict__ v4, int64_t n4,
                                                       float* __restrict__ wt,
                                                       const float* __restrict__ gt,
                                                       float* __restrict__ vt, int tail, float lr,
                                                       float mu, float wd, float inv_b,
                                                       const FcSegs segs, int64_t elem0,
                                                       FcLrDev* lrs) {
    if (lrs) {  // firecaffe_sgd_step_sched: the schedule at its current iteration
        __shared__ float s_lr;
        if (threadIdx.x == 0) s_lr = fc_lr_dev(lrs);
        __syncthreads();
        lr = s_lr;
    }
    const int64_t T = blockDim.x;
    const int64_t stride = (int64_t)gridDim.x * T * U;
    auto load = [&](int64_t base, float4* g, float4* w, float4* v) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = base + j * T;
            if (i < n4) {
                g[j] = ld_stream(g4 + i);
                w[j] = ld_rw(w4 + i);
                v[j] = ld_rw(v4 + i);
            }
        }
    };
    auto update = [&](int64_t base, float4* g, float4* w, float4* v) {
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = base + j * T;
            if (i < n4) {
                sgd4_any(segs, elem0 + 4 * i, g[j], w[j], v[j], lr, mu, wd, inv_b);
                st_na(w4 + i, w[j]);
                st_na(v4 + i, v[j]);
            }
        }
    };
    int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x;
    if constexpr (DB) {
        float4 g[U], w[U], v[U];
        load(base, g, w, v);
        while (base < n4) {
            float4 g2[U], w2[U], v2[U];
            load(base + stride, g2, w2, v2);
            update(base, g, w, v);
#pragma unroll
            for (int j = 0; j < U; ++j) {
                g[j] = g2[j];
                w[j] = w2[j];
                v[j] = v2[j];
            }
            base += stride;
        }
    } else {
        for (; base < n4; base += stride) {
            float4 g[U], w[U], v[U];
            load(base, g, w, v);
            update(base, g, w, v);
        }
    }
    // the n % 4 trailing elements
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x < tail) {
        const int t = threadIdx.x;
        float w = wt[t], v = vt[t];
        sgd1_any(segs, elem0 + 4 * n4 + t, gt[t], w, v, lr, mu, wd, inv_b);
        wt[t] = w;
        vt[t] = v;
    }
    if (lrs) {  // the last CTA to finish advances the iteration (all CTAs read it at entry)
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&lrs->done, 1u) + 1u == gridDim.x) {
                lrs->done = 0u;
                lrs->iter = lrs->iter + 1;
                __threadfence();
            }
        }
    }
}

// bf16-gradient variant: grad holds bf16 (upcast exactly to fp32),
// w and mom fp32; 4 elements per unit (8 B of gradient, 16 B of w and of mom),
// every access coalesced; U units per thread in flight.
template <int U>
__global__ void __launch_bounds__(256) sgd_step_bf16_kernel(float4* __restrict__ w4,
                                                            const uint2* __restrict__ g4,
                                                            float4* __restrict__ v4, int64_t n4,
                                                            int64_t n, float lr, float mu, float wd,
                                                            float inv_b, const FcSegs segs) {
    const int64_t T = blockDim.x;
    const int64_t stride = (int64_t)gridDim.x * T * U;
    for (int64_t b0 = (int64_t)blockIdx.x * T * U + threadIdx.x; b0 < n4; b0 += stride) {
        uint2 g[U];
        float4 w[U], v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = b0 + j * T;
            if (i < n4) {
                asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                             : "=r"(g[j].x), "=r"(g[j].y)
                             : "l"(g4 + i));
                w[j] = ld_rw(w4 + i);
                v[j] = ld_rw(v4 + i);
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = b0 + j * T;
            if (i < n4) {
                const float4 S = make_float4(__uint_as_float(g[j].x << 16), __uint_as_float(g[j].x & 0xffff0000u),
                                             __uint_as_float(g[j].y << 16), __uint_as_float(g[j].y & 0xffff0000u));
                sgd4_any(segs, 4 * i, S, w[j], v[j], lr, mu, wd, inv_b);
                st_na(w4 + i, w[j]);
                st_na(v4 + i, v[j]);
            }
        }
    }
    // the n % 4 trailing elements
    const int tail = (int)(n - 4 * n4);
    if (blockIdx.x == gridDim.x - 1 && (int)threadIdx.x < tail) {
        const int64_t e = 4 * n4 + threadIdx.x;
        float* wf = reinterpret_cast<float*>(w4);
        float* vf = reinterpret_cast<float*>(v4);
        const uint16_t h = reinterpret_cast<const uint16_t*>(g4)[e];
        float ww = wf[e], vv = vf[e];
        sgd1_any(segs, e, __uint_as_float((uint32_t)h << 16), ww, vv, lr, mu, wd, inv_b);
        wf[e] = ww;
        vf[e] = vv;
    }
}

cudaError_t launch_sgd_step_bf16(float* w, const uint16_t* grad, float* mom, int64_t n, float lr,
                                 float mu, float wd, float inv_b, const FcSegs& segs,
                                 cudaStream_t st) {
    constexpr int U = 4, T = 256;
    const int64_t n4 = n / 4;
    int occ = 0;
    occ = occupancy((const void*)sgd_step_bf16_kernel<U>, T);
    int64_t want = (n4 + (int64_t)T * U - 1) / ((int64_t)T * U);
    int64_t cap = (int64_t)dev_info().sms * (occ > 0 ? occ : 1);
    int64_t grid = want < cap ? want : cap;
    if (grid < 1) grid = 1;
    sgd_step_bf16_kernel<U><<<(unsigned)grid, T, 0, st>>>((float4*)w, (const uint2*)grad,
                                                          (float4*)mom, n4, n, lr, mu, wd, inv_b,
                                                          segs);
    return cudaGetLastError();
}

// 0 = automatic: register double-buffered, U = 2 below 32 M params and U = 1
// above (measured on B200, scripts/gpu_sgd_db.sh, profiles/r01_sgd_db.jsonl:
// NiN 22.6 vs 22.9 us, AlexNet 186 vs 192 us, VGG-19 445 vs 463 us against
// the single-buffered U = 4 kernel); tune_sgd_unroll(u) forces one shape.
static int g_sgd_unroll = 0;

cudaError_t launch_sgd_step(float* w, const float* grad, float* mom, int64_t n, float lr, float mu,
                            float wd, float inv_b, const FcSegs& segs, cudaStream_t st, FcLrDev* lrs) {
    return launch_sgd_step_range(w, grad, mom, 0, n, lr, mu, wd, inv_b, segs, st, lrs);
}

// Elements [off, off + len) (off a multiple of 4); blob lookups use absolute indices.
cudaError_t launch_sgd_step_range(float* w0, const float* grad0, float* mom0, int64_t off,
                                  int64_t len, float lr, float mu, float wd, float inv_b,
                                  const FcSegs& segs, cudaStream_t st, FcLrDev* lrs) {
    float* w = w0 + off;
    const float* grad = grad0 + off;
    float* mom = mom0 + off;
    const int64_t n = len;
    const int64_t n4 = n / 4;
    const int tail = (int)(n - n4 * 4);
    const int T = 256;
    const DevInfo& di = dev_info();
    auto run = [&](auto kern, int U) -> cudaError_t {
        int occ = 0;
        occ = occupancy((const void*)kern, T);
        int64_t want = (n4 + (int64_t)T * U - 1) / ((int64_t)T * U);
        int64_t cap = (int64_t)di.sms * (occ > 0 ? occ : 1);
        int64_t grid = want < cap ? want : cap;
        if (grid < 1) grid = 1;
        kern<<<(unsigned)grid, T, 0, st>>>((float4*)w, (const float4*)grad, (float4*)mom, n4,
                                           w + n4 * 4, grad + n4 * 4, mom + n4 * 4, tail, lr, mu,
                                           wd, inv_b, segs, off, lrs);
        return cudaGetLastError();
    };
    const int u = g_sgd_unroll != 0 ? g_sgd_unroll : (n < ((int64_t)32 << 20) ? -2 : -1);
    switch (u) {  // < 0: double-buffered with |u|
        case 1: return run(sgd_step_kernel<1, false>, 1);
        case 2: return run(sgd_step_kernel<2, false>, 2);
        case 8: return run(sgd_step_kernel<8, false>, 8);
        case -1: return run(sgd_step_kernel<1, true>, 1);
        case -2: return run(sgd_step_kernel<2, true>, 2);
        case -4: return run(sgd_step_kernel<4, true>, 4);
        default: return run(sgd_step_kernel<4, false>, 4);
    }
}

void set_sgd_unroll(int u) { g_sgd_unroll = u; }

}  // namespace fc
