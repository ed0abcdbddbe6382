// Host-buffer entry points: the 1-GPU fused SGD with the gradient coming from
// (pinned) host memory and the updated weights going back to it, pipelined in
// chunks over three streams so that the H2D copy of chunk i+1, the SGD kernel
// of chunk i and the D2H copy of chunk i-1 overlap (PCIe is full duplex: the
// two copy directions run on separate copy engines).
#include <cuda_runtime.h>
#include <stdint.h>

#include "fc_device.cuh"
#include "fc_launch.h"

namespace fc {

// Zero-copy variant: ONE kernel reads the gradient straight from pinned host
// memory over PCIe (UVA-mapped), keeps a device copy in `grad_dev`, applies the
// SGD against w/mom in HBM and writes the new weights both to HBM and straight
// back to pinned host memory.  PCIe reads (gradient) and posted writes
// (weights) stream concurrently in both directions with no copy-engine stages
// to fill or drain.
template <int U>
__global__ void __launch_bounds__(256) sgd_step_hostio_kernel(
    float4* __restrict__ w4, const float4* __restrict__ gh4, float4* __restrict__ gd4,
    float4* __restrict__ v4, float4* __restrict__ wh4, int64_t n4, int64_t n, float lr, float mu,
    float wd, float inv_b, const FcSegs segs, int64_t elem0) {
    const int64_t T = blockDim.x;
    const int64_t stride = (int64_t)gridDim.x * T * U;
    for (int64_t b0 = (int64_t)blockIdx.x * T * U + threadIdx.x; b0 < n4; b0 += stride) {
        float4 g[U], w[U], v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = b0 + j * T;
            if (i < n4) {
                g[j] = gh4[i];  // PCIe read of pinned host memory
                w[j] = ld_rw(w4 + i);
                v[j] = ld_rw(v4 + i);
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = b0 + j * T;
            if (i < n4) {
                if (gd4) st_na(gd4 + i, g[j]);
                sgd4_any(segs, elem0 + 4 * i, g[j], w[j], v[j], lr, mu, wd, inv_b);
                st_na(w4 + i, w[j]);
                st_na(v4 + i, v[j]);
                wh4[i] = w[j];  // PCIe posted write to pinned host memory
            }
        }
    }
    const int tail = (int)(n - 4 * n4);
    if (blockIdx.x == gridDim.x - 1 && (int)threadIdx.x < tail) {
        const int64_t e = 4 * n4 + threadIdx.x;
        const float gg = reinterpret_cast<const float*>(gh4)[e];
        float* wf = reinterpret_cast<float*>(w4);
        float* vf = reinterpret_cast<float*>(v4);
        if (gd4) reinterpret_cast<float*>(gd4)[e] = gg;
        float ww = wf[e], vv = vf[e];
        sgd1_any(segs, elem0 + e, gg, ww, vv, lr, mu, wd, inv_b);
        wf[e] = ww;
        vf[e] = vv;
        reinterpret_cast<float*>(wh4)[e] = ww;
    }
}

cudaError_t launch_sgd_step_hostio(float* w, const float* grad_host, float* grad_dev, float* mom,
                                   float* w_host, int64_t n, float lr, float mu, float wd,
                                   float inv_b, const FcSegs& segs, cudaStream_t st) {
    constexpr int U = 4, T = 256;
    const int64_t n4 = n / 4;
    int occ = 0;
    occ = occupancy((const void*)sgd_step_hostio_kernel<U>, T);
    int64_t want = (n4 + (int64_t)T * U - 1) / ((int64_t)T * U);
    int64_t cap = (int64_t)dev_info().sms * (occ > 0 ? occ : 1);
    int64_t grid = want < cap ? want : cap;
    if (grid < 1) grid = 1;
    sgd_step_hostio_kernel<U><<<(unsigned)grid, T, 0, st>>>(
        (float4*)w, (const float4*)grad_host, (float4*)grad_dev, (float4*)mom, (float4*)w_host, n4,
        n, lr, mu, wd, inv_b, segs, 0);
    return cudaGetLastError();
}



struct PipeCtx {
    bool ready = false;
    cudaStream_t s[3];             // 0: H2D, 1: compute, 2: D2H
    cudaEvent_t start;             // user stream -> internal streams
    cudaEvent_t h2d[kPipeDepth], comp[kPipeDepth], d2h[kPipeDepth];
};

static PipeCtx g_pipe[64];

static cudaError_t pipe_ctx(PipeCtx** out) {
    int d = 0;
    cudaError_t e = cudaGetDevice(&d);
    if (e != cudaSuccess) return e;
    if (d < 0 || d >= 64) return cudaErrorInvalidDevice;
    PipeCtx& p = g_pipe[d];
    if (!p.ready) {
        for (int i = 0; i < 3; ++i)
            if ((e = cudaStreamCreateWithFlags(&p.s[i], cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming)) != cudaSuccess) return e;
        for (int i = 0; i < kPipeDepth; ++i) {
            if ((e = cudaEventCreateWithFlags(&p.h2d[i], cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&p.comp[i], cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&p.d2h[i], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        p.ready = true;
    }
    *out = &p;
    return cudaSuccess;
}

cudaError_t launch_sgd_step_host(float* w, const float* grad_host, float* grad_dev, float* mom,
                                 float* w_host, int64_t n, float lr, float mu, float wd,
                                 float inv_b, const FcSegs& segs, int64_t chunk,
                                 cudaStream_t user) {
    PipeCtx* p = nullptr;
    cudaError_t e = pipe_ctx(&p);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(p->start, user)) != cudaSuccess) return e;
    for (int i = 0; i < 3; ++i)
        if ((e = cudaStreamWaitEvent(p->s[i], p->start, 0)) != cudaSuccess) return e;
    // Uniform stages (measured on B200, NiN: 2M-float stages 0.84 ms; 0.5M 0.96 ms;
    // a small-first/small-last ramp did not help; H2D || D2H alone is 0.66 ms).
    const int64_t nst = (n + chunk - 1) / chunk;
    int64_t off = 0;
    for (int64_t k = 0; k < nst; ++k) {
        const int64_t len = off + chunk <= n ? chunk : n - off;
        const int slot = (int)(k % kPipeDepth);
        // H2D of chunk k (reuses staging only through grad_dev, which is per-chunk disjoint)
        if ((e = cudaMemcpyAsync(grad_dev + off, grad_host + off, len * 4, cudaMemcpyHostToDevice,
                                 p->s[0])) != cudaSuccess)
            return e;
        if ((e = cudaEventRecord(p->h2d[slot], p->s[0])) != cudaSuccess) return e;
        // SGD on chunk k
        if ((e = cudaStreamWaitEvent(p->s[1], p->h2d[slot], 0)) != cudaSuccess) return e;
        // (the blob table is indexed by absolute element; the range launcher passes `off`)
        if ((e = launch_sgd_step_range(w, grad_dev, mom, off, len, lr, mu, wd, inv_b, segs, p->s[1])) !=
            cudaSuccess)
            return e;
        if ((e = cudaEventRecord(p->comp[slot], p->s[1])) != cudaSuccess) return e;
        // D2H of chunk k's updated weights
        if ((e = cudaStreamWaitEvent(p->s[2], p->comp[slot], 0)) != cudaSuccess) return e;
        if ((e = cudaMemcpyAsync(w_host + off, w + off, len * 4, cudaMemcpyDeviceToHost, p->s[2])) !=
            cudaSuccess)
            return e;
        if ((e = cudaEventRecord(p->d2h[slot], p->s[2])) != cudaSuccess) return e;
        off += len;
    }
    // the user's stream continues after every copy has landed
    if ((e = cudaEventRecord(p->start, p->s[2])) != cudaSuccess) return e;
    return cudaStreamWaitEvent(user, p->start, 0);
}

}  // namespace fc

namespace fc {

// Hybrid pipeline: the copy engine brings each stage's gradient in (H2D), the
// SGD kernel of that stage writes the new weights straight to pinned host
// memory (SM posted writes), so the two PCIe directions run concurrently
// without a D2H copy stage.
cudaError_t launch_sgd_step_hybrid(float* w, const float* grad_host, float* grad_dev, float* mom,
                                   float* w_host_dev, int64_t n, float lr, float mu, float wd,
                                   float inv_b, const FcSegs& segs, int64_t chunk,
                                   cudaStream_t user) {
    PipeCtx* p = nullptr;
    cudaError_t e = pipe_ctx(&p);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(p->start, user)) != cudaSuccess) return e;
    for (int i = 0; i < 2; ++i)
        if ((e = cudaStreamWaitEvent(p->s[i], p->start, 0)) != cudaSuccess) return e;
    constexpr int U = 4, T = 256;
    const int occ = occupancy((const void*)sgd_step_hostio_kernel<U>, T);
    const int64_t cap = (int64_t)dev_info().sms * (occ > 0 ? occ : 1);
    const int64_t nst = (n + chunk - 1) / chunk;
    int64_t off = 0;
    for (int64_t k = 0; k < nst; ++k) {
        const int64_t len = off + chunk <= n ? chunk : n - off;
        const int slot = (int)(k % kPipeDepth);
        if ((e = cudaMemcpyAsync(grad_dev + off, grad_host + off, len * 4, cudaMemcpyHostToDevice,
                                 p->s[0])) != cudaSuccess)
            return e;
        if ((e = cudaEventRecord(p->h2d[slot], p->s[0])) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(p->s[1], p->h2d[slot], 0)) != cudaSuccess) return e;
        const int64_t n4 = len / 4;
        int64_t grid = (n4 + (int64_t)T * U - 1) / ((int64_t)T * U);
        if (grid > cap) grid = cap;
        if (grid < 1) grid = 1;
        sgd_step_hostio_kernel<U><<<(unsigned)grid, T, 0, p->s[1]>>>(
            (float4*)(w + off), (const float4*)(grad_dev + off), nullptr, (float4*)(mom + off),
            (float4*)(w_host_dev + off), n4, len, lr, mu, wd, inv_b, segs, off);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        off += len;
    }
    if ((e = cudaEventRecord(p->start, p->s[1])) != cudaSuccess) return e;
    return cudaStreamWaitEvent(user, p->start, 0);
}

}  // namespace fc
