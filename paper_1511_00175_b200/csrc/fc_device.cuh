// Device primitives for libfirecaffe (sm_100a).
//
// - 128-bit vector loads/stores with explicit cache policy (inline PTX).
// - System-scope release/acquire flags for cross-GPU synchronisation over
//   NVLink peer memory (flags live in the reserved prefix of each rank's heap).
// - The fp32 SGD rule with explicit round-to-nearest intrinsics so that nvcc
//   cannot contract or reorder it (the rounding sequence is part of the
//   contract, R6 / R11).
#pragma once
#include <stdint.h>

#include "fc_internal.h"

namespace fc {

// ---------------------------------------------------------------- loads ----
// Streaming load of data that nobody writes during the kernel (grad in the
// 1-GPU step): non-coherent path, no L1 allocation.
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
// Load of data this thread later overwrites (w, mom): coherent, no L1 allocation.
__device__ __forceinline__ float4 ld_rw(const float4* p) {
    float4 r;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
// Load of data another GPU (or another CTA) produced during this kernel, or of
// a peer GPU's memory: cache at L2 only (.cg), never L1 (L1 is not coherent).
__device__ __forceinline__ float4 ld_cg(const float4* p) {
    float4 r;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ float ld_cg1(const float* p) {
    float r;
    asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}
// ---------------------------------------------------------------- stores ---
__device__ __forceinline__ void st_na(float4* p, float4 v) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_cs(float4* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st1(float* p, float v) {
    asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

// ---------------------------------------------------------------- flags ----
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// System-scope fence of the exit / flag publication.  fence.sc is the stronger
// fence (it implies acq_rel), and measured 0.2-0.45 us cheaper than
// fence.acq_rel.sys on B200 with and without outstanding stores
// (profiles/r01_fence_bench.txt), so the stronger one is used.
__device__ __forceinline__ void fence_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ uint64_t ld_relaxed_sys64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_acquire_sys64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys64(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// flag >= epoch, modulo 2^32 (flags are monotonic epoch stamps, never reset)
__device__ __forceinline__ bool reached(uint32_t flag, uint32_t epoch) {
    return (int32_t)(flag - epoch) >= 0;
}

// Spin until *f has reached `epoch`.  Polls with relaxed sys-scope loads and
// performs ONE acquire load once the stamp is seen (acquire: later loads of
// the producer's data cannot be satisfied before the flag).  Bounded by
// timeout_ns of %globaltimer; on timeout records FC_ERR_TIMEOUT in *status
// and returns false.  Also gives up once any CTA has recorded an error (so one
// missing peer does not cost one timeout per wait).
__device__ __forceinline__ bool wait_flag(const uint32_t* f, uint32_t epoch, uint64_t timeout_ns,
                                          int* status) {
    if (reached(ld_acquire_sys(f), epoch)) return true;
    const uint64_t t0 = globaltimer();
    uint32_t spins = 0;
    while (true) {
        if (reached(ld_relaxed_sys(f), epoch)) {
            (void)ld_acquire_sys(f);
            return true;
        }
        if ((++spins & 63u) == 0) {
            if (*(volatile int*)status != FC_OK) return false;
            if (globaltimer() - t0 > timeout_ns) {
                atomicCAS(status, FC_OK, FC_ERR_TIMEOUT);
                return false;
            }
        }
    }
}

// ---------------------------------------------------------------- math -----
// One SGD element (R6): g = S*inv_b; d = fma(wd,w,g);
// v' = fma(mu, v, lr*d); w' = w - v'.  Explicit _rn intrinsics: no contraction.
__device__ __forceinline__ void sgd1(float S, float& w, float& v, float lr, float mu, float wd,
                                     float inv_b) {
    const float g = __fmul_rn(S, inv_b);
    const float d = __fmaf_rn(wd, w, g);
    const float t = __fmul_rn(lr, d);
    const float vn = __fmaf_rn(mu, v, t);
    w = __fsub_rn(w, vn);
    v = vn;
}
__device__ __forceinline__ void sgd4(const float4& S, float4& w, float4& v, float lr, float mu,
                                     float wd, float inv_b) {
    sgd1(S.x, w.x, v.x, lr, mu, wd, inv_b);
    sgd1(S.y, w.y, v.y, lr, mu, wd, inv_b);
    sgd1(S.z, w.z, v.z, lr, mu, wd, inv_b);
    sgd1(S.w, w.w, v.w, lr, mu, wd, inv_b);
}

// ---- Caffe per-blob multipliers (R20) ---------------------------
// Blob containing element e: largest k with begin[k] <= e (begin[0] == 0).
__device__ __forceinline__ int seg_find(const FcSegs& s, int64_t e) {
    int lo = 0, hi = s.nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(s.begin + mid) <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}
__device__ __forceinline__ void sgd1_seg(const FcSegs& s, int64_t e, float S, float& w, float& v,
                                         float lr, float mu, float wd, float inv_b) {
    const int k = seg_find(s, e);
    sgd1(S, w, v, __fmul_rn(lr, __ldg(s.lrm + k)), mu, __fmul_rn(wd, __ldg(s.dm + k)), inv_b);
}
// Four consecutive elements e..e+3; one lookup unless a blob boundary falls inside.
__device__ __forceinline__ void sgd4_seg(const FcSegs& s, int64_t e, const float4& S, float4& w,
                                         float4& v, float lr, float mu, float wd, float inv_b) {
    const int k = seg_find(s, e);
    const bool whole = (k + 1 >= s.nseg) || (__ldg(s.begin + k + 1) > e + 3);
    if (whole) {
        sgd4(S, w, v, __fmul_rn(lr, __ldg(s.lrm + k)), mu, __fmul_rn(wd, __ldg(s.dm + k)), inv_b);
    } else {
        sgd1_seg(s, e + 0, S.x, w.x, v.x, lr, mu, wd, inv_b);
        sgd1_seg(s, e + 1, S.y, w.y, v.y, lr, mu, wd, inv_b);
        sgd1_seg(s, e + 2, S.z, w.z, v.z, lr, mu, wd, inv_b);
        sgd1_seg(s, e + 3, S.w, w.w, v.w, lr, mu, wd, inv_b);
    }
}
// Dispatch: uniform fast path when no table is given.
__device__ __forceinline__ void sgd4_any(const FcSegs& s, int64_t e, const float4& S, float4& w,
                                         float4& v, float lr, float mu, float wd, float inv_b) {
    if (s.nseg > 0) sgd4_seg(s, e, S, w, v, lr, mu, wd, inv_b);
    else sgd4(S, w, v, lr, mu, wd, inv_b);
}
__device__ __forceinline__ void sgd1_any(const FcSegs& s, int64_t e, float S, float& w, float& v,
                                         float lr, float mu, float wd, float inv_b) {
    if (s.nseg > 0) sgd1_seg(s, e, S, w, v, lr, mu, wd, inv_b);
    else sgd1(S, w, v, lr, mu, wd, inv_b);
}

__device__ __forceinline__ float4 add4(const float4& a, const float4& b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                       __fadd_rn(a.w, b.w));
}

// k-nomial tree association over P register values, rooted at index 0, in
// absolute rank space (R1): at step s = K^l, node r (r % (K*s) == 0)
// absorbs r + j*s for j = 1..K-1 ascending.  Fully unrolled at compile time.
template <int P, int K>
__device__ __forceinline__ float4 tree_sum_regs(float4 (&x)[P]) {
#pragma unroll
    for (int s = 1; s < P; s *= K) {
#pragma unroll
        for (int r = 0; r < P; r += K * s) {
#pragma unroll
            for (int j = 1; j < K; ++j) {
                const int c = r + j * s;
                if (c < P) x[r] = add4(x[r], x[c]);
            }
        }
    }
    return x[0];
}
template <int P, int K>
__device__ __forceinline__ float tree_sum_regs1(float (&x)[P]) {
#pragma unroll
    for (int s = 1; s < P; s *= K) {
#pragma unroll
        for (int r = 0; r < P; r += K * s) {
#pragma unroll
            for (int j = 1; j < K; ++j) {
                const int c = r + j * s;
                if (c < P) x[r] = __fadd_rn(x[r], x[c]);
            }
        }
    }
    return x[0];
}

}  // namespace fc
