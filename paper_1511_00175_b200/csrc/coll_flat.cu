// FLAT-family collective kernels: the bf16-wire
// variant of the FLAT executor, the owned-slice all-gather, and the kernel
// table of the fp32 FLAT executor / parameter server (whose template is in
// coll_flat.cuh).  One persistent kernel per call, one CTA per SM; see
// coll_common.cuh for the synchronisation.
#include <stdlib.h>

#include "coll_flat.cuh"

namespace fc {

// ------------------------------------------------------------ FLAT, bf16 wire
// SURVEY §8 f4 (16-bit gradients on the wire).  Every rank's
// gradient is bf16; the owner upcasts each operand exactly to fp32 and then
// evaluates the same K-nomial tree in fp32 (R22), applies SGD in
// fp32 and pushes fp32 weights.  The reduce phase moves half the bytes.
__device__ __forceinline__ float bf16_to_f32(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }
__device__ __forceinline__ const uint16_t* gradh_of(const FcColl& c, int q) {
    return reinterpret_cast<const uint16_t*>(c.peers.heap[q] + c.off_grad);
}

// 4 elements per unit: 8-byte bf16 loads and float4 weight accesses are both
// fully coalesced per warp; U units per thread keep (P-1)*8*U remote bytes in
// flight per thread.  Work mapping: the plain grid stride (the fp32 FLAT
// kernel's dynamic claims were tried here too and measured equal at p = 2 and
// 1 % slower at p = 4, profiles/r02_bf16_dyn_vs_stride.txt; not kept).  p = 2: U = 6 is spill-free (U = 8 spilled 20 B/thread;
// measured NiN +2 %, AlexNet -1 % time vs U = 8, scripts/gpu_bf16_unroll.sh).
#define BF16_UNROLL(P) ((P) <= 2 ? 6 : (P) <= 4 ? 4 : 1)
__device__ __forceinline__ uint2 ld_cg_u2(const uint2* p) {
    uint2 r;
    asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ float4 bf16x4_to_f32(const uint2 u) {
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                       __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
}

template <int P, int K>
__global__ void __launch_bounds__(FLAT_T) flat_bf16_kernel(const __grid_constant__ FcColl c) {
    constexpr int U = BF16_UNROLL(P);
    const int rank = my_rank(c);
    epoch_begin(c);
    trace(c, 0);
    const bool ok = cta_barrier(c, rank, 0);
    trace(c, 1);
    if (ok) {
        const int64_t nch = (c.n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
        int64_t c0, c1;
        owned_chunks(rank, P, nch, false, &c0, &c1);
        const int64_t e0 = c0 * FC_CHUNK_FLOATS;
        const int64_t e1 = min(c1 * FC_CHUNK_FLOATS, c.n);
        if (e1 > e0) {
            const int64_t i0 = e0 / 4, i1 = e1 / 4;  // units of 4 elements (8 B of bf16)
            float4* w4 = reinterpret_cast<float4*>(w_of(c, rank));
            float4* v4 = reinterpret_cast<float4*>(mom_of(c, rank));
            const int64_t T = FLAT_T;
            const int64_t stride = (int64_t)gridDim.x * T * U;
            for (int64_t base = i0 + (int64_t)blockIdx.x * T * U + threadIdx.x; base < i1; base += stride) {
                uint2 x[U][P];
                float4 w[U], v[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int64_t i = base + j * T;
                    if (i < i1) {
#pragma unroll
                        for (int q = 0; q < P; ++q)
                            x[j][q] = ld_cg_u2(reinterpret_cast<const uint2*>(gradh_of(c, q)) + i);
                    }
                }
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int64_t i = base + j * T;
                    if (i < i1) {
                        w[j] = ld_rw(w4 + i);
                        v[j] = ld_rw(v4 + i);
                    }
                }
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int64_t i = base + j * T;
                    if (i < i1) {
                        float4 f[P];
#pragma unroll
                        for (int q = 0; q < P; ++q) f[q] = bf16x4_to_f32(x[j][q]);
                        const float4 S = tree_sum_regs<P, K>(f);
                        sgd4_any(c.segs, 4 * i, S, w[j], v[j], s_lr, c.mu, c.wd, c.inv_b);
                        st_na(v4 + i, v[j]);
#pragma unroll
                        for (int q = 0; q < P; ++q) st_na(reinterpret_cast<float4*>(w_of(c, q)) + i, w[j]);
                    }
                }
            }
            const int rem = (int)(e1 - 4 * i1);  // trailing n % 4 elements of the last slice
            if (blockIdx.x == 0 && (int)threadIdx.x < rem) {
                const int64_t e = 4 * i1 + threadIdx.x;
                float xs[P];
#pragma unroll
                for (int q = 0; q < P; ++q) xs[q] = bf16_to_f32(gradh_of(c, q)[e]);
                const float S = tree_sum_regs1<P, K>(xs);
                float ww = w_of(c, rank)[e], vv = mom_of(c, rank)[e];
                sgd1_any(c.segs, e, S, ww, vv, s_lr, c.mu, c.wd, c.inv_b);
                st1(mom_of(c, rank) + e, vv);
                for (int q = 0; q < P; ++q) st1(w_of(c, q) + e, ww);
            }
        }
    }
    trace(c, 2);
    finish_call(c, rank);
}

// ------------------------------------------------------------ ALLGATHER ----
// op FC_OP_ALLGATHER_OWNED: every rank pushes its owned slice of a symmetric
// buffer (off_grad) to every other rank, so all ranks end with the full vector
// (e.g. the sharded momentum of the fused update, for a checkpoint: R18).
template <int P>
__global__ void __launch_bounds__(FLAT_T) allgather_kernel(const __grid_constant__ FcColl c) {
    const int rank = my_rank(c);
    epoch_begin(c);
    trace(c, 0);
    const bool ok = cta_barrier(c, rank, 0);
    trace(c, 1);
    if (ok) {
        const int64_t nch = (c.n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
        int64_t c0, c1;
        owned_chunks(rank, P, nch, c.owner_single_root != 0, &c0, &c1);
        const int64_t e0 = c0 * FC_CHUNK_FLOATS;
        const int64_t e1 = min(c1 * FC_CHUNK_FLOATS, c.n);
        if (e1 > e0) {
            const int64_t i0 = e0 / 4, i1 = e1 / 4;
            const float4* src = reinterpret_cast<const float4*>(grad_of(c, rank));
            const int64_t stride = (int64_t)gridDim.x * FLAT_T * 2;
            for (int64_t base = i0 + (int64_t)blockIdx.x * FLAT_T * 2 + threadIdx.x; base < i1; base += stride) {
                float4 x[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int64_t i = base + j * FLAT_T;
                    if (i < i1) x[j] = ld_cg(src + i);
                }
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int64_t i = base + j * FLAT_T;
                    if (i < i1) {
#pragma unroll
                        for (int q = 0; q < P; ++q)
                            if (q != rank) st_na(reinterpret_cast<float4*>(grad_of(c, q)) + i, x[j]);
                    }
                }
            }
            const int rem = (int)(e1 - 4 * i1);
            if (blockIdx.x == 0 && (int)threadIdx.x < rem) {
                const int64_t e = 4 * i1 + threadIdx.x;
                const float v = ld_cg1(grad_of(c, rank) + e);
                for (int q = 0; q < P; ++q)
                    if (q != rank) st1(grad_of(c, q) + e, v);
            }
        }
    }
    trace(c, 2);
    finish_call(c, rank);
}

// ------------------------------------------------------------ kernel tables -
// Unroll override for tuning experiments (FC_FLAT_UNROLL=1|2|4; 0 = default).
static int flat_unroll_override() {
    static int u = -1;
    if (u < 0) {
        const char* e = getenv("FC_FLAT_UNROLL");
        u = e ? atoi(e) : 0;
    }
    return u;
}

const void* flat_kernel_for(int p, int arity) {
    switch (flat_unroll_override()) {
        case 1: return flat_kernel_u1(p, arity);
        case 2: return flat_kernel_u2(p, arity);
        case 4: return flat_kernel_u4(p, arity);
        default:
            switch (FLAT_UNROLL(p)) {
                case 4: return flat_kernel_u4(p, arity);
                case 2: return flat_kernel_u2(p, arity);
                default: return flat_kernel_u1(p, arity);
            }
    }
}

template <int P>
static const void* bf16_for(int K) {
    if (K >= P) K = P;
    switch (K) {
        case 2: return (const void*)flat_bf16_kernel<P, 2>;
#define FC_K(k) case k: if constexpr (P >= k) return (const void*)flat_bf16_kernel<P, k>; else return nullptr;
        FC_K(3) FC_K(4) FC_K(5) FC_K(6) FC_K(7) FC_K(8)
#undef FC_K
    }
    return nullptr;
}

const void* flat_bf16_kernel_for(int p, int arity) {
    switch (p) {
#define FC_P(PP) case PP: return bf16_for<PP>(arity);
        FC_P(2) FC_P(3) FC_P(4) FC_P(5) FC_P(6) FC_P(7) FC_P(8)
#undef FC_P
    }
    return nullptr;
}

const void* allgather_kernel_for(int p) {
    switch (p) {
#define FC_P(PP) case PP: return (const void*)allgather_kernel<PP>;
        FC_P(2) FC_P(3) FC_P(4) FC_P(5) FC_P(6) FC_P(7) FC_P(8)
#undef FC_P
    }
    return nullptr;
}

}  // namespace fc
