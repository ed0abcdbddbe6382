// Collective kernels of libfirecaffe: the reduction tree over NVLink peer
// memory: one persistent kernel per call (one wave of CTAs;
// a cooperative launch for virtual worlds, whose CTAs wait on each other).
//
// Every rank's heap is mapped into every process (CUDA IPC), so a kernel reads
// a peer GPU's gradient slice with ordinary 128-bit loads and writes a peer's
// weights with ordinary 128-bit stores; both cross NVLink / NVSwitch.  Order
// between GPUs comes from epoch-stamped flags in the heaps' reserved prefix
// (st.release.sys / ld.acquire.sys).  Producers PUSH flags to the consumer's
// heap so that every spin is on local memory.
//
// Schedules (include/firecaffe.h fc_sched) — all produce the same bits, the
// k-nomial association of DESIGN.md R1:
//   FLAT        each rank pulls its owner slice from all p ranks, evaluates
//               the whole tree in registers, applies SGD, pushes w' to all.
//   FOREST      recursive halving: at level l rank r pulls |W|/2^(l+1) from
//               r^2^l (the binomial tree of slice s is rooted at its owner);
//               SGD fused into the last level; tree or direct broadcast.
//   SINGLE_ROOT the paper's binomial tree rooted at rank 0 (Fig. P:312-315);
//               the root applies SGD to all of W, then broadcast.
//   PS          (op FC_OP_PS) rank 0 pulls everything, sequential sum, pushes.
// Static work mapping: chunk cc (FC_CHUNK_FLOATS floats) is always processed
// by CTA cc % gridDim.x, element k of a chunk always by the same thread, so a
// rank's own partial sums need no flags between levels (program order).
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "fc_device.cuh"
#include "fc_launch.h"

namespace fc {

constexpr int TREE_T = 256;                       // threads per CTA (tree schedules)
constexpr int FLAT_T = 512;                       // threads per CTA (FLAT / PS), one CTA per SM
// float4 per thread per operand in flight in FLAT: enough remote bytes in flight
// (148 CTAs x 512 thr x (P-1) x U x 16 B >= 2.4 MB) at <= 128 registers
// (measured: U = 4 best at p = 2, U = 2 at p = 4; profiles/r01_sweep_flat_unroll_*)
#define FLAT_UNROLL(P) ((P) <= 2 ? 4 : 2)
constexpr int C4 = FC_CHUNK_FLOATS / 4;           // float4 per chunk (1024)
constexpr int PER_T = C4 / TREE_T;                // float4 per thread per chunk (4)
static_assert(C4 % TREE_T == 0, "chunk must split evenly over the CTA");

// ------------------------------------------------------------ addressing ---
__device__ __forceinline__ int my_rank(const FcColl& c) {
    return c.rank >= 0 ? c.rank : (int)blockIdx.y;
}
__device__ __forceinline__ uint32_t* flag_base(const FcColl& c, int q) {
    return reinterpret_cast<uint32_t*>(c.peers.heap[q]);
}
__device__ __forceinline__ uint64_t* bar_flag(const FcColl& c, int owner, int slot, int cta,
                                              int src) {
    return reinterpret_cast<uint64_t*>(flag_base(c, owner)) +
           ((int64_t)(slot * FC_MAX_CTAS + cta) * FC_MAX_RANKS + src);
}
__device__ __forceinline__ uint32_t* red_flag(const FcColl& c, int owner, int l, int64_t cc) {
    return flag_base(c, owner) + c.bar_words + (int64_t)l * c.max_chunks + cc;
}
__device__ __forceinline__ uint32_t* av_flag(const FcColl& c, int owner, int64_t cc) {
    return flag_base(c, owner) + c.red_words + cc;
}
__device__ __forceinline__ float* grad_of(const FcColl& c, int q) {
    return reinterpret_cast<float*>(c.peers.heap[q] + c.off_grad);
}
__device__ __forceinline__ float* w_of(const FcColl& c, int q) {
    return reinterpret_cast<float*>(c.peers.heap[q] + c.off_w);
}
__device__ __forceinline__ float* mom_of(const FcColl& c, int q) {
    return c.off_mom >= 0 ? reinterpret_cast<float*>(c.peers.heap[q] + c.off_mom) : c.mom_local;
}

__device__ __forceinline__ void trace(const FcColl& c, int slot) {
    if (c.trace && threadIdx.x == 0)
        c.trace[((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * FC_TRACE_SLOTS + slot] = globaltimer();
}

// ------------------------------------------------------------ epochs -------
// The call counter lives in device memory (c.ctl[0] = epoch of the last
// completed call, c.ctl[1] = CTAs finished in the current call), so a call's
// kernel arguments never change from call to call and the collectives can be
// captured in a CUDA graph and replayed.  Every CTA reads the epoch at entry;
// the last CTA to finish publishes the next one (stream order makes it visible
// to the next launch).  All ranks make the same calls, so the counters agree.
__shared__ uint32_t s_epoch;

__device__ __forceinline__ void epoch_begin(const FcColl& c) {
    if (threadIdx.x == 0) s_epoch = *(volatile uint32_t*)c.ctl + 1u;
    __syncthreads();
}

__device__ __forceinline__ void epoch_end(const FcColl& c) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t total = gridDim.x * gridDim.y;
        const uint32_t done = atomicAdd(c.ctl + 1, 1u) + 1u;
        if (done == total) {
            c.ctl[1] = 0u;
            __threadfence();
            atomicExch(c.ctl, s_epoch);
        }
    }
}

// ------------------------------------------------------------ sync ---------
// All-to-all barrier among the CTAs with this blockIdx.x on every rank
// (slot 0 = entry, 1 = exit).  Thread q < p pushes "rank arrived" into rank q's
// heap, then spins on rank q's stamp in the local heap.
//  entry (slot 0): the stamp orders nothing the CTA wrote (the rank's inputs
//    were produced by earlier kernels, complete and coherent in its L2), so it
//    is a relaxed store: no fence on the critical path.
//  exit (slot 1): st.release.sys orders the CTA's earlier writes — peer stores
//    included; the __syncthreads orders the other threads' writes before it
//    (PTX causality through bar.sync) — ahead of the stamp.
// A stamp is one 64-bit word: epoch | signature << 32.  The signature hashes the
// call's op, n, executor and hyper-parameters; a peer whose signature differs
// made a different call (MPI/NCCL rule broken) -> sticky FC_ERR_MISMATCH on
// every rank and no data is touched.
__device__ bool cta_barrier(const FcColl& c, int rank, int slot) {
    __syncthreads();
    const int t = threadIdx.x;
    bool good = true;
    if (t < c.p && t != rank) {
        const uint64_t stamp = (uint64_t)s_epoch | ((uint64_t)c.sig << 32);
        uint64_t* dst = bar_flag(c, t, slot, blockIdx.x, rank);
        if (slot == 0) st_relaxed_sys64(dst, stamp);
        else st_release_sys64(dst, stamp);
        const uint64_t* f = bar_flag(c, rank, slot, blockIdx.x, t);
        uint64_t v = ld_acquire_sys64(f);
        if (!reached((uint32_t)v, s_epoch)) {
            const uint64_t t0 = globaltimer();
            uint32_t spins = 0;
            while (true) {
                v = ld_relaxed_sys64(f);
                if (reached((uint32_t)v, s_epoch)) {
                    v = ld_acquire_sys64(f);
                    break;
                }
                if ((++spins & 63u) == 0) {
                    if (*(volatile int*)c.status != FC_OK) { good = false; break; }
                    if (globaltimer() - t0 > c.timeout_ns) {
                        atomicCAS(c.status, FC_OK, FC_ERR_TIMEOUT);
                        good = false;
                        break;
                    }
                }
            }
        }
        if (good && (uint32_t)v == s_epoch && (uint32_t)(v >> 32) != c.sig) {
            atomicCAS(c.status, FC_OK, FC_ERR_MISMATCH);
            good = false;
        }
    }
    return __syncthreads_and(good) != 0;
}

// One thread waits for a flag; the CTA learns the outcome.
__device__ __forceinline__ bool wait_one(const FcColl& c, const uint32_t* f) {
    bool good = true;
    if (threadIdx.x == 0) good = wait_flag(f, s_epoch, c.timeout_ns, c.status);
    return __syncthreads_and(good) != 0;
}

// Publish the CTA's last `count` chunks (cc_last, cc_last - G, ...) after ONE
// sys-scope release fence: thread 0 fences (ordering every thread's chunk
// writes, sequenced before it by the bar.sync) and then writes the consumers'
// epoch stamps with relaxed stores (`stamp(cc)` does the stores for one
// chunk).  A sys fence costs 4-8 us on B200 (scripts/fence_bench.cu), so the
// tree schedules pay one per PUB chunks instead of one per chunk.
constexpr int PUB = 8;
template <typename Stamp>
__device__ __forceinline__ void publish_batch(const FcColl& c, int64_t cc_last, int G, int count,
                                              Stamp stamp) {
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_sys();
        for (int k = 0; k < count; ++k) stamp(cc_last - (int64_t)k * G);
    }
}

__device__ __forceinline__ int64_t first_chunk(int64_t lo, int G, int b) {
    const int64_t r = lo % G;
    return lo + ((b - r) % G + G) % G;
}

// ------------------------------------------------------------ chunk ops ----
// Level step on chunk cc: s = own partial + peer partial (R1: the
// lower rank group's partial plus the upper group's; fp32 addition commutes
// bitwise, so operand order is immaterial).  Not last: s -> own grad (in
// place).  Last (subtree root): fused -> SGD on w, mom; unfused -> s -> grad.
// `push`: bitmask of ranks that also receive the result right away (last level
// only): every other rank for a direct broadcast, the first broadcast hop for
// a tree broadcast, so the root's link sends while it still receives.
template <int P>
__device__ __forceinline__ void reduce_chunk(const FcColl& c, int rank, int64_t cc, float* own,
                                             const float* peer, bool last, bool fused,
                                             uint32_t push) {
    const int64_t e0 = cc * FC_CHUNK_FLOATS;
    const int64_t e1 = min(e0 + (int64_t)FC_CHUNK_FLOATS, c.n);
    const int nf4 = (int)((e1 - e0) >> 2);
    const int rem = (int)((e1 - e0) & 3);
    const int t = threadIdx.x;
    float4* own4 = reinterpret_cast<float4*>(own + e0);
    const float4* peer4 = reinterpret_cast<const float4*>(peer + e0);
    float4 a[PER_T], b[PER_T];
#pragma unroll
    for (int j = 0; j < PER_T; ++j) {
        const int k = j * TREE_T + t;
        if (k < nf4) {
            a[j] = ld_cg(own4 + k);
            b[j] = ld_cg(peer4 + k);
        }
    }
    if (!last || !fused) {
#pragma unroll
        for (int j = 0; j < PER_T; ++j) {
            const int k = j * TREE_T + t;
            if (k < nf4) {
                const float4 s = add4(a[j], b[j]);
                st_na(own4 + k, s);
                if (last && push) {
#pragma unroll
                    for (int q = 0; q < P; ++q)
                        if ((push >> q) & 1u) st_na(reinterpret_cast<float4*>(grad_of(c, q) + e0) + k, s);
                }
            }
        }
        if (t < rem) {
            const int64_t e = e0 + 4 * (int64_t)nf4 + t;
            const float s = __fadd_rn(ld_cg1(own + e), ld_cg1(peer + e));
            st1(own + e, s);
            if (last && push)
                for (int q = 0; q < P; ++q)
                    if ((push >> q) & 1u) st1(grad_of(c, q) + e, s);
        }
        return;
    }
    // last level, fused SGD: the reduced gradient lives only in registers
    float4* w4 = reinterpret_cast<float4*>(w_of(c, rank) + e0);
    float4* v4 = reinterpret_cast<float4*>(mom_of(c, rank) + e0);
    float4 w[PER_T], v[PER_T];
#pragma unroll
    for (int j = 0; j < PER_T; ++j) {
        const int k = j * TREE_T + t;
        if (k < nf4) {
            w[j] = ld_rw(w4 + k);
            v[j] = ld_rw(v4 + k);
        }
    }
#pragma unroll
    for (int j = 0; j < PER_T; ++j) {
        const int k = j * TREE_T + t;
        if (k < nf4) {
            const float4 s = add4(a[j], b[j]);
            sgd4_any(c.segs, e0 + 4 * (int64_t)k, s, w[j], v[j], c.lr, c.mu, c.wd, c.inv_b);
            st_na(w4 + k, w[j]);
            st_na(v4 + k, v[j]);
            if (push) {
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if ((push >> q) & 1u) st_na(reinterpret_cast<float4*>(w_of(c, q) + e0) + k, w[j]);
            }
        }
    }
    if (t < rem) {
        const int64_t e = e0 + 4 * (int64_t)nf4 + t;
        const float s = __fadd_rn(ld_cg1(own + e), ld_cg1(peer + e));
        float* wp = w_of(c, rank) + e;
        float* vp = mom_of(c, rank) + e;
        float ww = *wp, vv = *vp;
        sgd1_any(c.segs, e, s, ww, vv, c.lr, c.mu, c.wd, c.inv_b);
        st1(wp, ww);
        st1(vp, vv);
        if (push)
            for (int q = 0; q < P; ++q)
                if ((push >> q) & 1u) st1(w_of(c, q) + e, ww);
    }
}

// Copy chunk cc of `src` (local) to up to 3 destinations (peers).
__device__ __forceinline__ void copy_chunk(const FcColl& c, int64_t cc, const float* src,
                                           float* const* dst, int ndst) {
    const int64_t e0 = cc * FC_CHUNK_FLOATS;
    const int64_t e1 = min(e0 + (int64_t)FC_CHUNK_FLOATS, c.n);
    const int nf4 = (int)((e1 - e0) >> 2);
    const int rem = (int)((e1 - e0) & 3);
    const int t = threadIdx.x;
    const float4* s4 = reinterpret_cast<const float4*>(src + e0);
    float4 x[PER_T];
#pragma unroll
    for (int j = 0; j < PER_T; ++j) {
        const int k = j * TREE_T + t;
        if (k < nf4) x[j] = ld_cg(s4 + k);
    }
    for (int d = 0; d < ndst; ++d) {
        float4* d4 = reinterpret_cast<float4*>(dst[d] + e0);
#pragma unroll
        for (int j = 0; j < PER_T; ++j) {
            const int k = j * TREE_T + t;
            if (k < nf4) st_na(d4 + k, x[j]);
        }
    }
    if (t < rem) {
        const int64_t e = e0 + 4 * (int64_t)nf4 + t;
        const float v = ld_cg1(src + e);
        for (int d = 0; d < ndst; ++d) st1(dst[d] + e, v);
    }
}

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
// flight per thread.
#define BF16_UNROLL(P) ((P) <= 2 ? 8 : (P) <= 4 ? 4 : 1)
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
__global__ void __launch_bounds__(FLAT_T) flat_bf16_kernel(const FcColl c) {
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
                        sgd4_any(c.segs, 4 * i, S, w[j], v[j], c.lr, c.mu, c.wd, c.inv_b);
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
                sgd1_any(c.segs, e, S, ww, vv, c.lr, c.mu, c.wd, c.inv_b);
                st1(mom_of(c, rank) + e, vv);
                for (int q = 0; q < P; ++q) st1(w_of(c, q) + e, ww);
            }
        }
    }
    trace(c, 2);
    cta_barrier(c, rank, 1);
    trace(c, 3);
    epoch_end(c);
}

// ------------------------------------------------------------ ALLGATHER ----
// op FC_OP_ALLGATHER_OWNED: every rank pushes its owned slice of a symmetric
// buffer (off_grad) to every other rank, so all ranks end with the full vector
// (e.g. the sharded momentum of the fused update, for a checkpoint: R18).
template <int P>
__global__ void __launch_bounds__(FLAT_T) allgather_kernel(const FcColl c) {
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
    cta_barrier(c, rank, 1);
    trace(c, 3);
    epoch_end(c);
}

// ------------------------------------------------------------ FLAT / PS ----
// One communication level: the owner of slice [e0, e1) loads all P ranks'
// values, evaluates the K-nomial tree in registers (K = P: the parameter
// server's sequential order), then either applies SGD and pushes w' to every
// rank (fused) or pushes the sum to every rank's grad.
// Pull broadcast (FC_BCAST_PULL): copy every peer's published slice elements
// produced by the peer CTA with this CTA's index (same grid-stride mapping).
template <int P, int U>
__device__ __forceinline__ void pull_results(const FcColl& c, int rank) {
    const bool fused = c.op == FC_OP_ALLREDUCE_SGD;
    const int64_t nch = (c.n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
    int64_t b0[P], len4[P];
    int64_t maxlen = 0;
#pragma unroll
    for (int q = 0; q < P; ++q) {
        int64_t c0, c1;
        owned_chunks(q, P, nch, false, &c0, &c1);
        const int64_t e0 = c0 * FC_CHUNK_FLOATS, e1 = min(c1 * FC_CHUNK_FLOATS, c.n);
        b0[q] = e0 / 4;
        len4[q] = e1 > e0 ? e1 / 4 - e0 / 4 : 0;
        if (q != rank && len4[q] > maxlen) maxlen = len4[q];
    }
    const float4* src[P];
#pragma unroll
    for (int q = 0; q < P; ++q) src[q] = reinterpret_cast<const float4*>(fused ? w_of(c, q) : grad_of(c, q));
    float4* dst = reinterpret_cast<float4*>(fused ? w_of(c, rank) : grad_of(c, rank));
    const int64_t T = FLAT_T;
    const int64_t stride = (int64_t)gridDim.x * T * U;
    for (int64_t rel = (int64_t)blockIdx.x * T * U + threadIdx.x; rel < maxlen; rel += stride) {
        float4 x[U][P];
#pragma unroll
        for (int j = 0; j < U; ++j)
#pragma unroll
            for (int q = 0; q < P; ++q)
                if (q != rank && rel + j * T < len4[q]) x[j][q] = ld_cg(src[q] + b0[q] + rel + j * T);
#pragma unroll
        for (int j = 0; j < U; ++j)
#pragma unroll
            for (int q = 0; q < P; ++q)
                if (q != rank && rel + j * T < len4[q]) st_na(dst + b0[q] + rel + j * T, x[j][q]);
    }
    if (blockIdx.x == 0) {  // trailing n % 4 elements of the last slice
        for (int q = 0; q < P; ++q) {
            if (q == rank) continue;
            int64_t c0, c1;
            owned_chunks(q, P, nch, false, &c0, &c1);
            const int64_t e1 = min(c1 * FC_CHUNK_FLOATS, c.n);
            if (e1 <= c0 * FC_CHUNK_FLOATS) continue;
            const int64_t e = 4 * (b0[q] + len4[q]) + threadIdx.x;
            if (e < e1) {
                const float* s1 = fused ? w_of(c, q) : grad_of(c, q);
                float* d1 = fused ? w_of(c, rank) : grad_of(c, rank);
                st1(d1 + e, ld_cg1(s1 + e));
            }
        }
    }
}

template <int P, int K, int U>
__global__ void __launch_bounds__(FLAT_T) flat_kernel(const FcColl c) {
    const int rank = my_rank(c);
    const bool pull = c.bcast == FC_BCAST_PULL && c.op != FC_OP_PS;
    epoch_begin(c);
    trace(c, 0);
    const bool ok = cta_barrier(c, rank, 0);
    trace(c, 1);
    if (ok) {
        const int64_t nch = (c.n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
        int64_t c0, c1;
        owned_chunks(rank, P, nch, c.op == FC_OP_PS, &c0, &c1);
        const int64_t e0 = c0 * FC_CHUNK_FLOATS;
        const int64_t e1 = min(c1 * FC_CHUNK_FLOATS, c.n);
        const bool fused = c.op == FC_OP_ALLREDUCE_SGD;
        if (e1 > e0) {
            // push broadcast: results go to every rank's buffer now; pull broadcast:
            // only to the own buffer, the peers fetch them after the publish barrier
            const int64_t i0 = e0 / 4, i1 = e1 / 4;
            const int64_t T = FLAT_T;
            // grid-stride: all CTAs sweep the slice in lockstep, so at any moment the
            // GPU's remote reads fall in one few-MB window of each peer's heap (a
            // contiguous range per CTA measured ~10% slower: 444 scattered streams)
            const int64_t ce = i1;
            const int64_t stride = (int64_t)gridDim.x * T * U;
            for (int64_t base = i0 + (int64_t)blockIdx.x * T * U + threadIdx.x; base < ce;
                 base += stride) {
                float4 x[U][P];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int64_t i = base + j * T;
                    if (i < ce) {
#pragma unroll
                        for (int q = 0; q < P; ++q)
                            x[j][q] = ld_cg(reinterpret_cast<const float4*>(grad_of(c, q)) + i);
                    }
                }
                if (fused) {
                    float4 w[U], v[U];
                    float4* w4 = reinterpret_cast<float4*>(w_of(c, rank));
                    float4* v4 = reinterpret_cast<float4*>(mom_of(c, rank));
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const int64_t i = base + j * T;
                        if (i < ce) {
                            w[j] = ld_rw(w4 + i);
                            v[j] = ld_rw(v4 + i);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const int64_t i = base + j * T;
                        if (i < ce) {
                            const float4 S = tree_sum_regs<P, K>(x[j]);
                            sgd4_any(c.segs, 4 * i, S, w[j], v[j], c.lr, c.mu, c.wd, c.inv_b);
                            st_na(v4 + i, v[j]);
#pragma unroll
                            for (int q = 0; q < P; ++q)
                                if (!pull || q == rank) st_na(reinterpret_cast<float4*>(w_of(c, q)) + i, w[j]);
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const int64_t i = base + j * T;
                        if (i < ce) {
                            const float4 S = tree_sum_regs<P, K>(x[j]);
#pragma unroll
                            for (int q = 0; q < P; ++q)
                                if (!pull || q == rank) st_na(reinterpret_cast<float4*>(grad_of(c, q)) + i, S);
                        }
                    }
                }
            }
            // trailing n % 4 elements of the last slice
            const int rem = (int)(e1 - 4 * i1);
            if (blockIdx.x == 0 && (int)threadIdx.x < rem) {
                const int64_t e = 4 * i1 + threadIdx.x;
                float xs[P];
#pragma unroll
                for (int q = 0; q < P; ++q) xs[q] = ld_cg1(grad_of(c, q) + e);
                const float S = tree_sum_regs1<P, K>(xs);
                if (fused) {
                    float ww = w_of(c, rank)[e], vv = mom_of(c, rank)[e];
                    sgd1_any(c.segs, e, S, ww, vv, c.lr, c.mu, c.wd, c.inv_b);
                    st1(mom_of(c, rank) + e, vv);
                    for (int q = 0; q < P; ++q)
                        if (!pull || q == rank) st1(w_of(c, q) + e, ww);
                } else {
                    for (int q = 0; q < P; ++q)
                        if (!pull || q == rank) st1(grad_of(c, q) + e, S);
                }
            }
        }
    }
    trace(c, 2);
    // push: the exit barrier proves every peer's stores into this rank landed.
    // pull: the same barrier, now BEFORE the broadcast, publishes this CTA's
    // finished results (release after local stores only); then this CTA copies
    // the matching elements of every peer's slice (the ones that peer's CTA
    // with the same index produced) and the kernel ends with no remote writes.
    const bool ok2 = cta_barrier(c, rank, 1);
    if (pull && ok && ok2) pull_results<P, U>(c, rank);
    trace(c, 3);
    epoch_end(c);
}

// ------------------------------------------------------------ FOREST -------
template <int P>
__global__ void __launch_bounds__(TREE_T) forest_kernel(const FcColl c) {
    constexpr int M = (P >= 8) ? 3 : (P >= 4) ? 2 : (P >= 2) ? 1 : 0;
    static_assert((1 << M) == P, "forest needs a power-of-two world");
    const int rank = my_rank(c);
    const int G = gridDim.x, b = blockIdx.x;
    const int64_t nch = (c.n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
    const bool fused = c.op == FC_OP_ALLREDUCE_SGD;
    const bool direct = c.bcast == FC_BCAST_DIRECT;
    float* own = grad_of(c, rank);
    epoch_begin(c);
    trace(c, 0);
    bool ok = cta_barrier(c, rank, 0);
    trace(c, 1);

    // ---- reduce: recursive halving, level l pairs rank with rank ^ 2^l.  The
    // last level also sends each finished chunk straight on: to every rank
    // (direct) or to the first broadcast hop rank ^ 2^(M-1) (tree), so the
    // owner's link sends while it still receives.
    const uint32_t all_mask = ((1u << P) - 1u) & ~(1u << rank);
    const int bc0 = rank ^ (1 << (M - 1));  // first hop of the tree broadcast
    int64_t lo = 0, hi = nch;
    for (int l = 0; l < M && ok; ++l) {
        const int partner = rank ^ (1 << l);
        const int64_t mid = lo + (hi - lo + 1) / 2;
        if ((rank >> l) & 1) lo = mid; else hi = mid;
        const bool last = (l == M - 1);
        const int64_t mid_next = lo + (hi - lo + 1) / 2;
        const bool keep_lower_next = ((rank >> (l + 1)) & 1) == 0;
        const float* pg = grad_of(c, partner);
        const int next_partner = rank ^ (1 << (l + 1));
        const uint32_t push = !last ? 0u : (direct ? all_mask : (1u << bc0));
        const bool publish = !last || !direct;
        auto stamp = [&](int64_t cx) {
            if (!last) {  // next-level consumer of chunk cx is the partner
                if ((cx < mid_next) != keep_lower_next) st_relaxed_sys(red_flag(c, next_partner, l, cx), s_epoch);
            } else {      // chunk cx of the owned slice has reached the first broadcast hop
                st_relaxed_sys(av_flag(c, bc0, cx), s_epoch);
            }
        };
        int pend = 0;
        int64_t cc_last = -1;
        for (int64_t cc = first_chunk(lo, G, b); cc < hi; cc += G) {
            if (l >= 1 && !wait_one(c, red_flag(c, rank, l - 1, cc))) { ok = false; break; }
            reduce_chunk<P>(c, rank, cc, own, pg, last, fused, push);
            if (publish) {
                cc_last = cc;
                if (++pend == PUB) { publish_batch(c, cc_last, G, pend, stamp); pend = 0; }
            }
        }
        if (ok && pend) publish_batch(c, cc_last, G, pend, stamp);
    }

    // ---- broadcast back down the tree (recursive doubling), or direct
    trace(c, 2);
    if (!direct) {
        const int64_t o0 = lo, o1 = hi;  // owned slice
        float* mine = fused ? w_of(c, rank) : own;
        for (int j = 1; j < M && ok; ++j) {  // (level j = 0 was sent inside the last reduce level)
            const int l = M - 1 - j;
            const int partner = rank ^ (1 << l);
            int64_t rlo = 0, rhi = nch;  // region R_{l+1}(rank) held now
            for (int i = 0; i <= l; ++i) {
                const int64_t m2 = rlo + (rhi - rlo + 1) / 2;
                if ((rank >> i) & 1) rlo = m2; else rhi = m2;
            }
            float* dst = fused ? w_of(c, partner) : grad_of(c, partner);
            auto stamp = [&](int64_t cx) { st_relaxed_sys(av_flag(c, partner, cx), s_epoch); };
            int pend = 0;
            int64_t cc_last = -1;
            for (int64_t cc = first_chunk(rlo, G, b); cc < rhi; cc += G) {
                const bool owned = cc >= o0 && cc < o1;
                if (!owned && !wait_one(c, av_flag(c, rank, cc))) { ok = false; break; }
                copy_chunk(c, cc, mine, &dst, 1);
                cc_last = cc;
                if (++pend == PUB) { publish_batch(c, cc_last, G, pend, stamp); pend = 0; }
            }
            if (ok && pend) publish_batch(c, cc_last, G, pend, stamp);
        }
        if (ok && M > 0) {  // chunks that arrive at the last level are not forwarded: wait for them
            const int p0 = rank ^ 1;
            const int64_t m0 = (nch + 1) / 2;
            const int64_t rlo = (p0 & 1) ? m0 : 0, rhi = (p0 & 1) ? nch : m0;
            for (int64_t cc = first_chunk(rlo, G, b); cc < rhi; cc += G)
                if (!wait_one(c, av_flag(c, rank, cc))) break;
        }
    } else {
        cta_barrier(c, rank, 1);
    }
    trace(c, 3);
    epoch_end(c);
}

// ------------------------------------------------------------ SINGLE ROOT --
// The paper's binomial tree rooted at rank 0: level l, rank r with
// r % 2^(l+1) == 0 absorbs the whole partial of r + 2^l (if < p).
template <int P>
__global__ void __launch_bounds__(TREE_T) single_root_kernel(const FcColl c) {
    const int rank = my_rank(c);
    const int G = gridDim.x, b = blockIdx.x;
    const int64_t nch = (c.n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
    const bool fused = c.op == FC_OP_ALLREDUCE_SGD;
    const bool direct = c.bcast == FC_BCAST_DIRECT;
    float* own = grad_of(c, rank);
    epoch_begin(c);
    trace(c, 0);
    bool ok = cta_barrier(c, rank, 0);
    trace(c, 1);

    int send_level = -1, last_recv = -1, L = 0;
    for (int l = 0; (1 << l) < P; ++l, ++L) {
        if (rank % (2 << l) == 0) {
            if (rank + (1 << l) < P) last_recv = l;
        } else if (send_level < 0) {
            send_level = l;
        }
    }
    const int parent = send_level >= 0 ? rank - (1 << send_level) : -1;

    // The root's final level sends each finished chunk straight on: to every
    // rank (direct) or to its children (tree), overlapping its send and receive.
    uint32_t root_children = 0;
    for (int l = 0; l < L; ++l)
        if ((1 << l) < P) root_children |= 1u << (1 << l);
    const uint32_t all_mask = ((1u << P) - 1u) & ~1u;
    for (int l = 0; l < L && ok; ++l) {
        if (rank % (2 << l) != 0) break;  // sent at an earlier level: done reducing
        const int child = rank + (1 << l);
        if (child >= P) continue;
        const bool child_has_children = (l >= 1) && (child + 1 < P);
        const bool root_final = (rank == 0) && (l == L - 1);
        const bool signal_parent = (l == last_recv) && (parent >= 0);
        const bool publish = signal_parent || (root_final && !direct);
        const uint32_t push = root_final ? (direct ? all_mask : root_children) : 0u;
        const float* cg = grad_of(c, child);
        auto stamp = [&](int64_t cx) {
            if (signal_parent) {
                st_relaxed_sys(red_flag(c, parent, send_level, cx), s_epoch);
            } else {  // root, tree broadcast: the chunk has reached every child
                for (int q = 1; q < P; q <<= 1) st_relaxed_sys(av_flag(c, q, cx), s_epoch);
            }
        };
        int pend = 0;
        int64_t cc_last = -1;
        for (int64_t cc = b; cc < nch; cc += G) {
            if (child_has_children && !wait_one(c, red_flag(c, rank, l, cc))) { ok = false; break; }
            reduce_chunk<P>(c, rank, cc, own, cg, root_final, fused, push);
            if (publish) {
                cc_last = cc;
                if (++pend == PUB) { publish_batch(c, cc_last, G, pend, stamp); pend = 0; }
            }
        }
        if (ok && pend) publish_batch(c, cc_last, G, pend, stamp);
    }

    trace(c, 2);
    if (!direct) {
      if (rank != 0) {  // (the root sent to its children inside its final level)
        // receive from the parent at send_level, forward to children at levels send_level-1..0
        float* mine = fused ? w_of(c, rank) : own;
        float* dst[3];
        int nd = 0;
        const int top = rank == 0 ? L : send_level;
        for (int l = top - 1; l >= 0; --l)
            if (rank + (1 << l) < P) dst[nd++] = fused ? w_of(c, rank + (1 << l)) : grad_of(c, rank + (1 << l));
        auto stamp = [&](int64_t cx) {
            for (int l = top - 1; l >= 0; --l)
                if (rank + (1 << l) < P) st_relaxed_sys(av_flag(c, rank + (1 << l), cx), s_epoch);
        };
        int pend = 0;
        int64_t cc_last = -1;
        for (int64_t cc = b; cc < nch && ok; cc += G) {
            if (rank != 0 && !wait_one(c, av_flag(c, rank, cc))) { ok = false; break; }
            if (nd > 0) {
                copy_chunk(c, cc, mine, dst, nd);
                cc_last = cc;
                if (++pend == PUB) { publish_batch(c, cc_last, G, pend, stamp); pend = 0; }
            }
        }
        if (ok && pend) publish_batch(c, cc_last, G, pend, stamp);
      }
    } else {
        cta_barrier(c, rank, 1);
    }
    trace(c, 3);
    epoch_end(c);
}

// ------------------------------------------------------------ dispatch -----
template <int P, int U>
static const void* flat_for_u(int K) {
    switch (K) {
        case 2: return (const void*)flat_kernel<P, 2, U>;
#define FC_K(k) case k: if constexpr (P >= k) return (const void*)flat_kernel<P, k, U>; else return nullptr;
        FC_K(3) FC_K(4) FC_K(5) FC_K(6) FC_K(7) FC_K(8)
#undef FC_K
    }
    return nullptr;
}

// Unroll override for tuning experiments (FC_FLAT_UNROLL=1|2|4; 0 = default).
static int flat_unroll_override() {
    static int u = -1;
    if (u < 0) {
        const char* e = getenv("FC_FLAT_UNROLL");
        u = e ? atoi(e) : 0;
    }
    return u;
}

template <int P>
static const void* flat_for(int K) {
    // K >= P is the same association as K = P (one level, sequential)
    if (K >= P) K = P;
    switch (flat_unroll_override()) {
        case 1: return flat_for_u<P, 1>(K);
        case 2: return flat_for_u<P, 2>(K);
        case 4: return flat_for_u<P, 4>(K);
        default: return flat_for_u<P, FLAT_UNROLL(P)>(K);
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

template <int P>
static const void* forest_for() {
    if constexpr ((P & (P - 1)) == 0) return (const void*)forest_kernel<P>;
    else return nullptr;
}

struct KernelPick {
    const void* fn;
    int block;
    bool flat;
};

static KernelPick pick_kernel(int sched, int arity, int p, int op) {
    if (op == FC_OP_PS) arity = p;
    const bool bf16 = op == FC_OP_ALLREDUCE_SGD_BF16;  // always the FLAT executor
    const bool gather = op == FC_OP_ALLGATHER_OWNED;
    const bool flat = op == FC_OP_PS || sched == FC_SCHED_FLAT || bf16 || gather;
    KernelPick k{nullptr, flat ? FLAT_T : TREE_T, flat};
    switch (p) {
#define FC_P(PP)                                                                              \
    case PP:                                                                                  \
        if (gather) k.fn = (const void*)allgather_kernel<PP>;                                 \
        else if (bf16) k.fn = bf16_for<PP>(arity);                                            \
        else if (flat) k.fn = flat_for<PP>(arity);                                            \
        else if (sched == FC_SCHED_SINGLE_ROOT) k.fn = (const void*)single_root_kernel<PP>;   \
        else k.fn = forest_for<PP>();                                                         \
        break;
        FC_P(2) FC_P(3) FC_P(4) FC_P(5) FC_P(6) FC_P(7) FC_P(8)
#undef FC_P
    }
    return k;
}

// CTAs per rank.  FLAT: one wide CTA per SM — every CTA pays a sys-scope
// release fence at the exit barrier and that fence gets slower with the number
// of CTAs issuing it (4.4 us at 148 CTAs, 7.8 us at 444; scripts/fence_bench.cu,
// launch_bench.cu).  Tree schedules: as many 256-thread CTAs as fit (their
// chunk pipeline wants more independent CTAs).  Virtual worlds share one GPU.
int collective_grid(int sched, int arity, int p, bool virt, int op, int64_t n) {
    const KernelPick k = pick_kernel(sched, arity, p, op);
    if (!k.fn || p < 1) return 0;
    int occ = 0;
    occ = occupancy(k.fn, k.block);
    if (occ < 1) return 0;
    static int flat_per_sm = -1;
    if (flat_per_sm < 0) {
        const char* e = getenv("FC_FLAT_CTAS_PER_SM");
        flat_per_sm = e ? atoi(e) : 0;  // 0 = by size
    }
    if (k.flat) {
        // measured (p = 2, 4): 1 CTA/SM wins while the per-rank slice is small (the
        // fixed exit cost dominates), 2 CTAs/SM from ~32 MB slices on (more bytes in
        // flight): NiN p=2 63.5 vs 66.6 us, VGG-19 p=2 932 vs 879 us
        int want = flat_per_sm > 0 ? flat_per_sm : (n / p >= (int64_t)(8 << 20) ? 2 : 1);
        if (occ > want) occ = want;
    }
    int64_t cap = (int64_t)dev_info().sms * occ;
    if (virt) {
        int occ_all = 0;
        occ_all = occupancy(k.fn, k.block);
        cap = (int64_t)dev_info().sms * occ_all / p;
    }
    if (cap > FC_MAX_CTAS) cap = FC_MAX_CTAS;
    return (int)cap;
}

cudaError_t launch_collective(const FcColl& c, int sched, int arity, bool virt, int grid_x,
                              cudaStream_t st) {
    const KernelPick k = pick_kernel(sched, arity, c.p, c.op);
    if (!k.fn) return cudaErrorInvalidValue;
    dim3 grid(grid_x, virt ? c.p : 1), block(k.block);
    void* args[] = {(void*)&c};
    // A virtual world's CTAs wait on CTAs of the same launch: they must be
    // co-resident, which only a cooperative launch guarantees.  In a real world
    // CTA b only ever waits on CTA b of OTHER GPUs and the grid never exceeds one
    // resident wave, so a plain launch suffices;
    // FC_LAUNCH=coop forces the cooperative path for diagnosis.
    static int force_coop = -1;
    if (force_coop < 0) {
        const char* e = getenv("FC_LAUNCH");
        force_coop = (e && strcmp(e, "coop") == 0) ? 1 : 0;
    }
    if (virt || force_coop) return cudaLaunchCooperativeKernel(k.fn, grid, block, args, 0, st);
    return cudaLaunchKernel(k.fn, grid, block, args, 0, st);
}

}  // namespace fc
