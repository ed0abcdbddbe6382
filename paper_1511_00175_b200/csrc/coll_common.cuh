// Device-side building blocks shared by the collective executors
// (coll_flat.cu, coll_tree.cu): heap addressing, the device epoch counter,
// the cross-GPU CTA barrier, batched flag publication and the chunk
// operations of the tree schedules.  Included by exactly those .cu files.
//
// Every rank's heap is mapped into every process (CUDA IPC), so a kernel reads
// a peer GPU's gradient slice with ordinary 128-bit loads and writes a peer's
// weights with ordinary 128-bit stores; both cross NVLink / NVSwitch.  Order
// between GPUs comes from epoch-stamped flags in the heaps' reserved prefix
// (st.release.sys / ld.acquire.sys).  Producers PUSH flags to the consumer's
// heap so that every spin is on local memory.
#pragma once
#include <cuda_runtime.h>

#include "fc_device.cuh"
#include "fc_launch.h"

namespace fc {

constexpr int TREE_T = kTreeThreads;              // threads per CTA (tree schedules)
constexpr int FLAT_T = kFlatThreads;              // threads per CTA (FLAT / PS), one CTA per SM
// float4 per thread per operand in flight in FLAT (per claimed unit run of the
// dynamic mapping): U = 2 at p = 2, U = 1 from p = 3 on.  With the dynamic
// claims, smaller runs measured faster than round 1's U = 4 / 2 (finer claims,
// and 148 CTAs x 512 thr x (P-1) x U x 16 B is still >= 2.4 MB of remote loads
// in flight): p = 2 U = 2 vs 4 0-2 %, p = 4 U = 1 vs 2 0.7-2.2 % faster at
// NiN..AlexNet sizes (profiles/r02_flat_unroll_dyn.txt, A/B twice).  U = 2 at
// p >= 6 would exceed the 128 registers of a 512-thread CTA (spills).
#define FLAT_UNROLL(P) ((P) <= 2 ? 2 : 1)
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
// The call's learning rate: the argument, or (c.lrs, the *_sched entry points)
// the device-resident schedule at its current iteration, evaluated once per CTA.
__shared__ float s_lr;

__device__ __forceinline__ void epoch_begin(const FcColl& c) {
    if (threadIdx.x == 0) {
        s_epoch = *(volatile uint32_t*)c.ctl + 1u;
        s_lr = c.lrs ? fc_lr_dev(c.lrs) : c.lr;
    }
    __syncthreads();
}

// Last CTA of a call: the schedule's next call uses the next iteration (every
// CTA of this call read `iter` at entry, before arriving on the counter).
__device__ __forceinline__ void advance_lr(const FcColl& c) {
    if (c.lrs) c.lrs->iter = c.lrs->iter + 1;
}

__device__ __forceinline__ void epoch_end(const FcColl& c) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t total = gridDim.x * gridDim.y;
        const uint32_t done = atomicAdd(c.ctl + 1, 1u) + 1u;
        if (done == total) {
            c.ctl[1] = 0u;
            for (int r = 0; r < FC_MAX_RANKS; ++r) c.ctl[FC_CTL_CLAIM + r] = 0u;
            advance_lr(c);
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
static __device__ bool cta_barrier(const FcColl& c, int rank, int slot) {
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

// Rank-level exit (c.rank_exit = 1 or 2): instead of an all-to-all barrier per
// CTA (every CTA paying a sys-scope fence; the fence gets slower the more CTAs
// issue it), every CTA orders its writes — local and peer — with a gpu-scope
// fence and arrives on the call's CTA counter (ctl[1]); the LAST CTA to arrive
// on this GPU makes all of them visible system-wide with ONE sys fence and
// writes its exit stamp, then waits for every peer's stamp (written by that
// peer's last CTA after all of ITS CTAs arrived).  When the kernel ends, every
// store any peer made into this rank's heap has landed.  Memory-model chain
// (PTX causality order is transitive): CTA stores -> fence.gpu + counter
// increment -> last CTA's increment + fence.gpu (same GPU) -> fence.sys +
// stamp -> the peer's acquire.sys of the stamp.  The other CTAs leave at once.
// Where the stamp goes:
//   1 (push, default): into every peer's heap; each rank polls its own heap
//     (local loads).
//   2 (poll): into the rank's OWN heap; the last CTA's threads q < p poll
//     peer q's stamp word over NVLink with acquire loads, in parallel, so no
//     remote store follows the fence.  Measured the same as push at p = 2
//     (profiles/r02_exit_push_vs_poll.txt): the stamps are not what makes
//     the kernel's completion slower than an empty kernel's.
// Then the epoch advances as in epoch_end.  Virtual worlds: the last CTA of
// the whole grid already follows every rank's CTAs, no stamps needed.
// `cta_slot`: which slot-1 stamp word carries the exit (0; the FLAT pull path,
// whose per-CTA slot-1 barrier already used the low indices this call, passes
// FC_EXIT_CTA_SLOT, an index no grid reaches).
__shared__ uint32_t s_last;
static __device__ __forceinline__ void exit_rank(const FcColl& c, int rank, int cta_slot = 0) {
    __syncthreads();
    const int t = threadIdx.x;
    if (t == 0) {
        __threadfence();
        const uint32_t total = gridDim.x * gridDim.y;
        s_last = atomicAdd(c.ctl + 1, 1u) + 1u == total;
    }
    __syncthreads();
    if (!s_last) {
        // c.clean_exit (default): a CTA that is not the last one fences at system
        // scope AFTER arriving -- off the last CTA's critical path, concurrent with
        // its remaining work -- so that when the grid ends only the last CTA's SM
        // has peer accesses not yet made system-visible, and the end-of-grid flush
        // is short: completion ~6 instead of ~9 us, net 0.6-2 us per call
        // (scripts/gap_bench.cu, profiles/r02_gap_bench.txt, r02_exit_clean.txt).
        // Not needed for correctness (the last CTA's fence covers every CTA's
        // stores through the counter).
        if (c.clean_exit && c.rank >= 0 && t == 0) fence_sys();
        return;
    }
    if (c.rank >= 0) {
        const uint64_t stamp = (uint64_t)s_epoch | ((uint64_t)c.sig << 32);
        const bool poll = c.rank_exit == 2;
        if (t == 0) {
            fence_sys();  // (sc.sys subsumes the gpu-scope acquire fence after the counter)
            if (poll) {
                st_relaxed_sys64(bar_flag(c, rank, 1, cta_slot, rank), stamp);
            } else {
                for (int q = 0; q < c.p; ++q)
                    if (q != rank) st_relaxed_sys64(bar_flag(c, q, 1, cta_slot, rank), stamp);
            }
        }
        if (poll) __syncthreads();  // thread q polls only after the fence and the own stamp
        bool good = true;
        if (t < c.p && t != rank) {
            // poll: peer t's own stamp word in ITS heap (remote acquire loads);
            // push: the word peer t wrote into this rank's heap (local loads)
            const uint64_t* f = poll ? bar_flag(c, t, 1, cta_slot, t) : bar_flag(c, rank, 1, cta_slot, t);
            const uint64_t t0 = globaltimer();
            uint32_t spins = 0;
            while (!reached((uint32_t)(poll ? ld_acquire_sys64(f) : ld_relaxed_sys64(f)), s_epoch)) {
                if ((++spins & (poll ? 7u : 63u)) == 0) {
                    if (*(volatile int*)c.status != FC_OK) { good = false; break; }
                    if (globaltimer() - t0 > c.timeout_ns) {
                        atomicCAS(c.status, FC_OK, FC_ERR_TIMEOUT);
                        good = false;
                        break;
                    }
                }
            }
            if (good && !poll) (void)ld_acquire_sys64(f);
        }
        __syncthreads();
    }
    if (t == 0) {
        c.ctl[1] = 0u;
        for (int r = 0; r < FC_MAX_RANKS; ++r) c.ctl[FC_CTL_CLAIM + r] = 0u;
        advance_lr(c);
        __threadfence();
        atomicExch(c.ctl, s_epoch);
    }
}

// Per-CTA exit with LOCAL stamps (c.rank_exit == 3, real worlds): every CTA
// makes its own writes — local and peer — visible system-wide with its own
// `fence.sys` and writes its exit stamp into its OWN heap (a release pattern at
// sys scope whose write is local); thread q < p then polls peer q's stamp of
// the CTA with this index over NVLink with acquire loads (each a release/
// acquire pair at sys scope: peer q's CTA's pushes into this heap
// happen-before this CTA's exit).  All CTAs of a rank together observe every
// CTA of every peer, so when the kernel ends every store any peer made into
// this heap has landed.  No remote store follows a fence: a kernel whose CTAs
// each issued `fence.sys` after their peer stores completes ~3.3 us sooner
// than one with only gpu-scope fences and one last-CTA sys fence
// (scripts/gap_bench.cu, profiles/r02_gap_bench.txt), and the fences of the 148
// CTAs overlap each other.  Then the epoch advances as in epoch_end.
static __device__ __forceinline__ void exit_cta_poll(const FcColl& c, int rank) {
    __syncthreads();
    const int t = threadIdx.x;
    const uint64_t stamp = (uint64_t)s_epoch | ((uint64_t)c.sig << 32);
    if (t == 0) {
        fence_sys();
        st_relaxed_sys64(bar_flag(c, rank, 1, blockIdx.x, rank), stamp);
    }
    bool good = true;
    if (t < c.p && t != rank) {
        const uint64_t* f = bar_flag(c, t, 1, blockIdx.x, t);
        const uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        uint64_t v;
        while (!reached((uint32_t)(v = ld_acquire_sys64(f)), s_epoch)) {
            __nanosleep(64);
            if ((++spins & 7u) == 0) {
                if (*(volatile int*)c.status != FC_OK) { good = false; break; }
                if (globaltimer() - t0 > c.timeout_ns) {
                    atomicCAS(c.status, FC_OK, FC_ERR_TIMEOUT);
                    good = false;
                    break;
                }
            }
        }
        if (good && (uint32_t)v == s_epoch && (uint32_t)(v >> 32) != c.sig) atomicCAS(c.status, FC_OK, FC_ERR_MISMATCH);
    }
    __syncthreads();
}

// End of a collective whose data phase may have written into peers' heaps:
// the exit barrier (per CTA, or per rank with c.rank_exit), then the epoch.
__device__ __forceinline__ void finish_call(const FcColl& c, int rank) {
    if (c.rank_exit == 3 && c.rank >= 0) {
        exit_cta_poll(c, rank);
        trace(c, 3);
        epoch_end(c);
        return;
    }
    if (c.rank_exit) {
        exit_rank(c, rank);
        trace(c, 3);
        return;
    }
    cta_barrier(c, rank, 1);
    trace(c, 3);
    epoch_end(c);
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
            sgd4_any(c.segs, e0 + 4 * (int64_t)k, s, w[j], v[j], s_lr, c.mu, c.wd, c.inv_b);
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
        sgd1_any(c.segs, e, s, ww, vv, s_lr, c.mu, c.wd, c.inv_b);
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

}  // namespace fc
