// The fp32 FLAT executor kernel template: one
// NVSwitch round per call.  Instantiated once per unroll factor U in
// coll_flat_u{1,2,4}.cu (FC_FLAT_TABLE below) so the ~80 <P, K, U> variants
// compile in parallel; see coll_common.cuh for the synchronisation.
#pragma once
#include "coll_common.cuh"

namespace fc {

// ------------------------------------------------------------ FLAT / PS ----
// One communication level: the owner of slice [e0, e1) loads all P ranks'
// values, evaluates the K-nomial tree in registers (K = P: the parameter
// server's sequential order), then either applies SGD and pushes w' to every
// rank (fused) or pushes the sum to every rank's grad.
// Pull broadcast (FC_BCAST_PULL): copy every peer's published slice elements
// produced by the peer CTA with this CTA's index — the per-CTA barrier only
// orders that CTA's writes, so this must enumerate exactly the element set the
// data phase gives CTA blockIdx.x (balanced: me + s*G*T for every slab s;
// c.flat_map == 1: the plain grid stride; the pull path never uses the dynamic map).
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
    const int64_t GT = (int64_t)gridDim.x * T;
    const int64_t me = c.flat_map == 1 ? (int64_t)blockIdx.x * T * U + threadIdx.x : (int64_t)blockIdx.x * T + threadIdx.x;
    const int64_t step = c.flat_map == 1 ? T : GT;  // between this thread's U elements of one pass
    for (int64_t rel = me; rel < maxlen; rel += GT * U) {
        float4 x[U][P];
#pragma unroll
        for (int j = 0; j < U; ++j)
#pragma unroll
            for (int q = 0; q < P; ++q)
                if (q != rank && rel + j * step < len4[q]) x[j][q] = ld_cg(src[q] + b0[q] + rel + j * step);
#pragma unroll
        for (int j = 0; j < U; ++j)
#pragma unroll
            for (int q = 0; q < P; ++q)
                if (q != rank && rel + j * step < len4[q]) st_na(dst + b0[q] + rel + j * step, x[j][q]);
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

// One "row" of the FLAT data phase for this thread: elements rb + j*step for
// j < nv (and < ce), U float4 per rank in flight.  Loads the P ranks' values,
// evaluates the K-nomial tree in registers (R1), then (fused) applies SGD and
// stores v' locally and w' to every rank (pull: only locally), or (allreduce /
// PS) stores the sum to every rank's grad (pull: only locally).
template <int P, int K, int U>
__device__ __forceinline__ void flat_row(const FcColl& c, int rank, int64_t rb, int nv, int64_t step,
                                         int64_t ce, bool fused, bool pull) {
#define FC_IX(j) ((j) < nv ? rb + (int64_t)(j) * step : ce)
    float4 x[U][P];
#pragma unroll
    for (int j = 0; j < U; ++j) {
        const int64_t i = FC_IX(j);
        if (i < ce) {
#pragma unroll
            for (int q = 0; q < P; ++q) x[j][q] = ld_cg(reinterpret_cast<const float4*>(grad_of(c, q)) + i);
        }
    }
    if (fused) {
        float4 w[U], v[U];
        float4* w4 = reinterpret_cast<float4*>(w_of(c, rank));
        float4* v4 = reinterpret_cast<float4*>(mom_of(c, rank));
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = FC_IX(j);
            if (i < ce) {
                w[j] = ld_rw(w4 + i);
                v[j] = ld_rw(v4 + i);
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = FC_IX(j);
            if (i < ce) {
                const float4 S = tree_sum_regs<P, K>(x[j]);
                sgd4_any(c.segs, 4 * i, S, w[j], v[j], s_lr, c.mu, c.wd, c.inv_b);
                st_na(v4 + i, v[j]);
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if (!pull || q == rank) st_na(reinterpret_cast<float4*>(w_of(c, q)) + i, w[j]);
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = FC_IX(j);
            if (i < ce) {
                const float4 S = tree_sum_regs<P, K>(x[j]);
#pragma unroll
                for (int q = 0; q < P; ++q)
                    if (!pull || q == rank) st_na(reinterpret_cast<float4*>(grad_of(c, q)) + i, S);
            }
        }
    }
#undef FC_IX
}

// Dynamic work claims (c.flat_map == 2, push broadcast): the slice is cut into
// units of T consecutive float4 (one per thread, coalesced); CTAs claim runs
// of g <= U consecutive units from a per-rank counter (ctl[FC_CTL_CLAIM +
// rank], zeroed again by the call's last CTA), g shrinking towards 1 as the
// slice runs out (guided: about remaining / 2G units per claim), so the CTAs
// that the NVLink/switch serves faster take more work and all of them finish
// within about one unit's time of each other.  Thread 0 issues the next claim
// right after the current row's loads are in flight, so its latency hides
// behind the row.  All CTAs still sweep the slice front to back together.
__shared__ int64_t s_claim[2];
__shared__ int s_claim_n[2];
__device__ __forceinline__ int guided_units(int64_t total, int64_t next, int G, int gmax) {
    const int64_t rem = total - next;
    int64_t g = rem / (2 * (int64_t)G);
    return (int)(g < 1 ? 1 : g > gmax ? gmax : g);
}

template <int P, int K, int U>
__global__ void __launch_bounds__(FLAT_T) flat_kernel(const __grid_constant__ FcColl c) {
    const int rank = my_rank(c);
    const bool pull = c.bcast == FC_BCAST_PULL && c.op != FC_OP_PS;
    const bool dyn = c.flat_map == 2 && !pull;  // pull pairs elements with the peer CTA's: static only
    epoch_begin(c);
    trace(c, 0);
    const int64_t nch = (c.n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
    int64_t c0, c1;
    owned_chunks(rank, P, nch, c.op == FC_OP_PS, &c0, &c1);
    const int64_t e0 = c0 * FC_CHUNK_FLOATS;
    const int64_t e1 = min(c1 * FC_CHUNK_FLOATS, c.n);
    // dyn: the CTA's first work claim touches only this rank's counter, so it is
    // issued BEFORE the entry barrier (by a thread the barrier does not use) and
    // its latency hides behind the barrier's stamp round trip
    constexpr int CLAIM_T = 32;
    uint32_t first_claim = 0;
    int first_g = 0;
    const bool pre = c.preclaim != 0;
    if (dyn && pre && e1 > e0 && threadIdx.x == CLAIM_T) {
        int64_t a = e0 / 4, b = e1 / 4;
        if (c.win_s > 1) window_range(e0 / 4, e1 / 4, c.win_k, c.win_s, &a, &b);
        first_g = guided_units((b - a + FLAT_T - 1) / FLAT_T, 0, gridDim.x, U);
        first_claim = atomicAdd(c.ctl + FC_CTL_CLAIM + rank, (uint32_t)first_g);
    }
    const bool ok = cta_barrier(c, rank, 0);
    trace(c, 1);
    if (ok) {
        const bool fused = c.op == FC_OP_ALLREDUCE_SGD;
        if (e1 > e0) {
            // push broadcast: results go to every rank's buffer now; pull broadcast:
            // only to the own buffer, the peers fetch them after the publish barrier
            const int64_t i1 = e1 / 4;
            const int64_t T = FLAT_T;
            // stage window (c.win_s > 1, the pipelined host entry point): only
            // window win_k of win_s of this rank's slice; the n % 4 tail goes with
            // the last window
            int64_t i0 = e0 / 4, ce = i1;
            if (c.win_s > 1) window_range(e0 / 4, i1, c.win_k, c.win_s, &i0, &ce);
            const bool tail_here = c.win_s <= 1 || c.win_k == c.win_s - 1;
            const int64_t GT = (int64_t)gridDim.x * T;
            const int64_t M = ce - i0;
            // Static work mapping.  A "slab" is G*T consecutive float4s (one per
            // thread of the grid, coalesced); the slice is nslab slabs.  Default
            // (balanced): rows of <= U slabs, the slabs spread evenly over
            // ceil(nslab / U) rows, so every CTA does the same work in every row.
            // c.flat_map == 1 (FC_FLAT_MAP=stride): the plain grid stride, where the
            // last partial row of G*T*U belongs to the first CTAs and the others idle.
            // Either way all CTAs sweep the slice in lockstep, so at any moment the
            // GPU's remote reads fall in one few-MB window of each peer's heap (a
            // contiguous range per CTA measured ~10% slower: 444 scattered streams).
            // Dynamic (dyn): rows are the claimed runs of units (above).
            const bool stride = c.flat_map == 1;
            const int64_t nslab = (M + GT - 1) / GT;
            const int64_t rows = stride ? (M + GT * U - 1) / (GT * U) : (nslab + U - 1) / U;
            const int64_t me = stride ? (int64_t)blockIdx.x * T * U + threadIdx.x
                                      : (int64_t)blockIdx.x * T + threadIdx.x;
            // dyn: the counter counts units of T float4; a claim of g units covers
            // g*T consecutive float4 and thread t takes base + t + j*T (j < g).
            // (Quarter units -- short last rows of a quarter of the threads -- were
            // built and measured: the CTAs then end within ~3 us instead of ~9 us at
            // p = 4, but the last CTA ends no sooner (the link is saturated to the
            // end) and p = 2 got 3 % slower; profiles/r02_flat_quarter_claims.txt.)
            constexpr int QU = 1;
            const int64_t TQ = T / QU;
            const int64_t total = (M + TQ - 1) / TQ;
            const int G = gridDim.x;
            uint32_t* ctr = c.ctl + FC_CTL_CLAIM + rank;
            if (dyn) {
                if (!pre && threadIdx.x == CLAIM_T) {  // FC_FLAT_PRECLAIM=0: claim after the barrier
                    first_g = guided_units(total, 0, G, QU * U);
                    first_claim = atomicAdd(ctr, (uint32_t)first_g);
                }
                if (threadIdx.x == CLAIM_T) {
                    s_claim[0] = (int64_t)first_claim;
                    s_claim_n[0] = first_g;
                }
                __syncthreads();
            }
            int64_t s0 = 0;
            for (int64_t r = 0;; ++r) {
                // element j of this thread in row r: rb + j * step, for j < nv (and < lim)
                int64_t rb, step, lim = ce;
                int nv;
                uint32_t next = 0;
                int gnext = 0;
                if (dyn) {
                    const int64_t q0 = s_claim[r & 1];
                    if (q0 >= total) break;
                    const int64_t g = min((int64_t)s_claim_n[r & 1], total - q0);
                    rb = i0 + q0 * TQ + threadIdx.x;
                    step = T;
                    nv = U;
                    lim = min(ce, i0 + (q0 + g) * TQ);
                    if (threadIdx.x == 0) {  // the next claim; its result is needed only after this row
                        gnext = guided_units(total, q0 + g, G, QU * U);
                        next = atomicAdd(ctr, (uint32_t)gnext);
                    }
                } else {
                    if (r >= rows) break;
                    const int64_t s1 = stride ? 0 : nslab * (r + 1) / rows;
                    rb = stride ? i0 + r * GT * U + me : i0 + s0 * GT + me;
                    nv = stride ? U : (int)(s1 - s0);
                    step = stride ? T : GT;
                    s0 = s1;
                }
                flat_row<P, K, U>(c, rank, rb, nv, step, lim, fused, pull);
                if (dyn) {
                    if (threadIdx.x == 0) {
                        s_claim[(r + 1) & 1] = (int64_t)next;
                        s_claim_n[(r + 1) & 1] = gnext;
                    }
                    __syncthreads();
                }
            }
            // trailing n % 4 elements of the last slice
            const int rem = (int)(e1 - 4 * i1);
            if (tail_here && blockIdx.x == 0 && (int)threadIdx.x < rem) {
                const int64_t e = 4 * i1 + threadIdx.x;
                float xs[P];
#pragma unroll
                for (int q = 0; q < P; ++q) xs[q] = ld_cg1(grad_of(c, q) + e);
                const float S = tree_sum_regs1<P, K>(xs);
                if (fused) {
                    float ww = w_of(c, rank)[e], vv = mom_of(c, rank)[e];
                    sgd1_any(c.segs, e, S, ww, vv, s_lr, c.mu, c.wd, c.inv_b);
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
    // with the same index produced).  The kernel then still needs the
    // rank-level exit: peers may be pulling from THIS rank's published slice,
    // and once the kernel ends the caller may overwrite it (the next backward
    // writes grad) — without the exit a slow peer reads the new values (found
    // by the shared-GPU world test, tests/test_multi_gpu.py).
    if (!pull) {
        finish_call(c, rank);
        return;
    }
    const bool ok2 = cta_barrier(c, rank, 1);
    if (ok && ok2) pull_results<P, U>(c, rank);
    trace(c, 3);
    exit_rank(c, rank, FC_EXIT_CTA_SLOT);
}

// Kernel table of one unroll factor: flat_kernel<p, arity, U> (arity >= p is
// the same association as arity = p: one level, sequential).
#define FC_FLAT_TABLE(U)                                                                     \
    template <int P>                                                                         \
    static const void* flat_for_##U(int K) {                                                 \
        if (K >= P) K = P;                                                                   \
        switch (K) {                                                                         \
            case 2: return (const void*)flat_kernel<P, 2, U>;                                \
            case 3: if constexpr (P >= 3) return (const void*)flat_kernel<P, 3, U>; break;   \
            case 4: if constexpr (P >= 4) return (const void*)flat_kernel<P, 4, U>; break;   \
            case 5: if constexpr (P >= 5) return (const void*)flat_kernel<P, 5, U>; break;   \
            case 6: if constexpr (P >= 6) return (const void*)flat_kernel<P, 6, U>; break;   \
            case 7: if constexpr (P >= 7) return (const void*)flat_kernel<P, 7, U>; break;   \
            case 8: if constexpr (P >= 8) return (const void*)flat_kernel<P, 8, U>; break;   \
        }                                                                                    \
        return nullptr;                                                                      \
    }                                                                                        \
    const void* flat_kernel_u##U(int p, int arity) {                                         \
        switch (p) {                                                                         \
            case 2: return flat_for_##U<2>(arity);                                           \
            case 3: return flat_for_##U<3>(arity);                                           \
            case 4: return flat_for_##U<4>(arity);                                           \
            case 5: return flat_for_##U<5>(arity);                                           \
            case 6: return flat_for_##U<6>(arity);                                           \
            case 7: return flat_for_##U<7>(arity);                                           \
            case 8: return flat_for_##U<8>(arity);                                           \
        }                                                                                    \
        return nullptr;                                                                      \
    }

const void* flat_kernel_u1(int p, int arity);
const void* flat_kernel_u2(int p, int arity);
const void* flat_kernel_u4(int p, int arity);

}  // namespace fc
