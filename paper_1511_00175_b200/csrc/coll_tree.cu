// Tree-schedule collective kernels: FOREST — the
// XOR-rotated binomial forest / recursive halving, one binomial tree per
// owner slice, SGD fused into the last level, tree or direct broadcast — and
// SINGLE_ROOT, the paper's binomial tree rooted at rank 0.  Chunks
// of FC_CHUNK_FLOATS flow level to level behind per-chunk epoch flags; see
// coll_common.cuh for the synchronisation.
#include "coll_common.cuh"

namespace fc {

// ------------------------------------------------------------ FOREST -------
template <int P, int MINB>
__global__ void __launch_bounds__(TREE_T, MINB) forest_kernel(const __grid_constant__ FcColl c) {
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
        finish_call(c, rank);
        return;
    }
    trace(c, 3);
    epoch_end(c);
}

// ------------------------------------------------------------ SINGLE ROOT --
// The paper's binomial tree rooted at rank 0: level l, rank r with
// r % 2^(l+1) == 0 absorbs the whole partial of r + 2^l (if < p).
template <int P, int MINB>
__global__ void __launch_bounds__(TREE_T, MINB) single_root_kernel(const __grid_constant__ FcColl c) {
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
        finish_call(c, rank);
        return;
    }
    trace(c, 3);
    epoch_end(c);
}

// ------------------------------------------------------------ kernel tables -
// Two register budgets per kernel (MINB = resident CTAs per SM the compiler
// must allow): MINB = 1 lets a 256-thread CTA use ~160 registers with no
// spills; MINB = 2 caps it at 128 and spills 8-76 B/thread (ptxas -v) but
// doubles the CTAs in the chunk pipeline.  coll_dispatch.cu picks by slice size.
template <int P, int MINB>
static const void* forest_for() {
    if constexpr ((P & (P - 1)) == 0) return (const void*)forest_kernel<P, MINB>;
    else return nullptr;
}

const void* forest_kernel_for(int p, int ctas_per_sm) {
    switch (p) {
#define FC_P(PP) case PP: return ctas_per_sm >= 2 ? forest_for<PP, 2>() : forest_for<PP, 1>();
        FC_P(2) FC_P(3) FC_P(4) FC_P(5) FC_P(6) FC_P(7) FC_P(8)
#undef FC_P
    }
    return nullptr;
}

const void* single_root_kernel_for(int p, int ctas_per_sm) {
    switch (p) {
#define FC_P(PP)                                                                              \
    case PP:                                                                                  \
        return ctas_per_sm >= 2 ? (const void*)single_root_kernel<PP, 2> : (const void*)single_root_kernel<PP, 1>;
        FC_P(2) FC_P(3) FC_P(4) FC_P(5) FC_P(6) FC_P(7) FC_P(8)
#undef FC_P
    }
    return nullptr;
}

}  // namespace fc
