// Internal host/device structures of libfirecaffe (not part of the C ABI).
#pragma once
#include <math.h>
#include <stdint.h>

#include "../../include/firecaffe.h"

#define FC_MAX_RANKS 8
#define FC_MAX_CTAS 1024
#define FC_EXIT_CTA_SLOT (FC_MAX_CTAS - 1)  // exit stamp word of the FLAT pull path; grids stay below it
#define FC_MAX_LEVELS 3          // log2(FC_MAX_RANKS)
#define FC_CHUNK_FLOATS 4096     // flag granularity of the level-structured schedules (16 KB)
#define FC_BAR_SLOTS 2           // 0 = entry barrier, 1 = exit barrier

// Layout of the flag area at the start of every rank's heap (uint32 words):
//   bar[FC_BAR_SLOTS][FC_MAX_CTAS][FC_MAX_RANKS]   per-CTA all-to-all barriers, uint64 each:
//                                                  epoch | call signature << 32 (2 words)
//   red[FC_MAX_LEVELS][max_chunks]                 "partial of chunk c for level l+1 ready"
//   av[max_chunks]                                 "broadcast value of chunk c has arrived"
// All flags hold the epoch of the call that last wrote them (monotonic, never reset).
struct FcFlagLayout {
    int64_t max_chunks;
    int64_t bar_words;   // offset of red[] in words
    int64_t red_words;   // offset of av[] in words
    int64_t total_bytes; // reserved prefix, rounded to 64 KB
};

static inline FcFlagLayout fc_flag_layout(int64_t heap_bytes) {
    FcFlagLayout L;
    L.max_chunks = heap_bytes / (4 * (int64_t)FC_CHUNK_FLOATS) + 1;
    L.bar_words = 2 * (int64_t)FC_BAR_SLOTS * FC_MAX_CTAS * FC_MAX_RANKS;
    L.red_words = L.bar_words + (int64_t)FC_MAX_LEVELS * L.max_chunks;
    int64_t words = L.red_words + L.max_chunks;
    int64_t bytes = words * 4;
    L.total_bytes = (bytes + 65535) / 65536 * 65536;
    return L;
}

// Device copy of a Caffe per-blob multiplier table (nseg == 0: uniform update).
struct FcSegs {
    const int64_t* begin;
    const float* lrm;
    const float* dm;
    int nseg;
};

// Device-resident schedule state of the *_sched entry points (R21).
// The learning rate the schedule gives at every reachable "level" is computed
// ONCE on the host, by the same definition the oracle writes (factor by
// std::pow in double, one rounding of base_lr * factor to fp32), and uploaded
// as a table; the kernels only map the iteration to its level and load the
// fp32 value, so host and device give identical bits for every valid schedule.
//   FIXED      level 0
//   STEP       level floor(iter / stepsize)          (table ends where the value
//   MULTISTEP  level #{steps[j] <= iter}              stops changing: 0, inf, or
//   POLY       level min(iter, max_iter)              gamma == 1; clamped beyond)
// `iter` is the iteration the next call uses; `done` is the CTA arrival counter
// with which the last CTA of a call advances it (stream order publishes it).
struct FcLrDev {
    int policy;
    int nsteps;
    int64_t stepsize;
    int64_t max_iter;
    int64_t steps[FC_LR_MAX_STEPS];
    const float* table;  // device: lr of level 0 .. nlevels-1
    int64_t nlevels;
    int64_t iter;
    uint32_t done;
};

#ifdef __CUDACC__
__device__ __forceinline__ float fc_lr_dev(const FcLrDev* d) {
    const int64_t it = *(volatile const int64_t*)&d->iter;
    int64_t k = 0;
    switch (d->policy) {
        case FC_LR_STEP: k = it / d->stepsize; break;
        case FC_LR_MULTISTEP:
            for (int j = 0; j < d->nsteps; ++j) k += d->steps[j] <= it;
            break;
        case FC_LR_POLY: k = it < d->max_iter ? it : d->max_iter; break;
        default: k = 0;
    }
    if (k >= d->nlevels) k = d->nlevels - 1;
    return d->table[k];
}
#endif

// Everything a collective kernel needs to find every rank's buffers.
struct FcPeers {
    char* heap[FC_MAX_RANKS];  // each rank's heap base, as mapped in this process
};

struct FcColl {
    FcPeers peers;
    int rank;          // >= 0: this process's rank; -1: virtual world, rank = blockIdx.y
    int p;             // world size
    uint32_t* ctl;     // device call counter: [0] last completed epoch, [1] CTAs done
    uint32_t sig;      // hash of (op, n, schedule, hyper-parameters): must match on every rank
    int op;            // FcOp
    uint64_t timeout_ns;
    int* status;       // sticky device status (FC_OK until a timeout)
    int64_t n;         // floats
    int64_t off_grad;  // byte offsets of the symmetric buffers inside each heap
    int64_t off_w;
    int64_t off_mom;   // >= 0: mom is symmetric in the heap; < 0: use mom_local
    float* mom_local;
    float lr, mu, wd, inv_b;
    FcLrDev* lrs;      // non-null: lr = the schedule at lrs->iter (device), advanced once per call
    FcSegs segs;       // per-blob multipliers for the fused update
    int bcast;         // fc_bcast
    int owner_single_root;  // ownership of the single-root schedule (rank 0 owns all)
    int64_t bar_words, red_words, max_chunks;
    uint64_t* trace;   // optional: per-CTA %globaltimer stamps [rank][cta][FC_TRACE_SLOTS]
    int rank_exit;     // 1: rank-level exit (one sys fence per GPU), 0: per-CTA exit barrier
    int win_k, win_s;  // FLAT push only: process window win_k of win_s of the owned slice (win_s <= 1: all)
    int flat_map;      // FLAT work mapping: 0 = balanced slab rows, 1 = plain grid stride, 2 = dynamic claims
    int preclaim;      // FLAT dyn: 1 = the first claim is issued before the entry barrier (default)
    int clean_exit;    // rank-level exit: 1 = non-last CTAs fence at sys scope after arriving (default)
};

#define FC_TRACE_SLOTS 4
// device call-control words (fc_world::d_ctl): [0] epoch of the last completed call,
// [1] CTAs finished in the current call, [FC_CTL_CLAIM + r] rank r's FLAT work-claim
// counter (dynamic mapping); the call's last CTA zeroes [1] and the claim counters
#define FC_CTL_CLAIM 2
#define FC_CTL_WORDS (FC_CTL_CLAIM + FC_MAX_RANKS)  // kernel entry, after entry barrier, after the data phase, exit

enum FcOp {
    FC_OP_ALLREDUCE = 0,
    FC_OP_ALLREDUCE_SGD = 1,
    FC_OP_PS = 2,
    FC_OP_ALLREDUCE_SGD_BF16 = 3,
    FC_OP_ALLGATHER_OWNED = 4
};
