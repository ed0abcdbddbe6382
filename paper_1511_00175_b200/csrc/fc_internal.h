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

#ifdef __CUDACC__
#define FC_HD __host__ __device__
#else
#define FC_HD
#endif

// Learning-rate factor of the paper's schedules at iteration `iter` (DESIGN.md
// R21), the same arithmetic on the host (firecaffe_lr_at) and on the device
// (the *_sched entry points): STEP / MULTISTEP gamma^k by binary powering in
// double (k = 1, 2: gamma, fl(gamma^2)); POLY (1 - iter/max_iter)^power in
// double, power 0.5 (the paper's) as the correctly rounded sqrt, power
// 1 as the base itself, others through pow; 0 at and after max_iter.  The
// caller validates the schedule.
FC_HD inline double fc_lr_factor(const fc_lr_schedule& s, int64_t iter) {
    int64_t k = 0;
    switch (s.policy) {
        case FC_LR_STEP:
            k = iter / s.stepsize;
            break;
        case FC_LR_MULTISTEP:
            for (int j = 0; j < s.nsteps; ++j) k += s.steps[j] <= iter;
            break;
        case FC_LR_POLY: {
            if (iter >= s.max_iter) return 0.0;
            const double x = 1.0 - (double)iter / (double)s.max_iter;
            if (s.power == 0.5f) return sqrt(x);
            if (s.power == 1.0f) return x;
            return pow(x, (double)s.power);
        }
        default:
            return 1.0;
    }
    double f = 1.0, b = (double)s.gamma;
    while (k > 0) {
        if (k & 1) f *= b;
        k >>= 1;
        if (k) b *= b;
    }
    return f;
}

// fl32(base_lr * factor): one rounding of the double product to fp32
FC_HD inline float fc_lr_value(const fc_lr_schedule& s, int64_t iter) {
    return (float)((double)s.base_lr * fc_lr_factor(s, iter));
}

// Device-resident schedule state of the *_sched entry points: the schedule,
// the iteration the next call uses, and the CTA arrival counter with which the
// last CTA of a call advances `iter` (stream order publishes it to the next call).
struct FcLrDev {
    fc_lr_schedule s;
    int64_t iter;
    uint32_t done;
};

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
    int map_stride;    // FLAT: 1 = plain grid-stride work mapping, 0 = balanced slab rows (default)
};

#define FC_TRACE_SLOTS 4  // kernel entry, after entry barrier, after the data phase, exit

enum FcOp {
    FC_OP_ALLREDUCE = 0,
    FC_OP_ALLREDUCE_SGD = 1,
    FC_OP_PS = 2,
    FC_OP_ALLREDUCE_SGD_BF16 = 3,
    FC_OP_ALLGATHER_OWNED = 4
};
