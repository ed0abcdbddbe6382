// The C ABI of libfirecaffe (include/firecaffe.h): argument validation,
// the symmetric heap, world creation (CUDA IPC peer mapping over NVLink or a
// virtual world on one GPU), executor selection and kernel launch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>
#include <mutex>
#include <vector>

#include "fc_internal.h"
#include "fc_launch.h"

#define FC_VERSION_STR "firecaffe-b200 0.1.0 sm_100a"
#define FC_HOST_MAX_STAGES 16

struct fc_segments {
    int nseg;
    int64_t n;
    int device;
    uint32_t hash;  // of the host table: part of the collective call signature
    int64_t* d_begin;
    float* d_lrm;
    float* d_dm;
};

struct fc_lr_state {
    FcLrDev* d;         // device copy of the schedule + the iteration counter
    float* table;       // device: the lr of every schedule level (FcLrDev::table)
    fc_lr_schedule s;   // host copy (validation, call signature)
    int device;
    uint32_t hash;      // of the schedule: part of the collective call signature
};

struct fc_world {
    int rank;  // -1 for a virtual world
    int p;
    int device;
    int virt;
    char* heap_local;      // this rank's heap (virtual: rank 0's)
    int64_t heap_bytes;    // per rank
    char* peer[FC_MAX_RANKS];
    bool opened[FC_MAX_RANKS];
    uint32_t* d_ctl;  // device call counter (graph-capturable epochs)
    uint64_t timeout_ns;
    int* d_status;
    int arity;
    fc_sched sched;
    fc_bcast bcast;
    FcFlagLayout layout;
    uint64_t* trace;
    int64_t trace_cap;
    int last_grid;
    int max_ctas;  // 0 = automatic
    // staged host entry point (firecaffe_tree_allreduce_sgd_host), created on first use
    bool hp_ready;
    cudaStream_t hp_s[3];  // H2D, collective, D2H
    cudaEvent_t hp_start, hp_h2d[FC_HOST_MAX_STAGES], hp_coll[FC_HOST_MAX_STAGES];
};

namespace fc {
const DevInfo& dev_info() {
    static DevInfo cache[64];
    static bool have[64];
    int d = 0;
    cudaGetDevice(&d);
    if (d < 0 || d >= 64) d = 0;
    if (!have[d]) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
        cache[d].device = d;
        cache[d].sms = sms > 0 ? sms : 1;
        have[d] = true;
    }
    return cache[d];
}

// Resident CTAs per SM of (kernel, block size) on the current device, cached:
// the occupancy query costs microseconds and sits on every call's host path.
int occupancy(const void* fn, int block) {
    struct Entry {
        const void* fn;
        int block, device, occ;
    };
    static Entry table[512];
    static int used = 0;
    static std::mutex mu;
    const int dev = dev_info().device;
    std::lock_guard<std::mutex> lock(mu);
    for (int i = 0; i < used; ++i)
        if (table[i].fn == fn && table[i].block == block && table[i].device == dev) return table[i].occ;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, 0) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (used < 512) table[used++] = Entry{fn, block, dev, occ};
    return occ;
}
}  // namespace fc

using namespace fc;

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static bool overlap(const void* a, const void* b, int64_t bytes) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + (uintptr_t)bytes && y < x + (uintptr_t)bytes;
}

static fc_status check_hyper(float lr, float mu, float wd, int64_t batch) {
    if (!(lr > 0.0f) || !std::isfinite(lr)) return FC_ERR_INVALID_ARG;
    if (!(mu >= 0.0f && mu < 1.0f)) return FC_ERR_INVALID_ARG;
    if (!(wd >= 0.0f) || !std::isfinite(wd)) return FC_ERR_INVALID_ARG;
    if (batch < 1) return FC_ERR_INVALID_ARG;
    return FC_OK;
}

static fc_status check_vec(const void* p, int64_t n) {
    if (n > 0 && (!p || !aligned16(p))) return FC_ERR_INVALID_ARG;
    return FC_OK;
}

// float inv_b = 1 / (float)batch, one fp32 rounding (R7)
static float inv_batch(int64_t batch) {
    const volatile float one = 1.0f;
    const volatile float b = (float)batch;
    return one / b;
}

// Exit protocol of the collectives (coll_common.cuh exit_rank): rank-level,
// the last CTA per GPU does one sys fence and pushes its stamp into every
// peer's heap (default, FC_EXIT=push); the same with the stamp written into
// its own heap and polled by the peers over NVLink (FC_EXIT=poll: measured
// equal, profiles/r02_exit_push_vs_poll.txt); or, with FC_EXIT=cta, the
// per-CTA exit barrier (profiles/r01_sweep_exit_*).
// Part of the call signature, so ranks that disagree fail with FC_ERR_MISMATCH
// at entry instead of waiting on stamps that never come.
static int exit_mode() {
    static int m = -1;
    if (m < 0) {
        const char* e = getenv("FC_EXIT");
        m = (e && strcmp(e, "cta") == 0) ? 0 : (e && strcmp(e, "poll") == 0) ? 2
            : (e && strcmp(e, "ctapoll") == 0) ? 3 : 1;
    }
    return m;
}

// FLAT work mapping (coll_flat.cuh): dynamic guided claims from a per-rank
// counter (default, FC_FLAT_MAP=dyn; push broadcast only, the pull path pairs
// elements statically and uses the balanced rows), balanced static slab rows
// (balanced, round 1's default) or the plain grid stride (stride).  Measured
// (profiles/r02_flat_map_p2.txt): dyn 0.9-2.2 % faster than balanced at
// p = 2 from NiN to AlexNet size.  Value-neutral (every element is processed
// once, same arithmetic), so not part of the call signature.
static int flat_map() {
    static int m = -1;
    if (m < 0) {
        const char* e = getenv("FC_FLAT_MAP");
        m = (e && strcmp(e, "stride") == 0) ? 1 : (e && strcmp(e, "balanced") == 0) ? 0 : 2;
    }
    return m;
}

// FLAT dynamic mapping: issue each CTA's first claim before the entry barrier
// (default) or after it (FC_FLAT_PRECLAIM=0, A/B only).  Value-neutral.
static int flat_preclaim() {
    static int m = -1;
    if (m < 0) {
        const char* e = getenv("FC_FLAT_PRECLAIM");
        m = (e && strcmp(e, "0") == 0) ? 0 : 1;
    }
    return m;
}

// Rank-level exit: the CTAs that are not last issue a sys-scope fence after
// arriving (default) or leave at once (FC_CLEAN_EXIT=0, round 1's exit).
// Measured (profiles/r02_exit_clean.txt, A/B three times): the kernel's
// completion drops from ~9 to ~6 us (an empty kernel's), the span grows by
// 1.2-1.6 us (the concurrent fences), net NiN p = 4 -2.0 us, p = 2 -0.6 us,
// GoogLeNet / AlexNet -1.0..-1.6 us.  Value-neutral.
static int clean_exit() {
    static int m = -1;
    if (m < 0) {
        const char* e = getenv("FC_CLEAN_EXIT");
        m = (e && strcmp(e, "0") == 0) ? 0 : 1;
    }
    return m;
}

extern "C" {

const char* firecaffe_version(void) { return FC_VERSION_STR; }

const char* firecaffe_status_str(fc_status s) {
    switch (s) {
        case FC_OK: return "ok";
        case FC_ERR_INVALID_ARG: return "invalid argument";
        case FC_ERR_NOT_SYMMETRIC: return "buffer not in the symmetric heap";
        case FC_ERR_MISMATCH: return "world/device mismatch";
        case FC_ERR_TIMEOUT: return "timeout waiting for a peer";
        case FC_ERR_CUDA: return "CUDA error";
        case FC_ERR_UNSUPPORTED: return "unsupported schedule for this world";
    }
    return "unknown status";
}

float firecaffe_scale_lr(float base_lr, int64_t base_batch, int64_t batch) {
    if (base_batch < 1 || batch < 1) return 0.0f;
    return (float)((double)base_lr * (double)batch / (double)base_batch);
}

int64_t firecaffe_heap_reserved_bytes(int64_t heap_bytes) {
    if (heap_bytes < 0) return -1;
    return fc_flag_layout(heap_bytes).total_bytes;
}

fc_status firecaffe_heap_alloc(int64_t bytes, void** heap) {
    if (!heap || bytes <= 0) return FC_ERR_INVALID_ARG;
    *heap = nullptr;
    void* p = nullptr;
    if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) return FC_ERR_CUDA;
    if (cudaMemset(p, 0, (size_t)bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        cudaFree(p);
        return FC_ERR_CUDA;
    }
    *heap = p;
    return FC_OK;
}

fc_status firecaffe_heap_free(void* heap) {
    if (!heap) return FC_OK;
    return cudaFree(heap) == cudaSuccess ? FC_OK : FC_ERR_CUDA;
}

fc_status firecaffe_heap_export(void* heap, uint8_t* handle_out) {
    if (!heap || !handle_out) return FC_ERR_INVALID_ARG;
    static_assert(sizeof(cudaIpcMemHandle_t) == FC_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, heap) != cudaSuccess) return FC_ERR_CUDA;
    memcpy(handle_out, &h, sizeof(h));
    return FC_OK;
}

static void default_config(fc_world* w) {
    w->arity = 2;
    // measured fastest on B200 at p = 2, 4: one NVSwitch round per call
    w->sched = FC_SCHED_FLAT;
    w->bcast = FC_BCAST_DIRECT;
}

static fc_status world_common(fc_world* w, int world_size, int dev, int64_t heap_bytes,
                              uint64_t timeout_ns) {
    w->p = world_size;
    w->device = dev;
    w->heap_bytes = heap_bytes;
    w->timeout_ns = timeout_ns ? timeout_ns : 30ull * 1000000000ull;
    w->layout = fc_flag_layout(heap_bytes);
    if (w->layout.total_bytes >= heap_bytes) return FC_ERR_INVALID_ARG;
    if (cudaMalloc(&w->d_status, sizeof(int)) != cudaSuccess) return FC_ERR_CUDA;
    if (cudaMemset(w->d_status, 0, sizeof(int)) != cudaSuccess) return FC_ERR_CUDA;
    if (cudaMalloc(&w->d_ctl, FC_CTL_WORDS * sizeof(uint32_t)) != cudaSuccess) return FC_ERR_CUDA;
    if (cudaMemset(w->d_ctl, 0, FC_CTL_WORDS * sizeof(uint32_t)) != cudaSuccess) return FC_ERR_CUDA;
    default_config(w);
    return FC_OK;
}

fc_status firecaffe_world_create(int rank, int world_size, int cuda_device, void* local_heap,
                                 const uint8_t* handles, int64_t heap_bytes, uint64_t timeout_ns,
                                 fc_world** out) {
    if (!out) return FC_ERR_INVALID_ARG;
    *out = nullptr;
    if (world_size < 1 || world_size > FC_MAX_RANKS || rank < 0 || rank >= world_size)
        return FC_ERR_INVALID_ARG;
    if (!local_heap || heap_bytes <= 0 || (world_size > 1 && !handles)) return FC_ERR_INVALID_ARG;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return FC_ERR_CUDA;
    if (cur != cuda_device) return FC_ERR_MISMATCH;
    fc_world* w = new fc_world();
    memset(w, 0, sizeof(*w));
    w->rank = rank;
    w->virt = 0;
    w->heap_local = (char*)local_heap;
    fc_status st = world_common(w, world_size, cuda_device, heap_bytes, timeout_ns);
    if (st != FC_OK) {
        firecaffe_world_destroy(w);
        return st;
    }
    for (int q = 0; q < world_size; ++q) {
        if (q == rank) {
            w->peer[q] = (char*)local_heap;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, handles + (size_t)q * FC_IPC_HANDLE_BYTES, sizeof(h));
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            firecaffe_world_destroy(w);
            return FC_ERR_CUDA;
        }
        w->peer[q] = (char*)p;
        w->opened[q] = true;
    }
    *out = w;
    return FC_OK;
}

fc_status firecaffe_world_create_virtual(int world_size, int cuda_device, void* heap,
                                         int64_t heap_bytes_per_rank, uint64_t timeout_ns,
                                         fc_world** out) {
    if (!out) return FC_ERR_INVALID_ARG;
    *out = nullptr;
    if (world_size < 1 || world_size > FC_MAX_RANKS || !heap || heap_bytes_per_rank <= 0 ||
        (heap_bytes_per_rank & 255) != 0)
        return FC_ERR_INVALID_ARG;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return FC_ERR_CUDA;
    if (cur != cuda_device) return FC_ERR_MISMATCH;
    fc_world* w = new fc_world();
    memset(w, 0, sizeof(*w));
    w->rank = -1;
    w->virt = 1;
    w->heap_local = (char*)heap;
    fc_status st = world_common(w, world_size, cuda_device, heap_bytes_per_rank, timeout_ns);
    if (st != FC_OK) {
        firecaffe_world_destroy(w);
        return st;
    }
    for (int q = 0; q < world_size; ++q) w->peer[q] = (char*)heap + (int64_t)q * heap_bytes_per_rank;
    *out = w;
    return FC_OK;
}

fc_status firecaffe_world_destroy(fc_world* w) {
    if (!w) return FC_OK;
    fc_status st = FC_OK;
    for (int q = 0; q < FC_MAX_RANKS; ++q)
        if (w->opened[q] && cudaIpcCloseMemHandle(w->peer[q]) != cudaSuccess) st = FC_ERR_CUDA;
    if (w->d_status) cudaFree(w->d_status);
    if (w->d_ctl) cudaFree(w->d_ctl);
    if (w->hp_ready) {
        for (int i = 0; i < 3; ++i) cudaStreamDestroy(w->hp_s[i]);
        cudaEventDestroy(w->hp_start);
        for (int i = 0; i < FC_HOST_MAX_STAGES; ++i) {
            cudaEventDestroy(w->hp_h2d[i]);
            cudaEventDestroy(w->hp_coll[i]);
        }
    }
    delete w;
    return st;
}

fc_status firecaffe_world_config(fc_world* w, int arity, fc_sched sched, fc_bcast bcast) {
    if (!w) return FC_ERR_INVALID_ARG;
    if (arity < 2 || (bcast != FC_BCAST_TREE && bcast != FC_BCAST_DIRECT && bcast != FC_BCAST_PULL))
        return FC_ERR_INVALID_ARG;
    if (bcast == FC_BCAST_PULL && sched != FC_SCHED_FLAT) return FC_ERR_UNSUPPORTED;
    if (sched != FC_SCHED_FOREST && sched != FC_SCHED_SINGLE_ROOT && sched != FC_SCHED_FLAT)
        return FC_ERR_INVALID_ARG;
    if (sched == FC_SCHED_FOREST && (arity != 2 || !is_pow2(w->p))) return FC_ERR_UNSUPPORTED;
    if (sched == FC_SCHED_SINGLE_ROOT && arity != 2) return FC_ERR_UNSUPPORTED;
    w->arity = arity;
    w->sched = sched;
    w->bcast = bcast;
    return FC_OK;
}

fc_status firecaffe_world_get_config(const fc_world* w, int* arity, fc_sched* sched,
                                     fc_bcast* bcast) {
    if (!w) return FC_ERR_INVALID_ARG;
    if (arity) *arity = w->arity;
    if (sched) *sched = w->sched;
    if (bcast) *bcast = w->bcast;
    return FC_OK;
}

fc_status firecaffe_world_poll(fc_world* w) {
    if (!w) return FC_ERR_INVALID_ARG;
    if (cudaDeviceSynchronize() != cudaSuccess) return FC_ERR_CUDA;
    int s = 0;
    if (cudaMemcpy(&s, w->d_status, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
        return FC_ERR_CUDA;
    return (fc_status)s;
}

fc_status firecaffe_plan_owned_range(int world_size, fc_sched sched, int rank, int64_t n,
                                     int64_t* begin, int64_t* end) {
    if (!begin || !end || world_size < 1 || world_size > FC_MAX_RANKS || rank < 0 ||
        rank >= world_size || n < 0)
        return FC_ERR_INVALID_ARG;
    if (world_size == 1) {
        *begin = 0;
        *end = n;
        return FC_OK;
    }
    const int64_t nch = (n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
    int64_t c0, c1;
    owned_chunks(rank, world_size, nch, sched == FC_SCHED_SINGLE_ROOT, &c0, &c1);
    int64_t b = c0 * FC_CHUNK_FLOATS, e = c1 * FC_CHUNK_FLOATS;
    if (b > n) b = n;
    if (e > n) e = n;
    if (e < b) e = b;
    *begin = b;
    *end = e;
    return FC_OK;
}

fc_status firecaffe_owned_range(const fc_world* w, int rank, int64_t n, int64_t* begin,
                                int64_t* end) {
    if (!w) return FC_ERR_INVALID_ARG;
    return firecaffe_plan_owned_range(w->p, w->sched, rank, n, begin, end);
}

static fc_status sgd_impl(float* w, const float* grad, float* mom, int64_t n, float lr, float mu,
                          float wd, int64_t batch, const fc_segments* segs, void* stream,
                          const fc_lr_state* lrst = nullptr);

fc_status firecaffe_sgd_step(float* w, const float* grad, float* mom, int64_t n, float lr,
                             float mu, float wd, int64_t batch, void* stream) {
    return sgd_impl(w, grad, mom, n, lr, mu, wd, batch, nullptr, stream);
}

fc_status firecaffe_sgd_step_segments(float* w, const float* grad, float* mom, int64_t n, float lr,
                                      float mu, float wd, int64_t batch, const fc_segments* segs,
                                      void* stream) {
    if (!segs) return FC_ERR_INVALID_ARG;
    return sgd_impl(w, grad, mom, n, lr, mu, wd, batch, segs, stream);
}

static fc_status check_segs(const fc_segments* segs, int64_t n, FcSegs* out) {
    out->begin = nullptr;
    out->lrm = nullptr;
    out->dm = nullptr;
    out->nseg = 0;
    if (!segs) return FC_OK;
    if (segs->n != n) return FC_ERR_INVALID_ARG;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return FC_ERR_CUDA;
    if (cur != segs->device) return FC_ERR_MISMATCH;
    out->begin = segs->d_begin;
    out->lrm = segs->d_lrm;
    out->dm = segs->d_dm;
    out->nseg = segs->nseg;
    return FC_OK;
}

static fc_status check_lr_state(const fc_lr_state* lrst) {
    if (!lrst) return FC_OK;
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return FC_ERR_CUDA;
    return cur == lrst->device ? FC_OK : FC_ERR_MISMATCH;
}

static fc_status sgd_impl(float* w, const float* grad, float* mom, int64_t n, float lr, float mu,
                          float wd, int64_t batch, const fc_segments* segs, void* stream,
                          const fc_lr_state* lrst) {
    if (n < 0) return FC_ERR_INVALID_ARG;
    fc_status st = check_hyper(lr, mu, wd, batch);
    if (st != FC_OK) return st;
    if (n == 0) return segs && segs->n != 0 ? FC_ERR_INVALID_ARG : FC_OK;
    if (check_vec(w, n) || check_vec(grad, n) || check_vec(mom, n)) return FC_ERR_INVALID_ARG;
    const int64_t bytes = n * 4;
    if (overlap(w, grad, bytes) || overlap(w, mom, bytes) || overlap(grad, mom, bytes))
        return FC_ERR_INVALID_ARG;
    FcSegs sd;
    st = check_segs(segs, n, &sd);
    if (st != FC_OK) return st;
    if ((st = check_lr_state(lrst)) != FC_OK) return st;
    cudaError_t e = launch_sgd_step(w, grad, mom, n, lr, mu, wd, inv_batch(batch), sd,
                                    (cudaStream_t)stream, lrst ? lrst->d : nullptr);
    return e == cudaSuccess ? FC_OK : FC_ERR_CUDA;
}

// Offset of a symmetric buffer inside this rank's heap, or -1.
static int64_t heap_offset(const fc_world* w, const void* p, int64_t n) {
    const char* c = (const char*)p;
    const int64_t off = c - w->heap_local;
    if (c < w->heap_local || off < w->layout.total_bytes) return -1;
    if (off + n * 4 > w->heap_bytes) return -1;
    return off;
}

static fc_status collective(fc_world* w, int op, float* wt, float* grad, float* mom, int64_t n,
                            float lr, float mu, float wd, int64_t batch,
                            const fc_segments* segs, void* stream, int win_k = 0, int win_s = 1,
                            const fc_lr_state* lrst = nullptr) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return FC_ERR_CUDA;
    if (cur != w->device) return FC_ERR_MISMATCH;
    FcColl c;
    memset(&c, 0, sizeof(c));
    const bool bf16 = op == FC_OP_ALLREDUCE_SGD_BF16;
    // (bf16 gradients: half the bytes; heap_offset checks n*4, which covers them)
    c.off_grad = heap_offset(w, grad, bf16 ? (n + 1) / 2 : n);
    if (c.off_grad < 0) return FC_ERR_NOT_SYMMETRIC;
    c.off_w = 0;
    c.off_mom = -1;
    uint32_t seg_hash = 0;
    if (op == FC_OP_ALLREDUCE_SGD || bf16) {
        c.off_w = heap_offset(w, wt, n);
        if (c.off_w < 0) return FC_ERR_NOT_SYMMETRIC;
        if (w->virt) {
            c.off_mom = heap_offset(w, mom, n);
            if (c.off_mom < 0) return FC_ERR_NOT_SYMMETRIC;
        }
        c.mom_local = mom;
        c.lr = lr;
        c.mu = mu;
        c.wd = wd;
        c.inv_b = inv_batch(batch);
        fc_status st = check_segs(segs, n, &c.segs);
        if (st != FC_OK) return st;
        if (segs) seg_hash = segs->hash;
        if ((st = check_lr_state(lrst)) != FC_OK) return st;
        if (lrst) {
            c.lrs = lrst->d;
            c.lr = 0.0f;
            seg_hash ^= lrst->hash * 0x9e3779b1u;  // the schedule replaces lr in the signature
        }
    }
    for (int q = 0; q < w->p; ++q) c.peers.heap[q] = w->peer[q];
    c.rank = w->virt ? -1 : w->rank;
    c.p = w->p;
    c.ctl = w->d_ctl;
    {  // call signature (FNV-1a): every rank must make the same call
        uint32_t h = 2166136261u;
        auto mix = [&h](const void* p, size_t len) {
            const unsigned char* b = (const unsigned char*)p;
            for (size_t i = 0; i < len; ++i) h = (h ^ b[i]) * 16777619u;
        };
        const int sched_used = op == FC_OP_PS ? -1 : (int)w->sched;
        const int bc = (int)w->bcast;
        mix(&op, sizeof op);
        mix(&n, sizeof n);
        mix(&w->p, sizeof w->p);
        mix(&sched_used, sizeof sched_used);
        mix(&w->arity, sizeof w->arity);
        mix(&bc, sizeof bc);
        mix(&c.lr, sizeof c.lr);
        mix(&c.mu, sizeof c.mu);
        mix(&c.wd, sizeof c.wd);
        mix(&c.inv_b, sizeof c.inv_b);
        mix(&seg_hash, sizeof seg_hash);
        const int rx = exit_mode();
        mix(&rx, sizeof rx);
        mix(&win_k, sizeof win_k);
        mix(&win_s, sizeof win_s);
        // the buffers' heap offsets: a peer's buffer is addressed at THIS
        // rank's offset, so ranks that disagree must fail, not read garbage
        mix(&c.off_grad, sizeof c.off_grad);
        mix(&c.off_w, sizeof c.off_w);
        mix(&c.off_mom, sizeof c.off_mom);
        // the flag layout (red/av offsets) derives from each rank's own heap size and
        // is applied to the peers' heaps: ranks whose heaps differ must fail at the
        // entry barrier (its stamps sit at fixed offsets) before any such flag is used
        mix(&w->heap_bytes, sizeof w->heap_bytes);
        c.sig = h;
    }
    c.op = op;
    c.rank_exit = exit_mode();
    c.win_k = win_k;
    c.win_s = win_s;
    c.flat_map = flat_map();
    c.preclaim = flat_preclaim();
    c.clean_exit = clean_exit();
    c.owner_single_root = w->sched == FC_SCHED_SINGLE_ROOT ? 1 : 0;
    c.timeout_ns = w->timeout_ns;
    c.status = w->d_status;
    c.n = n;
    c.bcast = w->bcast;
    c.bar_words = w->layout.bar_words;
    c.red_words = w->layout.red_words;
    c.max_chunks = w->layout.max_chunks;
    const int sched = (op == FC_OP_PS || bf16) ? FC_SCHED_FLAT : w->sched;
    int grid = collective_grid(sched, w->arity, w->p, w->virt != 0, op, n);
    if (grid < 1) return FC_ERR_UNSUPPORTED;
    if (w->max_ctas > 0 && grid > w->max_ctas) grid = w->max_ctas;
    w->last_grid = grid;
    // the grid is part of the call: the barriers pair CTAs by index across ranks
    c.sig = (c.sig ^ (uint32_t)grid) * 16777619u;
    const int64_t need = (int64_t)grid * (w->virt ? w->p : 1) * FC_TRACE_SLOTS;
    c.trace = (w->trace && w->trace_cap >= need) ? w->trace : nullptr;
    cudaError_t e = launch_collective(c, sched, w->arity, w->virt != 0, grid, (cudaStream_t)stream);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return FC_ERR_CUDA;
    }
    return FC_OK;
}

fc_status firecaffe_tree_allreduce(float* grad, int64_t n, fc_world* w, void* stream) {
    if (!w || n < 0) return FC_ERR_INVALID_ARG;
    if (n == 0 || w->p == 1) return FC_OK;
    if (check_vec(grad, n)) return FC_ERR_INVALID_ARG;
    return collective(w, FC_OP_ALLREDUCE, nullptr, grad, nullptr, n, 0, 0, 0, 1, nullptr, stream);
}

fc_status firecaffe_allgather_owned(float* buf, int64_t n, fc_world* w, void* stream) {
    if (!w || n < 0) return FC_ERR_INVALID_ARG;
    if (n == 0 || w->p == 1) return FC_OK;
    if (check_vec(buf, n)) return FC_ERR_INVALID_ARG;
    return collective(w, FC_OP_ALLGATHER_OWNED, nullptr, buf, nullptr, n, 0, 0, 0, 1, nullptr, stream);
}

fc_status firecaffe_ps_allreduce(float* grad, int64_t n, fc_world* w, void* stream) {
    if (!w || n < 0) return FC_ERR_INVALID_ARG;
    if (n == 0 || w->p == 1) return FC_OK;
    if (check_vec(grad, n)) return FC_ERR_INVALID_ARG;
    return collective(w, FC_OP_PS, nullptr, grad, nullptr, n, 0, 0, 0, 1, nullptr, stream);
}

static fc_status fused_impl(float* wt, float* grad, float* mom, int64_t n, float lr, float mu,
                            float wd, int64_t batch, const fc_segments* segs, fc_world* w,
                            void* stream, const fc_lr_state* lrst = nullptr) {
    if (!w || n < 0) return FC_ERR_INVALID_ARG;
    fc_status st = check_hyper(lr, mu, wd, batch);
    if (st != FC_OK) return st;
    if (n == 0) return segs && segs->n != 0 ? FC_ERR_INVALID_ARG : FC_OK;
    if (check_vec(wt, n) || check_vec(grad, n) || check_vec(mom, n)) return FC_ERR_INVALID_ARG;
    const int64_t bytes = n * 4;
    if (overlap(wt, grad, bytes) || overlap(wt, mom, bytes) || overlap(grad, mom, bytes))
        return FC_ERR_INVALID_ARG;
    if (w->p == 1) return sgd_impl(wt, grad, mom, n, lr, mu, wd, batch, segs, stream, lrst);
    return collective(w, FC_OP_ALLREDUCE_SGD, wt, grad, mom, n, lr, mu, wd, batch, segs, stream, 0, 1,
                      lrst);
}

fc_status firecaffe_tree_allreduce_sgd(float* wt, float* grad, float* mom, int64_t n, float lr,
                                       float mu, float wd, int64_t batch, fc_world* w,
                                       void* stream) {
    return fused_impl(wt, grad, mom, n, lr, mu, wd, batch, nullptr, w, stream);
}

fc_status firecaffe_tree_allreduce_sgd_segments(float* wt, float* grad, float* mom, int64_t n,
                                                float lr, float mu, float wd, int64_t batch,
                                                const fc_segments* segs, fc_world* w,
                                                void* stream) {
    if (!segs) return FC_ERR_INVALID_ARG;
    return fused_impl(wt, grad, mom, n, lr, mu, wd, batch, segs, w, stream);
}

static bool overlap2(const void* a, int64_t abytes, const void* b, int64_t bbytes) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + (uintptr_t)bbytes && y < x + (uintptr_t)abytes;
}

static fc_status check_bf16_args(float* wt, const uint16_t* grad, float* mom, int64_t n, float lr,
                                 float mu, float wd, int64_t batch) {
    if (n < 0) return FC_ERR_INVALID_ARG;
    fc_status st = check_hyper(lr, mu, wd, batch);
    if (st != FC_OK) return st;
    if (n == 0) return FC_OK;
    if (check_vec(wt, n) || check_vec(grad, n) || check_vec(mom, n)) return FC_ERR_INVALID_ARG;
    if (overlap2(wt, 4 * n, grad, 2 * n) || overlap2(wt, 4 * n, mom, 4 * n) ||
        overlap2(grad, 2 * n, mom, 4 * n))
        return FC_ERR_INVALID_ARG;
    return FC_OK;
}

fc_status firecaffe_sgd_step_bf16(float* wt, const uint16_t* grad, float* mom, int64_t n, float lr,
                                  float mu, float wd, int64_t batch, const fc_segments* segs,
                                  void* stream) {
    fc_status st = check_bf16_args(wt, grad, mom, n, lr, mu, wd, batch);
    if (st != FC_OK || n == 0) return st;
    FcSegs sd;
    st = check_segs(segs, n, &sd);
    if (st != FC_OK) return st;
    cudaError_t e = launch_sgd_step_bf16(wt, grad, mom, n, lr, mu, wd, inv_batch(batch), sd,
                                         (cudaStream_t)stream);
    return e == cudaSuccess ? FC_OK : FC_ERR_CUDA;
}

fc_status firecaffe_tree_allreduce_sgd_bf16(float* wt, uint16_t* grad, float* mom, int64_t n,
                                            float lr, float mu, float wd, int64_t batch,
                                            const fc_segments* segs, fc_world* w, void* stream) {
    if (!w) return FC_ERR_INVALID_ARG;
    fc_status st = check_bf16_args(wt, grad, mom, n, lr, mu, wd, batch);
    if (st != FC_OK || n == 0) return st;
    if (w->p == 1) return firecaffe_sgd_step_bf16(wt, grad, mom, n, lr, mu, wd, batch, segs, stream);
    return collective(w, FC_OP_ALLREDUCE_SGD_BF16, wt, (float*)grad, mom, n, lr, mu, wd, batch, segs,
                      stream);
}

fc_status firecaffe_segments_create(const fc_segment* segs, int nseg, int64_t n,
                                    fc_segments** out) {
    if (!out) return FC_ERR_INVALID_ARG;
    *out = nullptr;
    if (!segs || nseg < 1 || nseg > 65536 || n < 1) return FC_ERR_INVALID_ARG;
    if (segs[0].begin != 0) return FC_ERR_INVALID_ARG;
    for (int s = 0; s < nseg; ++s) {
        if (s > 0 && segs[s].begin <= segs[s - 1].begin) return FC_ERR_INVALID_ARG;
        if (segs[s].begin >= n) return FC_ERR_INVALID_ARG;
        if (!(segs[s].lr_mult >= 0.0f) || !std::isfinite(segs[s].lr_mult)) return FC_ERR_INVALID_ARG;
        if (!(segs[s].decay_mult >= 0.0f) || !std::isfinite(segs[s].decay_mult))
            return FC_ERR_INVALID_ARG;
    }
    fc_segments* t = new fc_segments();
    memset(t, 0, sizeof(*t));
    t->nseg = nseg;
    t->n = n;
    if (cudaGetDevice(&t->device) != cudaSuccess) {
        delete t;
        return FC_ERR_CUDA;
    }
    int64_t* hb = new int64_t[nseg];
    float* hl = new float[nseg];
    float* hd = new float[nseg];
    uint32_t h = 2166136261u;
    for (int s = 0; s < nseg; ++s) {
        hb[s] = segs[s].begin;
        hl[s] = segs[s].lr_mult;
        hd[s] = segs[s].decay_mult;
        const unsigned char* b = (const unsigned char*)&segs[s];
        for (size_t i = 0; i < sizeof(fc_segment); ++i) h = (h ^ b[i]) * 16777619u;
    }
    t->hash = h;
    bool ok = cudaMalloc(&t->d_begin, nseg * sizeof(int64_t)) == cudaSuccess &&
              cudaMalloc(&t->d_lrm, nseg * sizeof(float)) == cudaSuccess &&
              cudaMalloc(&t->d_dm, nseg * sizeof(float)) == cudaSuccess &&
              cudaMemcpy(t->d_begin, hb, nseg * sizeof(int64_t), cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(t->d_lrm, hl, nseg * sizeof(float), cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaMemcpy(t->d_dm, hd, nseg * sizeof(float), cudaMemcpyHostToDevice) == cudaSuccess;
    delete[] hb;
    delete[] hl;
    delete[] hd;
    if (!ok) {
        firecaffe_segments_destroy(t);
        return FC_ERR_CUDA;
    }
    *out = t;
    return FC_OK;
}

fc_status firecaffe_segments_destroy(fc_segments* t) {
    if (!t) return FC_OK;
    if (t->d_begin) cudaFree(t->d_begin);
    if (t->d_lrm) cudaFree(t->d_lrm);
    if (t->d_dm) cudaFree(t->d_dm);
    delete t;
    return FC_OK;
}

// Device address of page-locked host memory (UVA-mapped), or null.
static void* device_view(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

static bool pinned_host(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

fc_status firecaffe_sgd_step_host(float* w, float* grad, float* mom, const float* grad_host,
                                  float* w_host, int64_t n, float lr, float mu, float wd,
                                  int64_t batch, const fc_segments* segs, void* stream) {
    if (n < 0) return FC_ERR_INVALID_ARG;
    fc_status st = check_hyper(lr, mu, wd, batch);
    if (st != FC_OK) return st;
    if (n == 0) return FC_OK;
    if (check_vec(w, n) || check_vec(grad, n) || check_vec(mom, n)) return FC_ERR_INVALID_ARG;
    if (!grad_host || !w_host || !pinned_host(grad_host) || !pinned_host(w_host))
        return FC_ERR_INVALID_ARG;
    const int64_t bytes = n * 4;
    if (overlap(w, grad, bytes) || overlap(w, mom, bytes) || overlap(grad, mom, bytes) ||
        overlap(grad_host, w_host, bytes))
        return FC_ERR_INVALID_ARG;
    FcSegs sd;
    st = check_segs(segs, n, &sd);
    if (st != FC_OK) return st;
    // Three host paths (scripts/pcie_bench.py, NiN, B200; PCIe H2D || D2H ceiling 0.66 ms):
    //   hybrid (default): copy-engine H2D per 4 MB stage, the SGD kernel writes the new
    //                     weights straight to pinned host memory            0.79 ms
    //   zc   : one zero-copy kernel (PCIe reads + writes from the SMs)      0.84 ms
    //   pipe : H2D || SGD || D2H over three streams, 8 MB stages            0.83 ms
    // FC_HOST_MODE / FC_PIPE_CHUNK override (tuning only; all give the same bits).
    static int mode = -1;
    static int64_t chunk = 0;  // floats per stage
    if (mode < 0) {
        const char* m = getenv("FC_HOST_MODE");
        mode = (m && strcmp(m, "pipe") == 0) ? 1 : (m && strcmp(m, "zc") == 0) ? 0 : 2;
        const char* e = getenv("FC_PIPE_CHUNK");
        chunk = e ? atoll(e) : (mode == 1 ? ((int64_t)1 << 21) : ((int64_t)1 << 20));
        chunk = (chunk + 3) / 4 * 4;
        if (chunk < 4096) chunk = 4096;
    }
    cudaError_t e;
    const float* gdev = (const float*)device_view(grad_host);
    float* wdev = (float*)device_view(w_host);
    const bool mapped = gdev && wdev && aligned16(gdev) && aligned16(wdev);
    if (mode == 0 && mapped) {
        e = launch_sgd_step_hostio(w, gdev, grad, mom, wdev, n, lr, mu, wd, inv_batch(batch), sd,
                                   (cudaStream_t)stream);
    } else if (mode == 2 && mapped) {
        e = launch_sgd_step_hybrid(w, grad_host, grad, mom, wdev, n, lr, mu, wd, inv_batch(batch), sd,
                                   chunk, (cudaStream_t)stream);
    } else {
        e = launch_sgd_step_host(w, grad_host, grad, mom, w_host, n, lr, mu, wd, inv_batch(batch), sd,
                                 chunk, (cudaStream_t)stream);
    }
    return e == cudaSuccess ? FC_OK : FC_ERR_CUDA;
}

// Stages of the pipelined host entry point (FC_HOST_STAGES, default 4; 1 = serial).
static int host_stages() {
    static int s = -1;
    if (s < 0) {
        const char* e = getenv("FC_HOST_STAGES");
        s = e ? atoi(e) : 4;
        if (s < 1) s = 1;
        if (s > FC_HOST_MAX_STAGES) s = FC_HOST_MAX_STAGES;
    }
    return s;
}

static fc_status host_pipe_ready(fc_world* w) {
    if (w->hp_ready) return FC_OK;
    for (int i = 0; i < 3; ++i)
        if (cudaStreamCreateWithFlags(&w->hp_s[i], cudaStreamNonBlocking) != cudaSuccess) return FC_ERR_CUDA;
    if (cudaEventCreateWithFlags(&w->hp_start, cudaEventDisableTiming) != cudaSuccess) return FC_ERR_CUDA;
    for (int i = 0; i < FC_HOST_MAX_STAGES; ++i)
        if (cudaEventCreateWithFlags(&w->hp_h2d[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&w->hp_coll[i], cudaEventDisableTiming) != cudaSuccess)
            return FC_ERR_CUDA;
    w->hp_ready = true;
    return FC_OK;
}

// Elements [x, y) that stage k of s of the FLAT collective processes in owner
// r's slice (the kernel's window_range on float4 units; the n % 4 tail rides
// with the last stage).
static void stage_range(int r, int p, int64_t n, int k, int s, int64_t* x, int64_t* y) {
    const int64_t nch = (n + FC_CHUNK_FLOATS - 1) / FC_CHUNK_FLOATS;
    int64_t c0, c1;
    owned_chunks(r, p, nch, false, &c0, &c1);
    const int64_t e0 = c0 * FC_CHUNK_FLOATS;
    const int64_t e1 = c1 * FC_CHUNK_FLOATS < n ? c1 * FC_CHUNK_FLOATS : n;
    if (e1 <= e0) {
        *x = *y = e0;
        return;
    }
    int64_t a, b;
    window_range(e0 / 4, e1 / 4, k, s, &a, &b);
    *x = 4 * a;
    *y = k == s - 1 ? e1 : 4 * b;
}

fc_status firecaffe_tree_allreduce_sgd_host(float* w, float* grad, float* mom,
                                            const float* grad_host, float* w_host, int64_t n,
                                            float lr, float mu, float wd, int64_t batch,
                                            const fc_segments* segs, fc_world* world,
                                            void* stream) {
    if (!world || n < 0) return FC_ERR_INVALID_ARG;
    if (world->virt) return FC_ERR_UNSUPPORTED;  // one host buffer cannot feed p virtual ranks
    if (world->p == 1)
        return firecaffe_sgd_step_host(w, grad, mom, grad_host, w_host, n, lr, mu, wd, batch, segs,
                                       stream);
    if (n == 0) return FC_OK;
    if (!grad_host || !w_host || !pinned_host(grad_host) || !pinned_host(w_host))
        return FC_ERR_INVALID_ARG;
    fc_status st = check_hyper(lr, mu, wd, batch);
    if (st != FC_OK) return st;
    if (check_vec(grad, n) || check_vec(w, n) || check_vec(mom, n)) return FC_ERR_INVALID_ARG;
    const int64_t bytes = n * 4;
    if (overlap(w, grad, bytes) || overlap(w, mom, bytes) || overlap(grad, mom, bytes) ||
        overlap(grad_host, w_host, bytes))
        return FC_ERR_INVALID_ARG;
    FcSegs sd;
    if ((st = check_segs(segs, n, &sd)) != FC_OK) return st;
    if (heap_offset(world, grad, n) < 0 || heap_offset(world, w, n) < 0) return FC_ERR_NOT_SYMMETRIC;
    cudaStream_t user = (cudaStream_t)stream;
    const int S = host_stages();
    const int p = world->p;
    const bool staged = S > 1 && world->sched == FC_SCHED_FLAT && world->bcast != FC_BCAST_PULL &&
                        n >= (int64_t)S * p * FC_CHUNK_FLOATS;
    if (!staged) {  // serial: H2D, the fused collective, D2H on the caller's stream
        if (cudaMemcpyAsync(grad, grad_host, bytes, cudaMemcpyHostToDevice, user) != cudaSuccess)
            return FC_ERR_CUDA;
        st = fused_impl(w, grad, mom, n, lr, mu, wd, batch, segs, world, stream);
        if (st != FC_OK) return st;
        if (cudaMemcpyAsync(w_host, w, bytes, cudaMemcpyDeviceToHost, user) != cudaSuccess)
            return FC_ERR_CUDA;
        return FC_OK;
    }
    // Staged (S stages, three internal streams): stage k's gradient windows come
    // in on the H2D copy engine while stage k-1's collective runs over NVLink and
    // stage k-2's weights go out on the D2H copy engine.  Stage k of the FLAT
    // collective covers window k of EVERY owner's slice, so the momentum
    // ownership and the bits equal one full call (tested).
    if ((st = host_pipe_ready(world)) != FC_OK) return st;
    cudaStream_t* hs = world->hp_s;
    if (cudaEventRecord(world->hp_start, user) != cudaSuccess) return FC_ERR_CUDA;
    for (int i = 0; i < 3; ++i)
        if (cudaStreamWaitEvent(hs[i], world->hp_start, 0) != cudaSuccess) return FC_ERR_CUDA;
    for (int k = 0; k < S; ++k) {
        for (int r = 0; r < p; ++r) {
            int64_t x, y;
            stage_range(r, p, n, k, S, &x, &y);
            if (y > x && cudaMemcpyAsync(grad + x, grad_host + x, (y - x) * 4, cudaMemcpyHostToDevice,
                                         hs[0]) != cudaSuccess)
                return FC_ERR_CUDA;
        }
        if (cudaEventRecord(world->hp_h2d[k], hs[0]) != cudaSuccess ||
            cudaStreamWaitEvent(hs[1], world->hp_h2d[k], 0) != cudaSuccess)
            return FC_ERR_CUDA;
        st = collective(world, FC_OP_ALLREDUCE_SGD, w, grad, mom, n, lr, mu, wd, batch, segs, hs[1], k, S);
        if (st != FC_OK) return st;
        if (cudaEventRecord(world->hp_coll[k], hs[1]) != cudaSuccess ||
            cudaStreamWaitEvent(hs[2], world->hp_coll[k], 0) != cudaSuccess)
            return FC_ERR_CUDA;
        for (int r = 0; r < p; ++r) {
            int64_t x, y;
            stage_range(r, p, n, k, S, &x, &y);
            if (y > x &&
                cudaMemcpyAsync(w_host + x, w + x, (y - x) * 4, cudaMemcpyDeviceToHost, hs[2]) != cudaSuccess)
                return FC_ERR_CUDA;
        }
    }
    // the caller's stream continues after the last weights are on the host
    if (cudaEventRecord(world->hp_start, hs[2]) != cudaSuccess) return FC_ERR_CUDA;
    return cudaStreamWaitEvent(user, world->hp_start, 0) == cudaSuccess ? FC_OK : FC_ERR_CUDA;
}

// The paper's learning-rate schedules, R21:
// STEP gamma^floor(iter/stepsize), MULTISTEP gamma^#{steps <= iter}, POLY
// (1 - min(iter, max_iter)/max_iter)^power; the factor in double by std::pow,
// lr = one rounding of base_lr * factor to fp32.  Domain: base_lr > 0, gamma > 0,
// power >= 0 (all finite), stepsize >= 1, max_iter >= 1, 0 <= nsteps <= 16.
static bool valid_schedule(const fc_lr_schedule* s) {
    if (!s || !(s->base_lr > 0.0f) || !std::isfinite(s->base_lr)) return false;
    switch (s->policy) {
        case FC_LR_FIXED:
            return true;
        case FC_LR_STEP:
            return s->stepsize >= 1 && s->gamma > 0.0f && std::isfinite(s->gamma);
        case FC_LR_MULTISTEP:
            return s->nsteps >= 0 && s->nsteps <= FC_LR_MAX_STEPS && s->gamma > 0.0f &&
                   std::isfinite(s->gamma);
        case FC_LR_POLY:
            return s->max_iter >= 1 && s->power >= 0.0f && std::isfinite(s->power);
    }
    return false;
}

// lr of schedule level k (FcLrDev, fc_internal.h): STEP / MULTISTEP k = the
// number of decays so far, POLY k = the (clamped) iteration, FIXED k = 0.
static float lr_of_level(const fc_lr_schedule& s, int64_t k) {
    double f = 1.0;
    if (s.policy == FC_LR_STEP || s.policy == FC_LR_MULTISTEP)
        f = std::pow((double)s.gamma, (double)k);
    else if (s.policy == FC_LR_POLY)
        f = std::pow(1.0 - (double)k / (double)s.max_iter, (double)s.power);
    return (float)((double)s.base_lr * f);
}

static int64_t level_of(const fc_lr_schedule& s, int64_t iter) {
    switch (s.policy) {
        case FC_LR_STEP: return iter / s.stepsize;
        case FC_LR_MULTISTEP: {
            int64_t k = 0;
            for (int j = 0; j < s.nsteps; ++j) k += s.steps[j] <= iter;
            return k;
        }
        case FC_LR_POLY: return iter < s.max_iter ? iter : s.max_iter;
    }
    return 0;
}

float firecaffe_lr_at(const fc_lr_schedule* s, int64_t iter) {
    if (!valid_schedule(s) || iter < 0) return -1.0f;
    return lr_of_level(*s, level_of(*s, iter));
}

// Largest level table an fc_lr_state uploads (64 MB).
#define FC_LR_MAX_LEVELS ((int64_t)1 << 24)

// Every level's lr, host-computed (lr_of_level).  STEP: the levels are
// unbounded, but gamma^k is monotone, so once the fp32 value is 0 (gamma < 1)
// or inf (gamma > 1), or gamma == 1, every later level has the same value and
// the device clamps to the last entry.
static fc_status lr_levels(const fc_lr_schedule& s, std::vector<float>* out) {
    out->clear();
    switch (s.policy) {
        case FC_LR_FIXED: out->push_back(s.base_lr); return FC_OK;
        case FC_LR_MULTISTEP:
            for (int64_t k = 0; k <= s.nsteps; ++k) out->push_back(lr_of_level(s, k));
            return FC_OK;
        case FC_LR_POLY:
            if (s.max_iter + 1 > FC_LR_MAX_LEVELS) return FC_ERR_UNSUPPORTED;
            out->resize((size_t)s.max_iter + 1);
            for (int64_t k = 0; k <= s.max_iter; ++k) (*out)[(size_t)k] = lr_of_level(s, k);
            return FC_OK;
        case FC_LR_STEP:
            for (int64_t k = 0;; ++k) {
                if (k >= FC_LR_MAX_LEVELS) return FC_ERR_UNSUPPORTED;
                const float v = lr_of_level(s, k);
                out->push_back(v);
                if (s.gamma == 1.0f || v == 0.0f || std::isinf(v)) return FC_OK;
            }
    }
    return FC_ERR_INVALID_ARG;
}

fc_status firecaffe_lr_state_create(const fc_lr_schedule* sched, int64_t first_iter,
                                    fc_lr_state** out) {
    if (!out) return FC_ERR_INVALID_ARG;
    *out = nullptr;
    if (!valid_schedule(sched) || first_iter < 0) return FC_ERR_INVALID_ARG;
    fc_lr_schedule s = *sched;
    if (s.policy != FC_LR_MULTISTEP) s.nsteps = 0;
    for (int j = s.nsteps; j < FC_LR_MAX_STEPS; ++j) s.steps[j] = 0;
    std::vector<float> levels;
    fc_status st = lr_levels(s, &levels);
    if (st != FC_OK) return st;
    fc_lr_state* t = new fc_lr_state();
    memset(t, 0, sizeof(*t));
    t->s = s;
    uint32_t h = 2166136261u;
    const unsigned char* b = (const unsigned char*)&t->s;
    for (size_t i = 0; i < sizeof(t->s); ++i) h = (h ^ b[i]) * 16777619u;
    t->hash = h;
    FcLrDev init;
    memset(&init, 0, sizeof(init));
    init.policy = s.policy;
    init.nsteps = s.nsteps;
    init.stepsize = s.stepsize;
    init.max_iter = s.max_iter;
    for (int j = 0; j < FC_LR_MAX_STEPS; ++j) init.steps[j] = s.steps[j];
    init.nlevels = (int64_t)levels.size();
    init.iter = first_iter;
    const size_t tb = levels.size() * sizeof(float);
    if (cudaGetDevice(&t->device) != cudaSuccess || cudaMalloc(&t->table, tb) != cudaSuccess ||
        cudaMemcpy(t->table, levels.data(), tb, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMalloc(&t->d, sizeof(FcLrDev)) != cudaSuccess) {
        cudaGetLastError();
        firecaffe_lr_state_destroy(t);
        return FC_ERR_CUDA;
    }
    init.table = t->table;
    if (cudaMemcpy(t->d, &init, sizeof(init), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        firecaffe_lr_state_destroy(t);
        return FC_ERR_CUDA;
    }
    *out = t;
    return FC_OK;
}

fc_status firecaffe_lr_state_destroy(fc_lr_state* t) {
    if (!t) return FC_OK;
    if (t->d) cudaFree(t->d);
    if (t->table) cudaFree(t->table);
    delete t;
    return FC_OK;
}

fc_status firecaffe_lr_state_get_iter(const fc_lr_state* t, int64_t* iter) {
    if (!t || !iter) return FC_ERR_INVALID_ARG;
    if (cudaDeviceSynchronize() != cudaSuccess) return FC_ERR_CUDA;
    return cudaMemcpy(iter, &t->d->iter, sizeof(int64_t), cudaMemcpyDeviceToHost) == cudaSuccess
               ? FC_OK
               : FC_ERR_CUDA;
}

fc_status firecaffe_lr_state_set_iter(fc_lr_state* t, int64_t iter) {
    if (!t || iter < 0) return FC_ERR_INVALID_ARG;
    if (cudaDeviceSynchronize() != cudaSuccess) return FC_ERR_CUDA;
    return cudaMemcpy(&t->d->iter, &iter, sizeof(int64_t), cudaMemcpyHostToDevice) == cudaSuccess
               ? FC_OK
               : FC_ERR_CUDA;
}

fc_status firecaffe_sgd_step_sched(float* w, const float* grad, float* mom, int64_t n,
                                   fc_lr_state* lr, float mu, float wd, int64_t batch,
                                   const fc_segments* segs, void* stream) {
    if (!lr) return FC_ERR_INVALID_ARG;
    return sgd_impl(w, grad, mom, n, 1.0f, mu, wd, batch, segs, stream, lr);
}

fc_status firecaffe_tree_allreduce_sgd_sched(float* wt, float* grad, float* mom, int64_t n,
                                             fc_lr_state* lr, float mu, float wd, int64_t batch,
                                             const fc_segments* segs, fc_world* w, void* stream) {
    if (!lr) return FC_ERR_INVALID_ARG;
    return fused_impl(wt, grad, mom, n, 1.0f, mu, wd, batch, segs, w, stream, lr);
}

void firecaffe_tune_sgd_unroll(int u) { set_sgd_unroll(u); }

fc_status firecaffe_world_set_trace(fc_world* w, uint64_t* buf, int64_t capacity) {
    if (!w || capacity < 0) return FC_ERR_INVALID_ARG;
    w->trace = buf;
    w->trace_cap = buf ? capacity : 0;
    return FC_OK;
}

int firecaffe_world_last_grid(const fc_world* w) { return w ? w->last_grid : 0; }

fc_status firecaffe_world_set_max_ctas(fc_world* w, int max_ctas) {
    if (!w || max_ctas < 0 || max_ctas >= FC_EXIT_CTA_SLOT) return FC_ERR_INVALID_ARG;
    w->max_ctas = max_ctas;
    return FC_OK;
}

}  // extern "C"
