/* firecaffe.h — C ABI of the B200-native FireCaffe data-parallel hot path.
 *
 * FireCaffe (Iandola et al., arXiv 1511.00175; PAPER.md = the paper's text,
 * cited as P:line) trains with data parallelism: every worker computes the SUM
 * of the weight gradients over its part of the batch, the
 * per-worker sums are added across workers ("identical numerical
 * results as ... a single GPU") through a reduction tree (§6.2,
 * P:276-303) instead of a parameter server (§6.1), the sums go
 * "back down the tree", and every replica applies the SGD update
 * with momentum and weight decay.
 *
 * This library implements that per-iteration aggregation + update for one
 * NVSwitch node of B200 GPUs (1..8 ranks, one process per GPU):
 *   firecaffe_sgd_step            1-GPU fused SGD (the update alone)
 *   firecaffe_tree_allreduce      reduction-tree sum, result on every rank
 *   firecaffe_tree_allreduce_sgd  tree sum fused with the SGD update at each
 *                                 subtree root + broadcast of the new weights
 *   firecaffe_ps_allreduce        the paper's parameter server (baseline)
 *
 * Conventions (all functions):
 *   - All float buffers are fp32, in DEVICE memory, 16-byte aligned, and must
 *     not overlap.  The caller owns all memory; the library allocates device
 *     memory only in firecaffe_heap_alloc / firecaffe_world_create*.
 *   - Calls that take a `stream` (a cudaStream_t, passed as void*) are
 *     asynchronous: they validate on the host, enqueue one kernel and return.
 *     Host-detectable errors are returned synchronously and nothing is
 *     enqueued.  Device-side errors (a peer that never arrives) are sticky and
 *     returned by firecaffe_world_poll.
 *   - Collective calls (tree_*, ps_*) must be issued by every rank of the
 *     world in the same order with the same n and hyper-parameters (the
 *     MPI/NCCL convention).  Their `grad`, `w` (and, for a virtual world,
 *     `mom`) must lie inside the world's heap at the SAME byte offset on every
 *     rank (symmetric allocation), at or after firecaffe_heap_reserved_bytes().
 *     Ranks whose calls differ in any of these (op, n, executor, hyper-
 *     parameters, blob table, buffer offsets) all fail with a sticky
 *     FC_ERR_MISMATCH before any data moves.
 *   - Every device-side call (all but the *_host entry points' host checks) can
 *     be captured in a CUDA graph and replayed: kernel arguments do not change
 *     between calls (the collectives' call counter lives in device memory).
 *   - Numerics: round-to-nearest-even fp32, no FTZ, no fast-math; the summation
 *     association is fixed (documented per call) so results are bitwise
 *     deterministic and identical on every rank.  Inputs must be
 *     finite (NaN payloads are not reproducible across CPU/GPU).
 */
#ifndef FIRECAFFE_H
#define FIRECAFFE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FC_OK = 0,
    FC_ERR_INVALID_ARG = 1,   /* null/misaligned pointer, n < 0, lr <= 0, mu not in [0,1), wd < 0, batch < 1, overlap */
    FC_ERR_NOT_SYMMETRIC = 2, /* a collective buffer is outside the heap or inside its reserved prefix */
    FC_ERR_MISMATCH = 3,      /* world/device mismatch (called on another device), or, sticky from
                                 firecaffe_world_poll, ranks that made different collective calls
                                 (op, n, executor, hyper-parameters, blob table, buffer offsets) */
    FC_ERR_TIMEOUT = 4,       /* a peer did not arrive within the world's timeout (sticky) */
    FC_ERR_CUDA = 5,          /* a CUDA runtime call failed */
    FC_ERR_UNSUPPORTED = 6    /* schedule/arity not available for this world size */
} fc_status;

/* Who executes the reduction tree.  The VALUE never depends on it: every
 * schedule computes the same k-nomial association (see firecaffe_tree_allreduce). */
typedef enum {
    FC_SCHED_FOREST = 0,      /* XOR-rotated binomial forest: p owner slices, slice s reduced by a
                                 binomial tree rooted at rank s; level l pulls |W|/2^(l+1) from rank
                                 r^2^l over NVLink (recursive halving).  p power of two, arity 2. */
    FC_SCHED_SINGLE_ROOT = 1, /* the paper's single binomial tree rooted at rank 0 (Fig. P:312-315):
                                 level l, rank r (r mod 2^(l+1) == 0) pulls all of |W| from r+2^l. arity 2 */
    FC_SCHED_FLAT = 2         /* every rank pulls its owner slice from all p-1 peers at once and evaluates
                                 the tree in registers (one communication level); any p, any arity */
} fc_sched;

/* How the result goes "back down the tree". Bytes only: value-neutral. */
typedef enum {
    FC_BCAST_TREE = 0,        /* mirror of the reduce levels (recursive doubling for the forest) */
    FC_BCAST_DIRECT = 1,      /* each owner pushes its slice to every peer in one level */
    FC_BCAST_PULL = 2         /* FC_SCHED_FLAT only: owners publish their slice behind a per-CTA
                                 barrier, every rank pulls the others (no remote stores); the
                                 rank-level exit then keeps each published slice stable until
                                 every peer has pulled it */
} fc_bcast;

typedef struct fc_world fc_world; /* opaque; one per process (or one per virtual world) */

#define FC_IPC_HANDLE_BYTES 64

/* ---------------------------------------------------------------- heap ----
 * The symmetric heap: one device allocation per rank whose first
 * firecaffe_heap_reserved_bytes() bytes hold the library's synchronisation
 * flags.  Collective buffers are carved from the rest at identical offsets on
 * every rank (the caller does the carving).
 */

/* Bytes reserved at the start of a heap of `heap_bytes` (flag area; depends only
 * on heap_bytes).  User buffers must start at or after this offset. */
int64_t firecaffe_heap_reserved_bytes(int64_t heap_bytes);

/* cudaMalloc `bytes` on the current device and zero them.  *heap receives the
 * device pointer (256-byte aligned).  Free with firecaffe_heap_free. */
fc_status firecaffe_heap_alloc(int64_t bytes, void** heap);
fc_status firecaffe_heap_free(void* heap);

/* Export a heap for other processes of the node: writes FC_IPC_HANDLE_BYTES
 * opaque bytes (a cudaIpcMemHandle_t) to handle_out.  `heap` must be a pointer
 * returned by firecaffe_heap_alloc. */
fc_status firecaffe_heap_export(void* heap, uint8_t* handle_out);

/* --------------------------------------------------------------- world ----
 * firecaffe_world_create: the real world, one process per GPU.
 *   rank, world_size : this process's rank in [0, world_size), world_size in 1..8
 *   cuda_device      : the device this rank uses (must be current on the calling thread)
 *   local_heap       : this rank's heap from firecaffe_heap_alloc (heap_bytes bytes);
 *                      EVERY rank must pass the same heap_bytes: buffers and flags are
 *                      addressed in a peer's heap at this rank's offsets (the size is
 *                      part of every collective's call signature, so ranks whose sizes
 *                      differ fail with FC_ERR_MISMATCH at the entry barrier, whose
 *                      stamps sit at offsets that do not depend on the size)
 *   handles          : world_size * FC_IPC_HANDLE_BYTES bytes, rank-ordered exports of every
 *                      rank's heap (entry `rank` is ignored); exchanged by the caller
 *                      (e.g. torch.distributed all_gather_object)
 *   timeout_ns       : bound on every device-side wait (0 -> 30 s)
 * Opens every peer heap with CUDA IPC (peer access over NVLink).  Collective:
 * every rank must call it.  The flag area of local_heap must still be zero
 * (fresh firecaffe_heap_alloc) — flags are never reset afterwards.
 *
 * firecaffe_world_create_virtual: p ranks emulated on ONE GPU, for testing the
 * multi-rank schedules on a single device.  `heap` holds world_size consecutive
 * rank heaps of heap_bytes_per_rank bytes each (allocate with firecaffe_heap_alloc
 * (world_size * heap_bytes_per_rank)).  Collective calls on a virtual world take
 * rank 0's buffer pointers; rank r's are at + r * heap_bytes_per_rank, for grad, w
 * AND mom.  One cooperative kernel runs all ranks (rank = blockIdx.y).
 */
fc_status firecaffe_world_create(int rank, int world_size, int cuda_device, void* local_heap,
                                 const uint8_t* handles, int64_t heap_bytes, uint64_t timeout_ns,
                                 fc_world** out);
fc_status firecaffe_world_create_virtual(int world_size, int cuda_device, void* heap,
                                         int64_t heap_bytes_per_rank, uint64_t timeout_ns,
                                         fc_world** out);
fc_status firecaffe_world_destroy(fc_world* world);

/* Select the executor.  arity k (2..world_size) is the tree's branching factor
 * ("the base of log(p) depends on the branching factor"); arity > 2 and
 * FC_SCHED_FOREST needs arity 2 and a power-of-two world size, FC_SCHED_SINGLE_ROOT
 * needs arity 2; other combinations give FC_ERR_UNSUPPORTED and leave the
 * configuration unchanged.  The default chosen at world creation (the fastest
 * measured executor) is reported by firecaffe_world_get_config. */
fc_status firecaffe_world_config(fc_world* world, int arity, fc_sched sched, fc_bcast bcast);
fc_status firecaffe_world_get_config(const fc_world* world, int* arity, fc_sched* sched,
                                     fc_bcast* bcast);

/* Cap the CTAs per rank of the collective kernels (0 = automatic: one wave
 * over all SMs; at most 1022).  A small cap (e.g. 16) lets a collective
 * overlap other work on the GPU (bucketed overlap with the backward pass)
 * without taking every SM; every rank must use the same cap (a rank that
 * launches a different grid makes the call fail with FC_ERR_MISMATCH).
 * Value-neutral. */
fc_status firecaffe_world_set_max_ctas(fc_world* world, int max_ctas);

/* Synchronise the device and return the sticky device status (FC_OK, or
 * FC_ERR_TIMEOUT if any wait of any earlier call timed out). */
fc_status firecaffe_world_poll(fc_world* world);

/* The element range [*begin, *end) of the n-element vector whose momentum this
 * rank updates in firecaffe_tree_allreduce_sgd (its subtree-root slice): the
 * whole vector for world_size 1, rank 0's [0,n) for FC_SCHED_SINGLE_ROOT, an
 * owner slice for FOREST/FLAT.  Host-only; no GPU needed. */
fc_status firecaffe_owned_range(const fc_world* world, int rank, int64_t n, int64_t* begin,
                                int64_t* end);
/* Same, from (world_size, schedule) alone (host-only helper for tests/tools). */
fc_status firecaffe_plan_owned_range(int world_size, fc_sched sched, int rank, int64_t n,
                                     int64_t* begin, int64_t* end);

/* ----------------------------------------------------------------- ops ----
 * firecaffe_sgd_step — one SGD step with momentum and weight decay on one GPU
 * (mu, wd P:358/P:363; Caffe convention, R6).  For i < n:
 *     g  = fl(grad[i] * fl(1/batch))      grad is the gradient SUM over `batch` images
 *     d  = fma(wd, w[i], g)
 *     v' = fma(mu, mom[i], fl(lr * d))
 *     w' = fl(w[i] - v')
 * w and mom are updated in place; grad is read-only.  lr is used as given (already
 * scaled for the batch, see firecaffe_scale_lr).  n == 0 is a no-op.
 * Errors: FC_ERR_INVALID_ARG for null/unaligned pointers with n > 0, n < 0,
 * lr <= 0, mu outside [0,1), wd < 0, batch < 1, overlapping buffers.
 */
fc_status firecaffe_sgd_step(float* w, const float* grad, float* mom, int64_t n, float lr,
                             float mu, float wd, int64_t batch, void* stream);

/* firecaffe_tree_allreduce — in place: on return (stream order) every rank's
 * grad[0..n) holds the reduction-tree sum of all ranks' grad.
 * Association (R1): k-nomial tree rooted at rank 0 in absolute rank
 * space; at step s = k^l node r (r mod k*s == 0) adds r + j*s, j = 1..k-1 ascending.
 * k=2: p=4 -> (g0+g1)+(g2+g3);  p=8 -> ((g0+g1)+(g2+g3))+((g4+g5)+(g6+g7)).
 * Every schedule produces these bits.  world_size 1: no-op. */
fc_status firecaffe_tree_allreduce(float* grad, int64_t n, fc_world* world, void* stream);

/* firecaffe_tree_allreduce_sgd — the fused hot path: tree-reduce grad, apply the
 * firecaffe_sgd_step update to the reduced gradient inside the final tree level
 * (the sum never round-trips HBM), and broadcast the updated weights.  On return
 * every rank's w[0..n) holds identical updated weights, bitwise equal to
 * firecaffe_tree_allreduce followed by firecaffe_sgd_step.  mom is updated only on
 * this rank's firecaffe_owned_range (the optimizer state is sharded across the
 * subtree roots, R18); grad's contents are unspecified afterwards.
 * world_size 1: identical to firecaffe_sgd_step.  Argument errors as sgd_step. */
fc_status firecaffe_tree_allreduce_sgd(float* w, float* grad, float* mom, int64_t n, float lr,
                                       float mu, float wd, int64_t batch, fc_world* world,
                                       void* stream);

/* firecaffe_ps_allreduce — the paper's synchronous parameter server (P:246-250,
 * P:267-269) as the measured comparison: rank 0 (also a worker, R3)
 * pulls every rank's grad, sums them sequentially in ascending rank order
 * ((g0+g1)+g2)+..., and sends the sum to every rank: in place, every rank's grad
 * holds it on return.  Equal bitwise to firecaffe_tree_allreduce with arity p. */
fc_status firecaffe_ps_allreduce(float* grad, int64_t n, fc_world* world, void* stream);

/* ------------------------------------------------ Caffe per-blob multipliers
 * The flat parameter vector is a concatenation of blobs (layers' weights and
 * biases).  Caffe gives each blob an lr_mult and a decay_mult (settings
 * "consistent with the Caffe configuration files"; typical: biases lr_mult 2,
 * decay_mult 0).  Blob s covers [segs[s].begin, segs[s+1].begin) (the last up to
 * n); per element the update uses local_lr = fl(lr*lr_mult), local_wd =
 * fl(wd*decay_mult) in the firecaffe_sgd_step rule (R20).  All
 * multipliers 1 gives exactly firecaffe_sgd_step's bits.
 * firecaffe_segments_create validates the HOST table (segs[0].begin == 0,
 * strictly increasing, every begin < n, finite multipliers >= 0) and copies it
 * to the current device once; the handle is then passed to the *_segments
 * calls, whose n must equal the table's n.  1 <= nseg <= 65536. */
typedef struct {
    int64_t begin;
    float lr_mult;
    float decay_mult;
} fc_segment;
typedef struct fc_segments fc_segments;
fc_status firecaffe_segments_create(const fc_segment* segs, int nseg, int64_t n, fc_segments** out);
fc_status firecaffe_segments_destroy(fc_segments* segs);
fc_status firecaffe_sgd_step_segments(float* w, const float* grad, float* mom, int64_t n, float lr,
                                      float mu, float wd, int64_t batch, const fc_segments* segs,
                                      void* stream);
fc_status firecaffe_tree_allreduce_sgd_segments(float* w, float* grad, float* mom, int64_t n,
                                                float lr, float mu, float wd, int64_t batch,
                                                const fc_segments* segs, fc_world* world,
                                                void* stream);

/* ------------------------------------------------ bf16 gradient wire format
 * SURVEY §8 f4 (16-bit gradients on the wire).  `grad` holds n
 * bfloat16 values (uint16 bit patterns; for the collective: symmetric in the
 * heap), w and mom fp32.  Each gradient is upcast EXACTLY to fp32 and the rest
 * is the fp32 path: the same tree association (R1), the same SGD
 * (R6, with segs' multipliers if segs != NULL), fp32 weights broadcast.  So the
 * result equals firecaffe_tree_allreduce_sgd applied to the upcast gradients,
 * bit for bit; the reduce phase moves 2 instead of 4 bytes per parameter.
 * The collective always uses the FLAT executor (the world's schedule is
 * ignored); world_size 1 = firecaffe_sgd_step_bf16.  grad is read-only.
 * Errors as firecaffe_tree_allreduce_sgd. */
fc_status firecaffe_sgd_step_bf16(float* w, const uint16_t* grad, float* mom, int64_t n, float lr,
                                  float mu, float wd, int64_t batch, const fc_segments* segs,
                                  void* stream);
fc_status firecaffe_tree_allreduce_sgd_bf16(float* w, uint16_t* grad, float* mom, int64_t n,
                                            float lr, float mu, float wd, int64_t batch,
                                            const fc_segments* segs, fc_world* world,
                                            void* stream);

/* ------------------------------------------------ host-buffer entry points
 * The same operations fed from / returned to HOST memory, for callers whose
 * gradients live on the host (and for the end-to-end benchmark).  grad_host
 * and w_host must be page-locked (cudaMallocHost / cudaHostRegister), n floats
 * each; w, grad, mom are the usual device buffers (grad receives the copy).
 * firecaffe_sgd_step_host: chunked pipeline over internal streams (H2D of
 *   chunk i+1 || SGD of chunk i || D2H of chunk i-1; PCIe is full duplex);
 *   results identical to firecaffe_sgd_step.  Ordered after prior work on
 *   `stream`; later work on `stream` sees every copy complete.  Not re-entrant
 *   across host threads on the same device.
 * firecaffe_tree_allreduce_sgd_host: H2D into the symmetric grad, the fused
 *   collective, D2H of the updated weights.  With the FLAT executor (push
 *   broadcast) and n >= S*p*4096 it runs as an S-stage pipeline on internal
 *   streams (S = FC_HOST_STAGES, default 4): stage k's H2D || stage k-1's
 *   collective || stage k-2's D2H, stage k covering window k of every owner's
 *   slice, so w, mom (owned slice) and grad end bitwise as after one full
 *   call.  Otherwise serial on `stream`.  Either way ordered after prior work
 *   on `stream`, and later work on `stream` sees the weights on the host.
 * segs may be NULL (uniform multipliers).  Errors as the device versions, plus
 * FC_ERR_INVALID_ARG for host buffers that are not page-locked. */
fc_status firecaffe_sgd_step_host(float* w, float* grad, float* mom, const float* grad_host,
                                  float* w_host, int64_t n, float lr, float mu, float wd,
                                  int64_t batch, const fc_segments* segs, void* stream);
fc_status firecaffe_tree_allreduce_sgd_host(float* w, float* grad, float* mom,
                                            const float* grad_host, float* w_host, int64_t n,
                                            float lr, float mu, float wd, int64_t batch,
                                            const fc_segments* segs, fc_world* world,
                                            void* stream);

/* ------------------------------------------------ learning-rate schedules
 * The paper's schedules (R21): FIXED; STEP gamma^floor(iter/stepsize);
 * MULTISTEP gamma^#{steps[k] <= iter} ("reduce this by a factor of 10x twice",
 * P:407); POLY (1 - it/max_iter)^power with it = min(iter, max_iter) (P:451-452,
 * power 0.5; past max_iter the schedule stays at its end value, lr = 0 for
 * power > 0).  The factor is std::pow in double, then lr = fl32(base_lr *
 * factor) — the oracle's definition, bit for bit.
 * firecaffe_lr_at returns -1 for invalid input: iter < 0; base_lr <= 0; gamma
 * <= 0 (STEP, MULTISTEP); power < 0 (POLY); any of them not finite; stepsize
 * < 1 (STEP); max_iter < 1 (POLY); nsteps outside 0..FC_LR_MAX_STEPS. */
typedef enum { FC_LR_FIXED = 0, FC_LR_STEP = 1, FC_LR_MULTISTEP = 2, FC_LR_POLY = 3 } fc_lr_policy;
#define FC_LR_MAX_STEPS 16
typedef struct {
    int policy;       /* fc_lr_policy */
    float base_lr;
    float gamma;
    int64_t stepsize;
    float power;
    int64_t max_iter;
    int nsteps;
    int64_t steps[FC_LR_MAX_STEPS];
} fc_lr_schedule;
float firecaffe_lr_at(const fc_lr_schedule* sched, int64_t iter);

/* On-device schedules ("computed on device from an iteration
 * counter, so the step needs no host sync").  An fc_lr_state holds, on the
 * device current at creation, the schedule's lr at every level it can reach
 * (computed once by firecaffe_lr_at's arithmetic on the host: the number of
 * decays for STEP / MULTISTEP, the clamped iteration for POLY; a STEP table
 * ends where gamma^k has become 0 or inf in fp32, after which the value
 * cannot change) plus an iteration counter.  firecaffe_sgd_step_sched /
 * firecaffe_tree_allreduce_sgd_sched are firecaffe_sgd_step /
 * firecaffe_tree_allreduce_sgd with lr = firecaffe_lr_at(sched, iter), read by
 * the kernel from that table at the counter, which the same kernel then
 * advances by one (stream-ordered): a captured CUDA graph replays the training
 * step with the schedule moving on, no host involvement, and device and host
 * give identical bits.  A call that enqueues nothing (n = 0) does not advance
 * the counter.  Collective rule: every rank creates its state from the same
 * schedule and first_iter and makes the same calls (the schedule, not the
 * iteration, is part of the call signature).
 *   firecaffe_lr_state_create   first_iter >= 0; FC_ERR_INVALID_ARG for an
 *                               invalid schedule (as firecaffe_lr_at);
 *                               FC_ERR_UNSUPPORTED if the table would exceed
 *                               2^24 levels (POLY max_iter >= 2^24, or a STEP
 *                               gamma so close to 1 that gamma^k needs more
 *                               levels to reach 0 in fp32)
 *   firecaffe_lr_state_get_iter synchronous: waits for the device, then reads
 *   firecaffe_lr_state_set_iter synchronous: waits for the device, then writes
 *                               (resume from a checkpoint)
 * The state must be used on its device (else FC_ERR_MISMATCH) and by one
 * stream at a time. */
typedef struct fc_lr_state fc_lr_state;
fc_status firecaffe_lr_state_create(const fc_lr_schedule* sched, int64_t first_iter, fc_lr_state** out);
fc_status firecaffe_lr_state_destroy(fc_lr_state* state);
fc_status firecaffe_lr_state_get_iter(const fc_lr_state* state, int64_t* iter);
fc_status firecaffe_lr_state_set_iter(fc_lr_state* state, int64_t iter);
fc_status firecaffe_sgd_step_sched(float* w, const float* grad, float* mom, int64_t n,
                                   fc_lr_state* lr, float mu, float wd, int64_t batch,
                                   const fc_segments* segs, void* stream);
fc_status firecaffe_tree_allreduce_sgd_sched(float* w, float* grad, float* mom, int64_t n,
                                             fc_lr_state* lr, float mu, float wd, int64_t batch,
                                             const fc_segments* segs, fc_world* world, void* stream);

/* firecaffe_allgather_owned — every rank's firecaffe_owned_range slice of the
 * symmetric buffer `buf` is copied to every other rank, in place: afterwards all
 * ranks hold the owners' values everywhere.  Use it on the momentum before a
 * checkpoint (firecaffe_tree_allreduce_sgd keeps it sharded, R18) or
 * before changing the executor (ownership differs for FC_SCHED_SINGLE_ROOT).
 * Collective; `buf` must be symmetric in the heap.  world_size 1: no-op. */
fc_status firecaffe_allgather_owned(float* buf, int64_t n, fc_world* world, void* stream);

/* Linear learning-rate scaling with the batch size:
 * returns fl(base_lr * batch / base_batch) computed in double, e.g. (0.01, 256, 1024) -> 0.04.
 * Returns 0 for base_batch < 1 or batch < 1. */
float firecaffe_scale_lr(float base_lr, int64_t base_batch, int64_t batch);

const char* firecaffe_status_str(fc_status s);

/* Diagnostics: when `buf` (device memory, `capacity` uint64 words) is set, every
 * collective kernel writes four %globaltimer stamps per CTA (entry, after the
 * entry barrier, after the data phase, exit) to buf[(vrank*grid + cta)*4 + slot]
 * (vrank = 0 in a real world).  Pass NULL to disable.  Value-neutral.
 * firecaffe_world_last_grid returns the CTAs per rank of the last collective. */
fc_status firecaffe_world_set_trace(fc_world* world, uint64_t* buf, int64_t capacity);
int firecaffe_world_last_grid(const fc_world* world);

/* Tuning knob for firecaffe_sgd_step: float4s in flight per thread per operand
 * (1, 2, 4 or 8); -1, -2, -4: the same with the next iteration's loads issued
 * before the current math (register double buffering); 0 (default): automatic
 * (-2 below 32 M params, -1 above, the measured best on B200).  Process-wide;
 * value-neutral. */
void firecaffe_tune_sgd_unroll(int unroll);

/* Library build identifier ("firecaffe-b200 <version> sm_100a"). */
const char* firecaffe_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FIRECAFFE_H */
