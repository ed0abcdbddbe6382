// Host-side dispatch of the collective kernels:
// which executor runs a call, how many CTAs it gets and how it is launched.
//
// Executors (include/firecaffe.h fc_sched) — all produce the same bits, the
// k-nomial association of DESIGN.md R1:
//   FLAT        each rank pulls its owner slice from all p ranks, evaluates
//               the whole tree in registers, applies SGD, pushes w' to all
//               (coll_flat.cu).
//   FOREST      recursive halving: at level l rank r pulls |W|/2^(l+1) from
//               r^2^l (the binomial tree of slice s is rooted at its owner);
//               SGD fused into the last level; tree or direct broadcast
//               (coll_tree.cu).
//   SINGLE_ROOT the paper's binomial tree rooted at rank 0 (Fig. P:312-315);
//               the root applies SGD to all of W, then broadcast (coll_tree.cu).
//   PS          (op FC_OP_PS) rank 0 pulls everything, sequential sum, pushes
//               (the FLAT kernel with K = p and rank 0 owning everything).
// One persistent kernel per call, one wave of CTAs: a cooperative launch for
// virtual worlds (their CTAs wait on each other), a plain one otherwise.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include "fc_launch.h"

namespace fc {

struct KernelPick {
    const void* fn;
    int block;
    bool flat;
};

// Tree schedules: the spill-free 1-CTA/SM build while the per-rank slice is
// below 4M floats (16 MB), the 2-CTA/SM build above (measured, p = 2 and 4:
// NiN forest/direct 65.5 vs 67.6 us, single_root/tree p=4 174 vs 190 us;
// AlexNet forest/direct 0.377 vs 0.389 ms; profiles/r01_sweep_tree_launch_bounds_*,
// scripts/gpu_tree_lb.sh).
constexpr int64_t kTreeDenseSliceFloats = (int64_t)4 << 20;

static int tree_ctas_per_sm(int p, int64_t n) {
    static int force = -1;
    if (force < 0) {
        const char* e = getenv("FC_TREE_CTAS_PER_SM");
        force = e ? atoi(e) : 0;
    }
    if (force == 1 || force == 2) return force;
    return p > 0 && n / p >= kTreeDenseSliceFloats ? 2 : 1;
}

static KernelPick pick_kernel(int sched, int arity, int p, int op, int64_t n) {
    if (op == FC_OP_PS) arity = p;
    const bool bf16 = op == FC_OP_ALLREDUCE_SGD_BF16;  // always the FLAT executor
    const bool gather = op == FC_OP_ALLGATHER_OWNED;
    const bool flat = op == FC_OP_PS || sched == FC_SCHED_FLAT || bf16 || gather;
    KernelPick k{nullptr, flat ? kFlatThreads : kTreeThreads, flat};
    if (gather) k.fn = allgather_kernel_for(p);
    else if (bf16) k.fn = flat_bf16_kernel_for(p, arity);
    else if (flat) k.fn = flat_kernel_for(p, arity);
    else if (sched == FC_SCHED_SINGLE_ROOT) k.fn = single_root_kernel_for(p, tree_ctas_per_sm(p, n));
    else k.fn = forest_kernel_for(p, tree_ctas_per_sm(p, n));
    return k;
}

// CTAs per rank.  FLAT: one wide CTA per SM — every CTA pays a sys-scope
// release fence at the exit barrier and that fence gets slower with the number
// of CTAs issuing it (4.4 us at 148 CTAs, 7.8 us at 444; scripts/fence_bench.cu,
// launch_bench.cu).  Tree schedules: as many 256-thread CTAs as fit (their
// chunk pipeline wants more independent CTAs).  Virtual worlds share one GPU.
int collective_grid(int sched, int arity, int p, bool virt, int op, int64_t n) {
    const KernelPick k = pick_kernel(sched, arity, p, op, n);
    if (!k.fn || p < 1) return 0;
    int occ = occupancy(k.fn, k.block);
    if (occ < 1) return 0;
    static int flat_per_sm = -1;
    if (flat_per_sm < 0) {
        const char* e = getenv("FC_FLAT_CTAS_PER_SM");
        flat_per_sm = e ? atoi(e) : 0;  // 0 = by size
    }
    int64_t cap;
    if (virt) {
        cap = (int64_t)dev_info().sms * occ / p;
    } else {
        if (k.flat) {
            // measured (p = 2, 4): 1 CTA/SM wins while the per-rank slice is small (the
            // fixed exit cost dominates), 2 CTAs/SM from ~32 MB slices on (more bytes in
            // flight): NiN p=2 63.5 vs 66.6 us, VGG-19 p=2 932 vs 879 us
            const int want = flat_per_sm > 0 ? flat_per_sm : (n / p >= (int64_t)(8 << 20) ? 2 : 1);
            if (occ > want) occ = want;
        }
        cap = (int64_t)dev_info().sms * occ;
    }
    if (cap > FC_EXIT_CTA_SLOT) cap = FC_EXIT_CTA_SLOT;  // CTA indices < the reserved exit word
    return (int)cap;
}

cudaError_t launch_collective(const FcColl& c, int sched, int arity, bool virt, int grid_x,
                              cudaStream_t st) {
    const KernelPick k = pick_kernel(sched, arity, c.p, c.op, c.n);
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
