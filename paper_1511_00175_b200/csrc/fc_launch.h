// Host-side launch interface between the C ABI (api.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fc_internal.h"

namespace fc {

struct DevInfo {
    int device;
    int sms;
};
const DevInfo& dev_info();  // current device's SM count (cached per device)
int occupancy(const void* fn, int block);  // resident CTAs/SM, cached per (kernel, block, device)

// lrs non-null (firecaffe_sgd_step_sched): lr comes from the device-resident
// schedule at its current iteration, which the kernel advances by one.
cudaError_t launch_sgd_step(float* w, const float* grad, float* mom, int64_t n, float lr, float mu,
                            float wd, float inv_b, const FcSegs& segs, cudaStream_t st,
                            FcLrDev* lrs = nullptr);
cudaError_t launch_sgd_step_range(float* w, const float* grad, float* mom, int64_t off, int64_t len,
                                  float lr, float mu, float wd, float inv_b, const FcSegs& segs,
                                  cudaStream_t st, FcLrDev* lrs = nullptr);
void set_sgd_unroll(int u);
cudaError_t launch_sgd_step_bf16(float* w, const uint16_t* grad, float* mom, int64_t n, float lr,
                                 float mu, float wd, float inv_b, const FcSegs& segs,
                                 cudaStream_t st);

// Host-buffer paths (host_pipeline.cu): zero-copy kernel and copy-engine pipeline
cudaError_t launch_sgd_step_hybrid(float* w, const float* grad_host, float* grad_dev, float* mom,
                                   float* w_host_dev, int64_t n, float lr, float mu, float wd,
                                   float inv_b, const FcSegs& segs, int64_t chunk,
                                   cudaStream_t user);
cudaError_t launch_sgd_step_hostio(float* w, const float* grad_host_dev, float* grad_dev, float* mom,
                                   float* w_host_dev, int64_t n, float lr, float mu, float wd,
                                   float inv_b, const FcSegs& segs, cudaStream_t st);
constexpr int kPipeDepth = 4;
cudaError_t launch_sgd_step_host(float* w, const float* grad_host, float* grad_dev, float* mom,
                                 float* w_host, int64_t n, float lr, float mu, float wd,
                                 float inv_b, const FcSegs& segs, int64_t chunk,
                                 cudaStream_t user);

// Collective launch: `virt` -> one cooperative grid of (grid_x, p) CTAs that emulates all ranks.
cudaError_t launch_collective(const FcColl& c, int sched, int arity, bool virt, int grid_x,
                              cudaStream_t st);
// Max CTAs per rank that can be co-resident for this schedule (virt: divided by p).
int collective_grid(int sched, int arity, int p, bool virt, int op, int64_t n);

// Kernel tables (nullptr if no instantiation exists for that p / arity).
constexpr int kTreeThreads = 256;  // threads per CTA, FOREST / SINGLE_ROOT
constexpr int kFlatThreads = 512;  // threads per CTA, FLAT / PS / bf16 / all-gather
const void* flat_kernel_for(int p, int arity);       // coll_flat.cu (also PS: arity = p)
const void* flat_bf16_kernel_for(int p, int arity);  // coll_flat.cu
const void* allgather_kernel_for(int p);             // coll_flat.cu
const void* forest_kernel_for(int p, int ctas_per_sm);       // coll_tree.cu (register budget
const void* single_root_kernel_for(int p, int ctas_per_sm);  //   for 1 or 2 CTAs per SM)

// Window k of s of the index range [a, b): [a + L*k/s, a + L*(k+1)/s), L = b - a
// (host + device: the pipelined host entry point and the FLAT kernel agree on it).
__host__ __device__ inline void window_range(int64_t a, int64_t b, int k, int s, int64_t* wa,
                                             int64_t* wb) {
    const int64_t L = b - a;
    *wa = a + L * k / s;
    *wb = a + L * (k + 1) / s;
}

// Owned chunk range [c0, c1) (in FC_CHUNK_FLOATS units) of `rank` (host + device).
__host__ __device__ inline bool is_pow2(int p) { return p > 0 && (p & (p - 1)) == 0; }
__host__ __device__ inline void owned_chunks(int rank, int p, int64_t n_chunks, bool single_root,
                                             int64_t* c0, int64_t* c1) {
    if (single_root) {
        *c0 = 0;
        *c1 = rank == 0 ? n_chunks : 0;
        return;
    }
    if (is_pow2(p)) {  // recursive halving: level l keeps the half selected by bit l of rank
        int64_t lo = 0, hi = n_chunks;
        for (int l = 0; (1 << l) < p; ++l) {
            const int64_t mid = lo + (hi - lo + 1) / 2;
            if ((rank >> l) & 1) lo = mid; else hi = mid;
        }
        *c0 = lo;
        *c1 = hi;
    } else {
        *c0 = (int64_t)rank * n_chunks / p;
        *c1 = (int64_t)(rank + 1) * n_chunks / p;
    }
}

}  // namespace fc
