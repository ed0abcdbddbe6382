// Tiny helper for scripts/gap_coll.py: kernels that write %globaltimer, so the
// launch and completion gaps around a collective can be read on the same clock
// as the collective's own in-kernel trace.
//   nvcc -O3 -shared -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -o scripts/libstamp.so scripts/stamp.cu
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void stamp_kernel(uint64_t* dst) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *dst = t;
}

__global__ void empty_kernel(uint64_t* dst) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (threadIdx.x == 0) {
        atomicMin((unsigned long long*)dst, (unsigned long long)t);
        atomicMax((unsigned long long*)dst + 1, (unsigned long long)t);
    }
}

extern "C" int stamp(uint64_t* dst, void* stream) {
    stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(dst);
    return (int)cudaGetLastError();
}

extern "C" int empty(uint64_t* dst, int grid, int block, void* stream) {
    empty_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(dst);
    return (int)cudaGetLastError();
}
