// NVLink peer-access throughput on B200: every GPU simultaneously reads from,
// writes to, or both, all other GPUs' memory with 128-bit accesses.  Reports
// bytes crossing each GPU's link per direction / time.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/nvlink_bench scripts/nvlink_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct Ptrs { float4* p[8]; };

// mode 0: read peers (sum kept in a register, one store at the end)
// mode 1: write peers
// mode 2: read peers + write peers (half the elements each, like the fused tree)
template <int U>
__global__ void kern(Ptrs peers, int me, int np, float4* local, int64_t n4, int mode, float4* sink) {
    const int64_t T = blockDim.x;
    const int64_t stride = (int64_t)gridDim.x * T * U;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int64_t base = (int64_t)blockIdx.x * T * U + threadIdx.x; base < n4; base += stride) {
        for (int q = 1; q < np; ++q) {
            const int peer = (me + q) % np;
            float4* src = peers.p[peer];
            if (mode == 0 || mode == 2) {
                float4 x[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int64_t i = base + j * T;
                    if (i < n4) asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x[j].x), "=f"(x[j].y), "=f"(x[j].z), "=f"(x[j].w) : "l"(src + i));
                }
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int64_t i = base + j * T;
                    if (i < n4) { acc.x += x[j].x; acc.y += x[j].y; acc.z += x[j].z; acc.w += x[j].w; }
                }
            }
            if (mode == 1 || mode == 2) {
                float4* dst = peers.p[peer] + n4;  // second half of the peer buffer
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int64_t i = base + j * T;
                    if (i < n4) dst[i] = make_float4(1.f, 2.f, 3.f, (float)me);
                }
            }
        }
    }
    if (acc.x == 12345.f) sink[threadIdx.x] = acc;
}

// TMA (cp.async.bulk) variants.  mode 3: bulk stores smem -> peer global;
// mode 4: bulk loads peer global -> smem (STAGES-deep mbarrier ring).
// CH bytes per bulk op.
template <int CH, int STAGES>
__global__ void kern_tma(Ptrs peers, int me, int np, int64_t bytes, int mode, int ndir) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[STAGES];
    const int64_t nch = bytes / CH;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(smem);
    int issued = 0;
    uint32_t phase[STAGES] = {0};
    for (int q = 1; q < np; ++q) {
        const int peer = (me + q) % np;
        char* base = (char*)peers.p[peer] + (mode == 3 ? bytes : 0);
        for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
            char* g = base + c * CH;
            if (mode == 3) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sbase), "r"(CH) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES) : "memory");
            } else {
                const int s = issued % STAGES;
                const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
                if (issued >= STAGES) {  // wait for the previous use of this stage
                    uint32_t done = 0;
                    while (!done)
                        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                     : "=r"(done) : "r"(b), "r"(phase[s]) : "memory");
                    phase[s] ^= 1;
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(CH) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sbase + s * CH), "l"(g), "r"(CH), "r"(b) : "memory");
                ++issued;
            }
        }
    }
    if (mode == 3) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    else
        for (int s = 0; s < STAGES && s < issued; ++s) {
            const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
            uint32_t done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(b), "r"(phase[s]) : "memory");
        }
}

int main(int argc, char** argv) {
    int ng = 0;
    CK(cudaGetDeviceCount(&ng));
    const int64_t bytes = (argc > 1 ? atoll(argv[1]) : 256) << 20;  // per peer per direction
    const int64_t n4 = bytes / 16;
    for (int np = 2; np <= ng; np *= 2) {
        std::vector<float4*> buf(np), sink(np);
        std::vector<cudaStream_t> st(np);
        std::vector<cudaEvent_t> e0(np), e1(np);
        for (int d = 0; d < np; ++d) {
            CK(cudaSetDevice(d));
            for (int q = 0; q < np; ++q) if (q != d) { cudaError_t e = cudaDeviceEnablePeerAccess(q, 0); if (e != cudaSuccess) cudaGetLastError(); }
            CK(cudaMalloc(&buf[d], 2 * bytes));
            CK(cudaMemset(buf[d], 0, 2 * bytes));
            CK(cudaMalloc(&sink[d], 1 << 16));
            CK(cudaStreamCreate(&st[d]));
            CK(cudaEventCreate(&e0[d]));
            CK(cudaEventCreate(&e1[d]));
        }
        Ptrs P{};
        for (int d = 0; d < np; ++d) P.p[d] = buf[d];
        const char* mn[] = {"read", "write", "read+write"};
        for (int mode = 0; mode < 3; ++mode)
            for (int ctas_per_sm : {1, 2, 4})
                for (int U : {1, 2, 4}) {
                    float best = 1e9;
                    for (int rep = 0; rep < 4; ++rep) {
                        for (int d = 0; d < np; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
                        for (int d = 0; d < np; ++d) {
                            CK(cudaSetDevice(d));
                            CK(cudaEventRecord(e0[d], st[d]));
                            dim3 g(148 * ctas_per_sm), b(512 / ctas_per_sm > 128 ? 512 : 256);
                            if (U == 1) kern<1><<<g, b, 0, st[d]>>>(P, d, np, buf[d], n4, mode, sink[d]);
                            if (U == 2) kern<2><<<g, b, 0, st[d]>>>(P, d, np, buf[d], n4, mode, sink[d]);
                            if (U == 4) kern<4><<<g, b, 0, st[d]>>>(P, d, np, buf[d], n4, mode, sink[d]);
                            CK(cudaEventRecord(e1[d], st[d]));
                        }
                        float worst = 0;
                        for (int d = 0; d < np; ++d) {
                            CK(cudaSetDevice(d));
                            CK(cudaEventSynchronize(e1[d]));
                            float ms;
                            CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
                            if (ms > worst) worst = ms;
                        }
                        if (rep > 0 && worst < best) best = worst;
                    }
                    // bytes per direction per GPU: read: (np-1)*bytes in; write: (np-1)*bytes out;
                    // read+write: (np-1)*bytes each way from each op type -> 2x per direction
                    double per_dir = (double)(np - 1) * bytes * (mode == 2 ? 2 : 1);
                    printf("np=%d %-10s ctas/SM=%d U=%d  %.1f GB/s per direction per GPU  (%.3f ms)\n", np, mn[mode],
                           ctas_per_sm, U, per_dir / (best * 1e-3) / 1e9, best);
                }
        // TMA bulk variants
        const int CH = 16384, ST = 4;
        for (int d = 0; d < np; ++d) {
            CK(cudaSetDevice(d));
            CK(cudaFuncSetAttribute(kern_tma<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST));
        }
        for (int mode = 3; mode <= 4; ++mode)
            for (int ctas_per_sm : {1, 2, 3}) for (int uni = 0; uni < (np == 2 ? 2 : 1); ++uni) {
                float best = 1e9;
                for (int rep = 0; rep < 4; ++rep) {
                    for (int d = 0; d < np; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
                    for (int d = 0; d < (uni ? 1 : np); ++d) {
                        CK(cudaSetDevice(d));
                        CK(cudaEventRecord(e0[d], st[d]));
                        kern_tma<CH, ST><<<148 * ctas_per_sm, 32, CH * ST, st[d]>>>(P, d, np, bytes, mode, 1);
                        CK(cudaGetLastError());
                        CK(cudaEventRecord(e1[d], st[d]));
                    }
                    float worst = 0;
                    for (int d = 0; d < (uni ? 1 : np); ++d) {
                        CK(cudaSetDevice(d));
                        CK(cudaEventSynchronize(e1[d]));
                        float ms;
                        CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
                        if (ms > worst) worst = ms;
                    }
                    if (rep > 0 && worst < best) best = worst;
                }
                double per_dir = (double)(np - 1) * bytes;
                printf("np=%d %s %-10s ctas/SM=%d CH=%d  %.1f GB/s per direction per GPU  (%.3f ms)\n", np, uni ? "UNI" : "BI ",
                       mode == 3 ? "tma-write" : "tma-read", ctas_per_sm, CH, per_dir / (best * 1e-3) / 1e9, best);
            }
        for (int d = 0; d < np; ++d) {
            CK(cudaSetDevice(d));
            for (int q = 0; q < np; ++q) if (q != d) cudaDeviceDisablePeerAccess(q);
            cudaFree(buf[d]);
            cudaFree(sink[d]);
        }
    }
    return 0;
}
