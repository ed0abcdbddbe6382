/* Driving libfirecaffe from plain C (no Python): the 1-GPU fused SGD and the
 * fused tree allreduce + SGD over a 4-rank virtual world on one GPU.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_demo.c \
 *       -L paper_1511_00175_b200 -lfirecaffe -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1511_00175_b200 -o /tmp/c_abi_demo
 *   /tmp/c_abi_demo out.bin
 *
 * Writes (as raw float32): the inputs it generated and the results, so a test
 * can compare them with the CPU oracle:  [grad(p*n) | w0(n) | v0(n) |
 * w_sgd(n) | v_sgd(n) | w_tree(n)]  with p = 4, n = 10007.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "firecaffe.h"

#define CK(x)                                                                  \
    do {                                                                       \
        fc_status s_ = (x);                                                    \
        if (s_ != FC_OK) {                                                     \
            fprintf(stderr, "%s -> %s\n", #x, firecaffe_status_str(s_));       \
            return 1;                                                          \
        }                                                                      \
    } while (0)

static uint64_t rng = 151100175ull;
static float frand(void) { /* xorshift64*, uniform in [-1, 1) */
    rng ^= rng >> 12;
    rng ^= rng << 25;
    rng ^= rng >> 27;
    return (float)((double)((rng * 2685821657736338717ull) >> 11) / 9007199254740992.0 * 2.0 - 1.0);
}

int main(int argc, char** argv) {
    const int p = 4;
    const int64_t n = 10007;
    const float lr = 0.04f, mu = 0.9f, wd = 5e-4f;
    const int64_t batch = 1024;
    float* g = (float*)malloc(sizeof(float) * p * n);
    float* w0 = (float*)malloc(sizeof(float) * n);
    float* v0 = (float*)malloc(sizeof(float) * n);
    float* out = (float*)malloc(sizeof(float) * n * 3);
    for (int64_t i = 0; i < p * n; ++i) g[i] = frand();
    for (int64_t i = 0; i < n; ++i) {
        w0[i] = 0.01f * frand();
        v0[i] = 1e-4f * frand();
    }
    printf("%s\n", firecaffe_version());

    /* 1-GPU fused SGD on rank 0's gradient */
    float *dw, *dg, *dv;
    cudaMalloc((void**)&dw, n * 4);
    cudaMalloc((void**)&dg, n * 4);
    cudaMalloc((void**)&dv, n * 4);
    cudaMemcpy(dw, w0, n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dg, g, n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v0, n * 4, cudaMemcpyHostToDevice);
    CK(firecaffe_sgd_step(dw, dg, dv, n, lr, mu, wd, batch, NULL));
    cudaMemcpy(out, dw, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(out + n, dv, n * 4, cudaMemcpyDeviceToHost);

    /* fused tree allreduce + SGD over a 4-rank virtual world */
    const int64_t per_rank = 1 << 22;
    void* heap = NULL;
    CK(firecaffe_heap_alloc(p * per_rank, &heap));
    fc_world* world = NULL;
    CK(firecaffe_world_create_virtual(p, 0, heap, per_rank, 0, &world));
    const int64_t off = firecaffe_heap_reserved_bytes(per_rank);
    const int64_t off_g = off, off_w = off + 65536, off_v = off + 2 * 65536;
    for (int r = 0; r < p; ++r) {
        char* base = (char*)heap + r * per_rank;
        cudaMemcpy(base + off_g, g + r * n, n * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(base + off_w, w0, n * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(base + off_v, v0, n * 4, cudaMemcpyHostToDevice);
    }
    CK(firecaffe_tree_allreduce_sgd((float*)((char*)heap + off_w), (float*)((char*)heap + off_g),
                                    (float*)((char*)heap + off_v), n, lr, mu, wd, batch, world, NULL));
    CK(firecaffe_world_poll(world));
    for (int r = 1; r < p; ++r) { /* every virtual rank holds the same weights */
        float* wr = (float*)malloc(n * 4);
        cudaMemcpy(out + 2 * n, (char*)heap + off_w, n * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(wr, (char*)heap + r * per_rank + off_w, n * 4, cudaMemcpyDeviceToHost);
        for (int64_t i = 0; i < n; ++i)
            if (((uint32_t*)wr)[i] != ((uint32_t*)(out + 2 * n))[i]) {
                fprintf(stderr, "rank %d differs at %lld\n", r, (long long)i);
                return 1;
            }
        free(wr);
    }
    CK(firecaffe_world_destroy(world));
    CK(firecaffe_heap_free(heap));

    if (argc > 1) {
        FILE* f = fopen(argv[1], "wb");
        fwrite(g, 4, p * n, f);
        fwrite(w0, 4, n, f);
        fwrite(v0, 4, n, f);
        fwrite(out, 4, 3 * n, f);
        fclose(f);
    }
    printf("c_abi_demo ok\n");
    return 0;
}
