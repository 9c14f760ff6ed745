/* A plain C99 caller of the C-ABI (include/dfa2c.h): no C++, no torch —
 * what a cgo / JNI / N-API binding does underneath. One small layer
 * (cfg1 geometry) through dfa2c_mha_forward at t = 0 (all Full) and t = 1
 * (F A0 A2 C), the head cache, the RSE query and the error path (a Cached
 * head without a slot is DFA2C_CACHE_MISS before any work).
 * Build: gcc -std=c99 -O2 -Iinclude -I$CUDA/include capi_from_c.c
 *        -Lpaper_2503_22796_b200 -ldfa2_b200 -L$CUDA/lib64 -lcudart */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dfa2c.h"

#define CHECK(x)                                                                      \
    do {                                                                              \
        int rc_ = (x);                                                                \
        if (rc_ != DFA2C_OK) {                                                        \
            fprintf(stderr, "%s:%d %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_,     \
                    dfa2c_last_error());                                              \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

static uint16_t to_bf16(float f) { /* round to nearest even */
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
static float from_bf16(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main(void) {
    const int64_t H = 4, d = 64, nv = 1024, nt = 77, n = nv + nt, B = 128;
    const size_t elems = (size_t)(H * n * d), bytes = elems * 2;
    dfa2c_dims dims = {H, d, nv, nt, DFA2C_VISUAL_FIRST};
    uint16_t* host = (uint16_t*)malloc(bytes);
    void *q, *k, *v, *out0, *out1;
    if (cudaMalloc(&q, bytes) || cudaMalloc(&k, bytes) || cudaMalloc(&v, bytes) || cudaMalloc(&out0, bytes) ||
        cudaMalloc(&out1, bytes))
        return 2;
    void* bufs[3] = {q, k, v};
    uint32_t seed = 12345u;
    for (int b = 0; b < 3; ++b) {
        for (size_t i = 0; i < elems; ++i) {
            seed = seed * 1664525u + 1013904223u;
            host[i] = to_bf16(((float)(seed >> 8) / 16777216.0f - 0.5f) * 3.0f);
        }
        if (cudaMemcpy(bufs[b], host, bytes, cudaMemcpyHostToDevice))
            return 2;
    }
    dfa2c_cache* cache = NULL;
    CHECK(dfa2c_cache_create(1, H, 1, n, d, &cache));

    int32_t kinds1[4] = {DFA2C_FULL, DFA2C_ARROW, DFA2C_ARROW, DFA2C_CACHED};
    int64_t wins1[4] = {0, 0, 2, 0};
    /* a Cached head before any slot exists: rejected before any work */
    int rc = dfa2c_mha_forward(q, k, v, 1, &dims, B, kinds1, wins1, cache, 0, 0, out1, NULL);
    if (rc != DFA2C_CACHE_MISS) {
        fprintf(stderr, "expected DFA2C_CACHE_MISS, got %d\n", rc);
        return 1;
    }
    int32_t kinds0[4] = {DFA2C_FULL, DFA2C_FULL, DFA2C_FULL, DFA2C_FULL};
    int64_t wins0[4] = {0, 0, 0, 0};
    CHECK(dfa2c_mha_forward(q, k, v, 1, &dims, B, kinds0, wins0, cache, 0, 0, out0, NULL));
    CHECK(dfa2c_mha_forward(q, k, v, 1, &dims, B, kinds1, wins1, cache, 0, 1, out1, NULL));
    if (cudaDeviceSynchronize())
        return 2;

    int64_t produced = -1;
    CHECK(dfa2c_cache_produced_at(cache, 0, 3, &produced)); /* the Cached head kept t = 0 */
    if (produced != 0) {
        fprintf(stderr, "cached head produced_at %lld\n", (long long)produced);
        return 1;
    }
    CHECK(dfa2c_cache_produced_at(cache, 0, 0, &produced));
    if (produced != 1)
        return 1;
    /* the Cached head's output is the t = 0 Full output, bitwise; the
     * others are finite attention outputs */
    uint16_t* o0 = (uint16_t*)malloc(bytes);
    uint16_t* o1 = (uint16_t*)malloc(bytes);
    if (cudaMemcpy(o0, out0, bytes, cudaMemcpyDeviceToHost) || cudaMemcpy(o1, out1, bytes, cudaMemcpyDeviceToHost))
        return 2;
    const size_t hs = (size_t)(n * d);
    if (memcmp(o0 + 3 * hs, o1 + 3 * hs, hs * 2) != 0) {
        fprintf(stderr, "cached head differs from its slot\n");
        return 1;
    }
    if (memcmp(o0, o1, hs * 2) != 0) { /* head 0 is Full at both t: same bits */
        fprintf(stderr, "Full head not deterministic\n");
        return 1;
    }
    for (size_t i = 0; i < elems; ++i)
        if (!isfinite(from_bf16(o1[i]))) {
            fprintf(stderr, "non-finite output at %zu\n", i);
            return 1;
        }
    /* RSE of the Arrow(0) head against the Full output of the same head */
    double rse[1];
    CHECK(dfa2c_rse((const char*)out1 + 1 * hs * 2, (const char*)out0 + 1 * hs * 2, DFA2C_BF16, 1, (int64_t)hs,
                    DFA2C_RSE_STANDARD, rse, NULL));
    if (!(rse[0] > 0.0 && isfinite(rse[0]))) { /* a narrower window changes the output */
        fprintf(stderr, "rse %g\n", rse[0]);
        return 1;
    }
    int64_t flops = 0;
    CHECK(dfa2c_plan_flops(&dims, B, kinds1, wins1, &flops));
    CHECK(dfa2c_cache_destroy(cache));
    printf("capi from C ok: %s, plan flops %lld, rse(A0 vs F) %.6f\n", dfa2c_version(), (long long)flops, rse[0]);
    free(host);
    free(o0);
    free(o1);
    return 0;
}
