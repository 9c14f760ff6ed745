/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's fused
 * head-wise attention path (the checker; see oracle.h for the contract and
 * how it is pinned against the reference itself). Never part of the product.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>


#include <pthread.h>
#include <unistd.h>

/* Minimal static-chunk parallel-for over [0, n) (no OpenMP in this image);
 * results never depend on the split because every index writes disjoint
 * outputs. Threads: ORACLE_THREADS, else all online cores. */
typedef void (*orc_body)(int64_t i, void* ctx);
typedef struct { int64_t lo, hi; orc_body fn; void* ctx; } orc_chunk;
static void* orc_run_chunk(void* p) {
    orc_chunk* c = (orc_chunk*)p;
    for (int64_t i = c->lo; i < c->hi; ++i) c->fn(i, c->ctx);
    return NULL;
}
static void orc_parallel_for(int64_t n, orc_body fn, void* ctx) {
    const char* env = getenv("ORACLE_THREADS");
    long t = env ? atol(env) : sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > n) t = n;
    if (t <= 1) { for (int64_t i = 0; i < n; ++i) fn(i, ctx); return; }
    pthread_t th[256];
    orc_chunk ch[256];
    if (t > 256) t = 256;
    for (long w = 0; w < t; ++w) {
        /* interleaved assignment balances ragged per-index cost */
        ch[w].lo = n * w / t; ch[w].hi = n * (w + 1) / t; ch[w].fn = fn; ch[w].ctx = ctx;
        pthread_create(&th[w], NULL, orc_run_chunk, &ch[w]);
    }
    for (long w = 0; w < t; ++w) pthread_join(th[w], NULL);
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* /root/reference/proj/src/arrow.cpp:113-153 */
int64_t orc_arrow_mask(int64_t nv, int64_t nt, int order, int64_t B, int64_t w,
                       uint8_t* active) {
    if (nv < 1 || nt < 0 || B < 1 || w < 0)
        return -1;
    const int64_t n = nv + nt;
    const int64_t nb = ceil_div(n, B);
    /* text span: inc/tensor.hpp:65-70 */
    const int64_t text_lo = order ? 0 : nv;
    const int64_t text_hi = order ? nt : n;
    const int64_t nvb = ceil_div(nv, B);
    int64_t weff = nvb - 1 > 0 ? nvb - 1 : 0; /* arrow.cpp:135-137 */
    if (w < weff)
        weff = w;
    if (!active)
        return nb;
    uint8_t* is_text = (uint8_t*)malloc((size_t)nb);
    for (int64_t i = 0; i < nb; ++i) {
        const int64_t lo = i * B;
        const int64_t hi = lo + B < n ? lo + B : n;
        is_text[i] = (lo < text_hi && hi > text_lo) ? 1 : 0; /* arrow.cpp:131 */
    }
    for (int64_t i = 0; i < nb; ++i)
        for (int64_t j = 0; j < nb; ++j) {
            const int64_t dij = i > j ? i - j : j - i;
            active[i * nb + j] = (is_text[i] || is_text[j] || dij <= weff) ? 1 : 0;
        }
    free(is_text);
    return nb;
}

/* /root/reference/proj/src/arrow.cpp:90-104 */
int64_t orc_active_positions(const uint8_t* active, int64_t n, int64_t B) {
    const int64_t nb = ceil_div(n, B);
    int64_t total = 0;
    for (int64_t i = 0; i < nb; ++i) {
        const int64_t li = (i + 1) * B <= n ? B : n - i * B;
        for (int64_t j = 0; j < nb; ++j)
            if (active[i * nb + j]) {
                const int64_t lj = (j + 1) * B <= n ? B : n - j * B;
                total += li * lj;
            }
    }
    return total;
}

/* /root/reference/proj/src/dispatch.cpp:93-120 */
int64_t orc_plan_flops(int64_t H, int64_t d, int64_t nv, int64_t nt, int order,
                       int64_t B, const int32_t* kinds, const int64_t* windows) {
    const int64_t n = nv + nt;
    const int64_t nb = ceil_div(n, B);
    uint8_t* m = (uint8_t*)malloc((size_t)(nb * nb));
    int64_t total = 0;
    for (int64_t h = 0; h < H; ++h) {
        if (kinds[h] == 0) {
            total += 4 * d * n * n;
        } else if (kinds[h] == 1) {
            orc_arrow_mask(nv, nt, order, B, windows[h], m);
            total += 4 * d * orc_active_positions(m, n, B);
        }
    }
    free(m);
    return total;
}

static float dot_f32(const float* a, const float* b, int64_t d) {
    float acc = 0.0f;
    for (int64_t i = 0; i < d; ++i)
        acc += a[i] * b[i];
    return acc;
}

/* streaming_block_pass, /root/reference/proj/src/arrow.cpp:24-72, per query
 * block over active key blocks in ascending order (arrow.cpp:184-186). */
typedef struct {
    const float *q, *k, *v;
    float* out;
    int64_t n, d, B, nb;
    const uint8_t* active;
} sparse_ctx;

static void sparse_block(int64_t qb, void* p) {
    const sparse_ctx* c = (const sparse_ctx*)p;
    const int64_t n = c->n, d = c->d, B = c->B, nb = c->nb;
    const float scale = 1.0f / sqrtf((float)d); /* arrow.cpp:29 */
    const int64_t r0 = qb * B;
    const int64_t rows = B < n - r0 ? B : n - r0;
    float* acc = (float*)calloc((size_t)(rows * d), sizeof(float));
    float* mx = (float*)malloc(sizeof(float) * (size_t)rows);
    float* sm = (float*)calloc((size_t)rows, sizeof(float));
    float* sc = (float*)malloc(sizeof(float) * (size_t)B);
    for (int64_t r = 0; r < rows; ++r)
        mx[r] = -INFINITY;
    for (int64_t kb = 0; kb < nb; ++kb) {
        if (!c->active[qb * nb + kb])
            continue;
        const int64_t c0 = kb * B;
        const int64_t cols = B < n - c0 ? B : n - c0;
        for (int64_t r = 0; r < rows; ++r) {
            const float* qr = c->q + (r0 + r) * d;
            float bmax = -INFINITY;
            for (int64_t x = 0; x < cols; ++x) {
                const float s = dot_f32(qr, c->k + (c0 + x) * d, d) * scale;
                sc[x] = s;
                if (s > bmax)
                    bmax = s;
            }
            const float m_new = mx[r] > bmax ? mx[r] : bmax;
            if (mx[r] != -INFINITY && m_new != mx[r]) { /* arrow.cpp:53-57 */
                const float alpha = expf(mx[r] - m_new);
                sm[r] *= alpha;
                for (int64_t x = 0; x < d; ++x)
                    acc[r * d + x] *= alpha;
            }
            for (int64_t x = 0; x < cols; ++x) { /* arrow.cpp:58-62 */
                const float pr = expf(sc[x] - m_new);
                sm[r] += pr;
                const float* vc = c->v + (c0 + x) * d;
                for (int64_t y = 0; y < d; ++y)
                    acc[r * d + y] += pr * vc[y];
            }
            mx[r] = m_new;
        }
    }
    for (int64_t r = 0; r < rows; ++r) { /* arrow.cpp:67-71 */
        const float inv = 1.0f / sm[r];
        for (int64_t x = 0; x < d; ++x)
            c->out[(r0 + r) * d + x] = acc[r * d + x] * inv;
    }
    free(acc);
    free(mx);
    free(sm);
    free(sc);
}

int orc_sparse_forward_f32(const float* q, const float* k, const float* v, float* out,
                           int64_t n, int64_t d, const uint8_t* active, int64_t B) {
    const int64_t nb = ceil_div(n, B);
    for (int64_t i = 0; i < nb; ++i) { /* arrow.cpp:176-179 */
        int any = 0;
        for (int64_t j = 0; j < nb; ++j)
            any |= active[i * nb + j];
        if (!any)
            return 3;
    }
    sparse_ctx c = {q, k, v, out, n, d, B, nb, active};
    orc_parallel_for(nb, sparse_block, &c);
    return 0;
}

/* attention_head_impl<double>, /root/reference/proj/src/tensor.cpp:73-114 */
typedef struct {
    const float *q, *k, *v;
    int64_t n, d, B, nb;
    const uint8_t* active;
    const int64_t* rows;
    double* out;
    volatile int rc;
} rows_ctx;

static void attention_row(int64_t ri, void* p) {
    rows_ctx* c = (rows_ctx*)p;
    const int64_t n = c->n, d = c->d;
    const int64_t i = c->rows ? c->rows[ri] : ri;
    const double scale = 1.0 / sqrt((double)d); /* tensor.cpp:76 */
    double* w = (double*)malloc(sizeof(double) * (size_t)n);
    const float* qr = c->q + i * d;
    const int64_t qb = c->active ? i / c->B : 0;
    double mx = -INFINITY;
    for (int64_t j = 0; j < n; ++j) {
        if (c->active && !c->active[qb * c->nb + j / c->B]) {
            w[j] = -INFINITY;
            continue;
        }
        double s = 0.0;
        for (int64_t x = 0; x < d; ++x)
            s += (double)qr[x] * (double)c->k[j * d + x];
        s *= scale;
        w[j] = s;
        if (s > mx)
            mx = s;
    }
    double* o = c->out + ri * d;
    if (mx == -INFINITY) { /* tensor.cpp:93-95 */
        c->rc = 3;
        free(w);
        return;
    }
    double denom = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        if (w[j] == -INFINITY) {
            w[j] = 0.0;
            continue;
        }
        w[j] = exp(w[j] - mx);
        denom += w[j];
    }
    const double inv = 1.0 / denom;
    for (int64_t x = 0; x < d; ++x)
        o[x] = 0.0;
    for (int64_t j = 0; j < n; ++j) /* tensor.cpp:110-112 */
        if (w[j] != 0.0) {
            const double a = w[j] * inv;
            for (int64_t x = 0; x < d; ++x)
                o[x] += a * (double)c->v[j * d + x];
        }
    free(w);
}

int orc_attention_rows_f64(const float* q, const float* k, const float* v, int64_t n,
                           int64_t d, const uint8_t* active, int64_t B,
                           const int64_t* rows, int64_t nrows, double* out) {
    rows_ctx c = {q, k, v, n, d, B, active ? ceil_div(n, B) : 1, active, rows, out, 0};
    orc_parallel_for(rows ? nrows : n, attention_row, &c);
    return c.rc;
}

/* mean_of / sum_sq_dev / sum_sq_diff / rse,
 * /root/reference/proj/src/calibrate.cpp:18-87 (sequential double sums). */
int orc_rse_f32(const float* y_m, const float* y_o, int64_t numel, int mode, double* out) {
    if (numel < 1)
        return 1;
    double mean = 0.0;
    for (int64_t i = 0; i < numel; ++i)
        mean += (double)y_o[i];
    mean /= (double)numel;
    double den = 0.0;
    for (int64_t i = 0; i < numel; ++i) {
        const double dd = (double)y_o[i] - mean;
        den += dd * dd;
    }
    if (den <= 0.0)
        return 5;
    double num = 0.0;
    for (int64_t i = 0; i < numel; ++i) {
        const double dd = mode ? (double)y_m[i] - mean : (double)y_m[i] - (double)y_o[i];
        num += dd * dd;
    }
    *out = num / den;
    return 0;
}

static float bf16_to_f32(uint16_t b) {
    const uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int orc_rse_bf16(const uint16_t* y_m, const uint16_t* y_o, int64_t numel, int mode,
                 double* out) {
    float* a = (float*)malloc(sizeof(float) * (size_t)numel);
    float* b = (float*)malloc(sizeof(float) * (size_t)numel);
    for (int64_t i = 0; i < numel; ++i) {
        a[i] = bf16_to_f32(y_m[i]);
        b[i] = bf16_to_f32(y_o[i]);
    }
    const int rc = orc_rse_f32(a, b, numel, mode, out);
    free(a);
    free(b);
    return rc;
}

void orc_round_bf16(float* x, int64_t numel) {
    for (int64_t i = 0; i < numel; ++i) {
        uint32_t u;
        memcpy(&u, &x[i], 4);
        if ((u & 0x7f800000u) != 0x7f800000u) {
            const uint32_t lsb = (u >> 16) & 1u;
            u += 0x7fffu + lsb;
        }
        u &= 0xffff0000u;
        memcpy(&x[i], &u, 4);
    }
}
