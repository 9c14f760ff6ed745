// workload_sm100.cu — the synthetic MMDiT Q/K/V stream generated on the
// device (the model of /root/reference/proj/src/
// workload.cpp:120-228, at FLUX scale).
//
// Per (layer, head) the reference draws, at t = 0,
//   visual rows: q = 6 u + 0.3 g_q, k = 6 u + 0.3 g_k, u = sqrt(2/d) cos(omega_f i + phase_f)
//   text rows:   q = (3/sqrt(d)) g_q, k = (3/sqrt(d)) g_k
//   v = g_v
// and then a random walk, x_t = x_{t-1} + drift * g_t (drift 0: frozen).
// Here the positional features (omega, phase) are the reference's own
// mt19937_64 draws (host), and the per-element gaussians g come from a
// counter-based generator — Philox4x32-10 keyed by the reference's stream
// seed of (seed, layer, head, t, tag), counter = element index, Box-Muller —
// so any slot is a pure function of (seed, t, layer, head, element), the
// walk state lives in HBM as fp32 (as the reference accumulates in f32) and
// every slot is emitted as the bf16 tensors the attention call reads.
// HBM-bound: per element and tensor, 4 B state read + 4 B write + 2 B out.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gen_types.h"

namespace dfa2k {

namespace {

__device__ __forceinline__ void philox_round(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c[0]), lo0 = M0 * c[0];
    const uint32_t hi1 = __umulhi(M1, c[2]), lo1 = M1 * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
}

// Philox4x32-10 of counter (lo, hi, 0, 0) under key (k0, k1)
__device__ __forceinline__ void philox(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        philox_round(c, k0, k1);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// two standard normals from two uint32 (Box-Muller; u1 in (0, 1])
__device__ __forceinline__ float2 box_muller(uint32_t a, uint32_t b) {
    const float u1 = (static_cast<float>(a) + 1.0f) * 2.3283064365386963e-10f;
    const float u2 = static_cast<float>(b) * 2.3283064365386963e-10f;
    const float r = sqrtf(-2.0f * __logf(u1));
    float s, c;
    __sincosf(6.283185307179586f * u2, &s, &c);
    return make_float2(r * c, r * s);
}

// 4 gaussians for elements 4j .. 4j+3 of the stream keyed (k0, k1)
__device__ __forceinline__ void gauss4(uint64_t j, uint32_t k0, uint32_t k1, float (&g)[4]) {
    uint32_t c[4] = {static_cast<uint32_t>(j), static_cast<uint32_t>(j >> 32), 0u, 0u};
    philox(c, k0, k1);
    const float2 a = box_muller(c[0], c[1]), b = box_muller(c[2], c[3]);
    g[0] = a.x;
    g[1] = a.y;
    g[2] = b.x;
    g[3] = b.y;
}

}  // namespace


// t = 0: state[3][H][n][d] (fp32) and out_q/k/v [H][n][d] (bf16).
// features: per head, omega[d] then phase[d] (double, the reference's draws).
__global__ void gen_init_kernel(float* __restrict__ state, __nv_bfloat16* __restrict__ oq,
                                __nv_bfloat16* __restrict__ ok, __nv_bfloat16* __restrict__ ov,
                                const GenHead* __restrict__ heads, const double* __restrict__ features, int H, int n,
                                int d, int text_lo, int text_hi, float feat_scale, float text_scale) {
    const int64_t per_head = static_cast<int64_t>(n) * d;
    const int64_t quads = per_head / 4;  // d % 4 == 0
    const int64_t total = quads * H;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int h = static_cast<int>(i / quads);
        const int64_t j = i % quads;  // quad within the head
        const GenHead gh = heads[h];
        const int64_t e0 = j * 4;
        const int row = static_cast<int>(e0 / d), f0 = static_cast<int>(e0 % d);
        float gq[4], gk[4], gv[4];
        gauss4(j, gh.key[0][0], gh.key[0][1], gq);
        gauss4(j, gh.key[1][0], gh.key[1][1], gk);
        gauss4(j, gh.key[2][0], gh.key[2][1], gv);
        const bool text = row >= text_lo && row < text_hi;
        float q4[4], k4[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (text) {
                q4[e] = text_scale * gq[e];
                k4[e] = text_scale * gk[e];
            } else {
                const double om = features[gh.omega_off + f0 + e], ph = features[gh.omega_off + d + f0 + e];
                const float u = feat_scale * static_cast<float>(cos(om * static_cast<double>(row) + ph));
                q4[e] = 6.0f * u + 0.3f * gq[e];
                k4[e] = 6.0f * u + 0.3f * gk[e];
            }
        }
        const int64_t off = static_cast<int64_t>(h) * per_head + e0;
        float* sq = state + off;
        float* sk = state + static_cast<int64_t>(H) * per_head + off;
        float* sv = state + 2 * static_cast<int64_t>(H) * per_head + off;
        *reinterpret_cast<float4*>(sq) = make_float4(q4[0], q4[1], q4[2], q4[3]);
        *reinterpret_cast<float4*>(sk) = make_float4(k4[0], k4[1], k4[2], k4[3]);
        *reinterpret_cast<float4*>(sv) = make_float4(gv[0], gv[1], gv[2], gv[3]);
        __nv_bfloat162* bq = reinterpret_cast<__nv_bfloat162*>(oq + off);
        __nv_bfloat162* bk = reinterpret_cast<__nv_bfloat162*>(ok + off);
        __nv_bfloat162* bv = reinterpret_cast<__nv_bfloat162*>(ov + off);
        bq[0] = __floats2bfloat162_rn(q4[0], q4[1]);
        bq[1] = __floats2bfloat162_rn(q4[2], q4[3]);
        bk[0] = __floats2bfloat162_rn(k4[0], k4[1]);
        bk[1] = __floats2bfloat162_rn(k4[2], k4[3]);
        bv[0] = __floats2bfloat162_rn(gv[0], gv[1]);
        bv[1] = __floats2bfloat162_rn(gv[2], gv[3]);
    }
}

// t -> t + 1: state += drift * g (one drift stream per head: q elements
// first, then k, then v, as the reference draws them, src/workload.cpp:
// 214-222), then emit bf16. emit_only: no step, just re-emit the state.
__global__ void gen_step_kernel(float* __restrict__ state, __nv_bfloat16* __restrict__ oq,
                                __nv_bfloat16* __restrict__ ok, __nv_bfloat16* __restrict__ ov,
                                const GenHead* __restrict__ heads, int H, int n, int d, int emit_only) {
    const int64_t per_head = static_cast<int64_t>(n) * d;
    const int64_t quads = per_head / 4;
    const int64_t total = quads * H * 3;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t tq = i / (quads * H);  // tensor: 0 q, 1 k, 2 v
        const int64_t r = i % (quads * H);
        const int h = static_cast<int>(r / quads);
        const int64_t j = r % quads;
        const GenHead gh = heads[h];
        const int64_t off = tq * H * per_head + static_cast<int64_t>(h) * per_head + j * 4;
        float4 s = *reinterpret_cast<const float4*>(state + off);
        if (!emit_only && gh.drift != 0.0f) {
            float g[4];
            gauss4(static_cast<uint64_t>(tq) * static_cast<uint64_t>(quads) + j, gh.key[0][0], gh.key[0][1], g);
            s.x += gh.drift * g[0];
            s.y += gh.drift * g[1];
            s.z += gh.drift * g[2];
            s.w += gh.drift * g[3];
            *reinterpret_cast<float4*>(state + off) = s;
        }
        __nv_bfloat16* o = tq == 0 ? oq : tq == 1 ? ok : ov;
        __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(o + static_cast<int64_t>(h) * per_head + j * 4);
        b[0] = __floats2bfloat162_rn(s.x, s.y);
        b[1] = __floats2bfloat162_rn(s.z, s.w);
    }
}

cudaError_t launch_gen_init(float* state, void* q, void* k, void* v, const GenHead* heads, const double* features,
                            int H, int n, int d, int text_lo, int text_hi, float feat_scale, float text_scale, int sms,
                            cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(n) * d / 4 * H;
    const int64_t blocks = (total + 255) / 256;
    const int grid = static_cast<int>(blocks < 16LL * sms ? blocks : 16LL * sms);
    gen_init_kernel<<<grid, 256, 0, st>>>(state, static_cast<__nv_bfloat16*>(q), static_cast<__nv_bfloat16*>(k),
                                          static_cast<__nv_bfloat16*>(v), heads, features, H, n, d, text_lo, text_hi,
                                          feat_scale, text_scale);
    return cudaGetLastError();
}

cudaError_t launch_gen_step(float* state, void* q, void* k, void* v, const GenHead* heads, int H, int n, int d,
                            int emit_only, int sms, cudaStream_t st) {
    const int64_t total = static_cast<int64_t>(n) * d / 4 * H * 3;
    const int64_t blocks = (total + 255) / 256;
    const int grid = static_cast<int>(blocks < 16LL * sms ? blocks : 16LL * sms);
    gen_step_kernel<<<grid, 256, 0, st>>>(state, static_cast<__nv_bfloat16*>(q), static_cast<__nv_bfloat16*>(k),
                                          static_cast<__nv_bfloat16*>(v), heads, H, n, d, emit_only);
    return cudaGetLastError();
}

}  // namespace dfa2k
