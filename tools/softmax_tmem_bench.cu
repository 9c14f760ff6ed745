// Softmax step on TMEM data (sm_100a), no MMAs: each warp repeatedly loads
// its rows' scores from TMEM (tcgen05.ld 32x32b), takes the row max, computes
// exp2 (MUFU + every EMU-th pair on the FMA pipe), the row sum, packs P to
// bf16 and stores it back (tcgen05.st) — the fused kernel's per-tile softmax
// with the TMEM latency included. Compares 2 warps per SMSP with 128-key rows
// (the kernel's two lanes) against 4 warps per SMSP with 64-key rows (a
// 4-lane, 64-key-step layout), in SMSP clocks per 128 scores of one row.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_22796_b200/csrc tools/softmax_tmem_bench.cu -o build/smt
#include <cstdio>
#include <cstdint>

#include "sm100_ptx.cuh"
using namespace dfa2k;

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : DFA2_R8(0), DFA2_R8(8), DFA2_R8(16), DFA2_R8(24), DFA2_R8(32), DFA2_R8(40), DFA2_R8(48), DFA2_R8(56)
        : "r"(taddr));
}

template <int EL, int EMU, bool WIDE_LD = false>
__global__ void __launch_bounds__(EL == 128 ? 256 : 512, 1) step(float* out, long long* clk, int iters) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        tmem_alloc(smem_u32(&slot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    // warp w: TMEM lane quarter w % 4, column block (w / 4) * EL
    const uint32_t base = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * EL;
    {  // fill the scores
        uint32_t v[32];
        for (int c = 0; c < EL; c += 32) {
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(0.01f * ((lane * 7 + i + c) % 97) - 0.3f);
            tmem_st32(base + c, v);
        }
        tmem_st_wait();
    }
    float l = 0.f, m_ref = 0.f;
    const float sl2 = 0.127f;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t s[EL];
        if (WIDE_LD) {
#pragma unroll
            for (int c = 0; c < EL; c += 64)
                tmem_ld64(base + c, s + c);
        } else {
#pragma unroll
            for (int c = 0; c < EL; c += 32)
                tmem_ld32(base + c, s + c);
        }
        tmem_ld_wait();
        float mm[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            mm[j] = fmaxf(__uint_as_float(s[2 * j]), __uint_as_float(s[2 * j + 1]));
#pragma unroll
        for (int c = 16; c < EL; c += 16)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                mm[j] = fmaxf(mm[j], fmaxf(__uint_as_float(s[c + 2 * j]), __uint_as_float(s[c + 2 * j + 1])));
        const float mx = fmaxf(fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3])),
                               fmaxf(fmaxf(mm[4], mm[5]), fmaxf(mm[6], mm[7]))) * sl2;
        m_ref = fmaxf(m_ref, mx);
        const float2 scale2 = make_float2(sl2, sl2), neg_m = make_float2(-m_ref, -m_ref);
        float2 sum = make_float2(0.f, 0.f);
#pragma unroll
        for (int cc = 0; cc < EL / 32; ++cc) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[32 * cc + 2 * i]),
                                                        __uint_as_float(s[32 * cc + 2 * i + 1])),
                                            scale2, neg_m);
                float2 p;
                if (EMU > 0 && (i % (EMU > 0 ? EMU : 1)) == EMU - 1) {
                    const float2 xc = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
                    const float2 t = __fadd2_rd(xc, make_float2(12582912.f, 12582912.f));
                    const float2 tm = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
                    const float2 f = __ffma2_rn(tm, make_float2(-1.f, -1.f), xc);
                    float2 q = __ffma2_rn(make_float2(0.0770652f, 0.0770652f), f, make_float2(0.227647f, 0.227647f));
                    q = __ffma2_rn(q, f, make_float2(0.69511634f, 0.69511634f));
                    q = __ffma2_rn(q, f, make_float2(1.0f, 1.0f));
                    p = make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                                    __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
                } else {
                    p = make_float2(ex2_approx(x.x), ex2_approx(x.y));
                }
                sum = __fadd2_rn(sum, p);
                pk[i] = pack_bf16x2(p.x, p.y);
            }
            tmem_st16(base + 16 * cc, pk);  // P over the first half of the scores, as the kernel does
        }
        tmem_st_wait();
        l += sum.x + sum.y;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = l;
    if (lane == 0)
        clk[blockIdx.x * 16 + warp] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0)
        tmem_dealloc(tmem, 512);
}

template <int EL, int EMU, bool WIDE_LD = false>
void run(float* out, long long* clk, long long* h, int warps) {
    const int iters = 400;
    step<EL, EMU, WIDE_LD><<<148, warps * 32>>>(out, clk, iters);
    step<EL, EMU, WIDE_LD><<<148, warps * 32>>>(out, clk, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, 148 * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int b = 0; b < 148; ++b)
        for (int w = 0; w < warps; ++w) mx = h[b * 16 + w] > mx ? h[b * 16 + w] : mx;
    const double rows = warps / 4.0 * EL / 128.0;  // 128-score rows per SMSP per iteration
    std::printf("keys/row %3d EMU %d warps/SMSP %d ld %s: %.0f clk per iteration, %.0f SMSP clk per 128 scores\n", EL,
                EMU, warps / 4, WIDE_LD ? "x64" : "x32", mx / iters, mx / iters / rows);
}

int main() {
    float* out;
    long long *clk, h[148 * 16];
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&clk, 148 * 16 * 8);
    run<128, 3>(out, clk, h, 8);   // the kernel today: 2 lanes x 128-key rows
    run<128, 3, true>(out, clk, h, 8);
    run<128, 3>(out, clk, h, 4);
    run<128, 3, true>(out, clk, h, 4);
    run<64, 3>(out, clk, h, 16);   // 4 lanes x 64-key rows
    run<64, 3>(out, clk, h, 8);
    run<128, 8>(out, clk, h, 8);
    run<64, 4>(out, clk, h, 16);
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
