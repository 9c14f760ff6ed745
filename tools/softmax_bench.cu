// Softmax exp-phase microbenchmark (sm_100a): one 128-element score row per
// thread held in registers, the kernel's per-pair recipe (FFMA2 scale-sub,
// exp2 on MUFU or the FMA-pipe polynomial every EMU-th pair, FADD2 row sum,
// F2FP bf16 pack) repeated; clocks per row with 1 or 2 warps per SMSP (the
// softmax warps of one or both lanes). Sizes the exp share the fused kernel
// can move off MUFU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/softmax_bench.cu -o /tmp/smb && /tmp/smb
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
template <int DEG>
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    const float2 xc = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
    const float2 t = __fadd2_rd(xc, make_float2(12582912.f, 12582912.f));
    const float2 tm = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = __ffma2_rn(tm, make_float2(-1.f, -1.f), xc);
    float2 p;
    if (DEG == 3) {
        p = __ffma2_rn(make_float2(0.0770652f, 0.0770652f), f, make_float2(0.227647f, 0.227647f));
        p = __ffma2_rn(p, f, make_float2(0.69511634f, 0.69511634f));
        p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
    } else {  // degree 2 minimax on [0,1): max rel err ~1.7e-3
        p = __ffma2_rn(make_float2(0.3371894f, 0.3371894f), f, make_float2(0.6576363f, 0.6576363f));
        p = __ffma2_rn(p, f, make_float2(1.0017247f, 1.0017247f));
    }
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

template <int EMU, int DEG, int EL = 128>
__global__ void __launch_bounds__(512, 1) row_kernel(const float* in, float* out, long long* clk, int iters) {
    float s[EL];
#pragma unroll
    for (int i = 0; i < EL; ++i) s[i] = in[(threadIdx.x * 131 + i) & 4095];
    const float2 scale2 = make_float2(0.127f, 0.127f);
    float m = 0.5f;
    uint32_t acc = 0;
    float l = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const float2 neg_m = make_float2(-m, -m);
        float2 sum = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < EL / 2; ++i) {
            const float2 x = __ffma2_rn(make_float2(s[2 * i], s[2 * i + 1]), scale2, neg_m);
            float2 p;
            if (EMU > 0 && (i % (EMU > 0 ? EMU : 1)) == EMU - 1)
                p = ex2_poly2<DEG>(x);
            else
                p = make_float2(ex2_approx(x.x), ex2_approx(x.y));
            sum = __fadd2_rn(sum, p);
            acc ^= pack_bf16x2(p.x, p.y);
        }
        l += sum.x + sum.y;
        m = l * 1e-30f + 0.5f;  // loop-carried: the next row's exps depend on this one
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = l + __uint_as_float(acc & 0x3FFFFFFF) * 1e-30f;
    if (threadIdx.x % 32 == 0)
        clk[blockIdx.x * 16 + threadIdx.x / 32] = t1 - t0;
}

template <int EMU, int DEG, int EL = 128>
void run(const float* in, float* out, long long* clk, long long* h, int threads) {
    const int iters = 400;
    row_kernel<EMU, DEG, EL><<<148, threads>>>(in, out, clk, iters);
    row_kernel<EMU, DEG, EL><<<148, threads>>>(in, out, clk, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, 148 * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int b = 0; b < 148; ++b)
        for (int w = 0; w < threads / 32; ++w) mx = h[b * 16 + w] > mx ? h[b * 16 + w] : mx;
    // SMSP time per 128 elements of one row: (warps per SMSP) x EL elements per warp-iteration
    const double rows_per_iter = threads / 128.0 * EL / 128.0;
    printf("EMU %d deg %d  elems/thread %3d warps/SMSP %d : %.0f clk per 128-element row of SMSP time\n", EMU, DEG,
           EL, threads / 128, mx / iters / rows_per_iter);
}

int main() {
    float *in, *out;
    long long *clk, h[148 * 16];
    cudaMalloc(&in, 4096 * 4);
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&clk, 148 * 16 * 8);
    cudaMemset(in, 0, 4096 * 4);
    for (int th : {256, 512}) {
        run<3, 3, 64>(in, out, clk, h, th);
        run<4, 3, 64>(in, out, clk, h, th);
    }
    for (int th : {128, 256, 384, 512}) {
        run<3, 3>(in, out, clk, h, th);
        run<4, 3>(in, out, clk, h, th);
    }
    for (int th : {128, 256}) {
        run<0, 3>(in, out, clk, h, th);
        run<8, 3>(in, out, clk, h, th);
        run<4, 3>(in, out, clk, h, th);
        run<3, 3>(in, out, clk, h, th);
        run<2, 3>(in, out, clk, h, th);
        run<3, 2>(in, out, clk, h, th);
        run<2, 2>(in, out, clk, h, th);
    }
    return 0;
}
