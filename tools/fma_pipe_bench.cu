// FP32 pipe throughput on sm_100a: SMSP clocks per warp instruction for the
// instruction forms the softmax uses — FFMA with three registers vs with an
// immediate, the packed FFMA2 / FADD2, FADD, FMNMX / 3-input FMNMX3 and the
// F2FP bf16 pack — and for mixes with MUFU.EX2 (do they overlap?). Sizes the
// per-element cost of each softmax step (scale-sub, exp2 on MUFU or the FMA
// pipe, row sum, pack).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fma_pipe_bench.cu -o build/fma_pipe && build/fma_pipe
#include <cstdint>
#include <cstdio>

constexpr int CH = 16;  // independent chains per thread

#define LOOP(BODY)                                  \
    for (int it = 0; it < iters; ++it) {            \
        _Pragma("unroll") for (int i = 0; i < CH; ++i) { BODY; } \
    }

template <int OP>
__global__ void __launch_bounds__(512, 1) pipe_kernel(const float* in, float* out, long long* clk, int iters) {
    float a[CH], b[CH];
    const float x = in[threadIdx.x & 63], y = in[(threadIdx.x + 7) & 63], z = in[(threadIdx.x + 13) & 63];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        a[i] = x + i * 1e-3f;
        b[i] = y - i * 1e-3f;
    }
    uint32_t acc = 0;
    __syncthreads();
    const long long t0 = clock64();
    if (OP == 0) {  // FFMA, 3 registers
        LOOP(asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(y), "f"(z)))
    } else if (OP == 1) {  // FFMA, immediate multiplier
        LOOP(asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, %1;" : "+f"(a[i]) : "f"(z)))
    } else if (OP == 2) {  // FFMA2 (packed fp32x2), registers
        const uint64_t yy = (static_cast<uint64_t>(__float_as_uint(y)) << 32) | __float_as_uint(y);
        const uint64_t zz = (static_cast<uint64_t>(__float_as_uint(z)) << 32) | __float_as_uint(z);
        uint64_t p[CH / 2];
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) p[i] = (static_cast<uint64_t>(__float_as_uint(a[2 * i])) << 32) | __float_as_uint(a[2 * i + 1]);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < CH / 2; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(yy), "l"(zz));
#pragma unroll
            for (int i = 0; i < CH / 2; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(yy), "l"(zz));
        }
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) a[i] = __uint_as_float(static_cast<uint32_t>(p[i]));
    } else if (OP == 3) {  // FADD2
        const uint64_t yy = (static_cast<uint64_t>(__float_as_uint(y)) << 32) | __float_as_uint(y);
        uint64_t p[CH / 2];
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) p[i] = (static_cast<uint64_t>(__float_as_uint(a[2 * i])) << 32) | __float_as_uint(a[2 * i + 1]);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < CH / 2; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(yy));
#pragma unroll
            for (int i = 0; i < CH / 2; ++i) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(yy));
        }
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) a[i] = __uint_as_float(static_cast<uint32_t>(p[i]));
    } else if (OP == 4) {  // FADD registers
        LOOP(asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i])))
    } else if (OP == 5) {  // FADD immediate
        LOOP(asm volatile("add.rn.f32 %0, %0, 0f3A800000;" : "+f"(a[i])))
    } else if (OP == 6) {  // FMNMX (2-input)
        LOOP(asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i])))
    } else if (OP == 7) {  // FMNMX3 (3-input)
        LOOP(asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b[i]), "f"(z)))
    } else if (OP == 8) {  // F2FP bf16x2 pack
        LOOP(uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(b[i])); a[i] = __uint_as_float(r))
    } else if (OP == 9) {  // MUFU.EX2
        LOOP(asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])))
    } else if (OP == 10) {  // MUFU.EX2 + FFMA imm, 1:1
        LOOP(asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])); asm volatile("fma.rn.f32 %0, %0, 0f3F7FF000, %1;" : "+f"(b[i]) : "f"(z)))
    } else if (OP == 11) {  // MUFU.EX2 + FFMA2, 1:1
        const uint64_t yy = (static_cast<uint64_t>(__float_as_uint(y)) << 32) | __float_as_uint(y);
        const uint64_t zz = (static_cast<uint64_t>(__float_as_uint(z)) << 32) | __float_as_uint(z);
        uint64_t p[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) p[i] = (static_cast<uint64_t>(__float_as_uint(b[i])) << 32) | __float_as_uint(b[i]);
        LOOP(asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])); asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(yy), "l"(zz)))
#pragma unroll
        for (int i = 0; i < CH; ++i) b[i] = __uint_as_float(static_cast<uint32_t>(p[i]));
    } else if (OP == 12) {  // FMUL registers
        LOOP(asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(y)))
    } else if (OP == 13) {  // FMUL2 (packed)
        const uint64_t yy = (static_cast<uint64_t>(__float_as_uint(y)) << 32) | __float_as_uint(y);
        uint64_t p[CH / 2];
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) p[i] = (static_cast<uint64_t>(__float_as_uint(a[2 * i])) << 32) | __float_as_uint(a[2 * i + 1]);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < CH / 2; ++i) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(yy));
#pragma unroll
            for (int i = 0; i < CH / 2; ++i) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(p[i]) : "l"(yy));
        }
#pragma unroll
        for (int i = 0; i < CH / 2; ++i) a[i] = __uint_as_float(static_cast<uint32_t>(p[i]));
    } else if (OP == 14) {  // FFMA, 2 registers + immediate addend (c in constant bank)
        LOOP(asm volatile("fma.rn.f32 %0, %0, %1, 0f3F7FF000;" : "+f"(a[i]) : "f"(y)))
    } else if (OP == 15) {  // IADD (integer add, the poly's exponent insert)
        LOOP(uint32_t u = __float_as_uint(a[i]); asm volatile("add.u32 %0, %0, %1;" : "+r"(u) : "r"(__float_as_uint(b[i]))); a[i] = __uint_as_float(u))
    }
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += a[i] + b[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
    if ((threadIdx.x & 31) == 0)
        clk[blockIdx.x * 16 + (threadIdx.x >> 5)] = t1 - t0;
}

template <int OP>
void run(const char* name, const float* in, float* out, long long* clk, long long* h, int threads) {
    const int iters = 512;
    pipe_kernel<OP><<<148, threads>>>(in, out, clk, iters);
    pipe_kernel<OP><<<148, threads>>>(in, out, clk, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, 148 * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int b = 0; b < 148; ++b)
        for (int w = 0; w < threads / 32; ++w) mx = h[b * 16 + w] > mx ? h[b * 16 + w] : mx;
    const int warps_per_smsp = threads / 128;
    // instructions per warp per iteration: CH (1 op per chain) or 2*CH for the mixes
    const double per_iter = (OP == 10 || OP == 11) ? 2.0 * CH : CH;
    std::printf("%-28s warps/SMSP %d: %.2f SMSP clk per warp instruction\n", name, warps_per_smsp,
                mx / iters / (per_iter * warps_per_smsp));
}

int main() {
    float *in, *out;
    long long *clk, h[148 * 16];
    cudaMalloc(&in, 64 * 4);
    cudaMalloc(&out, 148 * 512 * 4);
    cudaMalloc(&clk, 148 * 16 * 8);
    float hin[64];
    for (int i = 0; i < 64; ++i) hin[i] = 0.25f + 0.001f * i;
    cudaMemcpy(in, hin, sizeof hin, cudaMemcpyHostToDevice);
    for (int th : {128, 256, 512}) {
        run<0>("FFMA r,r,r", in, out, clk, h, th);
        run<1>("FFMA r,imm,r", in, out, clk, h, th);
        run<14>("FFMA r,r,imm", in, out, clk, h, th);
        run<2>("FFMA2 (f32x2)", in, out, clk, h, th);
        run<3>("FADD2 (f32x2)", in, out, clk, h, th);
        run<13>("FMUL2 (f32x2)", in, out, clk, h, th);
        run<4>("FADD r,r", in, out, clk, h, th);
        run<5>("FADD r,imm", in, out, clk, h, th);
        run<12>("FMUL r,r", in, out, clk, h, th);
        run<6>("FMNMX", in, out, clk, h, th);
        run<7>("FMNMX3", in, out, clk, h, th);
        run<8>("F2FP.BF16 pack", in, out, clk, h, th);
        run<15>("IADD", in, out, clk, h, th);
        run<9>("MUFU.EX2", in, out, clk, h, th);
        run<10>("MUFU.EX2 + FFMA imm (per instr)", in, out, clk, h, th);
        run<11>("MUFU.EX2 + FFMA2 (per instr)", in, out, clk, h, th);
    }
    std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
