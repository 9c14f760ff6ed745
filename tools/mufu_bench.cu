// MUFU exp2 throughput probe: f32 ex2.approx vs packed ex2.approx.f16x2 and
// ex2.approx.ftz.bf16x2 (elements per clock per SM), to size the softmax's
// exp budget; plus the f32 -> bf16x2 pack (cvt.rn.bf16x2.f32 = F2FP) alone,
// mixed with ex2 (do they share a pipe?), and an integer round-and-PRMT pack. nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_bench.cu -o /tmp/mufu
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

__global__ void f32_kernel(float* out, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f32 %0, %0;" : "+f"(a[i]));
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void f16x2_kernel(float* out, int iters) {
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.001f * threadIdx.x, -0.002f * i); a[i] = *reinterpret_cast<uint32_t*>(&h); }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
    float s = 0;
    for (int i = 0; i < 8; ++i) s += __half2float(reinterpret_cast<__half2*>(&a[i])->x);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void bf16x2_kernel(float* out, int iters) {
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) { __nv_bfloat162 h = __floats2bfloat162_rn(-0.001f * threadIdx.x, -0.002f * i); a[i] = *reinterpret_cast<uint32_t*>(&h); }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
    float s = 0;
    for (int i = 0; i < 8; ++i) s += __bfloat162float(reinterpret_cast<__nv_bfloat162*>(&a[i])->x);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// cvt.rn.bf16x2.f32 chains: 8 independent packs per iteration (feeding the
// result back through the float bits keeps each chain dependent)
__global__ void cvt_kernel(float* out, int iters) {
    float a[8], b[8];
    for (int i = 0; i < 8; ++i) { a[i] = 0.001f * (threadIdx.x + i); b[i] = 0.5f + i; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t r;
            asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(b[i]));
            a[i] = __uint_as_float(r);
        }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// one ex2 + one pack per element (the softmax's mix)
__global__ void mix_kernel(float* out, int iters) {
    float a[8], b[8];
    for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); b[i] = 0.5f + i; }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("ex2.approx.f32 %0, %0;" : "+f"(a[i]));
            uint32_t r;
            asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b[i]), "f"(a[i]));
            b[i] = __uint_as_float(r);
        }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + b[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// integer pack: round half up on the bit patterns (non-negative P), PRMT the high halves
__global__ void ipack_kernel(float* out, int iters) {
    uint32_t a[8], b[8];
    for (int i = 0; i < 8; ++i) { a[i] = __float_as_uint(0.001f * (threadIdx.x + i)); b[i] = __float_as_uint(0.5f + i); }
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            uint32_t r;
            asm volatile("{\n\t.reg .b32 x, y;\n\tadd.u32 x, %1, 0x8000;\n\tadd.u32 y, %2, 0x8000;\n\t"
                         "prmt.b32 %0, x, y, 0x7632;\n\t}" : "=r"(r) : "r"(a[i]), "r"(b[i]));
            a[i] = r;
        }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += __uint_as_float(a[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, sms * 4 * 1024 * 4);
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, void (*k)(float*, int), int elems_per_op) {
        k<<<sms * 4, 1024>>>(out, 16);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k<<<sms * 4, 1024>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = double(sms) * 4 * 1024 * iters * 8;
        const double per_clk_sm = ops * elems_per_op / (ms * 1e-3) / sms / (clk * 1e3);
        printf("%-8s %.3f ms  %.1f exp2/clk/SM (at %d MHz nominal)\n", name, ms, per_clk_sm, clk / 1000);
    };
    run("f32", f32_kernel, 1);
    run("f16x2", f16x2_kernel, 2);
    run("bf16x2", bf16x2_kernel, 2);
    printf("(below: packs or element-pairs per clk per SM)\n");
    run("cvt", cvt_kernel, 1);
    run("ex2+cvt", mix_kernel, 1);
    run("ipack", ipack_kernel, 1);
    return 0;
}
