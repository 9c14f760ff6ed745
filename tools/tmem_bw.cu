// TMEM read bandwidth probe (sm_100a): warps repeatedly read a 128-column
// fp32 row block (the softmax's S tile: 4 x tcgen05.ld.32x32b.x32 + wait) and
// fold it into a checksum; clocks per 128-column read with 4, 8 or 12 warps
// (1, 2, 3 per SMSP) — is reading S from TMEM a floor of the softmax?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_22796_b200/csrc tools/tmem_bw.cu -o build/tmem_bw
#include <cstdio>
#include <cstdint>

#include "sm100_ptx.cuh"
using namespace dfa2k;

__global__ void __launch_bounds__(384, 1) bw(uint32_t* out, long long* clk, int iters, int split) {
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
    const uint32_t lrow = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t col = static_cast<uint32_t>((warp >> 2) * 128) & 511u;
    uint32_t acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t a[32], b[32];
        if (split) {  // the kernel's pattern: two 64-column halves, wait after each
            tmem_ld32(tmem + lrow + col, a);
            tmem_ld32(tmem + lrow + col + 32, b);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += a[i] ^ b[i];
            tmem_ld32(tmem + lrow + col + 64, a);
            tmem_ld32(tmem + lrow + col + 96, b);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += a[i] ^ b[i];
        } else {
            uint32_t c[32], d[32];
            tmem_ld32(tmem + lrow + col, a);
            tmem_ld32(tmem + lrow + col + 32, b);
            tmem_ld32(tmem + lrow + col + 64, c);
            tmem_ld32(tmem + lrow + col + 96, d);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += a[i] ^ b[i] ^ c[i] ^ d[i];
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (lane == 0)
        clk[blockIdx.x * 12 + warp] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0)
        tmem_dealloc(tmem, 512);
}

int main() {
    uint32_t* out;
    long long *clk, h[148 * 12];
    cudaMalloc(&out, 148 * 384 * 4);
    cudaMalloc(&clk, 148 * 12 * 8);
    const int iters = 2000;
    for (int split : {0, 1})
        for (int warps : {4, 8, 12}) {
            bw<<<148, warps * 32>>>(out, clk, iters, split);
            bw<<<148, warps * 32>>>(out, clk, iters, split);
            cudaDeviceSynchronize();
            cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (int b = 0; b < 148; ++b)
                for (int w = 0; w < warps; ++w) mx = h[b * 12 + w] > mx ? h[b * 12 + w] : mx;
            const double per = mx / iters;  // clocks per 128-column read per warp
            std::printf("split %d warps %2d: %.0f clk per 128-col read per warp; SM reads %.0f B/clk\n", split,
                        warps, per, warps * 32 * 128 * 4 / per);
        }
    return cudaGetLastError() != cudaSuccess;
}
