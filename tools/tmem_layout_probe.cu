// Probe of the tcgen05.ld/st 16x256b and 16x128b data-path layouts on sm_100a:
// TMEM is filled through 32x32b stores (thread i = lane i) with
// value = lane * 1000 + column, then read back through the 16-lane shapes.
#include <cstdio>
#include <cstdint>
#include "../paper_2503_22796_b200/csrc/sm100_ptx.cuh"
using namespace dfa2k;

__global__ void probe(uint32_t* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        tmem_alloc(smem_u32(&slot), 64);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t lrow = static_cast<uint32_t>(warp * 32) << 16;
    uint32_t v[32];
    for (int c = 0; c < 32; ++c)
        v[c] = (warp * 32 + lane) * 1000 + c;
    tmem_st32(tmem + lrow, v);
    tmem_st_wait();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) {
        // 16x256b.x1 at lanes 32..47: 4 regs per thread
        uint32_t r[4];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tmem + lrow));
        tmem_ld_wait();
        for (int i = 0; i < 4; ++i) out[lane * 4 + i] = r[i];
        // 16x256b.x2 at lanes 48..63, columns 0..15: 8 regs per thread
        uint32_t s[8];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7])
                     : "r"(tmem + lrow + (16u << 16)));
        tmem_ld_wait();
        for (int i = 0; i < 8; ++i) out[128 + lane * 8 + i] = s[i];
        // 16x128b.x2 at lanes 32..47: 4 regs per thread
        uint32_t t[4];
        asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]) : "r"(tmem + lrow));
        tmem_ld_wait();
        for (int i = 0; i < 4; ++i) out[384 + lane * 4 + i] = t[i];
        // 16x128b.x2 STORE of (lane*100 + i) at lanes 32..47 cols 40..47, read back with 32x32b
        uint32_t w[4];
        for (int i = 0; i < 4; ++i) w[i] = 500000 + lane * 10 + i;
        asm volatile("tcgen05.st.sync.aligned.16x128b.x2.b32 [%0], {%1,%2,%3,%4};"
                     :: "r"(tmem + lrow + 40), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
        tmem_st_wait();
        uint32_t b[32];
        tmem_ld32(tmem + lrow + 32, b);
        tmem_ld_wait();
        for (int i = 0; i < 16; ++i) out[512 + lane * 16 + i] = b[8 + i];
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0)
        tmem_dealloc(tmem, 64);
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 4096 * 4);
    cudaMemset(d, 0xff, 4096 * 4);
    probe<<<1, 128>>>(d);
    uint32_t h[1024];
    cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(e));
    auto dec = [](uint32_t x) { static char b[32]; snprintf(b, 32, "L%u:c%u", x / 1000, x % 1000); return b; };
    printf("16x256b.x1 (lanes 32..):\n");
    for (int t = 0; t < 8; ++t) { printf(" t%d", t); for (int i = 0; i < 4; ++i) printf(" %s", dec(h[t * 4 + i])); printf("\n"); }
    printf(" t31"); for (int i = 0; i < 4; ++i) printf(" %s", dec(h[31 * 4 + i])); printf("\n");
    printf("16x256b.x2 (lanes 48..):\n");
    for (int t : {0, 1, 4, 31}) { printf(" t%d", t); for (int i = 0; i < 8; ++i) printf(" %s", dec(h[128 + t * 8 + i])); printf("\n"); }
    printf("16x128b.x2 (lanes 32..):\n");
    for (int t : {0, 1, 2, 3, 4, 31}) { printf(" t%d", t); for (int i = 0; i < 4; ++i) printf(" %s", dec(h[384 + t * 4 + i])); printf("\n"); }
    printf("16x128b.x2 store at col 40, read lanes 32.. cols 40..55 via 32x32b (value 500000+lane*10+reg):\n");
    for (int r : {0, 1, 8, 9, 15}) { printf(" lane%d", 32 + r); for (int i = 0; i < 10; ++i) printf(" %u", h[512 + r * 16 + i] >= 500000 && h[512 + r * 16 + i] < 600000 ? h[512 + r * 16 + i] - 500000 : 9999999); printf("\n"); }
    return 0;
}
