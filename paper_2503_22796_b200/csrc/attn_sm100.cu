// attn_sm100.cu — the fused head-wise attention kernel for B200 (sm_100a).
//
// Replaces, in ONE launch per joint-attention layer, the reference's phase-1
// loop of multi_strategy_attention (/root/reference/proj/src/dispatch.cpp:62-83)
// plus its phase-2 cache commit (:85-88):
//   Full heads  -> attention_head_impl      (src/tensor.cpp:73-114)
//   Arrow heads -> streaming_block_pass     (src/arrow.cpp:24-72) over only
//                  the KV tiles build_arrow_mask keeps (src/arrow.cpp:113-153)
//   Cached heads-> copy of the stored slot  (src/dispatch.cpp:77-81)
//
// Structure (persistent, one CTA per SM, static LPT work list built on the
// host, see dfa2c.cpp):
//   warp 0      TMA producer: Q tile (double-buffered) + K/V tiles (ring)
//   warp 1      tcgen05 issuer: S = Q K^T (SS, into TMEM, double-buffered)
//               and O += P V (TS: P read from TMEM, V from smem)
//   warp 2      TMEM allocator
//   warps 4-7   softmax warpgroup: one query row per thread; tcgen05.ld of
//               S, online softmax in the exp2 domain with lazy (threshold 8)
//               rescaling of O in TMEM, P written back to TMEM as bf16,
//               epilogue O/l -> bf16 -> out (+ cache slot); also executes the
//               Cached heads' copy items.
// TMEM (512 cols): S0 [0,128)  S1 [128,256)  O [256,256+D)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "attn_types.h"
#include "sm100_ptx.cuh"

namespace dfa2k {

template <int D>
struct Cfg {
    static constexpr int STAGES = D == 128 ? 2 : 4;
    static constexpr int BOXES = D / 64;                       // 128-byte column boxes
    static constexpr uint32_t BOX_BYTES = 128u * 128u;         // 128 rows x 128 B
    static constexpr uint32_t TILE_BYTES = BOXES * BOX_BYTES;  // one Q, K or V tile
    static constexpr uint32_t Q_OFF = 0;
    static constexpr uint32_t K_OFF = Q_OFF + 2 * TILE_BYTES;
    static constexpr uint32_t V_OFF = K_OFF + STAGES * TILE_BYTES;
    static constexpr uint32_t BAR_OFF = V_OFF + STAGES * TILE_BYTES;
    static constexpr int NBARS = 2 + 2 + 3 * STAGES + 2 + 2 + 2;
    static constexpr uint32_t SMEM_BYTES = BAR_OFF + NBARS * 8 + 16 + 1024;
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr uint32_t O_COL = 256;
};

namespace {

__device__ __forceinline__ uint32_t s_col(int sb) { return sb ? 128u : 0u; }

// Per-row 128-column validity bitmap for a partial tile: key < N and the
// (query block, key block) pair active in the head's block mask.
__device__ __forceinline__ void tile_valid_bits(const AttnArgs& a, const uint8_t* mask, int row,
                                                int k0, uint32_t (&vm)[4]) {
    vm[0] = vm[1] = vm[2] = vm[3] = 0u;
    const int B = a.block;
    const int rr = row < a.n ? row : a.n - 1;
    const uint8_t* mrow = mask + static_cast<size_t>(rr / B) * a.nb;
    const int kend = min(k0 + 128, a.n);
    for (int kb = k0 / B; kb * B < kend; ++kb) {
        if (!mrow[kb])
            continue;
        const int lo = max(kb * B, k0) - k0;
        const int hi = min(kb * B + B, kend) - k0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int a0 = max(lo, 32 * w), a1 = min(hi, 32 * w + 32);
            if (a1 > a0) {
                const int nbits = a1 - a0;
                const uint32_t bits = nbits == 32 ? 0xFFFFFFFFu : ((1u << nbits) - 1u);
                vm[w] |= bits << (a0 - 32 * w);
            }
        }
    }
}

}  // namespace

template <int D>
__global__ void __launch_bounds__(256, 1)
    attn_fwd_sm100(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                   const __grid_constant__ CUtensorMap tmv, const AttnArgs args) {
    using C = Cfg<D>;
    constexpr int S = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (sbase - raw);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    const uint32_t bars = sbase + C::BAR_OFF;
    auto q_full = [&](int i) { return bars + 8u * i; };
    auto q_empty = [&](int i) { return bars + 8u * (2 + i); };
    auto k_full = [&](int s) { return bars + 8u * (4 + s); };
    auto v_full = [&](int s) { return bars + 8u * (4 + S + s); };
    auto kv_empty = [&](int s) { return bars + 8u * (4 + 2 * S + s); };
    auto s_full = [&](int i) { return bars + 8u * (4 + 3 * S + i); };
    auto p_full = [&](int i) { return bars + 8u * (6 + 3 * S + i); };
    auto pv_done = [&](int i) { return bars + 8u * (8 + 3 * S + i); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::BAR_OFF + C::NBARS * 8);

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(q_full(i), 1);
            mbar_init(q_empty(i), 1);
            mbar_init(s_full(i), 1);
            mbar_init(p_full(i), 128);
            mbar_init(pv_done(i), 1);
        }
        for (int s = 0; s < S; ++s) {
            mbar_init(k_full(s), 1);
            mbar_init(v_full(s), 1);
            mbar_init(kv_empty(s), 1);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmq);
        tma_prefetch_desc(&tmk);
        tma_prefetch_desc(&tmv);
    }
    if (warp == 2) {
        tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int it0 = args.cta_begin[blockIdx.x];
    const int it1 = args.cta_begin[blockIdx.x + 1];

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t kv_it = 0, q_it = 0;
            for (int it = it0; it < it1; ++it) {
                const WorkItem w = args.items[it];
                if (w.flags & ITEM_COPY)
                    continue;
                const int qb = q_it & 1;
                mbar_wait(q_empty(qb), ((q_it >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(q_full(qb), C::TILE_BYTES);
#pragma unroll
                for (int b = 0; b < C::BOXES; ++b)
                    tma_load_3d(sbase + C::Q_OFF + qb * C::TILE_BYTES + b * C::BOX_BYTES, &tmq,
                                q_full(qb), b * 64, w.qtile * TILE_M, w.bh);
                ++q_it;
                for (int j = 0; j < w.n_tiles; ++j) {
                    const int kt = static_cast<int>(args.tiles[w.tile_begin + j] & TILE_INDEX_MASK);
                    const int st = kv_it % S;
                    const uint32_t ph = (kv_it / S) & 1;
                    mbar_wait(kv_empty(st), ph ^ 1);
                    mbar_arrive_expect_tx(k_full(st), C::TILE_BYTES);
#pragma unroll
                    for (int b = 0; b < C::BOXES; ++b)
                        tma_load_3d(sbase + C::K_OFF + st * C::TILE_BYTES + b * C::BOX_BYTES, &tmk,
                                    k_full(st), b * 64, kt * TILE_N, w.bh);
                    mbar_arrive_expect_tx(v_full(st), C::TILE_BYTES);
#pragma unroll
                    for (int b = 0; b < C::BOXES; ++b)
                        tma_load_3d(sbase + C::V_OFF + st * C::TILE_BYTES + b * C::BOX_BYTES, &tmv,
                                    v_full(st), b * 64, kt * TILE_N, w.bh);
                    ++kv_it;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        if (lane == 0) {
            constexpr uint32_t IDESC_S = idesc_bf16_f32(128, 128, false);
            constexpr uint32_t IDESC_O = idesc_bf16_f32(128, D, true);
            uint32_t kv_it = 0, q_it = 0, g = 0;
            for (int it = it0; it < it1; ++it) {
                const WorkItem w = args.items[it];
                if (w.flags & ITEM_COPY)
                    continue;
                const int qb = q_it & 1;
                mbar_wait(q_full(qb), (q_it >> 1) & 1);
                tc_fence_after();
                const uint32_t q_addr = sbase + C::Q_OFF + qb * C::TILE_BYTES;
                const int n = w.n_tiles;
                for (int j = 0; j <= n; ++j) {
                    if (j < n) {
                        // S_j = Q K_j^T  (M=128, N=128, K=D in steps of 16)
                        const uint32_t gj = g + j;
                        const int sb = gj & 1;
                        const uint32_t kv = kv_it + j;
                        const int st = kv % S;
                        mbar_wait(k_full(st), (kv / S) & 1);
                        tc_fence_after();
                        const uint32_t k_addr = sbase + C::K_OFF + st * C::TILE_BYTES;
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint32_t off = (kk >> 2) * C::BOX_BYTES + (kk & 3) * 32;
                            const uint64_t ad = smem_desc_sw128(q_addr + off, 16, 1024);
                            const uint64_t bd = smem_desc_sw128(k_addr + off, 16, 1024);
                            mma_bf16_ss(tmem + s_col(sb), ad, bd, IDESC_S, kk > 0 ? 1u : 0u);
                        }
                        mma_commit(s_full(sb));
                        if (j == n - 1)
                            mma_commit(q_empty(qb));
                    }
                    if (j >= 1) {
                        // O += P_{j-1} V_{j-1}  (M=128, N=D, K=128 keys in steps of 16)
                        const uint32_t gp = g + j - 1;
                        const int sb = gp & 1;
                        const uint32_t kv = kv_it + j - 1;
                        const int st = kv % S;
                        mbar_wait(p_full(sb), (gp >> 1) & 1);
                        mbar_wait(v_full(st), (kv / S) & 1);
                        tc_fence_after();
                        const uint32_t v_addr = sbase + C::V_OFF + st * C::TILE_BYTES;
#pragma unroll
                        for (int kk = 0; kk < 128 / 16; ++kk) {
                            const uint64_t bd = smem_desc_sw128(v_addr + kk * 2048, C::BOX_BYTES, 1024);
                            mma_bf16_ts(tmem + C::O_COL, tmem + s_col(sb) + kk * 8, bd, IDESC_O,
                                        (j > 1 || kk > 0) ? 1u : 0u);
                        }
                        mma_commit(kv_empty(st));
                        mma_commit(pv_done(sb));
                    }
                }
                g += n;
                kv_it += n;
                ++q_it;
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ softmax warpgroup
        const int wq = warp & 3;
        const int r = wq * 32 + lane;
        const uint32_t lrow = static_cast<uint32_t>(wq * 32) << 16;
        const float sl2 = args.scale_log2;
        const int N = args.n;
        uint32_t g = 0;
        for (int it = it0; it < it1; ++it) {
            const WorkItem w = args.items[it];
            const int row = w.qtile * TILE_M + r;
            if (w.flags & ITEM_COPY) {
                // Cached head: out <- stored slot, 16 B per thread-step.
                const int rows = min(TILE_M, N - w.qtile * TILE_M);
                const size_t base = (static_cast<size_t>(w.bh) * N + static_cast<size_t>(w.qtile) * TILE_M) * D;
                const uint4* src = reinterpret_cast<const uint4*>(args.cache + base);
                uint4* dst = reinterpret_cast<uint4*>(args.out + base);
                const int nvec = rows * D / 8;
                for (int i = r; i < nvec; i += 128)
                    dst[i] = src[i];
                continue;
            }
            const uint8_t* mask = args.masks + w.mask_off;
            float m_ref = -INFINITY;
            float l = 0.f;
            for (int j = 0; j < w.n_tiles; ++j, ++g) {
                const int sb = g & 1;
                const uint32_t word = args.tiles[w.tile_begin + j];
                mbar_wait(s_full(sb), (g >> 1) & 1);
                tc_fence_after();
                float s[128];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    tmem_ld32(tmem + lrow + s_col(sb) + 32 * c, reinterpret_cast<uint32_t*>(s) + 32 * c);
                tmem_ld_wait();
                if (word & TILE_PARTIAL) {
                    uint32_t vm[4];
                    tile_valid_bits(args, mask, row, static_cast<int>(word & TILE_INDEX_MASK) * TILE_N, vm);
#pragma unroll
                    for (int c = 0; c < 128; ++c)
                        if (!((vm[c >> 5] >> (c & 31)) & 1u))
                            s[c] = -INFINITY;
                }
                float m0 = s[0], m1 = s[1], m2 = s[2], m3 = s[3];
#pragma unroll
                for (int c = 4; c < 128; c += 4) {
                    m0 = fmaxf(m0, s[c]);
                    m1 = fmaxf(m1, s[c + 1]);
                    m2 = fmaxf(m2, s[c + 2]);
                    m3 = fmaxf(m3, s[c + 3]);
                }
                const float mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * sl2;
                float factor = 1.f;
                bool need = false;
                if (j == 0) {
                    m_ref = mx;
                } else if (mx > m_ref + 8.f) {
                    factor = (m_ref == -INFINITY) ? 0.f : ex2_approx(m_ref - mx);
                    m_ref = mx;
                    need = true;
                }
                l *= factor;
                if (__any_sync(0xFFFFFFFFu, need)) {
                    // O (through PV_{g-1}) must be final before rescaling it.
                    const uint32_t gp = g - 1;
                    mbar_wait(pv_done(gp & 1), (gp >> 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tmem + lrow + C::O_COL + 32 * c, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
                        tmem_st32(tmem + lrow + C::O_COL + 32 * c, o);
                    }
                    tmem_st_wait();
                }
                const float msub = (m_ref == -INFINITY) ? 0.f : m_ref;
                float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float p0 = ex2_approx(fmaf(s[32 * c + 2 * i], sl2, -msub));
                        const float p1 = ex2_approx(fmaf(s[32 * c + 2 * i + 1], sl2, -msub));
                        sum0 += p0;
                        sum1 += p1;
                        pk[i] = pack_bf16x2(p0, p1);
                    }
                    tmem_st16(tmem + lrow + s_col(sb) + 16 * c, pk);
                }
                l += sum0 + sum1;
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(p_full(sb));
            }
            // ---- epilogue: O / l -> bf16 -> out (+ cache slot)
            const uint32_t gp = g - 1;
            mbar_wait(pv_done(gp & 1), (gp >> 1) & 1);
            tc_fence_after();
            const float inv = 1.f / l;
            const bool valid = row < N;
            const size_t off = (static_cast<size_t>(w.bh) * N + row) * D;
            uint4* orow = reinterpret_cast<uint4*>(args.out + off);
            uint4* crow = (w.flags & ITEM_COMMIT) && args.cache
                              ? reinterpret_cast<uint4*>(args.cache + off)
                              : nullptr;
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tmem + lrow + C::O_COL + 32 * c, o);
                tmem_ld_wait();
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    pk[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
                if (valid) {
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        const uint4 val = make_uint4(pk[4 * v4], pk[4 * v4 + 1], pk[4 * v4 + 2], pk[4 * v4 + 3]);
                        orow[4 * c + v4] = val;
                        if (crow)
                            crow[4 * c + v4] = val;
                    }
                }
            }
            tc_fence_before();
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2)
        tmem_dealloc(tmem, C::TMEM_COLS);
}

template __global__ void attn_fwd_sm100<64>(const __grid_constant__ CUtensorMap,
                                            const __grid_constant__ CUtensorMap,
                                            const __grid_constant__ CUtensorMap, const AttnArgs);
template __global__ void attn_fwd_sm100<128>(const __grid_constant__ CUtensorMap,
                                             const __grid_constant__ CUtensorMap,
                                             const __grid_constant__ CUtensorMap, const AttnArgs);

// Host-side launcher (called from dfa2c.cpp).
cudaError_t launch_attn(int d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                        const AttnArgs& args, int grid, cudaStream_t stream) {
    if (d == 128) {
        using C = Cfg<128>;
        static bool init = false;
        if (!init) {
            cudaFuncSetAttribute(attn_fwd_sm100<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
            init = true;
        }
        attn_fwd_sm100<128><<<grid, 256, C::SMEM_BYTES, stream>>>(tq, tk, tv, args);
    } else {
        using C = Cfg<64>;
        static bool init = false;
        if (!init) {
            cudaFuncSetAttribute(attn_fwd_sm100<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
            init = true;
        }
        attn_fwd_sm100<64><<<grid, 256, C::SMEM_BYTES, stream>>>(tq, tk, tv, args);
    }
    return cudaGetLastError();
}

}  // namespace dfa2k
