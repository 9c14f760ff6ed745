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
// Structure: persistent, one CTA per SM, static LPT work list (dfa2c.cpp).
// A work item is a PAIR of 128-row query tiles (lanes A, B) of one head
// sharing one K/V stream (the union of their mask rows, ascending key order).
//   warp 0      TMA producer: Q_A/Q_B, K ring (runs ahead), V ring
//   warp 1      tcgen05 issuer, per union tile u and lane L:
//                 [wait P_L(u-1)] O_L += P_L V(u-1)   (TS: P from TMEM)
//                 S_L = Q_L K(u)^T                      (SS, into TMEM)
//               so one lane's MMAs overlap the other lane's softmax.
//               d = 64: P has its own TMEM columns, S_L(u) is issued first
//               (it waits only for the softmax to have read S_L(u-1)), and
//               warp 1 issues lane A's MMAs, warp 3 lane B's.
//   warp 2      TMEM allocator
//   warps 4-7   softmax lane A, warps 8-11 softmax lane B: one query row per
//               thread; S read from TMEM twice (row max, then exp2 -> bf16 P
//               written back over S), lazy rescale (threshold 2^8) of O in
//               TMEM, part of the exp2s on the FMA pipe (Cody-Waite +
//               degree-3 polynomial) to unload MUFU; epilogue O/l -> bf16 ->
//               out (+ cache slot); Cached heads' copy items.
// TMEM (512 cols), d=128: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512), P over S;
//   d=64: S_A, S_B as above, O_A [256,320) O_B [320,384) P_A [384,448) P_B [448,512)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>

#include "attn_types.h"
#include "sm100_ptx.cuh"

namespace dfa2k {

#ifndef DFA2_SEP_P64
#define DFA2_SEP_P64 1
#endif
#ifndef DFA2_SPLIT_MMA64
#define DFA2_SPLIT_MMA64 1
#endif
#ifndef DFA2_SPLIT_MMA128
#define DFA2_SPLIT_MMA128 0
#endif

template <int D>
struct Cfg {
#ifndef DFA2_KSTAGES128
#define DFA2_KSTAGES128 2
#endif
    // Q pair buffers: at d=64 a second one lets the next item's Q load while
    // the current item still computes (short arrow items switch often); at
    // d=128 shared memory has no room for it.
    static constexpr int QBUF = D == 128 ? 1 : 2;
    static constexpr int KSTAGES = D == 128 ? DFA2_KSTAGES128 : 4;
    static constexpr int VSTAGES = D == 128 ? 2 : 4;
    static constexpr int BOXES = D / 64;                       // 128-byte column boxes
    static constexpr uint32_t BOX_BYTES = 128u * 128u;         // 128 rows x 128 B
    static constexpr uint32_t TILE_BYTES = BOXES * BOX_BYTES;  // one Q, K or V tile
    static constexpr uint32_t Q_OFF = 0;                       // [QBUF] x (Q_A, Q_B)
    static constexpr uint32_t K_OFF = QBUF * 2 * TILE_BYTES;
    static constexpr uint32_t V_OFF = K_OFF + KSTAGES * TILE_BYTES;
    // two 16 KB staging boxes (128 rows x 64 cols bf16, 128B swizzle), one per
    // lane: O epilogue and cached-head copies go smem -> TMA bulk store
    static constexpr uint32_t STG_OFF = V_OFF + VSTAGES * TILE_BYTES;
    static constexpr uint32_t BAR_OFF = STG_OFF + 2 * BOX_BYTES;
    // d = 64: S 2x128 + O 2x64 columns leave 128 TMEM columns, so P gets
    // its own 64 columns per lane and a lane's next S no longer waits for
    // the PV that reads the current P (S_L(u+1) is issued as soon as the
    // softmax has read S_L(u)). At d = 128 P overwrites S in place.
    static constexpr bool SEP_P = D == 64 && DFA2_SEP_P64;
    // With P separate, each lane gets its own MMA-issuing warp (warp 1 lane
    // A, warp 3 lane B): a lane's S and PV then wait only on that lane.
    static constexpr bool SPLIT_MMA = (SEP_P && DFA2_SPLIT_MMA64) || (D == 128 && DFA2_SPLIT_MMA128);
    // copy tail: the CTA's trailing Cached-head copies run after all its
    // compute, through the whole freed window [0, 14 boxes): 7 per lane
    static constexpr int RING = 7;
    static_assert(2 * RING * BOX_BYTES <= BAR_OFF, "copy ring must fit below the barriers");
    static constexpr int NBARS = 2 * QBUF + 2 * KSTAGES + 2 * VSTAGES + 14 + 2 * RING;
    // The dynamic window starts 1024-aligned (the 1 KB system reservation
    // precedes it); the kernel traps otherwise, so no alignment slack.
    // HALVES items: per lane and row, the (reference max, row sum) exchanged
    // between the two lanes in the epilogue
    static constexpr uint32_t XCHG_OFF = BAR_OFF + NBARS * 8 + 16;
    static constexpr uint32_t SMEM_BYTES = XCHG_OFF + 2 * 2 * TILE_M * 4;
    static_assert(SMEM_BYTES <= 232448, "shared memory budget");
    static constexpr uint32_t TMEM_COLS = 512;
    static constexpr int THREADS = 384;
};

// Every EMU-th column pair of a 32-column chunk computes exp2 on the FMA
// pipe instead of MUFU (0 disables), per head dim: at d=64 the MMAs of a
// tile take half as long as at d=128 while the exp count is the same.
#ifndef DFA2_EMU_EVERY64
#define DFA2_EMU_EVERY64 3
#endif
#ifndef DFA2_EMU_EVERY128
#define DFA2_EMU_EVERY128 8
#endif

#ifndef DFA2_TRACE
#define DFA2_TRACE 0
#endif
// d = 128: commit V(u-1)'s "empty" barrier right after its last PV instead of
// after the step's last S MMA (the next V load then starts ~one S earlier)
#ifndef DFA2_EARLY_VFREE
#define DFA2_EARLY_VFREE 1
#endif

// Row max: keys 0..63 are loaded and reduced (8 chains) while keys 64..127
// are still in flight from TMEM (1), or everything loads first (0), per head
// dim (interleaved A/B: split 1% faster on FLUX68, unsplit 1.3-3.5% faster
// on SD3 layers). DFA2_SPLITLD sets both.
#ifdef DFA2_SPLITLD
#define DFA2_SPLITLD64 DFA2_SPLITLD
#define DFA2_SPLITLD128 DFA2_SPLITLD
#endif
#ifndef DFA2_SPLITLD64
#define DFA2_SPLITLD64 0
#endif
#ifndef DFA2_SPLITLD128
#define DFA2_SPLITLD128 1
#endif
template <int D>
constexpr bool SPLITLD = D == 64 ? DFA2_SPLITLD64 : DFA2_SPLITLD128;
// Keys 0..63 stay in registers from the max pass to their exps (1), or are
// re-read from TMEM after the keys-64..127 half (0), per head dim. Keeping
// them needs the softmax warpgroups' register budget raised (setmaxnreg,
// DFA2_REGS_*). Interleaved A/B (tools/ab_interleaved.py): d = 128 FLUX68
// -2.2%, all-Full -2.1%; d = 64 SD3 arrows +1.5% (so off there).
// Hardware warpgroup -> role (warpgroups 0,1,2 in hardware order):
// 0: control, lane A, lane B (lane B above lane A, control lowest);
// 1: lane A, lane B, control (control highest); 2: control, lane B, lane A;
// 3: lane B, lane A, control. Interleaved A/B: map 1 is 2% faster at d = 64
// (SD3), 2% slower at d = 128 than map 0.
// logical control warps of the producer and the TMEM allocator (0 and 2;
// the MMA issuers are 1, and 3 at d = 64): which SMSP each busy role sits on
#ifndef DFA2_PRODUCER_WARP
#define DFA2_PRODUCER_WARP 0
#endif
#ifndef DFA2_ALLOC_WARP
#define DFA2_ALLOC_WARP 2
#endif
#ifndef DFA2_WARPMAP64
#define DFA2_WARPMAP64 1
#endif
#ifndef DFA2_WARPMAP128
#define DFA2_WARPMAP128 0
#endif
template <int D>
constexpr int WARPMAP = D == 64 ? DFA2_WARPMAP64 : DFA2_WARPMAP128;
#ifndef DFA2_KEEPLO128
#define DFA2_KEEPLO128 1
#endif
#ifndef DFA2_KEEPLO64
#define DFA2_KEEPLO64 0
#endif
template <int D>
constexpr bool KEEPLO = D == 64 ? DFA2_KEEPLO64 : DFA2_KEEPLO128;
#ifndef DFA2_REGS_SOFTMAX
#define DFA2_REGS_SOFTMAX 216
#endif
#ifndef DFA2_REGS_OTHER
#define DFA2_REGS_OTHER 72
#endif
#ifndef DFA2_REGS_SOFTMAX64
#define DFA2_REGS_SOFTMAX64 DFA2_REGS_SOFTMAX
#endif
#ifndef DFA2_REGS_OTHER64
#define DFA2_REGS_OTHER64 DFA2_REGS_OTHER
#endif
// setmaxnreg split between the control and softmax warpgroups: always with
// KEEPLO, else on request (DFA2_REGSPLIT64)
#ifndef DFA2_REGSPLIT64
#define DFA2_REGSPLIT64 0
#endif
template <int D>
constexpr bool REGSPLIT = KEEPLO<D> || (D == 64 && DFA2_REGSPLIT64);
template <int D>
constexpr uint32_t REGS_SOFTMAX = D == 64 ? DFA2_REGS_SOFTMAX64 : DFA2_REGS_SOFTMAX;
template <int D>
constexpr uint32_t REGS_OTHER = D == 64 ? DFA2_REGS_OTHER64 : DFA2_REGS_OTHER;
static_assert(DFA2_REGS_OTHER64 + 2 * DFA2_REGS_SOFTMAX64 <= 3 * 168,
              "setmaxnreg must not ask for more than the CTA's 384 x 168 registers");
static_assert(DFA2_REGS_OTHER + 2 * DFA2_REGS_SOFTMAX <= 3 * 168,
              "setmaxnreg must not ask for more than the CTA's 384 x 168 registers");
// trace[((lane * 4096) + tile) * 8 + slot] = clock64() for CTA 0 (debug builds)
#define DFA2_STAMP(L_, j_, k_)                                                          \
    do {                                                                                \
        if (DFA2_TRACE && DFA2_TRACE != 4 && args.trace && blockIdx.x == 0 && (j_) < 4096) \
            if (DFA2_TRACE == 1 || DFA2_TRACE == 3 || (k_) < 3)                               \
                args.trace[((static_cast<int>(L_) * 4096) + static_cast<int>(j_)) * 8 + (k_)] = clock64(); \
    } while (0)

// Read-once / write-once TMA traffic (Q tiles, cached slots read for copies,
// outputs and cache commits) is tagged L2::evict_first so the K/V tiles that
// every query-tile pair of a head re-streams keep their L2 residency.
#ifndef DFA2_L2_HINTS
#define DFA2_L2_HINTS 1
#endif

namespace {

// the producer / MMA-issue warps' barrier waits (DFA2_CTL_SLEEP: hardware
// sleep until the phase completes, so they take no issue slots from the
// softmax warps of their SMSP while they wait)
#ifndef DFA2_CTL_SLEEP
#define DFA2_CTL_SLEEP 0
#endif
__device__ __forceinline__ void mbar_wait_ctl(uint32_t bar, uint32_t parity) {
    if (DFA2_CTL_SLEEP)
        mbar_wait_sleep(bar, parity);
    else
        mbar_wait(bar, parity);
}

__device__ __forceinline__ void tma_load_q(uint32_t dst, const CUtensorMap* map, uint32_t bar, int32_t c0, int32_t c1,
                                           int32_t c2) {
    if (DFA2_L2_HINTS)
        tma_load_3d_hint(dst, map, bar, c0, c1, c2, policy_evict_first());
    else
        tma_load_3d(dst, map, bar, c0, c1, c2);
}
__device__ __forceinline__ void tma_store_o(const CUtensorMap* map, uint32_t src, int32_t c0, int32_t c1, int32_t c2) {
    if (DFA2_L2_HINTS)
        tma_store_3d_hint(map, src, c0, c1, c2, policy_evict_first());
    else
        tma_store_3d(map, src, c0, c1, c2);
}

__device__ __forceinline__ uint32_t s_col(int lane) { return lane ? 128u : 0u; }
template <int D>
__device__ __forceinline__ uint32_t o_col(int lane) {
    return D == 64 ? 256u + 64u * lane : (lane ? 384u : 256u);
}
// P (bf16 pairs, 64 columns): its own columns at d = 64, else over S
template <int D>
__device__ __forceinline__ uint32_t p_col(int lane) {
    return D == 64 ? 384u + 64u * lane : s_col(lane);
}
// column offset of the P of keys 64..127 within the lane's P columns
template <int D>
constexpr uint32_t P_HI = D == 64 ? 32u : 64u;

#ifndef DFA2_SUM_CHAINS
#define DFA2_SUM_CHAINS 1
#endif
#ifndef DFA2_POLY_NOSEL
#define DFA2_POLY_NOSEL 1
#endif
// Two exp2s on the FMA/ALU pipes with packed fp32x2 arithmetic: x = j + f,
// j = floor(x) by the round-down magic-number add, 2^f by a degree-3
// minimax polynomial (max rel. error 8.6e-5, far below the bf16 rounding P
// is stored with), the exponent added as an integer; 0 below 2^-126, so
// masked (-inf) scores still give P == 0 exactly.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
    const float2 xc = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
    const float2 t = __fadd2_rd(xc, make_float2(12582912.f, 12582912.f));
    const float2 tm = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));  // floor(x)
    const float2 f = __ffma2_rn(tm, make_float2(-1.f, -1.f), xc);             // x - floor(x)
    float2 p = __ffma2_rn(make_float2(0.0770652f, 0.0770652f), f, make_float2(0.227647f, 0.227647f));
    p = __ffma2_rn(p, f, make_float2(0.69511634f, 0.69511634f));
    p = __ffma2_rn(p, f, make_float2(1.0f, 1.0f));
#if DFA2_POLY_NOSEL
    // no select: at the clamp (x <= -127) t = -127 and f = 0, so p = 1.0 and
    // the exponent add wraps 0x3F800000 + (-127 << 23) to exactly +0.0;
    // (-127, -126) gives denormals below 1.2e-38 (P rounds to bf16 anyway)
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
#else
    return make_float2(x.x < -126.f ? 0.f : __uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       x.y < -126.f ? 0.f : __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
#endif
}

// Per-row 128-column validity bitmap for a partial tile: key < N and the
// (query block, key block) pair active in the head's block mask.
__device__ __forceinline__ void tile_valid_bits(const AttnArgs& a, const uint8_t* mask, int row, int k0,
                                                uint32_t (&vm)[4]) {
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


// Partial tiles: overwrite the masked scores in TMEM with -inf before the
// common softmax pass (only tiles with block size != 128 or a ragged tail).
__device__ __forceinline__ void mask_tile_in_tmem(uint32_t sc, const uint32_t (&vm)[4]) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t s[32];
        tmem_ld32(sc + 32 * c, s);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (!((vm[c] >> i) & 1u))
                s[i] = 0xFF800000u;  // -inf
        tmem_st32(sc + 32 * c, s);
    }
    tmem_st_wait();
}

// One S tile of one lane. All 128 scores of the thread's row are loaded
// once (4 x tcgen05.ld, one wait): row max, lazy O rescale, then
// P = exp2(s*scale - m) as bf16 written back into the lane's S columns:
// keys 64..127 -> cols [64,96) (a region whose scores are already in
// registers) and signalled on p_half, so the MMA warp starts the first half
// of O += P V while keys 0..63 -> cols [0,32) are still being computed
// (signalled on p_full). Masked scores arrive as -inf and give P == 0
// exactly (MUFU ex2(-inf) = 0; the polynomial path selects 0 below 2^-126).
template <int D>
__device__ __forceinline__ void softmax_half(const uint32_t* s, float2 scale2, float2 neg_m, float2& sum,
                                             uint32_t dst) {
    constexpr int EMU = D == 64 ? DFA2_EMU_EVERY64 : DFA2_EMU_EVERY128;
    // DFA2_SUM_CHAINS independent row-sum accumulators (the FADD2 chain is
    // otherwise one dependency through every pair of the half)
    constexpr int NS = DFA2_SUM_CHAINS;
    float2 acc[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j)
        acc[j] = j == 0 ? sum : make_float2(0.f, 0.f);
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float2 x = __ffma2_rn(
                make_float2(__uint_as_float(s[32 * cc + 2 * i]), __uint_as_float(s[32 * cc + 2 * i + 1])), scale2,
                neg_m);
            float2 p;
            if (EMU > 0 && (i % (EMU > 0 ? EMU : 1)) == EMU - 1) {
                p = ex2_poly2(x);
            } else {
                p = make_float2(ex2_approx(x.x), ex2_approx(x.y));
            }
            acc[i % NS] = __fadd2_rn(acc[i % NS], p);
            pk[i] = pack_bf16x2(p.x, p.y);
        }
        tmem_st16(dst + 16 * cc, pk);
    }
#pragma unroll
    for (int j = 1; j < NS; ++j)
        acc[0] = __fadd2_rn(acc[0], acc[j]);
    sum = acc[0];
}

// DFA2_TRACE == 2: in-softmax stamps (slots 3..7 of the lane's trace rows)
#define DFA2_SSTAMP(k_)                                        \
    do {                                                       \
        if (DFA2_TRACE == 2 && stamp)                          \
            stamp[k_] = clock64();                             \
    } while (0)

// SEP_P (d = 64): P goes to the lane's own columns `pc`; bar_sfree is
// signalled once S is fully in registers (the lane's next S may overwrite
// it), and before the first P store / O rescale the lane waits for the PV
// of its previous tile (bar_pfree, parity pf_parity; < 0: no earlier tile).
template <int D>
__device__ __forceinline__ void softmax_tile(uint32_t sc, uint32_t oc, float sl2, float& m_ref, float& l,
                                             bool first, uint32_t bar_half, uint32_t bar_full, uint32_t pc,
                                             uint32_t bar_sfree, uint32_t bar_pfree, int pf_parity,
                                             long long* stamp = nullptr) {
    constexpr bool SEP = Cfg<D>::SEP_P;
#ifdef DFA2_FAKE_SOFTMAX  // timing experiment only: P is whatever S was (garbage)
    if (SEP) {
        tc_fence_before();
        mbar_arrive(bar_sfree);
    }
    if (SEP && pf_parity >= 0) mbar_wait(bar_pfree, static_cast<uint32_t>(pf_parity));
    tc_fence_before();
    mbar_arrive(bar_half);
    mbar_arrive(bar_full);
    l = 1.f;
    return;
#endif
    bool pfree_done = !SEP || pf_parity < 0;
    auto wait_pfree = [&] {
        if (!pfree_done) {
            mbar_wait(bar_pfree, static_cast<uint32_t>(pf_parity));
            tc_fence_after();
            pfree_done = true;
        }
    };
    uint32_t hi[64];
    float mx;
    uint32_t lo[64];  // keys 0..63 (re-loaded below unless KEEPLO<D>)
    {
        if constexpr (SPLITLD<D>) {
        // keys 0..63 first; their max chains run while keys 64..127 load
        tmem_ld32(sc, lo);
        tmem_ld32(sc + 32, lo + 32);
        tmem_ld_wait();
        tmem_ld32(sc + 64, hi);
        tmem_ld32(sc + 96, hi + 32);
        float mm[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
            mm[j] = fmaxf(__uint_as_float(lo[2 * j]), __uint_as_float(lo[2 * j + 1]));
#pragma unroll
        for (int c = 16; c < 64; c += 16)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                mm[j] = fmaxf(mm[j], fmaxf(__uint_as_float(lo[c + 2 * j]), __uint_as_float(lo[c + 2 * j + 1])));
        tmem_ld_wait();
        DFA2_SSTAMP(3);
#pragma unroll
        for (int c = 0; c < 64; c += 16)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                mm[j] = fmaxf(mm[j], fmaxf(__uint_as_float(hi[c + 2 * j]), __uint_as_float(hi[c + 2 * j + 1])));
        mx = fmaxf(fmaxf(fmaxf(mm[0], mm[1]), fmaxf(mm[2], mm[3])), fmaxf(fmaxf(mm[4], mm[5]), fmaxf(mm[6], mm[7]))) *
             sl2;
        } else {
        tmem_ld32(sc, lo);
        tmem_ld32(sc + 32, lo + 32);
        tmem_ld32(sc + 64, hi);
        tmem_ld32(sc + 96, hi + 32);
        tmem_ld_wait();
        DFA2_SSTAMP(3);
        float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 64; c += 4) {  // four independent 3-input max chains
            m0 = fmaxf(m0, fmaxf(__uint_as_float(lo[c]), __uint_as_float(lo[c + 1])));
            m1 = fmaxf(m1, fmaxf(__uint_as_float(hi[c]), __uint_as_float(hi[c + 1])));
            m2 = fmaxf(m2, fmaxf(__uint_as_float(lo[c + 2]), __uint_as_float(lo[c + 3])));
            m3 = fmaxf(m3, fmaxf(__uint_as_float(hi[c + 2]), __uint_as_float(hi[c + 3])));
        }
        mx = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * sl2;
        }
        if (KEEPLO<D> && SEP) {  // S fully in registers: the lane's next S may overwrite it
            tc_fence_before();
            mbar_arrive(bar_sfree);
        }
    }
    // lazy rescale: keep the reference max unless the tile max exceeds it by
    // more than 8 (P <= 2^8 stays exact in fp32 and representable in bf16)
    float factor = 1.f;
    bool need = false;
    if (first) {
        m_ref = mx;
    } else if (mx > m_ref + 8.f) {
        factor = (m_ref == -INFINITY) ? 0.f : ex2_approx(m_ref - mx);
        m_ref = mx;
        need = true;
    }
    l *= factor;
    DFA2_SSTAMP(4);
    if (__any_sync(0xFFFFFFFFu, need)) {
        // O holds every earlier PV of this lane: this S was issued after them,
        // so they completed before s_full fired (SEP_P: S is issued before
        // the previous PV, so wait for that PV explicitly).
        wait_pfree();
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(oc + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i)
                o[i] = __float_as_uint(__uint_as_float(o[i]) * factor);
            tmem_st32(oc + 32 * c, o);
        }
    }
    const float msub = (m_ref == -INFINITY) ? 0.f : m_ref;
    const float2 scale2 = make_float2(sl2, sl2);
    const float2 neg_m = make_float2(-msub, -msub);
    float2 sum = make_float2(0.f, 0.f);
    // keys 64..127 from registers -> P cols [64,96) (SEP_P: [32,64) of P): the
    // MMA warp starts on them
    wait_pfree();
    softmax_half<D>(hi, scale2, neg_m, sum, (SEP ? pc : sc) + P_HI<D>);
    DFA2_SSTAMP(5);
    tmem_st_wait();
    tc_fence_before();
    mbar_arrive(bar_half);
    DFA2_SSTAMP(6);
    // keys 0..63 re-read (cols [0,64) untouched so far) -> cols [0,32)
    if (!KEEPLO<D>) {
        tmem_ld32(sc, lo);
        tmem_ld32(sc + 32, lo + 32);
        tmem_ld_wait();
    }
    if (SEP && !KEEPLO<D>) {  // S fully read: the lane's next S may overwrite it
        tc_fence_before();
        mbar_arrive(bar_sfree);
    }
    DFA2_SSTAMP(7);
    softmax_half<D>(lo, scale2, neg_m, sum, SEP ? pc : sc);
    tmem_st_wait();
    tc_fence_before();
    mbar_arrive(bar_full);
    l += sum.x + sum.y;
}

// Flat cursor over the union tiles of a CTA's compute items.
struct Cursor {
    int it;
    int j;
};

__device__ __forceinline__ void skip_copies(const WorkItem* items, int it1, Cursor& c) {
    while (c.it < it1 && ((items[c.it].flags & ITEM_COPY) || items[c.it].n_tiles == 0)) {
        ++c.it;
        c.j = 0;
    }
}

__device__ __forceinline__ void advance(const WorkItem* items, int it1, Cursor& c) {
    if (++c.j >= items[c.it].n_tiles) {
        ++c.it;
        c.j = 0;
        skip_copies(items, it1, c);
    }
}

}  // namespace

template <int D>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_sm100(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                   const __grid_constant__ CUtensorMap tmv, const __grid_constant__ CUtensorMap tmo,
                   const __grid_constant__ CUtensorMap tmc, const AttnArgs args,
                   const __grid_constant__ PeerMaps peers) {
    using C = Cfg<D>;
    constexpr int KS = C::KSTAGES;
    constexpr int VS = C::VSTAGES;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    if (sbase & 1023u)
        __trap();

    // Logical warp roles: 0 producer, 1 (and 3 at d = 64) MMA issue, 2 TMEM
    // allocation, 4..7 softmax lane A, 8..11 lane B. The SMSP scheduler
    // favours the highest warp id among eligible warps, so which hardware
    // warpgroup takes which role sets the issue priority between the MMA
    // issuer and the two softmax warps sharing its SMSP (WARPMAP<D>). The
    // TMEM lane quarter of a softmax warp (hardware warp % 4) equals logical
    // warp % 4 under every map.
    const int hg = static_cast<int>(threadIdx.x >> 7);
    constexpr int WM = WARPMAP<D>;
    const int lg = WM == 0 ? hg : WM == 1 ? (hg + 1) % 3 : WM == 2 ? (hg == 0 ? 0 : 3 - hg) : 2 - hg;
    const int warp = lg * 4 + static_cast<int>((threadIdx.x >> 5) & 3);
    const int lane = threadIdx.x & 31;

    const uint32_t bars = sbase + C::BAR_OFF;
    constexpr int QB = 2 * C::QBUF;
    auto q_full = [&](int s) { return bars + 8u * s; };
    auto q_empty = [&](int s) { return bars + 8u * (C::QBUF + s); };
    auto k_full = [&](int s) { return bars + 8u * (QB + s); };
    auto k_empty = [&](int s) { return bars + 8u * (QB + KS + s); };
    auto v_full = [&](int s) { return bars + 8u * (QB + 2 * KS + s); };
    auto v_empty = [&](int s) { return bars + 8u * (QB + 2 * KS + VS + s); };
    auto s_full = [&](int l) { return bars + 8u * (QB + 2 * KS + 2 * VS + l); };
    auto p_full = [&](int l) { return bars + 8u * (QB + 2 + 2 * KS + 2 * VS + l); };
    auto o_full = [&](int l) { return bars + 8u * (QB + 4 + 2 * KS + 2 * VS + l); };
    auto p_half = [&](int l) { return bars + 8u * (QB + 6 + 2 * KS + 2 * VS + l); };
    auto c_full = [&](int l) { return bars + 8u * (QB + 8 + 2 * KS + 2 * VS + l); };  // copy-box landed
    auto s_free = [&](int l) { return bars + 8u * (QB + 10 + 2 * KS + 2 * VS + l); };  // SEP_P: S read
    auto p_free = [&](int l) { return bars + 8u * (QB + 12 + 2 * KS + 2 * VS + l); };  // SEP_P: PV done
    auto ring_full = [&](int l, int i) { return bars + 8u * (QB + 14 + 2 * KS + 2 * VS + l * C::RING + i); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::BAR_OFF + C::NBARS * 8);

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::QBUF; ++s) {
            mbar_init(q_full(s), 1);
            mbar_init(q_empty(s), C::SPLIT_MMA ? 2 : 1);
        }
        for (int s = 0; s < KS; ++s) {
            mbar_init(k_full(s), 1);
            mbar_init(k_empty(s), C::SPLIT_MMA ? 2 : 1);
        }
        for (int s = 0; s < VS; ++s) {
            mbar_init(v_full(s), 1);
            mbar_init(v_empty(s), C::SPLIT_MMA ? 2 : 1);
        }
        for (int l = 0; l < 2; ++l) {
            mbar_init(s_full(l), 1);
            mbar_init(p_full(l), 128);
            mbar_init(p_half(l), 128);
            mbar_init(c_full(l), 1);
            mbar_init(o_full(l), 1);
            mbar_init(s_free(l), 128);
            mbar_init(p_free(l), 1);
            for (int i = 0; i < C::RING; ++i)
                mbar_init(ring_full(l, i), 1);
        }
        fence_mbar_init();
    }
    if (warp == DFA2_PRODUCER_WARP && lane == 0) {
        tma_prefetch_desc(&tmq);
        tma_prefetch_desc(&tmk);
        tma_prefetch_desc(&tmv);
        tma_prefetch_desc(&tmo);
        tma_prefetch_desc(&tmc);
    }
    if (warp == DFA2_ALLOC_WARP) {
        tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // DFA2_TRACE == 4: per-CTA start / end (globaltimer ns) and the end of
    // each lane's softmax work, to see the schedule's tail
    auto gtime = [] {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return static_cast<long long>(t);
    };
    if (DFA2_TRACE == 4 && args.trace && threadIdx.x == 0)
        args.trace[blockIdx.x * 4 + 0] = gtime();

    const int it0 = args.cta_begin[blockIdx.x];
    const int it1 = args.cta_begin[blockIdx.x + 1];
    const WorkItem* items = args.items;

    if (warp < 4) {
    // warpgroup 0 (producer / MMA issue) hands registers to the softmax warpgroups
    if (REGSPLIT<D>)
        regs_dec<REGS_OTHER<D>>();
    if (warp == DFA2_PRODUCER_WARP) {
        // ------------------------------------------------ TMA producer
        // The whole warp walks the schedule (warp-uniform control flow keeps
        // coordinates in uniform registers); one elected lane issues.
        {
            Cursor kc{it0, 0}, vc{it0, 0};
            skip_copies(items, it1, kc);
            skip_copies(items, it1, vc);
            uint32_t kcount = 0, vcount = 0, qcount = 0, vitem = 0;
            while (vc.it < it1) {
                // K runs up to KS-1 tiles ahead of V, and into a later item
                // only while that item's Q pair buffer is free: at most QBUF
                // items ahead of V's item (each Q buffer is freed by its item's
                // last S, which needs that item's V stream)
                while (kc.it < it1 && kcount < vcount + (KS - 1) &&
                       !(kc.j == 0 && qcount - vitem >= static_cast<uint32_t>(C::QBUF))) {
                    const WorkItem& w = items[kc.it];
                    if (kc.j == 0) {
                        const int qs = qcount % C::QBUF;
                        const uint32_t qaddr = sbase + C::Q_OFF + qs * 2 * C::TILE_BYTES;
                        mbar_wait_ctl(q_empty(qs), ((qcount / C::QBUF) & 1) ^ 1);
                        const int nq = w.qtile_b >= 0 ? 2 : 1;
                        if (elect_one()) {
                            mbar_arrive_expect_tx(q_full(qs), nq * C::TILE_BYTES);
#pragma unroll
                            for (int b = 0; b < C::BOXES; ++b) {
                                tma_load_q(qaddr + b * C::BOX_BYTES, &tmq, q_full(qs), b * 64, w.qtile_a * TILE_M,
                                           w.bh);
                                if (nq == 2)
                                    tma_load_q(qaddr + C::TILE_BYTES + b * C::BOX_BYTES, &tmq, q_full(qs), b * 64,
                                                w.qtile_b * TILE_M, w.bh);
                            }
                        }
                        __syncwarp();
                        ++qcount;
                    }
                    const int kt = static_cast<int>(args.tiles[w.tile_begin + kc.j] & TILE_INDEX_MASK);
                    const int st = kcount % KS;
                    if (DFA2_TRACE == 3 && lane == 0) DFA2_STAMP(2, kcount, 0);
                    mbar_wait_ctl(k_empty(st), ((kcount / KS) & 1) ^ 1);
                    if (DFA2_TRACE == 3 && lane == 0) DFA2_STAMP(2, kcount, 1);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(k_full(st), C::TILE_BYTES);
#pragma unroll
                        for (int b = 0; b < C::BOXES; ++b)
                            tma_load_3d(sbase + C::K_OFF + st * C::TILE_BYTES + b * C::BOX_BYTES, &tmk, k_full(st),
                                        b * 64, kt * TILE_N, w.bh);
                    }
                    __syncwarp();
                    ++kcount;
                    advance(items, it1, kc);
                }
                const WorkItem& w = items[vc.it];
                const int kt = static_cast<int>(args.tiles[w.tile_begin + vc.j] & TILE_INDEX_MASK);
                const int st = vcount % VS;
                if (DFA2_TRACE == 3 && lane == 0) DFA2_STAMP(2, vcount, 2);
                mbar_wait_ctl(v_empty(st), ((vcount / VS) & 1) ^ 1);
                if (DFA2_TRACE == 3 && lane == 0) DFA2_STAMP(2, vcount, 3);
                if (elect_one()) {
                    mbar_arrive_expect_tx(v_full(st), C::TILE_BYTES);
#pragma unroll
                    for (int b = 0; b < C::BOXES; ++b)
                        tma_load_3d(sbase + C::V_OFF + st * C::TILE_BYTES + b * C::BOX_BYTES, &tmv, v_full(st),
                                    b * 64, kt * TILE_N, w.bh);
                }
                __syncwarp();
                ++vcount;
                advance(items, it1, vc);
                if (vc.j == 0)
                    ++vitem;
            }
        }
    } else if (C::SPLIT_MMA && (warp == 1 || warp == 3)) {
        // ------------------------------------------------ per-lane tcgen05 issuer
        // Both warps walk every union tile; a warp arrives on the K / V / Q
        // "empty" barriers (count 2) with a commit after its MMAs, or a plain
        // arrive, once the tile has landed, for tiles its lane does not fold.
        const int L = warp == 1 ? 0 : 1;
        const uint32_t need = L ? TILE_NEED_B : TILE_NEED_A;
        const uint32_t snapb = L ? TILE_SNAP_B : TILE_SNAP_A;
        constexpr uint32_t IDESC_S = idesc_bf16_f32(128, 128, false);
        constexpr uint32_t IDESC_O = idesc_bf16_f32(128, D, true);
        uint32_t kcount = 0, vcount = 0, qcount = 0, pcnt = 0, scount = 0;
        for (int it = it0; it < it1; ++it) {
            const WorkItem w = items[it];
            if ((w.flags & ITEM_COPY) || w.n_tiles == 0)
                continue;
            const int qs = qcount % C::QBUF;
            const uint32_t qbase = sbase + C::Q_OFF + qs * 2 * C::TILE_BYTES;
            mbar_wait_ctl(q_full(qs), (qcount / C::QBUF) & 1);
            tc_fence_after();
            const bool has_lane = L == 0 || w.qtile_b >= 0;
            bool first_pv = true, any_s = false;
            uint32_t prev = 0;
            const int U = w.n_tiles;
            uint32_t word_next = U > 0 ? __ldg(args.tiles + w.tile_begin) : 0u;
            for (int u = 0; u <= U; ++u) {
                // the next step's word is loaded a step ahead (its L2 latency
                // would otherwise sit on the issue path of every step)
                const uint32_t word = word_next;
                word_next = u + 1 < U ? __ldg(args.tiles + w.tile_begin + u + 1) : 0u;
                const int vst = vcount % VS;
                const int kst = kcount % KS;
                auto do_s = [&] {
                if (u < U) {
                    if (word & need) {
                        if (C::SEP_P && scount >= 1) {  // the lane's softmax has read its previous S
                            mbar_wait_ctl(s_free(L), (scount - 1) & 1);
                        }
                        mbar_wait_ctl(k_full(kst), (kcount / KS) & 1);
                        tc_fence_after();
                        const uint64_t qdesc = smem_desc_sw128(qbase + L * C::TILE_BYTES, 16, 1024);
                        const uint64_t kdesc = smem_desc_sw128(sbase + C::K_OFF + kst * C::TILE_BYTES, 16, 1024);
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < D / 16; ++kk) {
                                const uint32_t off = ((kk >> 2) * C::BOX_BYTES + (kk & 3) * 32) >> 4;
                                mma_bf16_ss(tmem + s_col(L), qdesc + off, kdesc + off, IDESC_S, kk > 0 ? 1u : 0u);
                            }
                            mma_commit(s_full(L));
                            mma_commit(k_empty(kst));
                            if (u == U - 1)
                                mma_commit(q_empty(qs));
                        }
                        __syncwarp();
                        ++scount;
                        any_s = true;
                    } else {
                        // the tile must be loaded before this use's arrival, or the
                        // arrival could complete the slot's previous phase
                        mbar_wait_ctl(k_full(kst), (kcount / KS) & 1);
                        if (elect_one()) {
                            mbar_arrive(k_empty(kst));
                            if (u == U - 1) {
                                if (any_s)
                                    mma_commit(q_empty(qs));
                                else
                                    mbar_arrive(q_empty(qs));
                            }
                        }
                        __syncwarp();
                    }
                }
                };
                auto do_pv = [&] {
                if (u >= 1) {
                    if (prev & need) {
                        mbar_wait_ctl(v_full(vst), (vcount / VS) & 1);
                        const uint64_t vdesc = smem_desc_sw128(sbase + C::V_OFF + vst * C::TILE_BYTES, C::BOX_BYTES, 1024);
                        mbar_wait_ctl(p_half(L), pcnt & 1);
                        tc_fence_after();
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 4; kk < 8; ++kk)
                                mma_bf16_ts(tmem + o_col<D>(L), tmem + p_col<D>(L) + P_HI<D> + (kk - 4) * 8,
                                            vdesc + (kk * 2048 >> 4), IDESC_O, (!first_pv || kk > 4) ? 1u : 0u);
                        }
                        __syncwarp();
                        mbar_wait_ctl(p_full(L), pcnt & 1);
                        tc_fence_after();
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                mma_bf16_ts(tmem + o_col<D>(L), tmem + p_col<D>(L) + kk * 8, vdesc + (kk * 2048 >> 4),
                                            IDESC_O, 1u);
                            if (prev & snapb)
                                mma_commit(o_full(L));
                            if (C::SEP_P)
                                mma_commit(p_free(L));
                            mma_commit(v_empty(vst));
                        }
                        __syncwarp();
                        first_pv = false;
                        ++pcnt;
                    } else {
                        mbar_wait_ctl(v_full(vst), (vcount / VS) & 1);
                        if (elect_one())
                            mbar_arrive(v_empty(vst));
                        __syncwarp();
                    }
                }
                };
                if (C::SEP_P) {  // S_L(u) first: it waits only for the softmax to have read S_L(u-1)
                    do_s();
                    do_pv();
                } else {  // P over S: the PV that reads P_L(u-1) goes first
                    do_pv();
                    do_s();
                }
                if (u >= 1)
                    ++vcount;
                if (u < U)
                    ++kcount;
                prev = word;
            }
            if (has_lane) {
                if (elect_one())
                    mma_commit(o_full(L));
                __syncwarp();
            }
            ++qcount;
        }
    } else if (warp == 1) {
        // ------------------------------------------------ tcgen05 issuer
        // Whole warp walks the schedule and waits; one elected lane (the same
        // lane every time, so tcgen05.commit tracks all its MMAs) issues.
        {
            constexpr uint32_t IDESC_S = idesc_bf16_f32(128, 128, false);
            constexpr uint32_t IDESC_O = idesc_bf16_f32(128, D, true);
            uint32_t kcount = 0, vcount = 0, qcount = 0;
            uint32_t pcnt[2] = {0, 0};
            uint32_t scount[2] = {0, 0};
            for (int it = it0; it < it1; ++it) {
                const WorkItem w = items[it];
                if ((w.flags & ITEM_COPY) || w.n_tiles == 0)
                    continue;
                const int qs = qcount % C::QBUF;
                const uint32_t qbase = sbase + C::Q_OFF + qs * 2 * C::TILE_BYTES;
                mbar_wait_ctl(q_full(qs), (qcount / C::QBUF) & 1);
                tc_fence_after();
                bool first_pv[2] = {true, true};
                uint32_t prev = 0;
                const int U = w.n_tiles;
                uint32_t word_next = U > 0 ? __ldg(args.tiles + w.tile_begin) : 0u;
                for (int u = 0; u <= U; ++u) {
                    // the next step's word is loaded a step ahead (its L2 latency
                    // would otherwise sit on the issue path of every step)
                    const uint32_t word = word_next;
                    word_next = u + 1 < U ? __ldg(args.tiles + w.tile_begin + u + 1) : 0u;
                    const int vst = vcount % VS;
                    const int kst = kcount % KS;
                    const uint32_t v_addr = sbase + C::V_OFF + vst * C::TILE_BYTES;
                    const uint32_t k_addr = sbase + C::K_OFF + kst * C::TILE_BYTES;
                    bool v_ready = false, k_ready = false, v_freed = false;
                    // lane by lane: O_L += P_L(u-1) V(u-1), then S_L = Q_L K(u)^T, so
                    // lane A's next S overlaps lane B's softmax and vice versa.
#pragma unroll
                    for (int L = 0; L < 2; ++L) {
                        const uint32_t need = L ? TILE_NEED_B : TILE_NEED_A;
                        auto issue_pv = [&] {
                            if (!v_ready) {
                                if (DFA2_TRACE == 3 && lane == 0) DFA2_STAMP(3, vcount, 0);
                                mbar_wait_ctl(v_full(vst), (vcount / VS) & 1);
                                v_ready = true;
                            }
                            if ((DFA2_TRACE == 1 || DFA2_TRACE == 3) && lane == 0) DFA2_STAMP(L, pcnt[L], 7);
                            // keys 64..127 (P in cols [64,96)) as soon as that half is ready,
                            // then keys 0..63 (cols [0,32))
                            const uint64_t vdesc = smem_desc_sw128(v_addr, C::BOX_BYTES, 1024);
                            mbar_wait_ctl(p_half(L), pcnt[L] & 1);
                            tc_fence_after();
                            if (lane == 0) DFA2_STAMP(L, pcnt[L], 3);
                            if (elect_one()) {
#pragma unroll
                                for (int kk = 4; kk < 8; ++kk)
                                    mma_bf16_ts(tmem + o_col<D>(L), tmem + p_col<D>(L) + P_HI<D> + (kk - 4) * 8,
                                                vdesc + (kk * 2048 >> 4), IDESC_O, (!first_pv[L] || kk > 4) ? 1u : 0u);
                            }
                            __syncwarp();
                            mbar_wait_ctl(p_full(L), pcnt[L] & 1);
                            tc_fence_after();
                            if (elect_one()) {
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)
                                    mma_bf16_ts(tmem + o_col<D>(L), tmem + p_col<D>(L) + kk * 8, vdesc + (kk * 2048 >> 4),
                                                IDESC_O, 1u);
                                // calibration snapshot: O_L is final for this band once
                                // these PVs complete (the lane's next PV waits for it)
                                if (prev & (L ? TILE_SNAP_B : TILE_SNAP_A))
                                    mma_commit(o_full(L));
                                if (C::SEP_P)
                                    mma_commit(p_free(L));  // P_L may be overwritten
                            }
                            __syncwarp();
                            if (lane == 0) DFA2_STAMP(L, pcnt[L], 4);
                            first_pv[L] = false;
                            ++pcnt[L];
                        };
                        auto issue_s = [&] {
                            if (C::SEP_P && scount[L] >= 1) {  // the lane's softmax has read its last S
                                mbar_wait_ctl(s_free(L), (scount[L] - 1) & 1);
                                tc_fence_after();
                            }
                            if (!k_ready) {
                                mbar_wait_ctl(k_full(kst), (kcount / KS) & 1);
                                k_ready = true;
                            }
                            if ((DFA2_TRACE == 1 || DFA2_TRACE == 3) && lane == 0) DFA2_STAMP(L, scount[L], 6);
                            tc_fence_after();
                            const uint64_t qdesc = smem_desc_sw128(qbase + L * C::TILE_BYTES, 16, 1024);
                            const uint64_t kdesc = smem_desc_sw128(k_addr, 16, 1024);
                            if (elect_one()) {
#pragma unroll
                                for (int kk = 0; kk < D / 16; ++kk) {
                                    const uint32_t off = ((kk >> 2) * C::BOX_BYTES + (kk & 3) * 32) >> 4;
                                    mma_bf16_ss(tmem + s_col(L), qdesc + off, kdesc + off, IDESC_S, kk > 0 ? 1u : 0u);
                                }
                                mma_commit(s_full(L));
                            }
                            __syncwarp();
                            if (lane == 0) DFA2_STAMP(L, scount[L], 5);
                            ++scount[L];
                        };
                        const bool do_pv = u >= 1 && (prev & need);
                        const bool do_s = u < U && (word & need);
                        if (C::SEP_P) {  // S_L(u) first: it only waits for the softmax to read S_L(u-1)
                            if (do_s)
                                issue_s();
                            if (do_pv)
                                issue_pv();
                        } else {
                            if (do_pv) {
                                issue_pv();
                                // V(u-1) is free once its last PV completes: release it
                                // before this lane's S so the producer's next V load
                                // does not also wait for that S
                                if (DFA2_EARLY_VFREE && (L == 1 || !(prev & TILE_NEED_B))) {
                                    if (elect_one())
                                        mma_commit(v_empty(vst));
                                    __syncwarp();
                                    v_freed = true;
                                }
                            }
                            if (do_s)
                                issue_s();
                        }
                    }
                    if (DFA2_TRACE == 3 && lane == 0) DFA2_STAMP(3, kcount, 1);
                    if (elect_one()) {
                        if (u >= 1 && !v_freed)
                            mma_commit(v_empty(vst));  // V(u-1) free once its PVs complete
                        if (u < U) {
                            mma_commit(k_empty(kst));  // K(u) free once its S MMAs complete
                            if (u == U - 1)
                                mma_commit(q_empty(qs));
                        }
                    }
                    __syncwarp();
                    if (DFA2_TRACE == 3 && lane == 0) DFA2_STAMP(3, kcount, 2);
                    if (u >= 1)
                        ++vcount;
                    if (u < U)
                        ++kcount;
                    prev = word;
                }
                // both lanes' O final once every MMA issued so far completes
                if (elect_one()) {
                    mma_commit(o_full(0));
                    if (w.qtile_b >= 0)
                        mma_commit(o_full(1));
                }
                __syncwarp();
                ++qcount;
            }
        }
    }
    } else {
        // ------------------------------------------------ softmax lanes
        if (REGSPLIT<D>)
            regs_inc<REGS_SOFTMAX<D>>();
        const int L = (warp - 4) >> 2;              // 0 = lane A, 1 = lane B
        const int wq = warp & 3;                    // TMEM lane quarter
        const int r = wq * 32 + lane;               // row within the query tile
        const uint32_t lrow = static_cast<uint32_t>(wq * 32) << 16;
        const uint32_t need_bit = L ? TILE_NEED_B : TILE_NEED_A;
        const uint32_t part_bit = L ? TILE_PART_B : TILE_PART_A;
        const float sl2 = args.scale_log2;
        const uint32_t sc = tmem + lrow + s_col(L);
        const uint32_t oc = tmem + lrow + o_col<D>(L);
        const uint32_t pc = tmem + lrow + p_col<D>(L);
        const uint32_t stg = sbase + C::STG_OFF + L * C::BOX_BYTES;  // this lane's staging box
        const bool issuer = r == 0;  // issues this lane's bulk copies / stores
        uint32_t scnt = 0, icnt = 0, ccnt = 0;
        uint32_t ring_phase[C::RING];  // copy tail: next phase parity of each ring barrier
#pragma unroll
        for (int i = 0; i < C::RING; ++i)
            ring_phase[i] = 0u;
        for (int it = it0; it < it1; ++it) {
            const WorkItem w = items[it];
            if (DFA2_TRACE == 4 && args.trace && L == 0 && r == 0 && it < 8192) {  // per-item start (lane A)
                long long* ti = args.trace + 148 * 4 + static_cast<size_t>(it) * 4;
                ti[0] = gtime();
                ti[1] = static_cast<long long>(w.n_tiles) | (static_cast<long long>(w.flags) << 16) |
                        (w.qtile_b < 0 ? (1ll << 30) : 0ll);
                ti[2] = blockIdx.x;
            }
            if ((w.flags & ITEM_COPY) && args.copies_last) {
                // Copy tail (the host guarantees every remaining item of this
                // CTA is a Cached-head copy): all compute of the CTA is done,
                // so the Q / K / V rings and the staging boxes are free. Both
                // lanes sync once (every pending store has read its staging),
                // then each lane streams its copy boxes through a ring of
                // RING 16 KB boxes: up to RING TMA loads in flight, each box
                // stored to out (and the peers) as it lands — HBM-rate
                // copies instead of one box at a time.
                if (issuer)
                    bulk_wait_read0();
                named_bar_sync(3, 256);
                if (issuer) {
                    // batches of up to RING boxes: all loads in flight, then each
                    // box stored as it lands (a continuous ring with lagged
                    // refills measured slower: 46.7 vs 41.7 us on an all-Cached
                    // FLUX layer)
                    int li = it, lb = 0;  // next box to load (item, column box)
                    while (li < it1) {
                        int got = 0;
                        int bq[C::RING], bbx[C::RING], bbh[C::RING];
                        bulk_wait_read0();  // the previous batch's stores have read the ring
                        while (li < it1 && got < C::RING) {
                            const WorkItem& cw = items[li];
                            const int cq = L ? cw.qtile_b : cw.qtile_a;
                            if (cq >= 0) {
                                const uint32_t addr = sbase + static_cast<uint32_t>(L * C::RING + got) * C::BOX_BYTES;
                                mbar_arrive_expect_tx(ring_full(L, got), C::BOX_BYTES);
                                tma_load_q(addr, &tmc, ring_full(L, got), lb * 64, cq * TILE_M, cw.bh);
                                bq[got] = cq;
                                bbx[got] = lb;
                                bbh[got] = cw.bh;
                                ++got;
                            }
                            if (cq < 0 || ++lb == D / 64) {
                                lb = 0;
                                ++li;
                            }
                        }
                        for (int i = 0; i < got; ++i) {
                            const uint32_t addr = sbase + static_cast<uint32_t>(L * C::RING + i) * C::BOX_BYTES;
                            mbar_wait(ring_full(L, i), ring_phase[i]);
                            ring_phase[i] ^= 1u;
                            tma_store_o(&tmo, addr, bbx[i] * 64, bq[i] * TILE_M, bbh[i]);
                            for (int p = 0; p < args.n_peers; ++p)
                                tma_store_o(&peers.m[p], addr, bbx[i] * 64, bq[i] * TILE_M, bbh[i]);
                            bulk_commit();
                        }
                    }
                }
                break;  // every remaining item was a copy
            }
            if (w.flags & ITEM_COPY) {
                // Cached head: out <- stored slot, one 128-row tile per lane,
                // 64-column boxes through the lane's staging buffer by TMA.
                const int qt = L ? w.qtile_b : w.qtile_a;
                if (issuer && qt >= 0) {
#pragma unroll
                    for (int b = 0; b < D / 64; ++b) {
                        bulk_wait_read0();  // staging free
                        mbar_arrive_expect_tx(c_full(L), C::BOX_BYTES);
                        tma_load_q(stg, &tmc, c_full(L), b * 64, qt * TILE_M, w.bh);
                        mbar_wait(c_full(L), ccnt & 1);
                        ++ccnt;
                        tma_store_o(&tmo, stg, b * 64, qt * TILE_M, w.bh);
                        for (int p = 0; p < args.n_peers; ++p)
                            tma_store_o(&peers.m[p], stg, b * 64, qt * TILE_M, w.bh);
                        bulk_commit();
                    }
                }
                continue;
            }
            const int qt = L ? w.qtile_b : w.qtile_a;
            if (qt < 0 || w.n_tiles == 0)
                continue;
            const int row = qt * TILE_M + r;
            const uint8_t* mask = args.masks + w.mask_off;
            float m_ref = -INFINITY;
            float l = 0.f;
            bool first = true;
            // ---- epilogue: O / l -> bf16 -> staging (128B swizzle) -> TMA
            // bulk stores to out and, for computed heads, the cache slot; for
            // calibration items (ITEM_MULTI) to every output in `dst`
            const bool commit = (w.flags & ITEM_COMMIT) && args.cache;
            const bool multi = (w.flags & ITEM_MULTI) != 0;
            auto store_box = [&](int b, const float* vals, float inv, uint32_t dst) {
                if (issuer)
                    bulk_wait_read0();  // previous store from this buffer has read smem
                named_bar_sync(1 + L, 128);
                const uint32_t rbase = stg + static_cast<uint32_t>(r) * 128u;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint32_t p0 = pack_bf16x2(vals[8 * c + 0] * inv, vals[8 * c + 1] * inv);
                    const uint32_t p1 = pack_bf16x2(vals[8 * c + 2] * inv, vals[8 * c + 3] * inv);
                    const uint32_t p2 = pack_bf16x2(vals[8 * c + 4] * inv, vals[8 * c + 5] * inv);
                    const uint32_t p3 = pack_bf16x2(vals[8 * c + 6] * inv, vals[8 * c + 7] * inv);
                    st_shared_v4(rbase + static_cast<uint32_t>((c ^ (r & 7)) * 16), p0, p1, p2, p3);
                }
                fence_proxy_async_smem();
                named_bar_sync(1 + L, 128);
                if (issuer) {
                    if (!multi) {
                        tma_store_o(&tmo, stg, b * 64, qt * TILE_M, w.bh);  // rows >= N are clipped
                        if (commit)
                            tma_store_o(&tmc, stg, b * 64, qt * TILE_M, w.bh);
                        for (int p = 0; p < args.n_peers; ++p)  // the other ranks' copies of the layer
                            tma_store_o(&peers.m[p], stg, b * 64, qt * TILE_M, w.bh);
                    } else {
                        if (dst & SNAP_ORIGINAL)
                            tma_store_3d(&tmc, stg, b * 64, qt * TILE_M, w.bh);
                        for (uint32_t m = dst & (SNAP_ORIGINAL - 1u); m; m &= m - 1u)
                            tma_store_3d(&tmo, stg, b * 64, qt * TILE_M, w.bh + (__ffs(m) - 1) * args.snap_stride);
                    }
                    bulk_commit();
                }
            };
            auto store_tile = [&](uint32_t dst) {
                const float inv = 1.f / l;
#pragma unroll
                for (int b = 0; b < D / 64; ++b) {
                    float o[64];
                    tmem_ld32(oc + 64 * b, reinterpret_cast<uint32_t*>(o));
                    tmem_ld32(oc + 64 * b + 32, reinterpret_cast<uint32_t*>(o) + 32);
                    tmem_ld_wait();
                    store_box(b, o, inv, dst);
                }
            };
            const uint32_t snap_bit = L ? TILE_SNAP_B : TILE_SNAP_A;
            int sidx = 0;
            uint32_t word_next = __ldg(args.tiles + w.tile_begin);
            for (int u = 0; u < w.n_tiles; ++u) {
                const uint32_t word = word_next;
                if (u + 1 < w.n_tiles)
                    word_next = __ldg(args.tiles + w.tile_begin + u + 1);
                if (!(word & need_bit))
                    continue;
                uint32_t vm[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
                const bool partial = (word & part_bit) != 0;
                if (partial)
                    tile_valid_bits(args, mask, row, static_cast<int>(word & TILE_INDEX_MASK) * TILE_N, vm);
                if (r == 0) DFA2_STAMP(L, scnt, 0);
                mbar_wait(s_full(L), scnt & 1);
                tc_fence_after();
                if (r == 0) DFA2_STAMP(L, scnt, 1);
                if (partial)
                    mask_tile_in_tmem(sc, vm);
                long long* stamp = nullptr;
                if (DFA2_TRACE == 2 && args.trace && blockIdx.x == 0 && r == 0 && scnt < 4096)
                    stamp = args.trace + ((L * 4096) + scnt) * 8;
                softmax_tile<D>(sc, oc, sl2, m_ref, l, first, p_half(L), p_full(L), pc, s_free(L), p_free(L),
                                scnt == 0 ? -1 : static_cast<int>((scnt - 1) & 1), stamp);
                if (r == 0) DFA2_STAMP(L, scnt, 2);
                if (DFA2_TRACE == 5 && lane == 0 && args.trace && blockIdx.x == 0 && scnt < 4096)
                    args.trace[((L * 4096) + scnt) * 8 + 4 + wq] = clock64();  // each warp's softmax end
                ++scnt;
                first = false;
                if (word & snap_bit) {
                    // the narrower candidate's window is complete: its output
                    // is this state, O / l (the reference's sparse pass over
                    // exactly these key blocks, src/arrow.cpp:24-72)
                    mbar_wait(o_full(L), icnt & 1);
                    ++icnt;
                    tc_fence_after();
                    store_tile(args.snap_slots[sidx++]);
                    tc_fence_before();
                }
            }
            mbar_wait(o_full(L), icnt & 1);
            ++icnt;
            tc_fence_after();
            if (w.flags & ITEM_HALVES) {
                // both lanes folded halves of this tile's keys: merge
                // O = (O_A 2^(m_A-M) + O_B 2^(m_B-M)) / (l_A 2^(m_A-M) + l_B 2^(m_B-M)),
                // lane L storing the 64-column boxes b = L, L + 2, ...
                float* xch = reinterpret_cast<float*>(smem + C::XCHG_OFF);
                xch[(L * 2 + 0) * TILE_M + r] = m_ref;
                xch[(L * 2 + 1) * TILE_M + r] = l;
                // the other lane's O completed on ITS o_full barrier: order our
                // cross-lane TMEM reads after it through the thread sync
                tc_fence_before();
                named_bar_sync(3, 256);
                tc_fence_after();
                const float mo = xch[((1 - L) * 2 + 0) * TILE_M + r], lo_ = xch[((1 - L) * 2 + 1) * TILE_M + r];
                const float mA = L ? mo : m_ref, lA = L ? lo_ : l, mB = L ? m_ref : mo, lB = L ? l : lo_;
                const float M = fmaxf(mA, mB);
                const float fA = exp2f(mA - M), fB = exp2f(mB - M);
                const float inv = 1.f / (lA * fA + lB * fB);
                for (int b = L; b < D / 64; b += 2) {
                    float oa[64], ob[64];
                    const uint32_t ca = tmem + lrow + o_col<D>(0) + 64 * b, cb = tmem + lrow + o_col<D>(1) + 64 * b;
                    tmem_ld32(ca, reinterpret_cast<uint32_t*>(oa));
                    tmem_ld32(ca + 32, reinterpret_cast<uint32_t*>(oa) + 32);
                    tmem_ld32(cb, reinterpret_cast<uint32_t*>(ob));
                    tmem_ld32(cb + 32, reinterpret_cast<uint32_t*>(ob) + 32);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        oa[i] = fmaf(oa[i], fA, ob[i] * fB);
                    store_box(b, oa, inv, 0u);
                }
                tc_fence_before();
                named_bar_sync(3, 256);  // both lanes have read O_A and O_B
                continue;
            }
            if (!(w.flags & ITEM_SPLIT)) {
                uint32_t dst = 0;
                if (multi)  // every snapshot not yet emitted: the full row covers them
                    for (int i = sidx; i < args.n_snap; ++i)
                        dst |= args.snap_slots[i];
                store_tile(dst);
                tc_fence_before();
                continue;
            }
            // ---- split item (one key chunk of a heavy query-tile pair):
            // publish this chunk's unnormalised O, reference max and row sum
            // ([slot][lane][col][row], coalesced over rows), then the CTA that
            // completes the group folds all chunks in chunk order (fixed, so
            // results do not depend on which CTA finishes last) and stores.
            {
                const size_t base = (static_cast<size_t>(w.part) * 2 + L);
                float* po = args.part_o + base * D * TILE_M;
#pragma unroll
                for (int b = 0; b < D / 64; ++b) {
                    uint32_t o[64];
                    tmem_ld32(oc + 64 * b, o);
                    tmem_ld32(oc + 64 * b + 32, o + 32);
                    tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 64; ++c)
                        po[(64 * b + c) * TILE_M + r] = __uint_as_float(o[c]);
                }
                args.part_ml[(base * 2 + 0) * TILE_M + r] = m_ref;
                args.part_ml[(base * 2 + 1) * TILE_M + r] = l;
            }
            tc_fence_before();
            __threadfence();
            named_bar_sync(1 + L, 128);
            int* flag = reinterpret_cast<int*>(smem + C::BAR_OFF + C::NBARS * 8 + 8) + L;
            if (r == 0)
                *flag = atomicAdd(args.counters + 2 * w.group + L, 1) == w.nchunk - 1;
            named_bar_sync(1 + L, 128);
            if (!*flag)
                continue;
            __threadfence();
            {
                const int slot0 = w.part - w.chunk;
                auto ml = [&](int c, int which) {
                    return __ldcg(args.part_ml + ((static_cast<size_t>(slot0 + c) * 2 + L) * 2 + which) * TILE_M + r);
                };
                // the first CW chunks' (max, sum) are loaded together and kept
                // in registers (a split pair has 2-4 chunks at FLUX sizes), so
                // the fold's global round trips do not serialise per chunk; the
                // arithmetic and its order are the same for every chunk count
                constexpr int CW = 8;
                const int nc = w.nchunk;
                float mcv[CW], lcv[CW];
#pragma unroll
                for (int c = 0; c < CW; ++c) {
                    mcv[c] = c < nc ? ml(c, 0) : -INFINITY;
                    lcv[c] = c < nc ? ml(c, 1) : 0.f;
                }
                float m = -INFINITY;
#pragma unroll
                for (int c = 0; c < CW; ++c)
                    m = fmaxf(m, mcv[c]);
                for (int c = CW; c < nc; ++c)
                    m = fmaxf(m, ml(c, 0));
                float lsum = 0.f;
#pragma unroll
                for (int c = 0; c < CW; ++c)
                    if (mcv[c] != -INFINITY)
                        lsum += exp2f(mcv[c] - m) * lcv[c];
                for (int c = CW; c < nc; ++c) {
                    const float mc = ml(c, 0);
                    if (mc != -INFINITY)
                        lsum += exp2f(mc - m) * ml(c, 1);
                }
#pragma unroll 1
                for (int b = 0; b < D / 64; ++b) {
                    float acc[64];
#pragma unroll
                    for (int i = 0; i < 64; ++i)
                        acc[i] = 0.f;
                    for (int c = 0; c < nc; ++c) {
                        float mc = -INFINITY;
#pragma unroll
                        for (int j = 0; j < CW; ++j)
                            if (j == c)
                                mc = mcv[j];
                        if (c >= CW)
                            mc = ml(c, 0);
                        if (mc == -INFINITY)
                            continue;  // this lane folded no tile in chunk c
                        const float wc = exp2f(mc - m);
                        const float* po = args.part_o + (static_cast<size_t>(slot0 + c) * 2 + L) * D * TILE_M;
#pragma unroll
                        for (int i = 0; i < 64; ++i)
                            acc[i] = fmaf(wc, __ldcg(po + (64 * b + i) * TILE_M + r), acc[i]);
                    }
                    store_box(b, acc, 1.f / lsum, 0u);
                }
            }
        }
        if (args.n_copy_tiles > 0) {
            // Copy pool: the layer's Cached-head copies are not in any CTA's
            // list; every CTA that has finished its compute drains the pool,
            // each lane claiming RING 64-column boxes at a time from one
            // counter, so copies fill whatever compute leaves idle and the
            // copy bandwidth evens out over the SMs (a static split left
            // the slowest CTAs 12% behind the average). Every box goes from
            // its cache slot to out (and the peers) through the lane's ring
            // in the freed Q / K / V window, as in the per-CTA copy tail.
            if (issuer)
                bulk_wait_read0();
            named_bar_sync(3, 256);  // both lanes' compute is done: the rings are free
            if (issuer) {
                // a tile's rows are contiguous in the [bh, N, d] layout of both
                // the cache and out: 1-D bulk copies of up to BOX_BYTES each
                const uint32_t tile_bytes = static_cast<uint32_t>(TILE_M * args.row_bytes);
                const int bpt = static_cast<int>((tile_bytes + C::BOX_BYTES - 1) / C::BOX_BYTES);
                const int total = args.n_copy_tiles * bpt;
                const uint64_t pol = policy_evict_first();
                const char* csrc = reinterpret_cast<const char*>(args.cache);
                for (;;) {
                    const int base = atomicAdd(args.copy_ctr, C::RING);
                    if (base >= total)
                        break;
                    const int got = min(C::RING, total - base);
                    int64_t boff[C::RING];
                    uint32_t blen[C::RING];
                    bulk_wait_read0();  // the previous batch's stores have read the ring
#pragma unroll
                    for (int i = 0; i < C::RING; ++i) {
                        blen[i] = 0;
                        if (i >= got)
                            continue;
                        const int box = base + i;
                        const int2 ct = args.copy_tiles[box / bpt];
                        const int rows = min(TILE_M, args.n - ct.y * TILE_M);
                        const int64_t off = static_cast<int64_t>(box % bpt) * C::BOX_BYTES;
                        const int64_t left = static_cast<int64_t>(rows) * args.row_bytes - off;
                        if (left <= 0)
                            continue;  // a ragged tile's missing box
                        blen[i] = static_cast<uint32_t>(left < static_cast<int64_t>(C::BOX_BYTES) ? left : static_cast<int64_t>(C::BOX_BYTES));
                        boff[i] = (static_cast<int64_t>(ct.x) * args.n + static_cast<int64_t>(ct.y) * TILE_M) *
                                      args.row_bytes + off;
                        const uint32_t addr = sbase + static_cast<uint32_t>(L * C::RING + i) * C::BOX_BYTES;
                        mbar_arrive_expect_tx(ring_full(L, i), blen[i]);
                        bulk_load_1d_hint(addr, csrc + boff[i], blen[i], ring_full(L, i), pol);
                    }
#pragma unroll
                    for (int i = 0; i < C::RING; ++i) {
                        if (blen[i] == 0)
                            continue;
                        const uint32_t addr = sbase + static_cast<uint32_t>(L * C::RING + i) * C::BOX_BYTES;
                        mbar_wait(ring_full(L, i), ring_phase[i]);
                        ring_phase[i] ^= 1u;
                        bulk_store_1d_hint(reinterpret_cast<char*>(args.out) + boff[i], addr, blen[i], pol);
                        for (int p = 0; p < args.n_peers; ++p)
                            bulk_store_1d_hint(static_cast<char*>(peers.ptr[p]) + boff[i], addr, blen[i], pol);
                        bulk_commit();
                    }
                }
            }
        }
        if (issuer)
            bulk_wait0();  // every bulk store of this lane has completed
    }

    if (DFA2_TRACE == 4 && args.trace && (warp == 4 || warp == 8) && lane == 0)
        args.trace[blockIdx.x * 4 + 1 + (warp >> 3)] = gtime();  // lane A / B softmax done
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (DFA2_TRACE == 4 && args.trace && threadIdx.x == 0)
        args.trace[blockIdx.x * 4 + 3] = gtime();
    if (args.n_copy_tiles > 0 && threadIdx.x == 0) {
        // the last CTA out re-zeroes this launch's pool counter slot (every
        // CTA's claims precede its increment here), ready for its next use
        __threadfence();
        if (atomicAdd(args.copy_ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
            atomicExch(args.copy_ctr, 0);
            atomicExch(args.copy_ctr + 1, 0);
        }
    }
    if (warp == DFA2_ALLOC_WARP)
        tmem_dealloc(tmem, C::TMEM_COLS);
}

#define DFA2_MAPS                                                                                 \
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,                     \
        const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap,                 \
        const __grid_constant__ CUtensorMap
template __global__ void attn_fwd_sm100<64>(DFA2_MAPS, const AttnArgs, const __grid_constant__ PeerMaps);
template __global__ void attn_fwd_sm100<128>(DFA2_MAPS, const AttnArgs, const __grid_constant__ PeerMaps);
#undef DFA2_MAPS

namespace {
template <int D>
cudaError_t launch_d(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const CUtensorMap& to,
                     const CUtensorMap& tc, const AttnArgs& args, const PeerMaps& peers, int grid,
                     cudaStream_t stream) {
    using C = Cfg<D>;
    // the smem attribute is per (function, device): set once per device; the
    // bitmask is atomic, so host threads driving different GPUs (one per
    // rank) never race on it (a redundant set is harmless)
    static std::atomic<uint64_t> configured{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = dev < 64 ? uint64_t{1} << dev : 0;
    if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
        const cudaError_t e =
            cudaFuncSetAttribute(attn_fwd_sm100<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
        if (e != cudaSuccess)
            return e;
        configured.fetch_or(bit, std::memory_order_acq_rel);
    }
    attn_fwd_sm100<D><<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(tq, tk, tv, to, tc, args, peers);
    return cudaGetLastError();
}
}  // namespace

// Host-side launcher (called from dfa2c.cpp). `to` / `tc` map the output and
// the cache layer buffer with the same [batch*H, N, d] geometry as q/k/v.
cudaError_t launch_attn(int d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                        const CUtensorMap& to, const CUtensorMap& tc, const AttnArgs& args, const PeerMaps& peers,
                        int grid, cudaStream_t stream) {
    return d == 128 ? launch_d<128>(tq, tk, tv, to, tc, args, peers, grid, stream)
                    : launch_d<64>(tq, tk, tv, to, tc, args, peers, grid, stream);
}

}  // namespace dfa2k
