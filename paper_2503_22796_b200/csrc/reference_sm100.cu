// reference_sm100.cu — attention_reference at the caller's precision.
//
// The reference's attention_reference (/root/reference/proj/src/tensor.cpp:
// 73-114, 268-295) is its f32 / f64 ground truth: masked scaled scores, the
// row max, exp(s - max), the row sum, and out = sum_j (w_j / sum) v_j, all in
// the tensor's own type. The drop-in keeps that contract on the GPU: this is
// a SIMT kernel in T = float or double (no bf16 rounding anywhere, no tensor
// cores), so a caller that uses attention_reference as an independent checker
// (run_bench's oracle gate, src/bench.cpp:126-134; cmd_verify) gets one.
//
// One warp per query row, two passes over the row's active keys:
//   1. s_j = (q . k_j) * (1/sqrt(d)), the row max (lanes own keys j = lane
//      mod 32, then a warp max);
//   2. w_j = exp(s_j - max); the row sum and sum_j w_j v_j, lanes owning
//      output columns c = lane + 32 i (each key's weight broadcast by shfl,
//      so the V row is read coalesced). out = acc / sum.
// Scores are recomputed in pass 2 rather than stored (an N-long row per warp
// would not fit on chip at FLUX sizes). The summation order differs from the
// reference's sequential loops, so results agree to rounding (~1e-6
// relative in f32, ~1e-15 in f64), not bitwise. K and V chunks of 32 keys are
// staged through shared memory and shared by the CTA's 8 rows.
#include <cuda_runtime.h>

#include <cstdint>

namespace dfa2k {

namespace {

constexpr int REF_WARPS = 8;   // query rows per CTA
constexpr int REF_KEYS = 32;   // keys per shared-memory chunk
constexpr int REF_MAXC = 16;   // output columns per lane: head_dim <= 512

template <typename T>
__device__ __forceinline__ T ex(T x);
template <>
__device__ __forceinline__ float ex<float>(float x) { return expf(x); }
template <>
__device__ __forceinline__ double ex<double>(double x) { return exp(x); }

// q, k, v, out: [H, N, d]; mask: nb*nb bytes or null; grid (ceil(N/8), H).
template <typename T>
__global__ void __launch_bounds__(REF_WARPS * 32)
attn_reference_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                      T* __restrict__ out, int n, int d, const uint8_t* __restrict__ mask, int block, int nb,
                      T scale) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sq = reinterpret_cast<T*>(smem_raw);               // [8][d]
    T* sk = sq + REF_WARPS * d;                           // [32][d + 1] (padded: lane j reads row j)
    T* sv = sk + REF_KEYS * (d + 1);                      // [32][d]
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t head = blockIdx.y;
    const int row = blockIdx.x * REF_WARPS + warp;
    const bool live = row < n;
    const T* qh = q + head * int64_t(n) * d;
    const T* kh = k + head * int64_t(n) * d;
    const T* vh = v + head * int64_t(n) * d;
    for (int c = lane; c < d; c += 32)
        sq[warp * d + c] = live ? qh[int64_t(row) * d + c] : T(0);
    const int qb = live && mask ? row / block : 0;
    const int row_lo = blockIdx.x * REF_WARPS, row_hi = min(n, row_lo + REF_WARPS);
    const T neg_inf = -__builtin_huge_val();

    // a key chunk is loaded when any row of the CTA keeps one of its keys
    auto chunk_needed = [&](int j0) {
        if (!mask)
            return true;
        const int j1 = min(n, j0 + REF_KEYS) - 1;
        for (int qbb = row_lo / block; qbb <= (row_hi - 1) / block; ++qbb)
            for (int kb = j0 / block; kb <= j1 / block; ++kb)
                if (mask[int64_t(qbb) * nb + kb])
                    return true;
        return false;
    };
    auto key_active = [&](int j) { return !mask || mask[int64_t(qb) * nb + j / block] != 0; };
    auto load_chunk = [&](int j0, bool with_v) {
        __syncthreads();
        for (int i = threadIdx.x; i < REF_KEYS * d; i += blockDim.x) {
            const int r = i / d, c = i % d, j = j0 + r;
            sk[r * (d + 1) + c] = j < n ? kh[int64_t(j) * d + c] : T(0);
            if (with_v)
                sv[r * d + c] = j < n ? vh[int64_t(j) * d + c] : T(0);
        }
        __syncthreads();
    };
    auto score = [&](int r) {
        T acc = T(0);
        const T* kr = sk + r * (d + 1);
        const T* qr = sq + warp * d;
        for (int c = 0; c < d; ++c)
            acc += qr[c] * kr[c];
        return acc * scale;
    };

    // pass 1: row max
    T mx = neg_inf;
    for (int j0 = 0; j0 < n; j0 += REF_KEYS) {
        if (!chunk_needed(j0))
            continue;
        load_chunk(j0, false);
        const int j = j0 + lane;
        if (live && j < n && key_active(j))
            mx = max(mx, score(lane));
    }
    for (int o = 16; o > 0; o >>= 1)
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));

    // pass 2: weights, row sum, weighted V
    T acc[REF_MAXC];
#pragma unroll
    for (int i = 0; i < REF_MAXC; ++i)
        acc[i] = T(0);
    T sum = T(0);
    for (int j0 = 0; j0 < n; j0 += REF_KEYS) {
        if (!chunk_needed(j0))
            continue;
        load_chunk(j0, true);
        const int j = j0 + lane;
        T w = T(0);
        if (live && j < n && key_active(j))
            w = ex<T>(score(lane) - mx);
        sum += w;
        for (int r = 0; r < REF_KEYS; ++r) {
            const T wr = __shfl_sync(0xffffffffu, w, r);
            if (wr == T(0))
                continue;  // masked or underflowed: contributes nothing (tensor.cpp:110-112)
#pragma unroll
            for (int i = 0; i < REF_MAXC; ++i) {
                const int c = lane + 32 * i;
                if (c < d)
                    acc[i] += wr * sv[r * d + c];
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1)
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (!live)
        return;
    const T inv = T(1) / sum;
    T* orow = out + (head * int64_t(n) + row) * d;
#pragma unroll
    for (int i = 0; i < REF_MAXC; ++i) {
        const int c = lane + 32 * i;
        if (c < d)
            orow[c] = acc[i] * inv;
    }
}

template <typename T>
cudaError_t launch_ref_t(const void* q, const void* k, const void* v, void* out, int64_t H, int64_t n, int64_t d,
                         const uint8_t* mask, int64_t block, int64_t nb, cudaStream_t st) {
    const size_t smem = sizeof(T) * (REF_WARPS * d + REF_KEYS * (d + 1) + REF_KEYS * d);
    auto kern = attn_reference_kernel<T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess)
        return e;
    const dim3 grid(static_cast<unsigned>((n + REF_WARPS - 1) / REF_WARPS), static_cast<unsigned>(H));
    const T scale = T(1) / sqrt(static_cast<T>(d));
    kern<<<grid, REF_WARPS * 32, smem, st>>>(static_cast<const T*>(q), static_cast<const T*>(k),
                                             static_cast<const T*>(v), static_cast<T*>(out), static_cast<int>(n),
                                             static_cast<int>(d), mask, static_cast<int>(block),
                                             static_cast<int>(nb), scale);
    return cudaGetLastError();
}

}  // namespace

int reference_max_head_dim() { return 32 * REF_MAXC; }

// dtype: 1 = f32, 2 = f64 (DFA2C_F32 / DFA2C_F64). mask: device bytes or null.
cudaError_t launch_attention_reference(const void* q, const void* k, const void* v, void* out, int dtype, int64_t H,
                                       int64_t n, int64_t d, const uint8_t* mask, int64_t block, int64_t nb,
                                       cudaStream_t stream) {
    if (dtype == 2)
        return launch_ref_t<double>(q, k, v, out, H, n, d, mask, block, nb, stream);
    return launch_ref_t<float>(q, k, v, out, H, n, d, mask, block, nb, stream);
}

}  // namespace dfa2k
