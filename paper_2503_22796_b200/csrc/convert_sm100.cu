// convert_sm100.cu — element-type conversion at the API boundary: the
// reference's operator API takes f32 / f64 host tensors
// (/root/reference/proj/include/dfa2/tensor.hpp:17-50) while the attention
// path computes on bf16. The C++ drop-in uploads f32 and converts on the
// device (round to nearest even, as __float2bfloat16_rn and the oracle's
// round_bf16) instead of converting element by element on the host.
// Grid-stride, 16-byte stores; HBM-bound.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

namespace dfa2k {

namespace {

template <typename S>
__device__ __forceinline__ float load_f(const S* p, int64_t i) {
    return static_cast<float>(p[i]);
}
template <>
__device__ __forceinline__ float load_f<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
    return __bfloat162float(p[i]);
}

template <typename S, typename T>
__device__ __forceinline__ void store_t(T* p, int64_t i, S x) {
    p[i] = static_cast<T>(x);
}

template <typename S, typename T>
__global__ void convert_kernel(const S* __restrict__ src, T* __restrict__ dst, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        if constexpr (std::is_same_v<T, __nv_bfloat16>)
            dst[i] = __float2bfloat16_rn(load_f(src, i));
        else if constexpr (std::is_same_v<S, double> && std::is_same_v<T, double>)
            dst[i] = src[i];
        else if constexpr (std::is_same_v<S, double>)
            dst[i] = static_cast<T>(src[i]);
        else
            dst[i] = static_cast<T>(load_f(src, i));
    }
}

template <typename S>
cudaError_t to(const void* src, int dst_dtype, void* dst, int64_t n, int grid, cudaStream_t st) {
    const S* s = static_cast<const S*>(src);
    switch (dst_dtype) {
    case 0: convert_kernel<S, __nv_bfloat16><<<grid, 256, 0, st>>>(s, static_cast<__nv_bfloat16*>(dst), n); break;
    case 1: convert_kernel<S, float><<<grid, 256, 0, st>>>(s, static_cast<float*>(dst), n); break;
    default: convert_kernel<S, double><<<grid, 256, 0, st>>>(s, static_cast<double*>(dst), n); break;
    }
    return cudaGetLastError();
}

}  // namespace

// dtype codes: 0 bf16, 1 f32, 2 f64 (DFA2C_BF16 / DFA2C_F32 / DFA2C_F64)
cudaError_t launch_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n, int sms,
                           cudaStream_t stream) {
    if (n <= 0)
        return cudaSuccess;
    const int64_t blocks = (n + 255) / 256;
    const int grid = static_cast<int>(blocks < 8LL * sms ? blocks : 8LL * sms);
    switch (src_dtype) {
    case 0: return to<__nv_bfloat16>(src, dst_dtype, dst, n, grid, stream);
    case 1: return to<float>(src, dst_dtype, dst, n, grid, stream);
    default: return to<double>(src, dst_dtype, dst, n, grid, stream);
    }
}

// ---- sharded layer: commit the rows other ranks computed ----------------
// After the all-gather every rank holds the whole layer output; the rows of
// computed heads outside this rank's own range [r0, r1) (flattened
// [batch*H*N] rows) are copied into this rank's cache layer, so every rank's
// cache is complete and a Cached head can be served by whichever rank owns
// its rows at a later timestep. 16-byte vectors, grid-stride; HBM-bound.
struct HeadBits {
    uint32_t w[32];  // computed heads (up to 1024)
};

__global__ void commit_rows_kernel(const uint4* __restrict__ out, uint4* __restrict__ cache, int64_t rows,
                                   int64_t r0, int64_t r1, int64_t n, int64_t H, int vec_per_row, HeadBits bits) {
    const int64_t outside = rows - (r1 - r0);
    const int64_t total = outside * vec_per_row;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        int64_t r = i / vec_per_row;
        r = r < r0 ? r : r + (r1 - r0);
        const int64_t h = (r / n) % H;
        if (!((bits.w[h >> 5] >> (h & 31)) & 1u))
            continue;
        const int64_t v = r * vec_per_row + i % vec_per_row;
        cache[v] = out[v];
    }
}

cudaError_t launch_commit_rows(const void* out, void* cache, int64_t rows, int64_t r0, int64_t r1, int64_t n,
                               int64_t H, int64_t d, const uint32_t* head_bits, int sms, cudaStream_t stream) {
    HeadBits b{};
    for (int i = 0; i < 32; ++i)
        b.w[i] = head_bits[i];
    const int vec = static_cast<int>(d * 2 / 16);
    const int64_t total = (rows - (r1 - r0)) * vec;
    if (total <= 0)
        return cudaSuccess;
    const int64_t blocks = (total + 255) / 256;
    const int grid = static_cast<int>(blocks < 8LL * sms ? blocks : 8LL * sms);
    commit_rows_kernel<<<grid, 256, 0, stream>>>(static_cast<const uint4*>(out), static_cast<uint4*>(cache), rows, r0,
                                                 r1, n, H, vec, b);
    return cudaGetLastError();
}

}  // namespace dfa2k
