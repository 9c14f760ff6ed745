// rse_sm100.cu — the calibration RSE query on B200.
//
// Replaces rse()/mean_of/sum_sq_dev/sum_sq_diff
// (/root/reference/proj/src/calibrate.cpp:18-87), which makes three
// sequential double passes over two [N, d] f32 tensors per (head, method),
// with ONE coalesced, 16-byte-vectorised pass per head:
//   K     = y_o[0]                       (shift for a cancellation-safe variance)
//   so1   = sum(y_o - K)     so2 = sum((y_o - K)^2)
//   sd2   = sum((y_m - y_o)^2)                      (standard numerator)
//   sm1   = sum(y_m - K)     sm2 = sum((y_m - K)^2) (literal numerator)
// all in fp64. Partials per CTA are written to a scratch array and a second
// tiny kernel folds them in a fixed order, so results are bitwise
// reproducible run to run (no atomics on values).
//   mean = K + so1/n,  den = so2 - so1^2/n
//   standard: num = sd2;  literal: num = sm2 - 2 (mean-K) sm1 + n (mean-K)^2
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace dfa2k {

namespace {

constexpr int RSE_THREADS = 256;
constexpr int NACC = 5;

template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
    static constexpr int W = 8;  // elements per 16-byte load
    __device__ static void load(const __nv_bfloat16* p, double (&x)[8]) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            x[2 * i] = static_cast<double>(__uint_as_float(w[i] << 16));
            x[2 * i + 1] = static_cast<double>(__uint_as_float(w[i] & 0xFFFF0000u));
        }
    }
    __device__ static double one(const __nv_bfloat16* p) { return static_cast<double>(__bfloat162float(*p)); }
};
template <>
struct Vec<float> {
    static constexpr int W = 4;
    __device__ static void load(const float* p, double (&x)[4]) {
        const float4 u = __ldg(reinterpret_cast<const float4*>(p));
        x[0] = u.x;
        x[1] = u.y;
        x[2] = u.z;
        x[3] = u.w;
    }
    __device__ static double one(const float* p) { return static_cast<double>(*p); }
};

template <>
struct Vec<double> {
    static constexpr int W = 2;
    __device__ static void load(const double* p, double (&x)[2]) {
        const double2 u = __ldg(reinterpret_cast<const double2*>(p));
        x[0] = u.x;
        x[1] = u.y;
    }
    __device__ static double one(const double* p) { return *p; }
};

__device__ __forceinline__ void accum(double m, double o, double K, double (&a)[NACC]) {
    const double dO = o - K;
    const double dM = m - K;
    const double dd = m - o;
    a[0] += dO;
    a[1] = fma(dO, dO, a[1]);
    a[2] = fma(dd, dd, a[2]);
    a[3] += dM;
    a[4] = fma(dM, dM, a[4]);
}

}  // namespace

// grid (nblk, H). Each CTA reduces one contiguous, vector-aligned chunk of one
// head and writes NACC partials to part[(h * nblk + b) * NACC].
template <typename T>
__global__ void __launch_bounds__(RSE_THREADS) rse_partial(const T* __restrict__ ym,
                                                           const T* __restrict__ yo, int64_t numel,
                                                           int64_t chunk, int vec_ok,
                                                           double* __restrict__ part) {
    constexpr int W = Vec<T>::W;
    const int h = blockIdx.y;
    const int b = blockIdx.x;
    const T* m = ym + static_cast<int64_t>(h) * numel;
    const T* o = yo + static_cast<int64_t>(h) * numel;
    const double K = Vec<T>::one(o);
    const int64_t lo = static_cast<int64_t>(b) * chunk;
    const int64_t hi = min(lo + chunk, numel);
    double a[NACC] = {0, 0, 0, 0, 0};
    // vec_ok (host-checked): 16-byte aligned bases and numel % W == 0; chunk is
    // a multiple of W. Otherwise scalar loads.
    if (vec_ok) {
        for (int64_t i = lo + static_cast<int64_t>(threadIdx.x) * W; i + W <= hi; i += RSE_THREADS * W) {
            double xm[W], xo[W];
            Vec<T>::load(m + i, xm);
            Vec<T>::load(o + i, xo);
#pragma unroll
            for (int e = 0; e < W; ++e)
                accum(xm[e], xo[e], K, a);
        }
    } else {
        for (int64_t i = lo + threadIdx.x; i < hi; i += RSE_THREADS)
            accum(Vec<T>::one(m + i), Vec<T>::one(o + i), K, a);
    }
    // fixed-pattern warp tree, then warps in index order
#pragma unroll
    for (int k = 0; k < NACC; ++k)
        for (int off = 16; off > 0; off >>= 1)
            a[k] += __shfl_xor_sync(0xFFFFFFFFu, a[k], off);
    __shared__ double red[RSE_THREADS / 32][NACC];
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < NACC; ++k)
            red[warp][k] = a[k];
    __syncthreads();
    if (threadIdx.x < NACC) {
        double t = 0.0;
        for (int w = 0; w < RSE_THREADS / 32; ++w)
            t += red[w][threadIdx.x];
        part[(static_cast<int64_t>(h) * gridDim.x + b) * NACC + threadIdx.x] = t;
    }
}

// One thread per head: fold partials in CTA order, finish the RSE.
template <typename T>
__global__ void rse_finalize(const T* __restrict__ yo, const double* __restrict__ part, int nblk,
                             int n_heads, int64_t numel, int mode, double* __restrict__ out) {
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= n_heads)
        return;
    double a[NACC] = {0, 0, 0, 0, 0};
    for (int b = 0; b < nblk; ++b)
#pragma unroll
        for (int k = 0; k < NACC; ++k)
            a[k] += part[(static_cast<int64_t>(h) * nblk + b) * NACC + k];
    const double K = Vec<T>::one(yo + static_cast<int64_t>(h) * numel);
    const double n = static_cast<double>(numel);
    const double dmean = a[0] / n;  // mean - K
    const double den = a[1] - a[0] * dmean;
    double num;
    if (mode == 0)
        num = a[2];
    else
        num = a[4] - 2.0 * dmean * a[3] + n * dmean * dmean;
    out[h] = den > 0.0 ? num / den : __longlong_as_double(0x7FF8000000000000ll);
}

cudaError_t launch_rse(const void* ym, const void* yo, int dtype, int64_t n_heads, int64_t numel,
                       int mode, double* out_dev, double* scratch, int nblk, cudaStream_t stream) {
    const int64_t W = dtype == 0 ? 8 : dtype == 1 ? 4 : 2;
    int64_t chunk = (numel + nblk - 1) / nblk;
    chunk = (chunk + W - 1) / W * W;
    const dim3 grid(nblk, static_cast<unsigned>(n_heads));
    const int vec_ok = (numel % W) == 0 && (reinterpret_cast<uintptr_t>(ym) % 16) == 0 &&
                       (reinterpret_cast<uintptr_t>(yo) % 16) == 0;
    const int fin_blocks = static_cast<int>((n_heads + 127) / 128);
    if (dtype == 0) {
        rse_partial<__nv_bfloat16><<<grid, RSE_THREADS, 0, stream>>>(
            static_cast<const __nv_bfloat16*>(ym), static_cast<const __nv_bfloat16*>(yo), numel, chunk, vec_ok, scratch);
        rse_finalize<__nv_bfloat16><<<fin_blocks, 128, 0, stream>>>(
            static_cast<const __nv_bfloat16*>(yo), scratch, nblk, static_cast<int>(n_heads), numel, mode, out_dev);
    } else if (dtype == 2) {
        rse_partial<double><<<grid, RSE_THREADS, 0, stream>>>(static_cast<const double*>(ym),
                                                              static_cast<const double*>(yo), numel, chunk, vec_ok,
                                                              scratch);
        rse_finalize<double><<<fin_blocks, 128, 0, stream>>>(static_cast<const double*>(yo), scratch, nblk,
                                                             static_cast<int>(n_heads), numel, mode, out_dev);
    } else {
        rse_partial<float><<<grid, RSE_THREADS, 0, stream>>>(static_cast<const float*>(ym),
                                                             static_cast<const float*>(yo), numel, chunk, vec_ok, scratch);
        rse_finalize<float><<<fin_blocks, 128, 0, stream>>>(static_cast<const float*>(yo), scratch, nblk,
                                                            static_cast<int>(n_heads), numel, mode, out_dev);
    }
    return cudaGetLastError();
}

}  // namespace dfa2k
