// rse_sm100.cu — the calibration RSE query on B200.
//
// Replaces rse()/mean_of/sum_sq_dev/sum_sq_diff
// (/root/reference/proj/src/calibrate.cpp:18-87), which makes three
// sequential double passes over two [N, d] f32 tensors per (head, method),
// with ONE streaming pass per head. Each CTA owns a contiguous chunk of one
// head; a producer warp moves it through a 4-stage shared-memory ring with
// 1-D bulk copies (cp.async.bulk, 8 KB per operand per stage, mbarrier
// completion), so HBM reads stay in flight while 8 consumer warps convert
// and accumulate from shared memory:
//   K     = y_o[0]                       (shift for a cancellation-safe variance)
//   so1   = sum(y_o - K)     so2 = sum((y_o - K)^2)
//   sd2   = sum((y_m - y_o)^2)                      (standard numerator)
//   sm1   = sum(y_m - K)     sm2 = sum((y_m - K)^2) (literal numerator)
// all in fp64. Partials per CTA are written to a scratch array and a second
// tiny kernel (one warp per head) folds them in a fixed order, so results
// are bitwise reproducible run to run (no atomics on values).
//   mean = K + so1/n,  den = so2 - so1^2/n
//   standard: num = sd2;  literal: num = sm2 - 2 (mean-K) sm1 + n (mean-K)^2
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

#include "sm100_ptx.cuh"

namespace dfa2k {

namespace {

constexpr int RSE_THREADS = 256;
constexpr int NACC = 5;

template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
    static constexpr int W = 8;  // elements per 16-byte load
    __device__ static void unpack(const uint4& u, double (&x)[8]) {
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
    __device__ static void unpack(const uint4& r, double (&x)[4]) {
        const float4 u = make_float4(__uint_as_float(r.x), __uint_as_float(r.y), __uint_as_float(r.z),
                                     __uint_as_float(r.w));
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
    __device__ static void unpack(const uint4& r, double (&x)[2]) {
        x[0] = __hiloint2double(static_cast<int>(r.y), static_cast<int>(r.x));
        x[1] = __hiloint2double(static_cast<int>(r.w), static_cast<int>(r.z));
    }
    __device__ static double one(const double* p) { return *p; }
};

template <bool LIT>
__device__ __forceinline__ void accum(double m, double o, double K, double (&a)[NACC]) {
    const double dO = o - K;
    const double dd = m - o;
    a[0] += dO;
    a[1] = fma(dO, dO, a[1]);
    a[2] = fma(dd, dd, a[2]);
    if (LIT) {  // literal numerator only: sum(y_m - K), sum((y_m - K)^2)
        const double dM = m - K;
        a[3] += dM;
        a[4] = fma(dM, dM, a[4]);
    }
}

#ifndef DFA2_RSE_STAGES
#define DFA2_RSE_STAGES 4
#endif
#ifndef DFA2_RSE_STAGE_KB
#define DFA2_RSE_STAGE_KB 8
#endif
#ifndef DFA2_RSE_CTAS
#define DFA2_RSE_CTAS 3
#endif
constexpr int RSE_STAGES = DFA2_RSE_STAGES;
constexpr uint32_t RSE_STAGE_BYTES = DFA2_RSE_STAGE_KB * 1024;  // per operand per stage
constexpr uint32_t RSE_BAR_OFF = RSE_STAGES * 2 * RSE_STAGE_BYTES;
constexpr uint32_t RSE_SMEM = RSE_BAR_OFF + 2 * RSE_STAGES * 8;

}  // namespace

// grid (nblk, H), RSE_THREADS consumer threads + 1 producer warp. CTA (b, h)
// reduces elements [b*chunk, min((b+1)*chunk, numel)) of head h and writes
// NACC partials to part[(h * nblk + b) * NACC]. vec_ok (host-checked): both
// bases 16-byte aligned, numel % W == 0 and chunk % W == 0; otherwise the
// whole chunk takes the scalar path. The order every value is folded in is
// fixed by (stage, thread, vector), so results are run-to-run bitwise stable.
template <typename T, bool LIT>
__global__ void __launch_bounds__(RSE_THREADS + 32) rse_partial(const T* __restrict__ ym,
                                                                const T* __restrict__ yo, int64_t numel,
                                                                int64_t chunk, int vec_ok,
                                                                double* __restrict__ part) {
    constexpr int W = Vec<T>::W;
    constexpr int64_t EPS = RSE_STAGE_BYTES / sizeof(T);  // elements per stage
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const uint32_t full0 = sbase + RSE_BAR_OFF, empty0 = full0 + 8 * RSE_STAGES;
    const int h = blockIdx.y;
    const int b = blockIdx.x;
    const T* m = ym + static_cast<int64_t>(h) * numel;
    const T* o = yo + static_cast<int64_t>(h) * numel;
    const int64_t lo = min(static_cast<int64_t>(b) * chunk, numel);
    const int64_t hi = min(lo + chunk, numel);
    const int64_t n_vec = vec_ok ? (hi - lo) / W * W : 0;  // staged through smem
    const int n_stage = static_cast<int>((n_vec + EPS - 1) / EPS);
    const int warp = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        for (int s = 0; s < RSE_STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, RSE_THREADS / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();

    double a[NACC] = {0, 0, 0, 0, 0};
    if (warp == RSE_THREADS / 32) {
        // ---- producer: one elected lane streams the chunk through the ring
        if (elect_one()) {
            for (int s = 0; s < n_stage; ++s) {
                const int slot = s % RSE_STAGES;
                if (s >= RSE_STAGES)
                    mbar_wait(empty0 + 8 * slot, ((s / RSE_STAGES) - 1) & 1);
                const int64_t e0 = lo + s * EPS;
                const uint32_t bytes = static_cast<uint32_t>(min(EPS, lo + n_vec - e0) * sizeof(T));
                const uint32_t dst = sbase + slot * 2 * RSE_STAGE_BYTES;
                mbar_arrive_expect_tx(full0 + 8 * slot, 2 * bytes);
                bulk_load_1d(dst, m + e0, bytes, full0 + 8 * slot);
                bulk_load_1d(dst + RSE_STAGE_BYTES, o + e0, bytes, full0 + 8 * slot);
            }
        }
        __syncwarp();
    } else {
        const double K = Vec<T>::one(o);
        // ---- consumers: W-element vectors, thread-strided within a stage
        for (int s = 0; s < n_stage; ++s) {
            const int slot = s % RSE_STAGES;
            mbar_wait(full0 + 8 * slot, (s / RSE_STAGES) & 1);
            const int64_t e_stage = min(EPS, n_vec - s * EPS);
            const uint32_t sm_m = sbase + slot * 2 * RSE_STAGE_BYTES;
            const uint32_t sm_o = sm_m + RSE_STAGE_BYTES;
#pragma unroll 2
            for (int64_t e = static_cast<int64_t>(threadIdx.x) * W; e < e_stage; e += RSE_THREADS * W) {
                const uint32_t off = static_cast<uint32_t>(e * sizeof(T));
                double xm[W], xo[W];
                Vec<T>::unpack(ld_shared_v4(sm_m + off), xm);
                Vec<T>::unpack(ld_shared_v4(sm_o + off), xo);
#pragma unroll
                for (int k = 0; k < W; ++k)
                    accum<LIT>(xm[k], xo[k], K, a);
            }
            __syncwarp();
            if ((threadIdx.x & 31) == 0)
                mbar_arrive(empty0 + 8 * slot);
        }
        // elements the ring does not cover (unaligned operands, sub-vector tail)
        for (int64_t i = lo + n_vec + threadIdx.x; i < hi; i += RSE_THREADS)
            accum<LIT>(Vec<T>::one(m + i), Vec<T>::one(o + i), K, a);
        // fixed-pattern warp tree
#pragma unroll
        for (int k = 0; k < NACC; ++k)
            for (int off = 16; off > 0; off >>= 1)
                a[k] += __shfl_xor_sync(0xFFFFFFFFu, a[k], off);
    }
    __shared__ double red[RSE_THREADS / 32][NACC];
    if (warp < RSE_THREADS / 32 && (threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < NACC; ++k)
            red[warp][k] = a[k];
    __syncthreads();
    if (threadIdx.x < NACC) {  // consumer warps in index order
        double t = 0.0;
        for (int w = 0; w < RSE_THREADS / 32; ++w)
            t += red[w][threadIdx.x];
        part[(static_cast<int64_t>(h) * gridDim.x + b) * NACC + threadIdx.x] = t;
    }
}

// ---- several candidates against one reference (influence_for_layer's
// per-layer RSE grid): y_o is streamed once per CTA and shared by up to
// RSE_MAXM candidate streams, so a layer's M RSEs read (M + 1) instead of
// 2M tensors. Same per-(candidate, head) partials as rse_partial, written as
// set m * H + h for rse_finalize.
constexpr int RSE_MAXM = 8;
constexpr int RSE_MULTI_STAGES = 2;
template <typename T>
struct CandPtrs {
    const T* p[RSE_MAXM];
};
constexpr uint32_t rse_multi_smem(int M) {
    return RSE_MULTI_STAGES * (M + 1) * RSE_STAGE_BYTES + 2 * RSE_MULTI_STAGES * 8;
}

template <typename T, bool LIT>
__global__ void __launch_bounds__(RSE_THREADS + 32) rse_multi_partial(CandPtrs<T> cands, int M,
                                                                      const T* __restrict__ yo, int64_t numel,
                                                                      int64_t chunk, int vec_ok,
                                                                      double* __restrict__ part) {
    constexpr int W = Vec<T>::W;
    constexpr int64_t EPS = RSE_STAGE_BYTES / sizeof(T);
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const uint32_t stage_bytes = static_cast<uint32_t>(M + 1) * RSE_STAGE_BYTES;
    const uint32_t full0 = sbase + RSE_MULTI_STAGES * stage_bytes, empty0 = full0 + 8 * RSE_MULTI_STAGES;
    const int h = blockIdx.y, H = gridDim.y;
    const int b = blockIdx.x;
    const T* o = yo + static_cast<int64_t>(h) * numel;
    const int64_t lo = min(static_cast<int64_t>(b) * chunk, numel);
    const int64_t hi = min(lo + chunk, numel);
    const int64_t n_vec = vec_ok ? (hi - lo) / W * W : 0;
    const int n_stage = static_cast<int>((n_vec + EPS - 1) / EPS);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < RSE_MULTI_STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, RSE_THREADS / 32);
        }
        fence_mbar_init();
    }
    __syncthreads();
    double ao[2] = {0, 0};
    double am[RSE_MAXM][3];
#pragma unroll
    for (int c = 0; c < RSE_MAXM; ++c)
        am[c][0] = am[c][1] = am[c][2] = 0.0;
    if (warp == RSE_THREADS / 32) {
        if (elect_one()) {
            for (int s = 0; s < n_stage; ++s) {
                const int slot = s % RSE_MULTI_STAGES;
                if (s >= RSE_MULTI_STAGES)
                    mbar_wait(empty0 + 8 * slot, ((s / RSE_MULTI_STAGES) - 1) & 1);
                const int64_t e0 = lo + s * EPS;
                const uint32_t bytes = static_cast<uint32_t>(min(EPS, lo + n_vec - e0) * sizeof(T));
                const uint32_t dst = sbase + slot * stage_bytes;
                mbar_arrive_expect_tx(full0 + 8 * slot, (M + 1) * bytes);
                bulk_load_1d(dst, o + e0, bytes, full0 + 8 * slot);
                for (int c = 0; c < M; ++c)
                    bulk_load_1d(dst + (c + 1) * RSE_STAGE_BYTES, cands.p[c] + static_cast<int64_t>(h) * numel + e0,
                                 bytes, full0 + 8 * slot);
            }
        }
        __syncwarp();
    } else {
        const double K = Vec<T>::one(o);
        for (int s = 0; s < n_stage; ++s) {
            const int slot = s % RSE_MULTI_STAGES;
            mbar_wait(full0 + 8 * slot, (s / RSE_MULTI_STAGES) & 1);
            const int64_t e_stage = min(EPS, n_vec - s * EPS);
            const uint32_t sm_o = sbase + slot * stage_bytes;
            for (int64_t e = static_cast<int64_t>(threadIdx.x) * W; e < e_stage; e += RSE_THREADS * W) {
                const uint32_t off = static_cast<uint32_t>(e * sizeof(T));
                double xo[W];
                Vec<T>::unpack(ld_shared_v4(sm_o + off), xo);
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const double dO = xo[k] - K;
                    ao[0] += dO;
                    ao[1] = fma(dO, dO, ao[1]);
                }
#pragma unroll
                for (int c = 0; c < RSE_MAXM; ++c) {
                    if (c >= M)
                        break;
                    double xm[W];
                    Vec<T>::unpack(ld_shared_v4(sm_o + (c + 1) * RSE_STAGE_BYTES + off), xm);
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const double dd = xm[k] - xo[k];
                        am[c][0] = fma(dd, dd, am[c][0]);
                        if (LIT) {
                            const double dM = xm[k] - K;
                            am[c][1] += dM;
                            am[c][2] = fma(dM, dM, am[c][2]);
                        }
                    }
                }
            }
            __syncwarp();
            if ((threadIdx.x & 31) == 0)
                mbar_arrive(empty0 + 8 * slot);
        }
        for (int64_t i = lo + n_vec + threadIdx.x; i < hi; i += RSE_THREADS) {
            const double xo = Vec<T>::one(o + i);
            const double dO = xo - K;
            ao[0] += dO;
            ao[1] = fma(dO, dO, ao[1]);
#pragma unroll
            for (int c = 0; c < RSE_MAXM; ++c) {
                if (c >= M)
                    break;
                const double xm = Vec<T>::one(cands.p[c] + static_cast<int64_t>(h) * numel + i);
                const double dd = xm - xo;
                am[c][0] = fma(dd, dd, am[c][0]);
                if (LIT) {
                    am[c][1] += xm - K;
                    am[c][2] = fma(xm - K, xm - K, am[c][2]);
                }
            }
        }
        for (int off = 16; off > 0; off >>= 1) {
            ao[0] += __shfl_xor_sync(0xFFFFFFFFu, ao[0], off);
            ao[1] += __shfl_xor_sync(0xFFFFFFFFu, ao[1], off);
        }
#pragma unroll
        for (int c = 0; c < RSE_MAXM; ++c)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                for (int off = 16; off > 0; off >>= 1)
                    am[c][k] += __shfl_xor_sync(0xFFFFFFFFu, am[c][k], off);
    }
    __shared__ double red[RSE_THREADS / 32][2 + 3 * RSE_MAXM];
    if (warp < RSE_THREADS / 32 && (threadIdx.x & 31) == 0) {
        red[warp][0] = ao[0];
        red[warp][1] = ao[1];
#pragma unroll
        for (int c = 0; c < RSE_MAXM; ++c)
#pragma unroll
            for (int k = 0; k < 3; ++k)
                red[warp][2 + 3 * c + k] = am[c][k];
    }
    __syncthreads();
    // thread j < 5M: candidate j / 5, slot j % 5 of the rse_finalize layout
    if (threadIdx.x < 5 * M) {
        const int c = threadIdx.x / 5, k = threadIdx.x % 5;
        const int src = k < 2 ? k : 2 + 3 * c + (k - 2);
        double t = 0.0;
        for (int w = 0; w < RSE_THREADS / 32; ++w)
            t += red[w][src];
        part[((static_cast<int64_t>(c) * H + h) * gridDim.x + b) * NACC + k] = t;
    }
}

// One warp per head: lane j folds partials j, j+32, ... in order, then a
// fixed xor tree; lane 0 finishes the RSE.
// n_heads partial sets; set i takes its reference shift from head i % ref_heads of yo
// (the multi-candidate kernel writes set m * H + h for candidate m, head h).
template <typename T>
__global__ void rse_finalize(const T* __restrict__ yo, const double* __restrict__ part, int nblk,
                             int n_heads, int ref_heads, int64_t numel, int mode, double* __restrict__ out) {
    // launched as a programmatic dependent of the partial kernel: resident
    // early, it waits here until every partial CTA has written its sums
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int h = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (h >= n_heads)
        return;
    double a[NACC] = {0, 0, 0, 0, 0};
    for (int b = lane; b < nblk; b += 32)
#pragma unroll
        for (int k = 0; k < NACC; ++k)
            a[k] += part[(static_cast<int64_t>(h) * nblk + b) * NACC + k];
#pragma unroll
    for (int k = 0; k < NACC; ++k)
        for (int off = 16; off > 0; off >>= 1)
            a[k] += __shfl_xor_sync(0xFFFFFFFFu, a[k], off);
    if (lane != 0)
        return;
    const double K = Vec<T>::one(yo + static_cast<int64_t>(h % ref_heads) * numel);
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

namespace {
// rse_finalize as a programmatic dependent launch: its launch latency
// overlaps the partial kernel's tail (griddepcontrol.wait orders its reads
// after every partial CTA's writes)
template <typename T>
void launch_finalize(int blocks, const T* yo, const double* part, int nblk, int n_heads, int ref_heads,
                     int64_t numel, int mode, double* out, cudaStream_t stream) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(blocks));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, rse_finalize<T>, yo, part, nblk, n_heads, ref_heads, numel, mode, out);
}

// true the first time a (kernel, device) pair is seen: the smem attribute is
// then set once instead of on every launch; thread-safe (one host thread per
// GPU), a rare duplicate set is harmless
template <int KIND>
bool needs_smem_attr(const void* fn) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> seen;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    return seen.insert({fn, dev}).second;
}

template <typename T, bool LIT>
void launch_partial(const dim3& grid, const T* m, const T* o, int64_t numel, int64_t chunk, int vec_ok,
                    double* scratch, cudaStream_t stream) {
    if (needs_smem_attr<0>(reinterpret_cast<const void*>(rse_partial<T, LIT>)))
        cudaFuncSetAttribute(rse_partial<T, LIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, RSE_SMEM);
    rse_partial<T, LIT><<<grid, RSE_THREADS + 32, RSE_SMEM, stream>>>(m, o, numel, chunk, vec_ok, scratch);
}

template <typename T>
void launch_typed(const void* ym, const void* yo, int64_t n_heads, int64_t numel, int mode, double* out_dev,
                  double* scratch, int nblk, int64_t chunk, int vec_ok, cudaStream_t stream) {
    const dim3 grid(nblk, static_cast<unsigned>(n_heads));
    const T* m = static_cast<const T*>(ym);
    const T* o = static_cast<const T*>(yo);
    if (mode == 0)
        launch_partial<T, false>(grid, m, o, numel, chunk, vec_ok, scratch, stream);
    else
        launch_partial<T, true>(grid, m, o, numel, chunk, vec_ok, scratch, stream);
    const int fin_blocks = static_cast<int>((n_heads + 7) / 8);
    launch_finalize<T>(fin_blocks, o, scratch, nblk, static_cast<int>(n_heads), static_cast<int>(n_heads), numel,
                       mode, out_dev, stream);
}
}  // namespace

int rse_ctas_per_sm() { return DFA2_RSE_CTAS; }  // 3 x (64 KB ring + bars) per SM by default
int rse_multi_max() { return RSE_MAXM; }

namespace {
template <typename T>
void launch_multi_typed(const void* const* ym, int M, const void* yo, int64_t n_heads, int64_t numel, int mode,
                        double* out_dev, double* scratch, int nblk, int64_t chunk, int vec_ok, cudaStream_t stream) {
    CandPtrs<T> c{};
    for (int i = 0; i < M; ++i)
        c.p[i] = static_cast<const T*>(ym[i]);
    const dim3 grid(nblk, static_cast<unsigned>(n_heads));
    const uint32_t smem = rse_multi_smem(M);
    auto kern = mode == 0 ? rse_multi_partial<T, false> : rse_multi_partial<T, true>;
    if (needs_smem_attr<1>(reinterpret_cast<const void*>(kern)))
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, rse_multi_smem(RSE_MAXM));
    kern<<<grid, RSE_THREADS + 32, smem, stream>>>(c, M, static_cast<const T*>(yo), numel, chunk, vec_ok, scratch);
    const int sets = static_cast<int>(M * n_heads);
    launch_finalize<T>((sets + 7) / 8, static_cast<const T*>(yo), scratch, nblk, sets, static_cast<int>(n_heads),
                       numel, mode, out_dev, stream);
}
}  // namespace

// out_dev[m * n_heads + h] = RSE(ym[m] head h, yo head h) for m < M <= rse_multi_max();
// scratch holds M * n_heads * nblk * 5 doubles.
cudaError_t launch_rse_multi(const void* const* ym, int M, const void* yo, int dtype, int64_t n_heads,
                             int64_t numel, int mode, double* out_dev, double* scratch, int nblk,
                             cudaStream_t stream) {
    const int64_t W = dtype == 0 ? 8 : dtype == 1 ? 4 : 2;
    int64_t chunk = (numel + nblk - 1) / nblk;
    chunk = (chunk + W - 1) / W * W;
    int vec_ok = (numel % W) == 0 && (reinterpret_cast<uintptr_t>(yo) % 16) == 0;
    for (int i = 0; i < M; ++i)
        vec_ok = vec_ok && (reinterpret_cast<uintptr_t>(ym[i]) % 16) == 0;
    if (dtype == 0)
        launch_multi_typed<__nv_bfloat16>(ym, M, yo, n_heads, numel, mode, out_dev, scratch, nblk, chunk, vec_ok,
                                          stream);
    else if (dtype == 2)
        launch_multi_typed<double>(ym, M, yo, n_heads, numel, mode, out_dev, scratch, nblk, chunk, vec_ok, stream);
    else
        launch_multi_typed<float>(ym, M, yo, n_heads, numel, mode, out_dev, scratch, nblk, chunk, vec_ok, stream);
    return cudaGetLastError();
}

cudaError_t launch_rse(const void* ym, const void* yo, int dtype, int64_t n_heads, int64_t numel,
                       int mode, double* out_dev, double* scratch, int nblk, cudaStream_t stream) {
    const int64_t W = dtype == 0 ? 8 : dtype == 1 ? 4 : 2;
    int64_t chunk = (numel + nblk - 1) / nblk;
    chunk = (chunk + W - 1) / W * W;
    const int vec_ok = (numel % W) == 0 && (reinterpret_cast<uintptr_t>(ym) % 16) == 0 &&
                       (reinterpret_cast<uintptr_t>(yo) % 16) == 0;
    if (dtype == 0)
        launch_typed<__nv_bfloat16>(ym, yo, n_heads, numel, mode, out_dev, scratch, nblk, chunk, vec_ok, stream);
    else if (dtype == 2)
        launch_typed<double>(ym, yo, n_heads, numel, mode, out_dev, scratch, nblk, chunk, vec_ok, stream);
    else
        launch_typed<float>(ym, yo, n_heads, numel, mode, out_dev, scratch, nblk, chunk, vec_ok, stream);
    return cudaGetLastError();
}

}  // namespace dfa2k
