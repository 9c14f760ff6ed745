// dfa2_api.cpp — the reference's C++ operator API (namespace dfa2,
// include/dfa2/*.hpp) implemented on top of the C-ABI (include/dfa2c.h).
//
// A caller of /root/reference/proj/include/dfa2/*.hpp relinks against
// libdfa2_b200.so and keeps its code: host f32 Tensors go in, the work runs
// on the sm_100a kernels (bf16 inputs, fp32 accumulation), f32 Tensors come
// back. Validation and the exception taxonomy follow the reference
// (src/dispatch.cpp:11-54, inc/errors.hpp:8-45).
#include <cuda_runtime.h>

#include <algorithm>
#include <immintrin.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdlib>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "dfa2/arrow.hpp"
#include "dfa2/cache.hpp"
#include "dfa2/calibrate.hpp"
#include "dfa2/dispatch.hpp"
#include "dfa2/errors.hpp"
#include "dfa2/plan.hpp"
#include "dfa2/tensor.hpp"
#include "dfa2c.h"

#define DFA2_API __attribute__((visibility("default")))

namespace dfa2 {

namespace detail {
namespace {
constexpr std::size_t kHuge = std::size_t{2} << 20;
// Freed large buffers are kept (up to 8 / 2 GB) and handed back for the same
// rounded size: the drop-in returns a fresh output Tensor every call, and
// without reuse each call re-faults (and the kernel re-zeroes) its 208 MB.
struct BigCache {
    std::mutex mu;
    std::vector<std::pair<std::size_t, void*>> free;
    std::size_t bytes = 0;
    static constexpr std::size_t kMaxBytes = std::size_t{2} << 30;
    static constexpr std::size_t kMaxEntries = 8;
    ~BigCache() {
        for (auto& [n, p] : free)
            std::free(p);
    }
};
BigCache& big_cache() {
    static BigCache* c = new BigCache;  // never destroyed: tensors may outlive static destruction
    return *c;
}
}  // namespace

DFA2_API void* host_alloc(std::size_t bytes) {
    if (bytes < kHuge) {
        void* p = std::malloc(bytes ? bytes : 1);
        if (!p)
            throw std::bad_alloc();
        return p;
    }
    const std::size_t rounded = (bytes + kHuge - 1) / kHuge * kHuge;
    {
        BigCache& c = big_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        for (std::size_t i = 0; i < c.free.size(); ++i)
            if (c.free[i].first == rounded) {
                void* p = c.free[i].second;
                c.bytes -= rounded;
                c.free.erase(c.free.begin() + static_cast<std::ptrdiff_t>(i));
                return p;
            }
    }
    void* p = std::aligned_alloc(kHuge, rounded);
    if (!p)
        throw std::bad_alloc();
    madvise(p, rounded, MADV_HUGEPAGE);  // advisory: transparent huge pages where enabled
    return p;
}
DFA2_API void host_free(void* p, std::size_t bytes) noexcept {
    if (p && bytes >= kHuge) {
        const std::size_t rounded = (bytes + kHuge - 1) / kHuge * kHuge;
        BigCache& c = big_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        if (c.free.size() < BigCache::kMaxEntries && c.bytes + rounded <= BigCache::kMaxBytes) {
            c.free.push_back({rounded, p});
            c.bytes += rounded;
            return;
        }
    }
    std::free(p);
}
}  // namespace detail

DFA2_API void throw_status(int status) {
    if (status == DFA2C_OK)
        return;
    const std::string msg = dfa2c_last_error();
    switch (status) {
    case DFA2C_SHAPE: throw ShapeError(msg);
    case DFA2C_NONFINITE: throw NonFiniteError(msg);
    case DFA2C_FULLY_MASKED: throw FullyMaskedRowError(msg);
    case DFA2C_CACHE_MISS: throw CacheMissError(msg);
    case DFA2C_DEGENERATE: throw DegenerateReferenceError(msg);
    case DFA2C_PLAN: throw PlanValidationError(msg);
    case DFA2C_IO: throw IoError(msg);
    case DFA2C_ORACLE: throw OracleError(msg);
    default: throw DeviceError(msg);
    }
}

namespace {

void check(int status) { throw_status(status); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

int64_t shape_numel(const std::vector<int64_t>& shape) {
    int64_t n = 1;
    for (int64_t d : shape) {
        if (d < 0)
            throw ShapeError("negative dimension");
        n *= d;
    }
    return n;
}

// Owning device buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    explicit DevBuf(size_t n) : bytes(n) { cuda_check(cudaMalloc(&p, n ? n : 16), "cudaMalloc"); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// Per-thread device staging for f32 transfers (grow-only).
struct Staging {
    void* p = nullptr;
    size_t bytes = 0;
    ~Staging() {
        if (p)
            cudaFree(p);
    }
    void* get(size_t n) {
        if (n > bytes) {
            if (p)
                cuda_check(cudaFree(p), "cudaFree");
            p = nullptr;
            cuda_check(cudaMalloc(&p, n), "cudaMalloc");
            bytes = n;
        }
        return p;
    }
};

// Persistent host worker pool: parallel_for(n, fn) runs fn(0..n-1) on
// up to hardware_concurrency threads (the caller included) and returns when
// all are done. Used to fill / drain pinned staging buffers.
class HostPool {
public:
    static HostPool& get() {
        static HostPool pool;
        return pool;
    }
    size_t size() const { return workers_.size() + 1; }
    template <class F>
    void parallel_for(size_t n, F&& fn) {
        if (n <= 1 || workers_.empty()) {
            for (size_t i = 0; i < n; ++i)
                fn(i);
            return;
        }
        std::function<void(size_t)> job(std::forward<F>(fn));
        std::lock_guard<std::mutex> one_job(call_mu_);  // callers on several threads take turns
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &job;
            n_ = n;
            next_ = 0;
            done_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        run_tasks();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return done_ == n_; });
        job_ = nullptr;
    }

private:
    HostPool() {
        const size_t hw = std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), 32));
        for (size_t i = 0; i + 1 < hw; ++i)
            workers_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (std::thread& t : workers_)
            t.join();
    }
    void run_tasks() {
        for (;;) {
            size_t i;
            const std::function<void(size_t)>* job;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (!job_ || next_ >= n_)
                    return;
                i = next_++;
                job = job_;
            }
            (*job)(i);
            std::lock_guard<std::mutex> lk(mu_);
            if (++done_ == n_)
                done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_)
                    return;
                seen = gen_;
            }
            run_tasks();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(size_t)>* job_ = nullptr;
    size_t n_ = 0, next_ = 0, done_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// Parallel host memcpy / zero fill over the worker pool (1 MB tasks).
void par_memcpy(void* dst, const void* src, size_t bytes) {
    const size_t task = size_t{1} << 20, n = (bytes + task - 1) / task;
    HostPool::get().parallel_for(n, [&](size_t t) {
        const size_t a = t * task, b = std::min(bytes, a + task);
        std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    });
}
void par_memset0(void* dst, size_t bytes) {
    const size_t task = size_t{1} << 20, n = (bytes + task - 1) / task;
    HostPool::get().parallel_for(n, [&](size_t t) {
        const size_t a = t * task, b = std::min(bytes, a + task);
        std::memset(static_cast<char*>(dst) + a, 0, b - a);
    });
}

// One contiguous host <-> device piece of a transfer.
struct Seg {
    const void* src;
    void* dst;
    size_t bytes;
};

// f32 -> bf16, round to nearest even (NaN -> 0x7FFF), bitwise what the
// device conversion (__float2bfloat16_rn, dfa2c_convert) gives.
void round_f32_to_bf16_scalar(const float* src, uint16_t* dst, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t u;
        std::memcpy(&u, src + i, 4);
        const bool nan = (u & 0x7FFFFFFFu) > 0x7F800000u;
        const uint32_t r = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
        dst[i] = nan ? uint16_t{0x7FFF} : static_cast<uint16_t>(r);
    }
}
void widen_bf16_to_f32_scalar(const uint16_t* src, float* dst, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        const uint32_t u = static_cast<uint32_t>(src[i]) << 16;
        std::memcpy(dst + i, &u, 4);
    }
}
// The same conversions 16 lanes at a time (AVX-512F/BW, picked at run time):
// the host side of the drop-in's f32 calling convention is bound by these
// passes over the tensors.
__attribute__((target("avx512f,avx512bw"))) void round_f32_to_bf16_avx512(const float* src, uint16_t* dst,
                                                                         size_t n) {
    const __m512i bias = _mm512_set1_epi32(0x7FFF), one = _mm512_set1_epi32(1);
    const __m512i absmask = _mm512_set1_epi32(0x7FFFFFFF), inf = _mm512_set1_epi32(0x7F800000);
    const __m512i qnan = _mm512_set1_epi32(0x7FFF);
    size_t i = 0;
    // streaming (non-temporal) stores once dst is 32-byte aligned: the pinned
    // chunk is read next by the DMA engine, not by this core
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31u); ++i)
        round_f32_to_bf16_scalar(src + i, dst + i, 1);
    for (; i + 16 <= n; i += 16) {
        const __m512i u = _mm512_loadu_si512(src + i);
        const __m512i lsb = _mm512_and_si512(_mm512_srli_epi32(u, 16), one);
        __m512i r = _mm512_srli_epi32(_mm512_add_epi32(_mm512_add_epi32(u, bias), lsb), 16);
        const __mmask16 nan = _mm512_cmpgt_epu32_mask(_mm512_and_si512(u, absmask), inf);
        r = _mm512_mask_mov_epi32(r, nan, qnan);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), _mm512_cvtepi32_epi16(r));
    }
    _mm_sfence();
    round_f32_to_bf16_scalar(src + i, dst + i, n - i);
}
__attribute__((target("avx512f,avx512bw"))) void widen_bf16_to_f32_avx512(const uint16_t* src, float* dst,
                                                                         size_t n) {
    size_t i = 0;
    // streaming stores into the caller's f32 tensor (no read-for-ownership of
    // the destination lines) once it is 64-byte aligned
    for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 63u); ++i)
        widen_bf16_to_f32_scalar(src + i, dst + i, 1);
    for (; i + 16 <= n; i += 16) {
        const __m256i h = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
        _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i), _mm512_slli_epi32(_mm512_cvtepu16_epi32(h), 16));
    }
    _mm_sfence();
    widen_bf16_to_f32_scalar(src + i, dst + i, n - i);
}
bool have_avx512bw() {
    static const bool ok = [] {
        __builtin_cpu_init();
        return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
    }();
    return ok;
}
void round_f32_to_bf16(const float* src, uint16_t* dst, size_t n) {
    if (have_avx512bw())
        round_f32_to_bf16_avx512(src, dst, n);
    else
        round_f32_to_bf16_scalar(src, dst, n);
}
void widen_bf16_to_f32(const uint16_t* src, float* dst, size_t n) {
    if (have_avx512bw())
        widen_bf16_to_f32_avx512(src, dst, n);
    else
        widen_bf16_to_f32_scalar(src, dst, n);
}

// Host <-> device mover for the reference's pageable host tensors: the
// segments are streamed in 32 MB chunks through three pinned buffers, each
// filled / drained by the worker pool while the neighbouring chunks are in
// flight on a copy stream. Synchronous for the caller, like the reference.
class HostMover {
public:
#ifndef DFA2_MOVER_CHUNK_MB
#define DFA2_MOVER_CHUNK_MB 32
#endif
#ifndef DFA2_MOVER_BUFS
#define DFA2_MOVER_BUFS 3
#endif
#ifndef DFA2_MOVER_TASK_KB
#define DFA2_MOVER_TASK_KB 1024
#endif
    static constexpr size_t kChunk = size_t{DFA2_MOVER_CHUNK_MB} << 20;
    static constexpr int kBufs = DFA2_MOVER_BUFS;
    ~HostMover() {
        for (int i = 0; i < kBufs; ++i) {
            if (pin_[i])
                cudaFreeHost(pin_[i]);
            if (ev_[i])
                cudaEventDestroy(ev_[i]);
        }
        if (st_)
            cudaStreamDestroy(st_);
    }
    // kRound: host f32 -> bf16 (round to nearest even) on the way up, bf16 ->
    // f32 on the way down, done by the pool while filling / draining the
    // pinned chunks; Seg::bytes then counts the bf16 (device-side) bytes.
    enum Mode { kCopy, kRound };
    void up(const void* src, void* dst_dev, size_t bytes) { move({Seg{src, dst_dev, bytes}}, true); }
    void down(const void* src_dev, void* dst, size_t bytes) { move({Seg{src_dev, dst, bytes}}, false); }
    // on_issued(hi, copy_stream): called after the DMAs of the flat bytes
    // [0, hi) have been enqueued (uploads), so a caller can order work on
    // another stream after them (an event on copy_stream) while the pool
    // keeps filling the next chunks.
    using Issued = std::function<void(size_t, cudaStream_t)>;
    void move(const std::vector<Seg>& segs, bool to_device, Mode mode = kCopy, const Issued& on_issued = {}) {
        init();
        cuda_check(cudaDeviceSynchronize(), "sync");  // device-side producers of the sources are done
        // the transfer as a flat byte range [0, total) over the segments
        std::vector<size_t> start(segs.size() + 1, 0);
        for (size_t i = 0; i < segs.size(); ++i)
            start[i + 1] = start[i] + segs[i].bytes;
        const size_t total = start.back();
        // pieces of [lo, hi): (segment, offset in segment, length)
        auto pieces = [&](size_t lo, size_t hi, auto&& f) {
            size_t i = static_cast<size_t>(std::upper_bound(start.begin(), start.end(), lo) - start.begin()) - 1;
            for (size_t pos = lo; pos < hi && i < segs.size(); ++i) {
                const size_t a = std::max(pos, start[i]), b = std::min(hi, start[i + 1]);
                if (b > a)
                    f(segs[i], a - start[i], b - a, a - lo);
                pos = b;
            }
        };
        HostPool& pool = HostPool::get();
        auto host_copy = [&](char* pinned, size_t lo, size_t hi, bool into_pinned) {
            // split the chunk into ~1 MB tasks over the pool
            const size_t len = hi - lo, task = size_t{DFA2_MOVER_TASK_KB} << 10;
            const size_t ntask = (len + task - 1) / task;
            pool.parallel_for(ntask, [&](size_t t) {
                const size_t a = lo + t * task, b = std::min(hi, a + task);
                pieces(a, b, [&](const Seg& sg, size_t off, size_t n, size_t at) {
                    char* pin = pinned + (a - lo) + at;
                    if (mode == kRound) {
                        if (into_pinned)
                            round_f32_to_bf16(static_cast<const float*>(sg.src) + off / 2,
                                              reinterpret_cast<uint16_t*>(pin), n / 2);
                        else
                            widen_bf16_to_f32(reinterpret_cast<const uint16_t*>(pin),
                                              static_cast<float*>(sg.dst) + off / 2, n / 2);
                    } else if (into_pinned) {
                        std::memcpy(pin, static_cast<const char*>(sg.src) + off, n);
                    } else {
                        std::memcpy(static_cast<char*>(sg.dst) + off, pin, n);
                    }
                });
            });
        };
        bool pending[kBufs] = {};
        size_t plo[kBufs] = {}, phi[kBufs] = {};
        int b = 0;
        for (size_t lo = 0; lo < total; lo += kChunk, b = (b + 1) % kBufs) {
            const size_t hi = std::min(total, lo + kChunk);
            if (pending[b]) {  // this pinned buffer's previous transfer must finish first
                cuda_check(cudaEventSynchronize(ev_[b]), "event");
                if (!to_device)
                    host_copy(pin_[b], plo[b], phi[b], false);
            }
            if (to_device) {
                host_copy(pin_[b], lo, hi, true);
                pieces(lo, hi, [&](const Seg& sg, size_t off, size_t n, size_t at) {
                    cuda_check(cudaMemcpyAsync(static_cast<char*>(sg.dst) + off, pin_[b] + at, n,
                                               cudaMemcpyHostToDevice, st_),
                               "upload");
                });
                if (on_issued)
                    on_issued(hi, st_);
            } else {
                pieces(lo, hi, [&](const Seg& sg, size_t off, size_t n, size_t at) {
                    cuda_check(cudaMemcpyAsync(pin_[b] + at, static_cast<const char*>(sg.src) + off, n,
                                               cudaMemcpyDeviceToHost, st_),
                               "download");
                });
            }
            cuda_check(cudaEventRecord(ev_[b], st_), "event");
            pending[b] = true;
            plo[b] = lo;
            phi[b] = hi;
        }
        for (int j = 0; j < kBufs; ++j) {  // drain, oldest first
            const int i = (b + j) % kBufs;
            if (!pending[i])
                continue;
            cuda_check(cudaEventSynchronize(ev_[i]), "event");
            if (!to_device)
                host_copy(pin_[i], plo[i], phi[i], false);
        }
    }

private:
    void init() {
        if (st_)
            return;
        cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
        for (int i = 0; i < kBufs; ++i) {
            void* p = nullptr;
            cuda_check(cudaMallocHost(&p, kChunk), "cudaMallocHost");
            pin_[i] = static_cast<char*>(p);
            cuda_check(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming), "event");
        }
    }
    cudaStream_t st_ = nullptr;
    char* pin_[kBufs] = {};
    cudaEvent_t ev_[kBufs] = {};
};
thread_local HostMover g_mover;

// f32 host values -> bf16 device buffer: the f32 bytes cross PCIe through
// pinned chunks and are rounded to bf16 on the device (dfa2c_convert).
void upload_bf16(const float* src, int64_t n, void* dst) {
    if (n <= 0)
        return;
    g_mover.move({Seg{src, dst, static_cast<size_t>(n) * 2}}, true, HostMover::kRound);
}

// Several (f32 host source, element count, bf16 device destination) pieces
// in ONE pipelined transfer.
struct UpPiece {
    const float* src;
    int64_t n;
    void* dst;
};
void upload_bf16_many(const std::vector<UpPiece>& ps, const HostMover::Issued& on_issued = {}) {
    // rounded to bf16 by the pool while it fills the pinned chunks: half the
    // PCIe bytes of an f32 upload, and no device-side conversion
    std::vector<Seg> segs;
    for (const UpPiece& p : ps)
        if (p.n > 0)
            segs.push_back(Seg{p.src, p.dst, static_cast<size_t>(p.n) * 2});
    if (!segs.empty())
        g_mover.move(segs, true, HostMover::kRound, on_issued);
}

void download_bf16(const void* src, int64_t n, float* dst) {
    if (n <= 0)
        return;
    // bf16 crosses PCIe; the pool widens it to f32 while draining the chunks
    g_mover.move({Seg{src, dst, static_cast<size_t>(n) * 2}}, false, HostMover::kRound);
}

// f32 view of a tensor (f64 narrowed).
std::vector<float> as_f32(const Tensor& t) {
    if (t.dtype() == Dtype::f32)
        return std::vector<float>(t.f32(), t.f32() + t.numel());
    std::vector<float> v(static_cast<size_t>(t.numel()));
    for (int64_t i = 0; i < t.numel(); ++i)
        v[i] = static_cast<float>(t.f64()[i]);
    return v;
}

dfa2c_dims cdims(const AttentionDims& d) {
    return dfa2c_dims{d.n_heads, d.head_dim, d.n_visual, d.n_text,
                      d.order == TokenOrder::visual_first ? DFA2C_VISUAL_FIRST : DFA2C_TEXT_FIRST};
}

void plan_arrays(const LayerPlan& plan, std::vector<int32_t>& kinds, std::vector<int64_t>& wins) {
    kinds.clear();
    wins.clear();
    for (const HeadStrategy& s : plan.strategies) {
        kinds.push_back(s.kind == StrategyKind::full ? DFA2C_FULL
                        : s.kind == StrategyKind::arrow ? DFA2C_ARROW
                                                        : DFA2C_CACHED);
        wins.push_back(s.window_blocks);
    }
}

}  // namespace

// ---------------------------------------------------------------- Tensor
DFA2_API Tensor Tensor::zeros(std::vector<int64_t> shape, Dtype dt) {
    Tensor t;
    const int64_t n = shape_numel(shape);
    t.shape_ = std::move(shape);
    t.dtype_ = dt;
    if (dt == Dtype::f32) {
        t.f32_.resize(static_cast<size_t>(n));
        par_memset0(t.f32_.data(), static_cast<size_t>(n) * sizeof(float));
    } else {
        t.f64_.resize(static_cast<size_t>(n));
        par_memset0(t.f64_.data(), static_cast<size_t>(n) * sizeof(double));
    }
    return t;
}
DFA2_API Tensor Tensor::from_f32(std::vector<int64_t> shape, std::vector<float> data) {
    if (shape_numel(shape) != static_cast<int64_t>(data.size()))
        throw ShapeError("data length does not match shape");
    Tensor t;
    t.shape_ = std::move(shape);
    t.f32_.resize(data.size());
    par_memcpy(t.f32_.data(), data.data(), data.size() * sizeof(float));
    return t;
}
DFA2_API Tensor Tensor::from_f64(std::vector<int64_t> shape, std::vector<double> data) {
    if (shape_numel(shape) != static_cast<int64_t>(data.size()))
        throw ShapeError("data length does not match shape");
    Tensor t;
    t.shape_ = std::move(shape);
    t.dtype_ = Dtype::f64;
    t.f64_.resize(data.size());
    par_memcpy(t.f64_.data(), data.data(), data.size() * sizeof(double));
    return t;
}
DFA2_API Tensor Tensor::uninitialized_f32(std::vector<int64_t> shape) {
    Tensor t;
    const int64_t n = shape_numel(shape);
    t.shape_ = std::move(shape);
    t.f32_.resize(static_cast<size_t>(n));
    return t;
}
DFA2_API int64_t Tensor::dim(int64_t i) const {
    if (i < 0 || i >= ndim())
        throw ShapeError("dimension index out of range");
    return shape_[static_cast<size_t>(i)];
}
DFA2_API int64_t Tensor::numel() const {
    return dtype_ == Dtype::f32 ? static_cast<int64_t>(f32_.size()) : static_cast<int64_t>(f64_.size());
}
DFA2_API float* Tensor::f32() {
    if (dtype_ != Dtype::f32)
        throw ShapeError("tensor is not float32");
    return f32_.data();
}
DFA2_API const float* Tensor::f32() const {
    if (dtype_ != Dtype::f32)
        throw ShapeError("tensor is not float32");
    return f32_.data();
}
DFA2_API double* Tensor::f64() {
    if (dtype_ != Dtype::f64)
        throw ShapeError("tensor is not float64");
    return f64_.data();
}
DFA2_API const double* Tensor::f64() const {
    if (dtype_ != Dtype::f64)
        throw ShapeError("tensor is not float64");
    return f64_.data();
}
DFA2_API Tensor Tensor::to_f64() const {
    if (dtype_ == Dtype::f64)
        return *this;
    Tensor t = zeros(shape_, Dtype::f64);
    for (size_t i = 0; i < f32_.size(); ++i)
        t.f64_[i] = static_cast<double>(f32_[i]);
    return t;
}
DFA2_API bool Tensor::operator==(const Tensor& o) const {
    if (dtype_ != o.dtype_ || shape_ != o.shape_)
        return false;
    if (dtype_ == Dtype::f32)
        return std::memcmp(f32_.data(), o.f32_.data(), f32_.size() * sizeof(float)) == 0;
    return std::memcmp(f64_.data(), o.f64_.data(), f64_.size() * sizeof(double)) == 0;
}
DFA2_API bool Tensor::all_finite() const {
    for (float v : f32_)
        if (!std::isfinite(v))
            return false;
    for (double v : f64_)
        if (!std::isfinite(v))
            return false;
    return true;
}
DFA2_API void Tensor::check_finite(const char* what) const {
    if (!all_finite())
        throw NonFiniteError(std::string(what) + ": non-finite scalar");
}

DFA2_API void AttentionDims::validate() const {
    if (n_heads < 1 || head_dim < 1)
        throw ShapeError("n_heads and head_dim must be >= 1");
    if (n_visual < 1 || n_text < 0)
        throw ShapeError("need n_visual >= 1 and n_text >= 0");
}

DFA2_API Tensor head_slice(const Tensor& x, int64_t head) {
    if (x.ndim() != 3)
        throw ShapeError("head_slice expects [H, N, d]");
    if (head < 0 || head >= x.dim(0))
        throw ShapeError("head index out of range");
    const int64_t n = x.dim(1), d = x.dim(2);
    Tensor s = Tensor::zeros({n, d}, x.dtype());
    if (x.dtype() == Dtype::f32)
        std::memcpy(s.f32(), x.f32() + head * n * d, sizeof(float) * n * d);
    else
        std::memcpy(s.f64(), x.f64() + head * n * d, sizeof(double) * n * d);
    return s;
}

DFA2_API void copy_into_head(Tensor& dst, int64_t head, const Tensor& src) {
    if (dst.ndim() != 3 || src.ndim() != 2)
        throw ShapeError("copy_into_head expects [H, N, d] and [N, d]");
    if (dst.dtype() != src.dtype())
        throw ShapeError("copy_into_head dtype mismatch");
    if (src.dim(0) != dst.dim(1) || src.dim(1) != dst.dim(2))
        throw ShapeError("copy_into_head shape mismatch");
    if (head < 0 || head >= dst.dim(0))
        throw ShapeError("head index out of range");
    const int64_t n = dst.dim(1), d = dst.dim(2);
    if (dst.dtype() == Dtype::f32)
        std::memcpy(dst.f32() + head * n * d, src.f32(), sizeof(float) * n * d);
    else
        std::memcpy(dst.f64() + head * n * d, src.f64(), sizeof(double) * n * d);
}

// ---------------------------------------------------------------- masks
DFA2_API BlockMask BlockMask::all_active(int64_t seq_len, int64_t block_size) {
    if (block_size < 1)
        throw ShapeError("block_size must be >= 1");
    if (seq_len < 1)
        throw ShapeError("seq_len must be >= 1");
    BlockMask m;
    m.block_size = block_size;
    m.seq_len = seq_len;
    m.n_query_blocks = (seq_len + block_size - 1) / block_size;
    m.n_key_blocks = m.n_query_blocks;
    m.active.assign(static_cast<size_t>(m.n_query_blocks * m.n_key_blocks), 1);
    return m;
}
DFA2_API int64_t BlockMask::block_len(int64_t i) const { return std::min(block_size, seq_len - i * block_size); }
DFA2_API int64_t BlockMask::active_positions() const {
    int64_t ap = 0;
    check(dfa2c_mask_stats(active.data(), seq_len, block_size, 1, &ap, nullptr, nullptr));
    return ap;
}
DFA2_API bool BlockMask::row_has_active(int64_t i) const {
    for (int64_t j = 0; j < n_key_blocks; ++j)
        if (is_active(i, j))
            return true;
    return false;
}

DFA2_API BlockMask build_arrow_mask(const ArrowSpec& spec) {
    const dfa2c_dims d = cdims(spec.dims);
    int64_t nb = 0;
    check(dfa2c_arrow_mask(&d, spec.block_size, spec.window_blocks, nullptr, &nb));
    BlockMask m;
    m.block_size = spec.block_size;
    m.seq_len = spec.dims.seq_len();
    m.n_query_blocks = m.n_key_blocks = nb;
    m.active.resize(static_cast<size_t>(nb * nb));
    check(dfa2c_arrow_mask(&d, spec.block_size, spec.window_blocks, m.active.data(), &nb));
    return m;
}
DFA2_API int64_t flops_count(const BlockMask& mask, int64_t head_dim) {
    int64_t f = 0;
    check(dfa2c_mask_stats(mask.active.data(), mask.seq_len, mask.block_size, head_dim, nullptr, &f, nullptr));
    return f;
}
DFA2_API int64_t dense_flops(int64_t seq_len, int64_t head_dim) { return dfa2c_dense_flops(seq_len, head_dim); }
DFA2_API double sparsity_ratio(const BlockMask& mask) {
    double s = 0.0;
    check(dfa2c_mask_stats(mask.active.data(), mask.seq_len, mask.block_size, 1, nullptr, nullptr, &s));
    return s;
}

// ---------------------------------------------------------------- attention
namespace {
void sparse_heads(const float* q, const float* k, const float* v, float* out, int64_t heads, int64_t n, int64_t d,
                  const BlockMask* mask) {
    const int64_t numel = heads * n * d;
    DevBuf dq(numel * 2), dk(numel * 2), dv(numel * 2), dout(numel * 2);
    upload_bf16(q, numel, dq.p);
    upload_bf16(k, numel, dk.p);
    upload_bf16(v, numel, dv.p);
    if (mask) {
        if (mask->seq_len != n)
            throw ShapeError("mask sequence length disagrees with tensors");
        check(dfa2c_sparse_attention_forward(dq.p, dk.p, dv.p, dout.p, heads, n, d, mask->active.data(),
                                             mask->block_size, nullptr));
    } else {
        check(dfa2c_dense_attention_forward(dq.p, dk.p, dv.p, dout.p, heads, n, d, nullptr));
    }
    download_bf16(dout.p, numel, out);
}
}  // namespace

DFA2_API void sparse_attention_forward(const float* q, const float* k, const float* v, float* out, int64_t n,
                                       int64_t d, const BlockMask& mask, bool /*parallel*/) {
    sparse_heads(q, k, v, out, 1, n, d, &mask);
}

DFA2_API Tensor sparse_attention_forward(const Tensor& q, const Tensor& k, const Tensor& v, const BlockMask& mask) {
    if (q.ndim() != 2 || k.ndim() != 2 || v.ndim() != 2)
        throw ShapeError("sparse attention expects per-head [N, d] tensors");
    if (q.shape() != k.shape() || q.shape() != v.shape())
        throw ShapeError("q/k/v shapes disagree");
    if (q.dtype() != Dtype::f32)
        throw ShapeError("sparse attention runs in float32");
    Tensor out = Tensor::zeros(q.shape(), Dtype::f32);
    sparse_attention_forward(q.f32(), k.f32(), v.f32(), out.f32(), q.dim(0), q.dim(1), mask);
    return out;
}

DFA2_API void dense_tiled_attention(const float* q, const float* k, const float* v, float* out, int64_t n, int64_t d,
                                    int64_t block_size, bool /*parallel*/) {
    if (block_size < 1)
        throw ShapeError("block_size must be >= 1");
    sparse_heads(q, k, v, out, 1, n, d, nullptr);
}

namespace {
// the reference's ground truth at the operands' own precision (SIMT kernel)
void reference_heads(const void* q, const void* k, const void* v, void* out, bool f64, int64_t heads, int64_t n,
                     int64_t d, const BlockMask* mask) {
    if (mask && mask->seq_len != n)
        throw ShapeError("mask sequence length disagrees with tensors");
    const size_t bytes = static_cast<size_t>(heads * n * d) * (f64 ? 8 : 4);
    DevBuf dq(bytes), dk(bytes), dv(bytes), dout(bytes);
    cuda_check(cudaMemcpy(dq.p, q, bytes, cudaMemcpyHostToDevice), "attention_reference upload");
    cuda_check(cudaMemcpy(dk.p, k, bytes, cudaMemcpyHostToDevice), "attention_reference upload");
    cuda_check(cudaMemcpy(dv.p, v, bytes, cudaMemcpyHostToDevice), "attention_reference upload");
    check(dfa2c_attention_reference(dq.p, dk.p, dv.p, dout.p, f64 ? DFA2C_F64 : DFA2C_F32, heads, n, d,
                                    mask ? mask->active.data() : nullptr, mask ? mask->block_size : 0, nullptr));
    cuda_check(cudaMemcpy(out, dout.p, bytes, cudaMemcpyDeviceToHost), "attention_reference download");
}
}  // namespace

DFA2_API Tensor attention_reference(const Tensor& q, const Tensor& k, const Tensor& v, const BlockMask* mask) {
    if (q.ndim() != 3 || k.ndim() != 3 || v.ndim() != 3)
        throw ShapeError("attention expects [H, N, d] tensors");
    if (q.shape() != k.shape() || q.shape() != v.shape())
        throw ShapeError("q/k/v shapes disagree");
    if (q.dtype() != k.dtype() || q.dtype() != v.dtype())
        throw ShapeError("q/k/v dtypes disagree");
    if (mask && mask->seq_len != q.dim(1))
        throw ShapeError("mask sequence length disagrees with tensors");
    q.check_finite("attention q");
    k.check_finite("attention k");
    v.check_finite("attention v");
    const bool f64 = q.dtype() == Dtype::f64;
    Tensor out = Tensor::zeros(q.shape(), q.dtype());
    if (f64)
        reference_heads(q.f64(), k.f64(), v.f64(), out.f64(), true, q.dim(0), q.dim(1), q.dim(2), mask);
    else
        reference_heads(q.f32(), k.f32(), v.f32(), out.f32(), false, q.dim(0), q.dim(1), q.dim(2), mask);
    out.check_finite("attention result");
    return out;
}

DFA2_API void attention_reference_head_f32(const float* q, const float* k, const float* v, float* out, int64_t n,
                                           int64_t d, const BlockMask* mask) {
    reference_heads(q, k, v, out, false, 1, n, d, mask);
}

// ---------------------------------------------------------------- cache
DFA2_API HeadCache::~HeadCache() { release_device(); }

void HeadCache::release_device() {
    if (dev_)
        dfa2c_cache_destroy(dev_);
    dev_ = nullptr;
    heads_ = n_ = d_ = layers_ = 0;
}

DFA2_API HeadCache::HeadCache(const HeadCache& other) { *this = other; }

DFA2_API HeadCache& HeadCache::operator=(const HeadCache& other) {
    if (this == &other)
        return *this;
    // deep copy: every entry as a host f32 tensor (device-only slots read
    // back first), uploaded to this cache's own slots on first GPU use
    std::map<std::pair<int64_t, int64_t>, Slot> copy;
    for (const auto& kv : other.slots_) {
        Slot s;
        s.produced_at = kv.second.produced_at;
        s.host = other.fetch(kv.first.first, kv.first.second);
        s.host_fresh = true;
        s.on_device = false;
        copy.emplace(kv.first, std::move(s));
    }
    release_device();
    slots_ = std::move(copy);
    return *this;
}

DFA2_API HeadCache::HeadCache(HeadCache&& other) noexcept { *this = std::move(other); }

DFA2_API HeadCache& HeadCache::operator=(HeadCache&& other) noexcept {
    if (this == &other)
        return *this;
    release_device();
    slots_ = std::move(other.slots_);
    other.slots_.clear();
    dev_ = other.dev_;
    heads_ = other.heads_;
    n_ = other.n_;
    d_ = other.d_;
    layers_ = other.layers_;
    other.dev_ = nullptr;
    other.heads_ = other.n_ = other.d_ = other.layers_ = 0;
    return *this;
}

DFA2_API dfa2c_cache* HeadCache::bind(int64_t n_heads, int64_t n, int64_t d) const {
    if (dev_) {
        if (n_heads != heads_ || n != n_ || d != d_)
            throw ShapeError("cached output shape disagrees with dims");
    } else {
        int64_t layers = 1;
        for (const auto& kv : slots_)
            layers = std::max(layers, kv.first.first + 1);
        check(dfa2c_cache_create(layers, n_heads, 1, n, d, &dev_));
        heads_ = n_heads;
        n_ = n;
        d_ = d;
        layers_ = layers;
    }
    for (auto& kv : slots_) {
        Slot& s = kv.second;
        if (s.on_device)
            continue;
        if (kv.first.second >= heads_)
            throw ShapeError("cached head index outside the layer's heads");
        if (s.host.ndim() != 2 || s.host.dim(0) != n || s.host.dim(1) != d)
            throw ShapeError("cached output shape disagrees with dims");
        DevBuf tmp(static_cast<size_t>(n * d) * 2);
        upload_bf16(s.host.f32(), n * d, tmp.p);
        check(dfa2c_cache_store(dev_, kv.first.first, kv.first.second, tmp.p, s.produced_at, nullptr));
        cuda_check(cudaDeviceSynchronize(), "cache upload");
        s.on_device = true;
        s.host_fresh = false;
    }
    return dev_;
}

DFA2_API void HeadCache::store(int64_t layer, int64_t head, Tensor output, int64_t t) {
    if (output.ndim() != 2)
        throw ShapeError("cache entries are per-head [N, d] tensors");
    Slot& s = slots_[{layer, head}];
    s.produced_at = t;
    s.host = output.dtype() == Dtype::f32 ? std::move(output)
                                          : Tensor::from_f32(output.shape(), as_f32(output));
    s.on_device = false;
    s.host_fresh = true;
    if (dev_)
        bind(heads_, n_, d_);  // upload now (bf16 slot)
}

DFA2_API HeadCache::Slot& HeadCache::slot(int64_t layer, int64_t head) const {
    const auto it = slots_.find({layer, head});
    if (it == slots_.end())
        throw CacheMissError("no cached output for layer " + std::to_string(layer) + ", head " + std::to_string(head));
    return it->second;
}

DFA2_API const Tensor& HeadCache::fetch(int64_t layer, int64_t head) const {
    Slot& s = slot(layer, head);
    if (!s.host_fresh) {
        DevBuf tmp(static_cast<size_t>(n_ * d_) * 2);
        check(dfa2c_cache_fetch(dev_, layer, head, tmp.p, nullptr));
        s.host = Tensor::zeros({n_, d_});
        download_bf16(tmp.p, n_ * d_, s.host.f32());
        s.host_fresh = true;
    }
    return s.host;
}

DFA2_API bool HeadCache::has(int64_t layer, int64_t head) const { return slots_.count({layer, head}) != 0; }
DFA2_API int64_t HeadCache::produced_at(int64_t layer, int64_t head) const { return slot(layer, head).produced_at; }
DFA2_API int64_t HeadCache::staleness(int64_t layer, int64_t head, int64_t t) const {
    return t - slot(layer, head).produced_at;
}
DFA2_API void HeadCache::clear() {
    slots_.clear();
    if (dev_)
        check(dfa2c_cache_clear(dev_));
}
DFA2_API int64_t HeadCache::size() const { return static_cast<int64_t>(slots_.size()); }

// Access for multi_strategy_attention / influence_for_layer.
class CacheAccess {
public:
    static void committed(HeadCache& c, int64_t layer, int64_t head, int64_t t) {
        HeadCache::Slot& s = c.slots_[{layer, head}];
        s.produced_at = t;
        s.on_device = true;
        s.host_fresh = false;
    }
};

// ---------------------------------------------------------------- dispatch
DFA2_API Tensor multi_strategy_attention(const Tensor& q, const Tensor& k, const Tensor& v, const LayerPlan& plan,
                                         HeadCache& cache, int64_t layer, int64_t t, const AttentionDims& dims,
                                         int64_t block_size) {
    // validate_plan_inputs (src/dispatch.cpp:11-26)
    dims.validate();
    if (block_size < 1)
        throw ShapeError("block_size must be >= 1");
    if (q.ndim() != 3 || q.shape() != k.shape() || q.shape() != v.shape())
        throw ShapeError("q/k/v must be identical [H, N, d] tensors");
    if (q.dtype() != Dtype::f32 || k.dtype() != Dtype::f32 || v.dtype() != Dtype::f32)
        throw ShapeError("multi-strategy attention runs in float32");
    if (q.dim(0) != dims.n_heads || q.dim(1) != dims.seq_len() || q.dim(2) != dims.head_dim)
        throw ShapeError("tensor shape disagrees with dims");
    if (plan.n_heads() != dims.n_heads)
        throw ShapeError("plan must assign exactly one strategy per head");
    // cached heads checked before any compute (src/dispatch.cpp:38-48)
    for (int64_t h = 0; h < plan.n_heads(); ++h)
        if (plan.strategies[h].kind == StrategyKind::cached && !cache.has(layer, h))
            throw CacheMissError("plan marks head " + std::to_string(h) + " Cached before it ever computed");
    const int64_t H = dims.n_heads, n = dims.seq_len(), d = dims.head_dim, numel = H * n * d;
    dfa2c_cache* dev = cache.bind(H, n, d);
    thread_local Staging sq, sk, sv, so;  // grow-only device buffers, reused call to call
    void* dq = sq.get(static_cast<size_t>(numel) * 2);
    void* dk = sk.get(static_cast<size_t>(numel) * 2);
    void* dv = sv.get(static_cast<size_t>(numel) * 2);
    void* dout = so.get(static_cast<size_t>(numel) * 2);
    // only computed heads' inputs cross PCIe (a Cached head reads its slot),
    // in ONE pipelined transfer ordered by head group: as soon as a group's
    // last chunk is enqueued, the group's launch is enqueued behind it (an
    // event on the copy stream), so the GPU computes group g while the host
    // rounds group g+1 and only the last group's compute is exposed
    const int64_t hs = n * d;
    std::vector<int32_t> kinds;
    std::vector<int64_t> wins;
    plan_arrays(plan, kinds, wins);
    const dfa2c_dims cd = cdims(dims);
    std::vector<int64_t> computed;
    for (int64_t h = 0; h < H; ++h)
        if (plan.strategies[h].kind != StrategyKind::cached)
            computed.push_back(h);
    constexpr size_t kGroups = 4;
    const size_t G = std::max<size_t>(1, std::min(kGroups, computed.size()));
    std::vector<UpPiece> ups;
    std::vector<size_t> group_end(G, 0);  // flat (bf16) bytes through each group
    std::vector<std::vector<int32_t>> group_kinds(G, kinds);
    size_t flat = 0;
    for (size_t g = 0; g < G; ++g) {
        std::vector<bool> in(static_cast<size_t>(H), g == 0);  // group 0 also copies the Cached heads
        for (int64_t h = 0; h < H; ++h)
            if (g == 0 && plan.strategies[h].kind != StrategyKind::cached)
                in[static_cast<size_t>(h)] = false;
        for (size_t i = computed.size() * g / G; i < computed.size() * (g + 1) / G; ++i) {
            const int64_t h = computed[i];
            in[static_cast<size_t>(h)] = true;
            for (const auto& [src, dst] :
                 {std::pair<const float*, void*>{q.f32(), dq}, {k.f32(), dk}, {v.f32(), dv}}) {
                ups.push_back({src + h * hs, hs, static_cast<char*>(dst) + h * hs * 2});
                flat += static_cast<size_t>(hs) * 2;
            }
        }
        group_end[g] = flat;
        for (int64_t h = 0; h < H; ++h)
            if (!in[static_cast<size_t>(h)])
                group_kinds[g][h] |= DFA2C_SKIP;
    }
    thread_local cudaEvent_t ev_group = [] {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        return e;
    }();
    size_t next = 0;
    auto launch_ready = [&](size_t issued, cudaStream_t copy_stream) {
        while (next < G && group_end[next] <= issued) {
            if (copy_stream) {
                cuda_check(cudaEventRecord(ev_group, copy_stream), "event");
                cuda_check(cudaStreamWaitEvent(nullptr, ev_group, 0), "wait");
            }
            check(dfa2c_mha_forward(dq, dk, dv, 1, &cd, block_size, group_kinds[next].data(), wins.data(), dev,
                                    layer, t, dout, nullptr));
            ++next;
        }
    };
    const bool prof = std::getenv("DFA2_HOST_PROFILE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    upload_bf16_many(ups, launch_ready);
    launch_ready(flat, nullptr);  // groups without uploads (all-Cached layers); move() already synced
    const auto t1 = now();
    if (prof) cudaDeviceSynchronize();
    const auto t2 = now();
    Tensor out = Tensor::uninitialized_f32(q.shape());  // the download writes every element
    const auto t3 = now();
    download_bf16(dout, numel, out.f32());
    const auto t4 = now();
    if (prof)
        std::fprintf(stderr, "[dfa2 host] upload + launches %.2f ms, rest of the kernels %.2f ms, out alloc %.2f ms, "
                     "download %.2f ms\n", ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
    for (int64_t h = 0; h < H; ++h)
        if (plan.strategies[h].kind != StrategyKind::cached)
            CacheAccess::committed(cache, layer, h, t);
    return out;
}

DFA2_API int64_t plan_flops(const LayerPlan& plan, const AttentionDims& dims, int64_t block_size) {
    if (plan.n_heads() != dims.n_heads)
        throw ShapeError("plan must assign exactly one strategy per head");
    std::vector<int32_t> kinds;
    std::vector<int64_t> wins;
    plan_arrays(plan, kinds, wins);
    const dfa2c_dims cd = cdims(dims);
    int64_t f = 0;
    check(dfa2c_plan_flops(&cd, block_size, kinds.data(), wins.data(), &f));
    return f;
}

// ---------------------------------------------------------------- calibration
DFA2_API double rse(const Tensor& y_m, const Tensor& y_o, RseMode mode) {
    if (y_m.shape() != y_o.shape() || y_m.dtype() != y_o.dtype())
        throw ShapeError("rse operands must share shape and dtype");
    if (y_m.numel() == 0)
        throw ShapeError("rse needs at least one element");
    const int64_t n = y_m.numel();
    const bool f64 = y_m.dtype() == Dtype::f64;
    const size_t bytes = static_cast<size_t>(n) * (f64 ? 8 : 4);
    DevBuf dm(bytes), dO(bytes);
    cuda_check(cudaMemcpy(dm.p, f64 ? static_cast<const void*>(y_m.f64()) : y_m.f32(), bytes, cudaMemcpyHostToDevice),
               "rse upload");
    cuda_check(cudaMemcpy(dO.p, f64 ? static_cast<const void*>(y_o.f64()) : y_o.f32(), bytes, cudaMemcpyHostToDevice),
               "rse upload");
    double out = 0.0;
    check(dfa2c_rse(dm.p, dO.p, f64 ? DFA2C_F64 : DFA2C_F32, 1, n,
                    mode == RseMode::standard ? DFA2C_RSE_STANDARD : DFA2C_RSE_LITERAL, &out, nullptr));
    return out;
}

DFA2_API std::string method_id(const HeadStrategy& s) {
    switch (s.kind) {
    case StrategyKind::arrow: return "arrow_w" + std::to_string(s.window_blocks);
    case StrategyKind::cached: return "cached";
    default: return "full";
    }
}

DFA2_API std::vector<MethodCandidate> make_candidates(const std::vector<int64_t>& windows, bool include_cached) {
    std::vector<MethodCandidate> methods;
    for (int64_t w : windows) {
        if (w < 0)
            throw ShapeError("window radii must be >= 0");
        methods.push_back({method_id(HeadStrategy::Arrow(w)), HeadStrategy::Arrow(w)});
    }
    if (include_cached)
        methods.push_back({"cached", HeadStrategy::Cached()});
    if (methods.empty())
        throw ShapeError("candidate set must be nonempty");
    return methods;
}

DFA2_API LayerInfluence influence_for_layer(const Tensor& q, const Tensor& k, const Tensor& v,
                                            const std::vector<MethodCandidate>& methods, const HeadCache& cache,
                                            int64_t layer, int64_t t, const AttentionDims& dims, int64_t block_size,
                                            RseMode mode, CalibrationStats* stats) {
    if (methods.empty())
        throw ShapeError("candidate set must be nonempty");
    // Candidates in any order, as in src/calibrate.cpp:216-251: Cached
    // entries measure the cache slots, every other kind is an arrow pass with
    // its window. The device call evaluates each distinct window once plus
    // the cached column; results are mapped back to the caller's order.
    std::vector<int64_t> windows;
    std::vector<int64_t> column;  // per method: device column
    bool cached = false;
    for (const MethodCandidate& m : methods) {
        if (m.strategy.kind == StrategyKind::cached) {
            cached = true;
            column.push_back(-1);
        } else {
            if (m.strategy.window_blocks < 0)
                throw ShapeError("window radii must be >= 0");
            windows.push_back(m.strategy.window_blocks);
            column.push_back(static_cast<int64_t>(windows.size()) - 1);
        }
    }
    const int64_t NW = static_cast<int64_t>(windows.size());
    for (int64_t& c : column)
        if (c < 0)
            c = NW;
    dims.validate();
    const int64_t H = dims.n_heads, n = dims.seq_len(), d = dims.head_dim, numel = H * n * d;
    const int64_t M = static_cast<int64_t>(methods.size());
    const int64_t MD = NW + (cached ? 1 : 0);  // device columns
    if (q.ndim() != 3 || q.dim(0) != H || q.dim(1) != n || q.dim(2) != d || q.shape() != k.shape() ||
        q.shape() != v.shape())
        throw ShapeError("tensor shape disagrees with dims");
    dfa2c_cache* dev = cache.size() > 0 ? cache.bind(H, n, d) : nullptr;
    DevBuf dq(numel * 2), dk(numel * 2), dv(numel * 2), dorig(numel * 2), douts(numel * 2 * MD);
    upload_bf16(as_f32(q).data(), numel, dq.p);
    upload_bf16(as_f32(k).data(), numel, dk.p);
    upload_bf16(as_f32(v).data(), numel, dv.p);
    std::vector<double> infl_dev(static_cast<size_t>(H * MD), 0.0);
    int64_t evals = 0;
    const dfa2c_dims cd = cdims(dims);
    check(dfa2c_influence_for_layer(dq.p, dk.p, dv.p, &cd, block_size, windows.data(), NW, cached ? 1 : 0, dev,
                                    layer, t, mode == RseMode::standard ? DFA2C_RSE_STANDARD : DFA2C_RSE_LITERAL,
                                    infl_dev.data(), dorig.p, douts.p, &evals, nullptr));
    LayerInfluence li;
    li.influence.assign(static_cast<size_t>(H * M), 0.0);
    for (int64_t h = 0; h < H; ++h)
        for (int64_t m = 0; m < M; ++m)
            li.influence[static_cast<size_t>(h * M + m)] = infl_dev[static_cast<size_t>(h * MD + column[m])];
    evals = 1 + M;  // one original + one evaluation per candidate (src/calibrate.cpp:207, 220-221)
    li.original = Tensor::zeros({H, n, d});
    download_bf16(dorig.p, numel, li.original.f32());
    li.method_outputs.resize(static_cast<size_t>(M));
    for (int64_t m = 0; m < M; ++m) {
        if (methods[m].strategy.kind == StrategyKind::cached && t == 0)
            continue;  // ineligible: left unset, as in the reference
        li.method_outputs[m] = Tensor::zeros({H, n, d});
        download_bf16(static_cast<const char*>(douts.p) + column[m] * numel * 2, numel, li.method_outputs[m].f32());
    }
    if (stats)
        stats->attention_evals += evals;
    return li;
}

// ---------------------------------------------------------------- plan
DFA2_API CompressionPlan CompressionPlan::all_full(const AttentionDims& dims, int64_t timesteps, int64_t layers,
                                                   int64_t block_size) {
    CompressionPlan p;
    p.dims = dims;
    p.n_timesteps = timesteps;
    p.n_layers = layers;
    p.block_size = block_size;
    p.layers.assign(static_cast<size_t>(timesteps * layers), LayerPlan::all_full(dims.n_heads));
    return p;
}
DFA2_API const LayerPlan& CompressionPlan::at(int64_t t, int64_t layer) const {
    return layers.at(static_cast<size_t>(t * n_layers + layer));
}
DFA2_API LayerPlan& CompressionPlan::at(int64_t t, int64_t layer) {
    return layers.at(static_cast<size_t>(t * n_layers + layer));
}

namespace {
void plan_flat(const CompressionPlan& p, std::vector<int32_t>& kinds, std::vector<int64_t>& wins) {
    if (static_cast<int64_t>(p.layers.size()) != p.n_timesteps * p.n_layers)
        throw PlanValidationError("plan must cover every (t, layer) exactly once");
    kinds.clear();
    wins.clear();
    for (const LayerPlan& lp : p.layers) {
        if (lp.n_heads() != p.dims.n_heads)
            throw PlanValidationError("head array length must equal H");
        std::vector<int32_t> k;
        std::vector<int64_t> w;
        plan_arrays(lp, k, w);
        kinds.insert(kinds.end(), k.begin(), k.end());
        wins.insert(wins.end(), w.begin(), w.end());
    }
}
}  // namespace

DFA2_API void CompressionPlan::validate() const {
    dims.validate();
    if (n_timesteps < 1 || n_layers < 1 || block_size < 1)
        throw PlanValidationError("plan needs T >= 1, L >= 1, block >= 1");
    if (!(delta >= 0.0))
        throw PlanValidationError("delta must be >= 0");
    if (!(coeff >= 1.0))
        throw PlanValidationError("coeff must be >= 1");
    std::vector<int32_t> kinds;
    std::vector<int64_t> wins;
    plan_flat(*this, kinds, wins);
    const dfa2c_dims cd = cdims(dims);
    check(dfa2c_plan_aggregate(&cd, n_timesteps, n_layers, block_size, kinds.data(), wins.data(), nullptr, nullptr,
                               nullptr));
}
DFA2_API int64_t CompressionPlan::flops_total() const {
    std::vector<int32_t> kinds;
    std::vector<int64_t> wins;
    plan_flat(*this, kinds, wins);
    const dfa2c_dims cd = cdims(dims);
    int64_t f = 0;
    check(dfa2c_plan_aggregate(&cd, n_timesteps, n_layers, block_size, kinds.data(), wins.data(), &f, nullptr,
                               nullptr));
    return f;
}
DFA2_API int64_t CompressionPlan::flops_dense_total() const {
    return n_timesteps * n_layers * dims.n_heads * dense_flops(dims.seq_len(), dims.head_dim);
}
DFA2_API double CompressionPlan::aggregate_sparsity() const {
    return 1.0 - static_cast<double>(flops_total()) / static_cast<double>(flops_dense_total());
}

DFA2_API bool CompressionPlan::operator==(const CompressionPlan& o) const {
    return dims.n_heads == o.dims.n_heads && dims.head_dim == o.dims.head_dim && dims.n_visual == o.dims.n_visual &&
           dims.n_text == o.dims.n_text && dims.order == o.dims.order && n_timesteps == o.n_timesteps &&
           n_layers == o.n_layers && block_size == o.block_size && delta == o.delta && coeff == o.coeff &&
           window_set == o.window_set && layers == o.layers && influence_digest == o.influence_digest;
}

// ---------------------------------------------------------------- plan files
DFA2_API std::string fnv1a_hex(const std::string& bytes) {
    char out[17];
    check(dfa2c_fnv1a_hex(bytes.data(), static_cast<int64_t>(bytes.size()), out));
    return out;
}

DFA2_API std::string plan_to_json(const CompressionPlan& plan) {
    const int64_t T = plan.n_timesteps, L = plan.n_layers, H = plan.dims.n_heads;
    std::vector<int32_t> kinds(static_cast<size_t>(std::max<int64_t>(T * L * H, 0)), DFA2C_FULL);
    std::vector<int64_t> wins(kinds.size(), 0);
    for (int64_t t = 0; t < T; ++t)
        for (int64_t l = 0; l < L; ++l) {
            const LayerPlan& lp = plan.at(t, l);
            if (lp.n_heads() != H)
                throw ShapeError("head array length must equal H");
            std::vector<int32_t> k;
            std::vector<int64_t> w;
            plan_arrays(lp, k, w);
            std::copy(k.begin(), k.end(), kinds.begin() + (t * L + l) * H);
            std::copy(w.begin(), w.end(), wins.begin() + (t * L + l) * H);
        }
    dfa2c_plan_header hdr{T, L, H, plan.dims.head_dim, plan.dims.n_visual, plan.dims.n_text, plan.block_size,
                          plan.delta, plan.coeff, static_cast<int64_t>(plan.window_set.size()), 0};
    int64_t len = 0;
    check(dfa2c_plan_to_json(&hdr, kinds.data(), wins.data(), plan.window_set.data(), plan.influence_digest.c_str(),
                             nullptr, 0, &len));
    std::string text(static_cast<size_t>(len) + 1, '\0');
    check(dfa2c_plan_to_json(&hdr, kinds.data(), wins.data(), plan.window_set.data(), plan.influence_digest.c_str(),
                             text.data(), len + 1, &len));
    text.resize(static_cast<size_t>(len));
    return text;
}

DFA2_API CompressionPlan plan_from_json(const std::string& text) {
    dfa2c_plan_header hdr{};
    check(dfa2c_plan_from_json(text.data(), static_cast<int64_t>(text.size()), &hdr, nullptr, nullptr, nullptr,
                               nullptr, 0));
    const int64_t T = hdr.n_timesteps, L = hdr.n_layers, H = hdr.n_heads;
    std::vector<int32_t> kinds(static_cast<size_t>(T * L * H));
    std::vector<int64_t> wins(kinds.size());
    std::vector<int64_t> ws(static_cast<size_t>(hdr.n_window_set) + 1);
    std::string digest(static_cast<size_t>(hdr.digest_len) + 1, '\0');
    check(dfa2c_plan_from_json(text.data(), static_cast<int64_t>(text.size()), &hdr, kinds.data(), wins.data(),
                               ws.data(), digest.data(), hdr.digest_len + 1));
    CompressionPlan p;
    p.dims.n_heads = H;
    p.dims.head_dim = hdr.head_dim;
    p.dims.n_visual = hdr.n_visual;
    p.dims.n_text = hdr.n_text;
    p.n_timesteps = T;
    p.n_layers = L;
    p.block_size = hdr.block_size;
    p.delta = hdr.delta;
    p.coeff = hdr.coeff;
    p.window_set.assign(ws.begin(), ws.begin() + hdr.n_window_set);
    digest.resize(static_cast<size_t>(hdr.digest_len));
    p.influence_digest = digest;
    p.layers.resize(static_cast<size_t>(T * L));
    for (int64_t i = 0; i < T * L; ++i)
        for (int64_t h = 0; h < H; ++h) {
            const size_t j = static_cast<size_t>(i * H + h);
            p.layers[static_cast<size_t>(i)].strategies.push_back(
                kinds[j] == DFA2C_ARROW ? HeadStrategy::Arrow(wins[j])
                                        : kinds[j] == DFA2C_CACHED ? HeadStrategy::Cached() : HeadStrategy::Full());
        }
    return p;
}

DFA2_API void save_plan(const CompressionPlan& plan, const std::string& path) {
    const std::string text = plan_to_json(plan);
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f)
        throw IoError("cannot open " + path + " for writing");
    const bool ok = std::fwrite(text.data(), 1, text.size(), f) == text.size();
    if (std::fclose(f) != 0 || !ok)
        throw IoError("failed writing " + path);
}

DFA2_API CompressionPlan load_plan(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f)
        throw IoError("cannot open " + path);
    std::string text;
    char buf[1 << 16];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof buf, f)) > 0)
        text.append(buf, got);
    std::fclose(f);
    return plan_from_json(text);
}

}  // namespace dfa2
