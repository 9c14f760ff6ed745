// dfa2c.cpp — host side of the C-ABI (include/dfa2c.h): bit-exact plan
// arithmetic, the per-head tile scheduler, the device-resident head cache,
// TMA descriptor creation and kernel launches. No CPU attention fallback
// exists here: every attention / RSE result comes from the sm_100a kernels.
#include "dfa2c.h"

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <queue>
#include <string>
#include <vector>

#include "attn_types.h"
#include "capi_status.h"
#include "nccl_dl.h"
#include "json_lite.h"

namespace dfa2k {
cudaError_t launch_attn(int d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                        const CUtensorMap& to, const CUtensorMap& tc, const AttnArgs& args, const PeerMaps& peers,
                        int grid, cudaStream_t stream);
int rse_ctas_per_sm();
cudaError_t launch_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n, int sms,
                           cudaStream_t stream);
cudaError_t launch_rse(const void* ym, const void* yo, int dtype, int64_t n_heads, int64_t numel,
                       int mode, double* out_dev, double* scratch, int nblk, cudaStream_t stream);
cudaError_t launch_rse_multi(const void* const* ym, int M, const void* yo, int dtype, int64_t n_heads,
                             int64_t numel, int mode, double* out_dev, double* scratch, int nblk,
                             cudaStream_t stream);
int rse_multi_max();
int reference_max_head_dim();
cudaError_t launch_commit_rows(const void* out, void* cache, int64_t rows, int64_t r0, int64_t r1, int64_t n,
                               int64_t H, int64_t d, const uint32_t* head_bits, int sms, cudaStream_t stream);
cudaError_t launch_attention_reference(const void* q, const void* k, const void* v, void* out, int dtype, int64_t H,
                                       int64_t n, int64_t d, const uint8_t* mask, int64_t block, int64_t nb,
                                       cudaStream_t stream);
}  // namespace dfa2k

using dfa2k::WorkItem;

namespace {

using dfa2c_detail::fail;
using dfa2c_detail::g_err;
using dfa2c_detail::guard;
long long* g_trace = nullptr;  // debug: per-tile timestamps (kernels built with -DDFA2_TRACE=1)
std::atomic<int64_t> g_launches{0};

#define DFA2C_CUDA_CHECK(expr)                                                             \
    do {                                                                                   \
        const cudaError_t e_ = (expr);                                                     \
        if (e_ != cudaSuccess)                                                             \
            fail(DFA2C_CUDA, std::string(#expr) + " failed: " + cudaGetErrorString(e_)); \
    } while (0)

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// AttentionDims::validate (src/tensor.cpp:225-230).
void validate_dims(const dfa2c_dims* d) {
    if (!d)
        fail(DFA2C_SHAPE, "dims must not be NULL");
    if (d->n_heads < 1 || d->head_dim < 1)
        fail(DFA2C_SHAPE, "n_heads and head_dim must be >= 1");
    if (d->n_visual < 1 || d->n_text < 0)
        fail(DFA2C_SHAPE, "need n_visual >= 1 and n_text >= 0");
    if (d->order != DFA2C_VISUAL_FIRST && d->order != DFA2C_TEXT_FIRST)
        fail(DFA2C_SHAPE, "unknown token order");
}

int64_t seq_len(const dfa2c_dims* d) { return d->n_visual + d->n_text; }
int64_t text_begin(const dfa2c_dims* d) { return d->order == DFA2C_VISUAL_FIRST ? d->n_visual : 0; }
int64_t text_end(const dfa2c_dims* d) { return d->order == DFA2C_VISUAL_FIRST ? seq_len(d) : d->n_text; }

// build_arrow_mask (src/arrow.cpp:113-153): a block is text if it overlaps
// the text span; the window clamps to the visual block count;
// active(i,j) = text(i) | text(j) | |i-j| <= w_eff.
std::vector<uint8_t> arrow_mask(const dfa2c_dims* dims, int64_t B, int64_t w) {
    validate_dims(dims);
    if (B < 1)
        fail(DFA2C_SHAPE, "block_size must be >= 1");
    if (w < 0)
        fail(DFA2C_SHAPE, "window_blocks must be >= 0");
    const int64_t n = seq_len(dims);
    const int64_t nb = ceil_div(n, B);
    const int64_t lo_t = text_begin(dims), hi_t = text_end(dims);
    std::vector<uint8_t> is_text(static_cast<size_t>(nb));
    for (int64_t i = 0; i < nb; ++i) {
        const int64_t lo = i * B, hi = std::min(lo + B, n);
        is_text[i] = (lo < hi_t && hi > lo_t) ? 1 : 0;
    }
    const int64_t weff = std::min(w, std::max<int64_t>(0, ceil_div(dims->n_visual, B) - 1));
    std::vector<uint8_t> m(static_cast<size_t>(nb * nb));
    for (int64_t i = 0; i < nb; ++i)
        for (int64_t j = 0; j < nb; ++j)
            m[i * nb + j] = (is_text[i] || is_text[j] || std::llabs(i - j) <= weff) ? 1 : 0;
    return m;
}

// BlockMask::active_positions (src/arrow.cpp:95-104).
int64_t active_positions(const uint8_t* m, int64_t n, int64_t B) {
    const int64_t nb = ceil_div(n, B);
    int64_t total = 0;
    for (int64_t i = 0; i < nb; ++i) {
        const int64_t li = std::min(B, n - i * B);
        for (int64_t j = 0; j < nb; ++j)
            if (m[i * nb + j])
                total += li * std::min(B, n - j * B);
    }
    return total;
}

void validate_plan(const dfa2c_dims* dims, const int32_t* kinds, const int64_t* windows) {
    if (!kinds)
        fail(DFA2C_SHAPE, "plan must assign exactly one strategy per head");
    for (int64_t h = 0; h < dims->n_heads; ++h) {
        const int32_t k = kinds[h] & ~DFA2C_SKIP;
        if ((kinds[h] & ~(DFA2C_SKIP | 3)) != 0 || k < DFA2C_FULL || k > DFA2C_CACHED)
            fail(DFA2C_SHAPE, "unknown strategy kind for head " + std::to_string(h));
        if (k == DFA2C_ARROW && (!windows || windows[h] < 0))
            fail(DFA2C_SHAPE, "window_blocks must be >= 0");
    }
}

int32_t kind_of(int32_t k) { return k & ~DFA2C_SKIP; }
bool skipped(int32_t k) { return (k & DFA2C_SKIP) != 0; }

// plan_flops (src/dispatch.cpp:93-120).
int64_t plan_flops(const dfa2c_dims* dims, int64_t B, const int32_t* kinds, const int64_t* windows) {
    validate_dims(dims);
    validate_plan(dims, kinds, windows);
    const int64_t n = seq_len(dims), d = dims->head_dim;
    std::map<int64_t, int64_t> arrow;
    int64_t total = 0;
    for (int64_t h = 0; h < dims->n_heads; ++h) {
        if (kind_of(kinds[h]) == DFA2C_FULL) {
            total += 4 * d * n * n;
        } else if (kind_of(kinds[h]) == DFA2C_ARROW) {
            auto it = arrow.find(windows[h]);
            if (it == arrow.end()) {
                const auto m = arrow_mask(dims, B, windows[h]);
                it = arrow.emplace(windows[h], 4 * d * active_positions(m.data(), n, B)).first;
            }
            total += it->second;
        }
    }
    return total;
}

// ------------------------------------------------------------ tile sets
// For every 128-row query tile, the 64-key KV tiles holding at least one
// active (query, key) pair, ascending (the reference folds key blocks in
// ascending order, src/arrow.cpp:184-186). A tile is PARTIAL when some pair
// inside [rows < n] x [keys < n] is inactive, or keys run past n.
struct TileSet {
    std::vector<int64_t> row_ptr;
    std::vector<uint32_t> cols;
};

TileSet build_tile_set(const uint8_t* m, int64_t n, int64_t B) {
    const int64_t nb = ceil_div(n, B);
    const int64_t nqt = ceil_div(n, dfa2k::TILE_M);
    const int64_t nkt = ceil_div(n, dfa2k::TILE_N);
    TileSet ts;
    ts.row_ptr.assign(static_cast<size_t>(nqt + 1), 0);
    for (int64_t i = 0; i < nqt; ++i) {
        const int64_t r0 = i * dfa2k::TILE_M, r1 = std::min(r0 + dfa2k::TILE_M, n);
        const int64_t qb0 = r0 / B, qb1 = (r1 - 1) / B;
        for (int64_t t = 0; t < nkt; ++t) {
            const int64_t c0 = t * dfa2k::TILE_N, c1 = std::min(c0 + dfa2k::TILE_N, n);
            const int64_t kb0 = c0 / B, kb1 = (c1 - 1) / B;
            bool any = false, all = true;
            for (int64_t qb = qb0; qb <= qb1; ++qb)
                for (int64_t kb = kb0; kb <= kb1; ++kb) {
                    const bool a = m[qb * nb + kb] != 0;
                    any |= a;
                    all &= a;
                }
            if (!any)
                continue;
            const bool partial = !all || (c1 - c0) < dfa2k::TILE_N;
            ts.cols.push_back(static_cast<uint32_t>(t) | (partial ? dfa2k::TILE_SET_PARTIAL : 0u));
        }
        ts.row_ptr[i + 1] = static_cast<int64_t>(ts.cols.size());
    }
    return ts;
}

void check_rows_nonempty(const uint8_t* m, int64_t nb) {
    for (int64_t i = 0; i < nb; ++i) {
        bool any = false;
        for (int64_t j = 0; j < nb && !any; ++j)
            any = m[i * nb + j] != 0;
        if (!any)
            fail(DFA2C_FULLY_MASKED, "query block " + std::to_string(i) + " has no active key blocks");
    }
}

// ------------------------------------------------------------ device plan
// A work list on the device: one stream-ordered block from the library pool
// holding the items, CTA ranges, tile words and masks. Every launch that
// reads it is fenced onto the device's retire stream (retire_after); on
// eviction the block is freed on that stream, after the upload (`ready`) and
// after every launch on any stream that was enqueued before the eviction, so
// building or dropping a plan never synchronises the device.
void plan_release(int device, void* dev, cudaEvent_t ready);
void retire_after(int device, cudaStream_t stream);
struct DevPlan {
    int grid = 0;
    int32_t n_groups = 0;  // split groups (counters per launch)
    int32_t n_slots = 0;   // partial-output slots (one per split chunk)
    bool copies_last = false;  // every CTA's copy items are the tail of its list
    int32_t n_copy_tiles = 0;  // copy pool: Cached-head tiles drained by every CTA
    int2* copy_tiles = nullptr;
    WorkItem* items = nullptr;
    int32_t* cta_begin = nullptr;
    uint32_t* tiles = nullptr;
    uint8_t* masks = nullptr;
    int32_t n_snap = 0;                                   // calibration plans: snapshots per query tile
    uint16_t snap_slots[dfa2k::MAX_SNAPS] = {};
    std::vector<int64_t> shard_rows;                      // sharded plans: [world + 1] flattened row bounds
    int device = 0;
    void* dev = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr;  // the upload (on the building call's stream) has landed
    ~DevPlan() { plan_release(device, dev, ready); }
    // a launch on any stream first orders itself after the upload
    void acquire(cudaStream_t stream) const { DFA2C_CUDA_CHECK(cudaStreamWaitEvent(stream, ready, 0)); }
    void release(cudaStream_t stream) const { retire_after(device, stream); }
};

// Head strategy for the scheduler: mask_id >= 0 => computed over that mask;
// JOB_COPY => cached (copy items); JOB_SKIP => not part of this launch.
constexpr int JOB_COPY = -1;
constexpr int JOB_SKIP = -2;
struct HeadJob {
    int mask_id;
    bool commit;
};

// Split-KV scheduling switch: dfa2c_set_split_kv(), default from the
// environment (DFA2_SPLIT_KV=1), process-wide.
std::atomic<int> g_split_kv{-1};
bool split_kv_enabled() {
    int v = g_split_kv.load();
    if (v < 0) {
        const char* e = std::getenv("DFA2_SPLIT_KV");
        v = (e && e[0] == '1') ? 1 : 0;
        int expect = -1;
        g_split_kv.compare_exchange_strong(expect, v);
        v = g_split_kv.load();
    }
    return v == 1;
}

int num_sms(int device) {
    int v = 0;
    DFA2C_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    return v;
}

// Stream-ordered scratch comes from a library-owned pool per device that
// never returns memory to the driver (release threshold = max), so
// steady-state calls allocate without driver round trips.
cudaMemPool_t scratch_pool(int device) {
    static std::mutex mu;
    static std::map<int, cudaMemPool_t> pools;
    std::lock_guard<std::mutex> lk(mu);
    auto it = pools.find(device);
    if (it != pools.end())
        return it->second;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool{};
    DFA2C_CUDA_CHECK(cudaMemPoolCreate(&pool, &props));
    uint64_t keep = std::numeric_limits<uint64_t>::max();
    DFA2C_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    pools[device] = pool;
    return pool;
}

template <class T>
void scratch_alloc(T** p, size_t bytes, cudaStream_t st) {
    int device = 0;
    DFA2C_CUDA_CHECK(cudaGetDevice(&device));
    DFA2C_CUDA_CHECK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, scratch_pool(device), st));
}

// Host staging for plan uploads: per device, a ring of pinned buffers, each
// reused once the copy that last read it has completed (its event), so a
// plan-cache miss costs host work and an asynchronous copy, not a device
// synchronisation.
struct PlanStaging {
    static constexpr int kSlots = 8;
    static constexpr size_t kBytes = size_t{8} << 20;
    char* buf[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
    int next = 0;
};
std::mutex g_staging_mu;
std::map<int, PlanStaging> g_staging;

template <class Fill>
void plan_upload(int device, cudaStream_t stream, void* dst, size_t bytes, Fill&& fill) {
    std::lock_guard<std::mutex> lk(g_staging_mu);
    PlanStaging& ps = g_staging[device];
    if (bytes > PlanStaging::kBytes) {  // oversized plan: pageable copy, in stream order
        std::vector<char> h(bytes);
        fill(h.data());
        DFA2C_CUDA_CHECK(cudaMemcpyAsync(dst, h.data(), bytes, cudaMemcpyHostToDevice, stream));
        DFA2C_CUDA_CHECK(cudaStreamSynchronize(stream));  // h goes out of scope
        return;
    }
    if (!ps.buf[0]) {  // one pinned allocation carved into the slots
        char* base = nullptr;
        DFA2C_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&base), PlanStaging::kSlots * PlanStaging::kBytes,
                                       cudaHostAllocPortable));
        for (int j = 0; j < PlanStaging::kSlots; ++j) {
            ps.buf[j] = base + j * PlanStaging::kBytes;
            DFA2C_CUDA_CHECK(cudaEventCreateWithFlags(&ps.ev[j], cudaEventDisableTiming));
        }
    }
    const int i = ps.next;
    ps.next = (ps.next + 1) % PlanStaging::kSlots;
    DFA2C_CUDA_CHECK(cudaEventSynchronize(ps.ev[i]));  // its previous upload has been read (no-op if unused)
    fill(ps.buf[i]);
    DFA2C_CUDA_CHECK(cudaMemcpyAsync(dst, ps.buf[i], bytes, cudaMemcpyHostToDevice, stream));
    DFA2C_CUDA_CHECK(cudaEventRecord(ps.ev[i], stream));
}

// Per device: the retire stream (frees of evicted plans) and one event used
// to fence launches onto it. cudaStreamWaitEvent captures the event's state
// at the call, so the event can be re-recorded by the next launch at once.
struct Retire {
    std::mutex mu;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev = nullptr;
};
Retire& retire_of(int device) {
    // never destroyed: plans evicted by static destruction at exit (g_plans)
    // still find their device's retire state
    static std::mutex* mu = new std::mutex;
    static auto* m = new std::map<int, std::unique_ptr<Retire>>;
    std::lock_guard<std::mutex> lk(*mu);
    auto& r = (*m)[device];
    if (!r) {
        r = std::make_unique<Retire>();
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        DFA2C_CUDA_CHECK(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
        DFA2C_CUDA_CHECK(cudaEventCreateWithFlags(&r->ev, cudaEventDisableTiming));
        cudaSetDevice(cur);
    }
    return *r;
}

void retire_after(int device, cudaStream_t stream) {
    Retire& r = retire_of(device);
    std::lock_guard<std::mutex> lk(r.mu);
    DFA2C_CUDA_CHECK(cudaEventRecord(r.ev, stream));
    DFA2C_CUDA_CHECK(cudaStreamWaitEvent(r.stream, r.ev, 0));
}

void plan_release(int device, void* dev, cudaEvent_t ready) {
    if (!dev && !ready)
        return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    Retire& r = retire_of(device);
    {
        std::lock_guard<std::mutex> lk(r.mu);
        if (ready)
            cudaStreamWaitEvent(r.stream, ready, 0);  // the upload itself (a plan never launched)
        if (dev)
            cudaFreeAsync(dev, r.stream);  // after every launch fenced so far, on any stream
    }
    if (ready)
        cudaEventDestroy(ready);
    cudaSetDevice(cur);
}

// Work entries of one mask: each is a pair of query tiles (lanes A, B)
// sharing the ascending union of their KV tile rows, every word tagged with
// the lanes that fold it; or, at d = 64, for a text query tile (every key
// tile for an arrow head: the longest chain of the layer), a HALVES entry:
// the tile on both lanes, lane A folding the first half of its key tiles
// and lane B the second, interleaved, merged in the epilogue. A lane folds
// its own tiles in ascending order either way, so pairing never changes a
// row's result; the halving is a fixed property of the geometry (text rows
// at d = 64, for every head and strategy), so each head's result is still
// a function of its own strategy alone.
struct PairSet {
    std::vector<int64_t> row_ptr;  // [entries + 1]
    std::vector<uint32_t> words;
    std::vector<int32_t> n_a, n_b;  // per entry: tiles lane A / lane B fold
    std::vector<int32_t> qa, qb;    // query tiles of lanes A / B (qb -1: single lane)
    std::vector<uint8_t> halves;    // HALVES entry
};

inline uint32_t tag_lane(uint32_t c, int lane) {
    const bool part = (c & dfa2k::TILE_SET_PARTIAL) != 0;
    return lane ? dfa2k::TILE_NEED_B | (part ? dfa2k::TILE_PART_B : 0u)
                : dfa2k::TILE_NEED_A | (part ? dfa2k::TILE_PART_A : 0u);
}

// text_tile[q]: query tile q runs as a HALVES entry candidate (empty: none)
// halve_single: a query tile left without a partner (odd tile count) runs as
// a HALVES entry too, so it keeps both lanes busy instead of folding its whole
// key row on one lane (d = 64, SD3's ragged 35th tile).
PairSet build_pair_set(const TileSet& ts, int64_t nqt, const std::vector<uint8_t>& text_tile, int64_t ratio,
                       bool halve_single) {
    PairSet ps;
    ps.row_ptr.push_back(0);
    ps.words.reserve(ts.cols.size());
    auto add_pair = [&](int64_t qa, int64_t qb) {
        // both rows are ascending: merge them (each tile once, tagged with its lanes)
        int64_t i = ts.row_ptr[qa], ie = ts.row_ptr[qa + 1];
        int64_t j = qb >= 0 ? ts.row_ptr[qb] : 0, je = qb >= 0 ? ts.row_ptr[qb + 1] : 0;
        ps.n_a.push_back(static_cast<int32_t>(ie - i));
        ps.n_b.push_back(static_cast<int32_t>(je - j));
        while (i < ie || j < je) {
            const uint32_t ca = i < ie ? ts.cols[i] : 0u, cb = j < je ? ts.cols[j] : 0u;
            const uint32_t ta = ca & ~dfa2k::TILE_SET_PARTIAL, tb = cb & ~dfa2k::TILE_SET_PARTIAL;
            if (j >= je || (i < ie && ta < tb)) {
                ps.words.push_back(ta | tag_lane(ca, 0));
                ++i;
            } else if (i >= ie || tb < ta) {
                ps.words.push_back(tb | tag_lane(cb, 1));
                ++j;
            } else {
                ps.words.push_back(ta | tag_lane(ca, 0) | tag_lane(cb, 1));
                ++i;
                ++j;
            }
        }
        ps.qa.push_back(static_cast<int32_t>(qa));
        ps.qb.push_back(static_cast<int32_t>(qb));
        ps.halves.push_back(0);
        ps.row_ptr.push_back(static_cast<int64_t>(ps.words.size()));
    };
    auto add_halves = [&](int64_t q) {
        const int64_t lo = ts.row_ptr[q], n = ts.row_ptr[q + 1] - lo, h = (n + 1) / 2;
        for (int64_t i = 0; i < h; ++i) {
            const uint32_t ca = ts.cols[lo + i];
            ps.words.push_back((ca & ~dfa2k::TILE_SET_PARTIAL) | tag_lane(ca, 0));
            if (i < n - h) {
                const uint32_t cb = ts.cols[lo + h + i];
                ps.words.push_back((cb & ~dfa2k::TILE_SET_PARTIAL) | tag_lane(cb, 1));
            }
        }
        ps.n_a.push_back(static_cast<int32_t>(h));
        ps.n_b.push_back(static_cast<int32_t>(n - h));
        ps.qa.push_back(static_cast<int32_t>(q));
        ps.qb.push_back(static_cast<int32_t>(q));
        ps.halves.push_back(1);
        ps.row_ptr.push_back(static_cast<int64_t>(ps.words.size()));
    };
    auto add_single = [&](int64_t q) {
        if (halve_single && ts.row_ptr[q + 1] - ts.row_ptr[q] >= 2)
            add_halves(q);
        else
            add_pair(q, -1);
    };
    if (text_tile.empty()) {
        for (int64_t q = 0; q < nqt; q += 2) {
            if (q + 1 < nqt)
                add_pair(q, q + 1);
            else
                add_single(q);
        }
        return ps;
    }
    // Halve only when the text rows are the mask's long pole: their key
    // chains are more than ratio/10 x the average chain of the other query tiles
    // (narrow arrow windows). A property of the mask alone, so heads with
    // the same strategy are treated alike and Full == Arrow(max) holds.
    int64_t other_len = 0, n_other = 0, text_len = 0;
    for (int64_t q = 0; q < nqt; ++q) {
        const int64_t len = ts.row_ptr[q + 1] - ts.row_ptr[q];
        if (text_tile[q])
            text_len = std::max(text_len, len);
        else {
            other_len += len;
            ++n_other;
        }
    }
    const bool halve = n_other > 0 && 10 * text_len * n_other > ratio * other_len;
    int64_t pending = -1;  // the other tiles pair up in order
    for (int64_t q = 0; q < nqt; ++q) {
        if (halve && text_tile[q] && ts.row_ptr[q + 1] - ts.row_ptr[q] >= 2) {
            add_halves(q);
        } else if (pending < 0) {
            pending = q;
        } else {
            add_pair(pending, q);
            pending = -1;
        }
    }
    if (pending >= 0)
        add_single(pending);
    return ps;
}

// Scheduling cost of a pair-set entry in lane-tile units: a step of the
// shared K/V stream costs one period whether one or both lanes fold it, so a
// pair costs 2 x its union length (a single-lane entry as much as a full
// pair); a HALVES entry's steps alternate between the lanes, each ~0.6 of a
// pair step (measured per item with -DDFA2_TRACE=4, tools/cta_tail.py
// --items: 1.05 vs 1.77 us per step at d = 64), so 1.2 per folded tile.
// +1 for the item's ramp.
double entry_cost(const PairSet& ps, size_t p) {
    if (ps.halves[p])
        return 1.2 * (ps.n_a[p] + ps.n_b[p]) + 1.0;
    return 2.0 * static_cast<double>(ps.row_ptr[p + 1] - ps.row_ptr[p]) + 1.0;
}

struct Cand {
    WorkItem w;
    double cost;
};
std::unique_ptr<DevPlan> schedule_items(int device, std::vector<Cand>& cands, const std::vector<uint32_t>& tiles,
                                        const std::vector<uint8_t>& mask_bytes, int32_t n_groups, int32_t n_slots,
                                        cudaStream_t stream);

// Builds the LPT-scheduled work list: each (sample, head, query-tile pair)
// is one item costing (#lane-A tiles + #lane-B tiles + 1) tile-units
// (compute) or #rows/128 (copy); items are sorted by cost (desc), then
// (bh, pair) so concurrently running CTAs share a head's K/V in L2, and
// greedily assigned to the least-loaded CTA. The schedule is static, so
// every run (and every GPU count) folds the same tiles in the same order:
// outputs are bitwise reproducible.
// Sharded launches (n_parts > 0; dfa2c_mha_forward_sharded): the layer's
// (sample, head, query-tile pair) sequence is cut into n_parts contiguous
// ranges of near-equal cost and this launch runs range `part`. Pairs are
// always (2p, 2p+1) (no HALVES entries), so every range is one contiguous
// span of the flattened [batch*H*N] output rows. Long pairs are split into
// key chunks against a fixed reference of kShardRefSMs SMs (an 8-GPU box),
// whatever the GPU count, so a head's bits are the same for every n_parts.
double shard_ref_sms() {
    static const double v = [] {
        const char* e = std::getenv("DFA2_SHARD_REF_SMS");  // A/B only
        return e ? std::atof(e) : 148.0 * 8;
    }();
    return v;
}

// DFA2_COPY_TAIL=0 keeps one staging box per lane for trailing copies (A/B)
bool copy_tail_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DFA2_COPY_TAIL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Cached-head copies as one pool drained by every CTA once its compute is
// done (DFA2_COPY_POOL=0: LPT places them as list items, copied in each
// CTA's tail).
#ifndef DFA2_COPY_POOL_DEFAULT
#define DFA2_COPY_POOL_DEFAULT 1
#endif
bool copy_pool_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DFA2_COPY_POOL");
        return e ? e[0] != '0' : DFA2_COPY_POOL_DEFAULT != 0;
    }();
    return on && copy_tail_enabled();
}

// Per-launch copy-pool counters: a ring of zeroed [claimed, done] pairs per
// device; launch k uses slot k mod kCopySlots and its last CTA re-zeroes it,
// so no memset sits between launches.
constexpr int kCopySlots = 1 << 16;
// The ring is allocated when the first plan with copies is built (never
// under CUDA-graph capture, which reuses built plans only).
int* copy_counter_base(int device) {
    static std::mutex mu;
    static int* base[64] = {};
    if (device < 0 || device >= 64)
        fail(DFA2C_UNSUPPORTED, "device index out of range");
    std::lock_guard<std::mutex> lk(mu);
    if (!base[device]) {
        int* p = nullptr;
        DFA2C_CUDA_CHECK(cudaMalloc(&p, sizeof(int) * 2 * kCopySlots));
        DFA2C_CUDA_CHECK(cudaMemset(p, 0, sizeof(int) * 2 * kCopySlots));
        DFA2C_CUDA_CHECK(cudaDeviceSynchronize());
        base[device] = p;
    }
    return base[device];
}
int* copy_counter_slot(int device) {
    static std::atomic<uint32_t> seq[64];
    int* base = copy_counter_base(device);
    return base + 2 * (seq[device].fetch_add(1) % kCopySlots);
}

// Key-chunk boundaries of a split pair: chunk c gets a share of the union
// tiles proportional to (nch - c), e.g. 1/2, 1/3, 1/6 for three chunks.
// Unequal chunks give the LPT assignment small items to fill the CTAs that
// the large ones leave short: a sharded rank whose range is all Full pairs
// (192 equal chunks on 148 SMs at 8 GPUs) otherwise ends one whole chunk
// late on a third of its SMs. Every chunk keeps at least one tile; the cut
// depends only on (U, nch), so results stay independent of the GPU count.
// Latency-mode split-KV (not sharded) keeps equal chunks: there the longest
// chunk is the launch's critical path (a single head: 1.03x dense-vs-arrow
// with unequal chunks against 1.5x+ with equal ones).
std::vector<int32_t> chunk_bounds(int32_t U, int32_t nch, bool unequal) {
    std::vector<int32_t> cut(static_cast<size_t>(nch) + 1, 0);
    const int64_t W = unequal ? int64_t{nch} * (nch + 1) / 2 : nch;
    int64_t acc = 0;
    for (int32_t c = 0; c < nch; ++c) {
        acc += unequal ? nch - c : 1;
        int64_t b = (acc * U + W / 2) / W;
        b = std::max<int64_t>(b, cut[c] + 1);            // non-empty
        b = std::min<int64_t>(b, U - (nch - 1 - c));      // room for the rest
        cut[c + 1] = static_cast<int32_t>(b);
    }
    cut[nch] = U;
    return cut;
}

// Host-side geometry of a work list: per-mask pair sets and their tile
// words, the split-KV chunking, and for sharded launches the partition.
struct PlanGeometry {
    std::vector<uint32_t> tiles;
    std::vector<uint8_t> mask_bytes;
    std::vector<int64_t> mask_tile_base, mask_off;
    std::vector<PairSet> sets;
    std::vector<std::vector<int32_t>> chunks_of;  // per mask, per pair: key chunks (1 = whole)
    std::vector<int64_t> shard_rows;              // sharded: [n_parts + 1] flattened row bounds
    std::vector<int32_t> pair_part;               // sharded: part of each (sample, head, pair)
};

PlanGeometry plan_geometry(int64_t batch, int64_t H, int64_t n, int64_t B,
                           const std::vector<std::vector<uint8_t>>& masks, const std::vector<HeadJob>& jobs,
                           const std::vector<int>& ref_jobs, int64_t text_lo, int64_t text_hi, int64_t halve_ratio,
                           int32_t n_parts) {
    const int64_t nqt = ceil_div(n, dfa2k::TILE_M);
    const int64_t np = (nqt + 1) / 2;  // copy items: pairs (2p, 2p+1)
    const bool sharded = n_parts > 0;
    PlanGeometry g;
    auto& tiles = g.tiles;
    auto& mask_bytes = g.mask_bytes;
    auto& mask_tile_base = g.mask_tile_base;
    auto& mask_off = g.mask_off;
    auto& sets = g.sets;
    auto& chunks_of = g.chunks_of;
    // text query tiles as HALVES entries (d = 64; not under split-KV, which
    // chunks the long rows its own way, nor in sharded launches)
    std::vector<uint8_t> text_tile;
    if (halve_ratio > 0 && !split_kv_enabled() && !sharded && text_hi > text_lo) {
        text_tile.assign(static_cast<size_t>(nqt), 0);
        for (int64_t q = 0; q < nqt; ++q) {
            const int64_t r0 = q * dfa2k::TILE_M, r1 = std::min(r0 + dfa2k::TILE_M, n);
            text_tile[q] = (r0 < text_hi && r1 > text_lo) ? 1 : 0;
        }
    }
    for (const auto& m : masks) {
        sets.push_back(build_pair_set(build_tile_set(m.data(), n, B), nqt, text_tile, halve_ratio,
                                      halve_ratio > 0 && !split_kv_enabled() && !sharded));
        mask_tile_base.push_back(static_cast<int64_t>(tiles.size()));
        tiles.insert(tiles.end(), sets.back().words.begin(), sets.back().words.end());
        mask_off.push_back(static_cast<int64_t>(mask_bytes.size()));
        mask_bytes.insert(mask_bytes.end(), m.begin(), m.end());
    }
    if (mask_bytes.empty())
        mask_bytes.push_back(0);
    if (tiles.empty())
        tiles.push_back(0);
    if (mask_bytes.size() > static_cast<size_t>(std::numeric_limits<int32_t>::max()) ||
        tiles.size() > static_cast<size_t>(std::numeric_limits<int32_t>::max()) || nqt > (1 << 24))
        fail(DFA2C_UNSUPPORTED, "work list too large");

    // Split-KV (opt-in, DFA2_SPLIT_KV=1): for latency-bound layers, e.g. a
    // late timestep with most heads Cached, where one text-row pair of an
    // arrow head (every key tile) outlasts everything else. The per-sample
    // load of the whole layer plan (ref_jobs: every head, including heads a
    // launch skips) is spread over a fixed reference of 148 SMs; a pair
    // costing more than that average becomes ceil(cost / average) key
    // chunks, combined in chunk order by the CTA that finishes the group's
    // last chunk. The decision is independent of the batch, of how a call is
    // split into launches (host-path groups; multi-GPU shards keep the plan
    // whole through DFA2C_SKIP) and of the device, so results are still
    // deterministic; but it depends on the other heads' strategies, which is
    // why it is off by default: with it off every head's result is a
    // function of its own strategy alone (head isolation, bitwise,
    // test_dispatch.cpp:98-109).
    const double kRefSMs = sharded ? shard_ref_sms() : 148.0;
    chunks_of.resize(sets.size());
    for (size_t mi = 0; mi < sets.size(); ++mi)
        chunks_of[mi].assign(sets[mi].qa.size(), 1);
    if (split_kv_enabled() || sharded) {
        double per_sample = 0.0;
        for (int64_t h = 0; h < H; ++h) {
            const int rj = ref_jobs.empty() ? jobs[h].mask_id : ref_jobs[h];
            if (rj < 0) {
                per_sample += static_cast<double>(n) / 128.0;  // a copy: ~1 unit per 128 rows
                continue;
            }
            const PairSet& ps = sets[rj];
            for (size_t p = 0; p < ps.qa.size(); ++p)
                per_sample += entry_cost(ps, p);
        }
        const double avg = std::max(per_sample / kRefSMs, 1.0);
        for (size_t mi = 0; mi < sets.size(); ++mi) {
            const PairSet& ps = sets[mi];
            for (size_t p = 0; p < ps.qa.size(); ++p) {
                const double cost = entry_cost(ps, p);
                const int64_t len = ps.row_ptr[p + 1] - ps.row_ptr[p];
                if (cost > avg && len >= 8)
                    chunks_of[mi][p] = static_cast<int32_t>(
                        std::min<int64_t>({static_cast<int64_t>(std::ceil(cost / avg)), len / 4, 32}));
            }
        }
    }
    // sharded: cost of every pair of the layer, in (sample, head, pair)
    // order, and the cut into n_parts near-equal contiguous ranges (a pair
    // belongs to the part containing the midpoint of its cost interval)
    auto& shard_rows = g.shard_rows;
    auto& pair_part = g.pair_part;
    if (sharded) {
        std::vector<double> cost;
        std::vector<int64_t> row_end;  // flattened end row of each pair
        for (int64_t b = 0; b < batch; ++b)
            for (int64_t h = 0; h < H; ++h) {
                const int rj = jobs[h].mask_id;
                if (rj == JOB_SKIP)
                    fail(DFA2C_SHAPE, "sharded launches take the whole layer (no skipped heads)");
                for (int64_t p = 0; p < np; ++p) {
                    const int64_t r1 = std::min<int64_t>(n, 256 * (p + 1));
                    if (rj == JOB_COPY) {
                        cost.push_back(static_cast<double>(r1 - 256 * p) / 128.0);
                    } else {
                        const PairSet& ps = sets[rj];
                        const int32_t nch = chunks_of[rj][p];
                        cost.push_back(entry_cost(ps, p) + (nch > 1 ? 0.5 * nch : 0.0));
                    }
                    row_end.push_back((b * H + h) * n + r1);
                }
            }
        double total = 0.0;
        for (double c : cost)
            total += c;
        shard_rows.assign(static_cast<size_t>(n_parts) + 1, 0);
        pair_part.resize(cost.size());
        double acc = 0.0;
        int32_t cur = 0;
        for (size_t i = 0; i < cost.size(); ++i) {
            const double mid = acc + 0.5 * cost[i];
            while (cur + 1 < n_parts && mid >= total * (cur + 1) / n_parts) {
                ++cur;
                shard_rows[static_cast<size_t>(cur)] = i ? row_end[i - 1] : 0;
            }
            pair_part[i] = cur;
            acc += cost[i];
        }
        for (int32_t c = cur + 1; c <= n_parts; ++c)
            shard_rows[static_cast<size_t>(c)] = batch * H * n;
    }

    return g;
}

std::unique_ptr<DevPlan> build_dev_plan(int device, int64_t batch, int64_t H, int64_t n, int64_t B,
                                        const std::vector<std::vector<uint8_t>>& masks,
                                        const std::vector<HeadJob>& jobs, const std::vector<int>& ref_jobs,
                                        int64_t text_lo, int64_t text_hi, int64_t halve_ratio, cudaStream_t stream,
                                        int32_t n_parts = 0, int32_t part = 0) {
    const int64_t nqt = ceil_div(n, dfa2k::TILE_M);
    const int64_t np = (nqt + 1) / 2;  // copy items: pairs (2p, 2p+1)
    const bool sharded = n_parts > 0;
    PlanGeometry g = plan_geometry(batch, H, n, B, masks, jobs, ref_jobs, text_lo, text_hi, halve_ratio, n_parts);
    auto& tiles = g.tiles;
    const auto& mask_bytes = g.mask_bytes;
    const auto& mask_tile_base = g.mask_tile_base;
    const auto& mask_off = g.mask_off;
    const auto& sets = g.sets;
    const auto& chunks_of = g.chunks_of;
    auto& shard_rows = g.shard_rows;
    const auto& pair_part = g.pair_part;
    int32_t n_groups = 0, n_slots = 0;

    std::vector<Cand> cands;
    cands.reserve(static_cast<size_t>(batch * H * np));
    int64_t pair_idx = -1;
    for (int64_t b = 0; b < batch; ++b)
        for (int64_t h = 0; h < H; ++h) {
            const HeadJob& j = jobs[h];
            if (j.mask_id == JOB_SKIP)
                continue;
            const int64_t n_entries =
                j.mask_id == JOB_COPY ? np : static_cast<int64_t>(sets[j.mask_id].qa.size());
            for (int64_t p = 0; p < n_entries; ++p) {
                ++pair_idx;
                if (sharded && pair_part[static_cast<size_t>(pair_idx)] != part)
                    continue;
                WorkItem w{};
                w.bh = static_cast<int32_t>(b * H + h);
                if (j.mask_id == JOB_COPY) {
                    w.qtile_a = static_cast<int32_t>(2 * p);
                    w.qtile_b = 2 * p + 1 < nqt ? static_cast<int32_t>(2 * p + 1) : -1;
                    w.flags = dfa2k::ITEM_COPY;
                    const int64_t rows = std::min<int64_t>(n, (w.qtile_b >= 0 ? w.qtile_b : w.qtile_a) * 128 + 128) -
                                         w.qtile_a * 128;
                    cands.push_back({w, static_cast<double>(rows) / 128.0});
                } else {
                    const PairSet& ps = sets[j.mask_id];
                    w.qtile_a = ps.qa[p];
                    w.qtile_b = ps.qb[p];
                    w.tile_begin = static_cast<int32_t>(mask_tile_base[j.mask_id] + ps.row_ptr[p]);
                    w.n_tiles = static_cast<int32_t>(ps.row_ptr[p + 1] - ps.row_ptr[p]);
                    w.mask_off = static_cast<int32_t>(mask_off[j.mask_id]);
                    w.flags = (j.commit ? dfa2k::ITEM_COMMIT : 0) | (ps.halves[p] ? dfa2k::ITEM_HALVES : 0);
                    if (ps.n_a[p] < 1)
                        fail(DFA2C_FULLY_MASKED, "query tile " + std::to_string(w.qtile_a) + " has no active key tiles");
                    if (w.qtile_b >= 0 && ps.n_b[p] < 1)
                        fail(DFA2C_FULLY_MASKED, "query tile " + std::to_string(w.qtile_b) + " has no active key tiles");
                    const int32_t nch = chunks_of[j.mask_id][p];
                    if (nch <= 1) {
                        cands.push_back({w, entry_cost(ps, p)});
                        continue;
                    }
                    const int32_t U = w.n_tiles, begin = w.tile_begin;
                    const std::vector<int32_t> cut = chunk_bounds(U, nch, sharded);
                    for (int32_t c = 0; c < nch; ++c) {
                        WorkItem cw = w;
                        const int32_t lo = cut[c], hi = cut[c + 1];
                        cw.tile_begin = begin + lo;
                        cw.n_tiles = hi - lo;
                        cw.flags |= dfa2k::ITEM_SPLIT;
                        cw.group = n_groups;
                        cw.chunk = c;
                        cw.nchunk = nch;
                        cw.part = n_slots + c;
                        // a chunk's steps cost one period each (split pairs are never HALVES)
                        cands.push_back({cw, 2.0 * cw.n_tiles + 1.5});
                    }
                    ++n_groups;
                    n_slots += nch;
                }
            }
        }
    if (cands.empty() && sharded) {  // an empty part: nothing to launch
        auto p = std::make_unique<DevPlan>();
        p->device = device;
        p->shard_rows = std::move(shard_rows);
        return p;
    }
    auto plan = schedule_items(device, cands, tiles, mask_bytes, n_groups, n_slots, stream);
    plan->shard_rows = std::move(shard_rows);
    return plan;
}

// LPT assignment of the work items to one persistent CTA per SM (cost desc,
// then (bh, pair) so concurrently running CTAs share a head's K/V in L2) and
// upload of the device plan.
// LPT leaves a tail when a CTA holds only ~3 items: the CTAs given one of
// the few long items (text-row pairs) later also receive a short one when
// everything else is full (SD3 Arrow(8): the costliest CTA 17% above the
// average). Improvement moves on the costliest CTA until none helps: move
// one of its items to a lightly loaded CTA, or swap it for a cheaper item
// there, whichever lowers the larger of the two loads the most. Only the
// item -> CTA assignment changes (every item's result is independent of
// where it runs), so results are bitwise unchanged. Deterministic: ties go
// to the lowest index.
void refine_schedule(std::vector<std::vector<const Cand*>>& bins, std::vector<double>& load) {
    const int m = static_cast<int>(bins.size());
    if (m < 2)
        return;
    size_t n_items = 0;
    for (const auto& b : bins)
        n_items += b.size();
    // Few items per CTA (SD3-size layers) is where LPT's tail is large and
    // the search is cheap: every CTA is a partner, and one item of the
    // costliest CTA may also trade for two cheaper ones (SD3 Arrow(8): 6.8%
    // -> 3.3% over the mean in the cost model). With many items per CTA
    // (FLUX) LPT is already within ~2%: the 16 lightest CTAs, single swaps.
    const bool deep = n_items <= static_cast<size_t>(6 * m);
    const int kLight = deep ? m : 16;  // lightest CTAs tried as partners
    const int max_iters = 4 * m;
    std::vector<int> order(static_cast<size_t>(m));
    for (int iter = 0; iter < max_iters; ++iter) {
        int cm = 0;
        for (int c = 1; c < m; ++c)
            if (load[c] > load[cm])
                cm = c;
        const double L = load[cm];
        for (int c = 0; c < m; ++c)
            order[c] = c;
        const int k = std::min(kLight, m);
        std::partial_sort(order.begin(), order.begin() + k, order.end(), [&](int a, int b) {
            return load[a] != load[b] ? load[a] < load[b] : a < b;
        });
        double best = L - 1e-9;
        int bi = -1, bc = -1, bj = -1, bk = -1;
        for (int i = 0; i < static_cast<int>(bins[cm].size()); ++i) {
            const double ci = bins[cm][i]->cost;
            for (int t = 0; t < k; ++t) {
                const int c = order[t];
                if (c == cm)
                    continue;
                const double mv = std::max(L - ci, load[c] + ci);
                if (mv < best) {
                    best = mv;
                    bi = i, bc = c, bj = -1, bk = -1;
                }
                const int nc = static_cast<int>(bins[c].size());
                for (int j = 0; j < nc; ++j) {
                    const double cj = bins[c][j]->cost;
                    if (cj >= ci)
                        continue;
                    const double sw = std::max(L - ci + cj, load[c] - cj + ci);
                    if (sw < best) {
                        best = sw;
                        bi = i, bc = c, bj = j, bk = -1;
                    }
                    if (!deep || nc > 8)
                        continue;
                    for (int q = j + 1; q < nc; ++q) {  // two of c's items for one of cm's
                        const double cjk = cj + bins[c][q]->cost;
                        if (cjk >= ci)
                            continue;
                        const double s2 = std::max(L - ci + cjk, load[c] - cjk + ci);
                        if (s2 < best) {
                            best = s2;
                            bi = i, bc = c, bj = j, bk = q;
                        }
                    }
                }
            }
        }
        if (bi < 0)
            return;
        const Cand* x = bins[cm][bi];
        bins[cm].erase(bins[cm].begin() + bi);
        load[cm] -= x->cost;
        if (bj >= 0) {
            // bk > bj: erase the later one first so bj stays valid
            if (bk >= 0) {
                const Cand* z = bins[bc][bk];
                bins[bc].erase(bins[bc].begin() + bk);
                load[bc] -= z->cost;
                bins[cm].push_back(z);
                load[cm] += z->cost;
            }
            const Cand* y = bins[bc][bj];
            bins[bc].erase(bins[bc].begin() + bj);
            load[bc] -= y->cost;
            bins[cm].push_back(y);
            load[cm] += y->cost;
        }
        bins[bc].push_back(x);
        load[bc] += x->cost;
    }
}

// LPT over `grid` CTAs of candidates already sorted costliest first, then
// (refine) the move / swap improvement above.
std::vector<std::vector<const Cand*>> assign_ctas(const std::vector<Cand>& cands, int grid, bool refine) {
    using Slot = std::pair<double, int>;
    std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> pq;
    for (int c = 0; c < grid; ++c)
        pq.push({0.0, c});
    std::vector<std::vector<const Cand*>> bins(static_cast<size_t>(grid));
    std::vector<double> load(static_cast<size_t>(grid), 0.0);
    for (const Cand& c : cands) {
        Slot s = pq.top();
        pq.pop();
        bins[s.second].push_back(&c);
        s.first += c.cost;
        load[s.second] = s.first;
        pq.push(s);
    }
    if (refine)
        refine_schedule(bins, load);
    return bins;
}

std::unique_ptr<DevPlan> schedule_items(int device, std::vector<Cand>& cands, const std::vector<uint32_t>& tiles,
                                        const std::vector<uint8_t>& mask_bytes, int32_t n_groups, int32_t n_slots,
                                        cudaStream_t stream) {
    std::stable_sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
        if (a.cost != b.cost)
            return a.cost > b.cost;
        if (a.w.bh != b.w.bh)
            return a.w.bh < b.w.bh;
        return a.w.qtile_a < b.w.qtile_a;
    });
    // copy pool: the Cached-head tiles leave the lists (LPT balances the
    // compute alone; every CTA drains the pool when its compute is done)
    std::vector<int2> copy_tiles;
    if (copy_pool_enabled()) {
        std::vector<Cand> compute;
        for (const Cand& c : cands) {
            if (c.w.flags & dfa2k::ITEM_COPY) {
                copy_tiles.push_back(make_int2(c.w.bh, c.w.qtile_a));
                if (c.w.qtile_b >= 0)
                    copy_tiles.push_back(make_int2(c.w.bh, c.w.qtile_b));
            } else {
                compute.push_back(c);
            }
        }
        cands.swap(compute);
    }
    const int64_t units = static_cast<int64_t>(cands.size() + copy_tiles.size());
    const int grid = static_cast<int>(std::min<int64_t>(num_sms(device), units));
    std::vector<std::vector<const Cand*>> bins = assign_ctas(cands, grid, true);
    std::vector<std::vector<WorkItem>> per_cta(static_cast<size_t>(grid));
    for (int c = 0; c < grid; ++c) {
        // costliest first within a CTA (LPT's order), copies last (the kernel's
        // copy tail streams a CTA's trailing copies through its freed rings)
        std::stable_sort(bins[c].begin(), bins[c].end(), [](const Cand* a, const Cand* b) {
            const bool ca = (a->w.flags & dfa2k::ITEM_COPY) != 0, cb = (b->w.flags & dfa2k::ITEM_COPY) != 0;
            return ca != cb ? cb : a->cost > b->cost;
        });
        for (const Cand* x : bins[c])
            per_cta[c].push_back(x->w);
    }
    std::vector<WorkItem> items;
    std::vector<int32_t> cta_begin(static_cast<size_t>(grid + 1), 0);
    bool copies_last = true;  // copies cost the least, so LPT leaves them at the end of every CTA
    for (int c = 0; c < grid; ++c) {
        bool seen_copy = false;
        for (const WorkItem& w : per_cta[c]) {
            const bool copy = (w.flags & dfa2k::ITEM_COPY) != 0;
            copies_last = copies_last && (copy || !seen_copy);
            seen_copy = seen_copy || copy;
        }
        items.insert(items.end(), per_cta[c].begin(), per_cta[c].end());
        cta_begin[c + 1] = static_cast<int32_t>(items.size());
    }

    auto p = std::make_unique<DevPlan>();
    p->grid = grid;
    p->copies_last = copies_last;
    p->n_copy_tiles = static_cast<int32_t>(copy_tiles.size());
    if (!copy_tiles.empty())
        copy_counter_base(device);
    p->n_groups = n_groups;
    p->n_slots = n_slots;
    p->device = device;
    // one block: [items | cta_begin | copy tiles | tiles | masks], 256-byte aligned parts
    auto up = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t o_items = 0, n_items = items.size() * sizeof(WorkItem);
    const size_t o_cta = up(o_items + n_items), n_cta = cta_begin.size() * sizeof(int32_t);
    const size_t o_copy = up(o_cta + n_cta), n_copy = copy_tiles.size() * sizeof(int2);
    const size_t o_tiles = up(o_copy + n_copy), n_tiles = tiles.size() * sizeof(uint32_t);
    const size_t o_masks = up(o_tiles + n_tiles), n_masks = mask_bytes.size();
    p->bytes = up(o_masks + n_masks);
    scratch_alloc(&p->dev, p->bytes, stream);
    char* d = static_cast<char*>(p->dev);
    p->items = reinterpret_cast<WorkItem*>(d + o_items);
    p->cta_begin = reinterpret_cast<int32_t*>(d + o_cta);
    p->copy_tiles = reinterpret_cast<int2*>(d + o_copy);
    p->tiles = reinterpret_cast<uint32_t*>(d + o_tiles);
    p->masks = reinterpret_cast<uint8_t*>(d + o_masks);
    plan_upload(device, stream, p->dev, p->bytes, [&](char* h) {
        std::memcpy(h + o_items, items.data(), n_items);
        std::memcpy(h + o_cta, cta_begin.data(), n_cta);
        if (n_copy)
            std::memcpy(h + o_copy, copy_tiles.data(), n_copy);
        std::memcpy(h + o_tiles, tiles.data(), n_tiles);
        std::memcpy(h + o_masks, mask_bytes.data(), n_masks);
    });
    DFA2C_CUDA_CHECK(cudaEventCreateWithFlags(&p->ready, cudaEventDisableTiming));
    DFA2C_CUDA_CHECK(cudaEventRecord(p->ready, stream));
    return p;
}

// Plans are cached per (device, geometry, plan) so steady-state calls only
// encode three tensor maps and launch.
std::mutex g_plan_mu;
std::map<std::string, std::shared_ptr<DevPlan>> g_plans;
std::deque<std::string> g_plan_order;  // insertion order, for eviction
size_t g_plan_bytes = 0;
// A calibrated FLUX schedule has one plan per (timestep, layer): 28 x 57 =
// 1,596 work lists of ~0.4 MB. Keep up to 8,192 plans / 4 GB.
constexpr size_t kMaxPlans = 8192;
constexpr size_t kMaxPlanBytes = size_t{4} << 30;
size_t max_plans() {  // DFA2_PLAN_CACHE_MAX overrides the count (tests exercise eviction with it)
    static const size_t v = [] {
        const char* e = std::getenv("DFA2_PLAN_CACHE_MAX");
        const long long x = e ? std::atoll(e) : 0;
        return x > 0 ? static_cast<size_t>(x) : kMaxPlans;
    }();
    return v;
}

bool stream_capturing(cudaStream_t stream) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    DFA2C_CUDA_CHECK(cudaStreamIsCapturing(stream, &st));
    return st != cudaStreamCaptureStatusNone;
}

// A plan captured into a CUDA graph: the graph orders itself after the
// plan's upload through an external event-wait node (a plain stream wait on
// an uncaptured event would invalidate the capture), and the plan stays
// allocated for the process lifetime.
std::mutex g_pinned_mu;
std::vector<std::shared_ptr<DevPlan>> g_pinned;
void pin_for_capture(const std::shared_ptr<DevPlan>& plan, cudaStream_t stream) {
    if (plan->ready)
        DFA2C_CUDA_CHECK(cudaStreamWaitEvent(stream, plan->ready, cudaEventWaitExternal));
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (std::find(g_pinned.begin(), g_pinned.end(), plan) == g_pinned.end())
        g_pinned.push_back(plan);
}

std::shared_ptr<DevPlan> plan_insert(const std::string& key, std::unique_ptr<DevPlan> p) {
    while (!g_plan_order.empty() && (g_plans.size() >= max_plans() || g_plan_bytes + p->bytes > kMaxPlanBytes)) {
        auto it = g_plans.find(g_plan_order.front());
        if (it != g_plans.end()) {
            g_plan_bytes -= it->second->bytes;
            g_plans.erase(it);
        }
        g_plan_order.pop_front();
    }
    g_plan_bytes += p->bytes;
    g_plan_order.push_back(key);
    std::shared_ptr<DevPlan> sp(std::move(p));
    g_plans.emplace(key, sp);
    return sp;
}

template <class T>
void put(std::string& key, const T& v) {
    key.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

// ------------------------------------------------------------ TMA maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q{};
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn)
        fail(DFA2C_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    return fn;
}

// [rows=batch*H][n][d] bf16, box {64 cols, box_rows rows, 1}, 128-byte
// swizzle: the canonical K-major SW128 UMMA layout (and MN-major for V).
CUtensorMap encode_map(const void* base, int64_t bh, int64_t n, int64_t d, int box_rows);

// Encoding is a pure host computation of the descriptor, and steady-state
// callers pass the same buffers every layer: a small per-thread cache keyed
// by (base, shape, box) saves ~0.5-1 us per map (five per launch).
CUtensorMap make_map(const void* base, int64_t bh, int64_t n, int64_t d, int box_rows) {
    struct Entry {
        const void* base;
        int64_t bh, n, d;
        int box;
        CUtensorMap m;
    };
    constexpr int kEntries = 16;
    thread_local Entry cache[kEntries];
    thread_local int next = 0;
    for (const Entry& e : cache)
        if (e.base == base && base && e.bh == bh && e.n == n && e.d == d && e.box == box_rows)
            return e.m;
    Entry& e = cache[next];
    next = (next + 1) % kEntries;
    e.m = encode_map(base, bh, n, d, box_rows);
    e.base = base;
    e.bh = bh;
    e.n = n;
    e.d = d;
    e.box = box_rows;
    return e.m;
}

CUtensorMap encode_map(const void* base, int64_t bh, int64_t n, int64_t d, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(n),
                                static_cast<cuuint64_t>(bh)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(d * 2), static_cast<cuuint64_t>(n * d * 2)};
    const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(DFA2C_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
    return m;
}

void check_ptr(const void* p, const char* what) {
    if (!p)
        fail(DFA2C_SHAPE, std::string(what) + " must not be NULL");
    if (reinterpret_cast<uintptr_t>(p) % 16 != 0)
        fail(DFA2C_SHAPE, std::string(what) + " must be 16-byte aligned");
}

}  // namespace

// ---------------------------------------------------------------- cache
struct dfa2c_cache {
    int64_t L = 0, H = 0, batch = 0, n = 0, d = 0;
    int device = 0;
    std::vector<void*> layer_buf;    // [L] -> [batch, H, n, d] bf16, lazily allocated
    std::vector<cudaEvent_t> layer_ready;  // [L] the buffer's allocation + zero fill has landed
    std::vector<int64_t> produced;   // [L*H], INT64_MIN = empty slot

    // Layer buffers come from the library's device pool (release threshold
    // max): a cache of 57 FLUX layers (5.9 GB) is created and destroyed in
    // microseconds instead of paying cudaMalloc / cudaFree (unmap) per layer.
    ~dfa2c_cache() {
        bool any = false;
        for (void* p : layer_buf)
            any |= p != nullptr;
        if (!any)
            return;
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaDeviceSynchronize();  // no launch may still read or write a slot
        for (void* p : layer_buf)
            if (p)
                cudaFreeAsync(p, nullptr);
        for (cudaEvent_t e : layer_ready)
            if (e)
                cudaEventDestroy(e);
        cudaSetDevice(cur);
    }
    size_t slot_elems() const { return static_cast<size_t>(n * d); }
    size_t layer_bytes() const { return static_cast<size_t>(batch * H * n * d) * 2; }
    // n_layers is a capacity hint: like the reference's map-backed HeadCache
    // (src/cache.cpp), any layer index >= 0 is accepted; storage grows.
    void ensure(int64_t layer) {
        if (layer >= L) {
            layer_buf.resize(static_cast<size_t>(layer + 1), nullptr);
            layer_ready.resize(static_cast<size_t>(layer + 1), nullptr);
            std::vector<int64_t> p(static_cast<size_t>((layer + 1) * H), std::numeric_limits<int64_t>::min());
            std::copy(produced.begin(), produced.end(), p.begin());
            produced.swap(p);
            L = layer + 1;
        }
    }
    void check(int64_t layer, int64_t head) {
        if (layer < 0 || head < 0 || head >= H)
            fail(DFA2C_SHAPE, "cache slot (" + std::to_string(layer) + ", " + std::to_string(head) +
                                  ") out of range");
        ensure(layer);
    }
    bool has(int64_t layer, int64_t head) const {
        return layer >= 0 && layer < L && head >= 0 && head < H &&
               produced[static_cast<size_t>(layer * H + head)] != std::numeric_limits<int64_t>::min();
    }
    // The layer's slot buffer, ordered on `st`: created (pool allocation +
    // zero fill) on the first caller's stream; a caller on any other stream
    // first waits for that to have landed.
    void* layer_ptr(int64_t layer, cudaStream_t st) {
        if (!layer_buf[layer]) {
            DFA2C_CUDA_CHECK(cudaMallocFromPoolAsync(&layer_buf[layer], layer_bytes(), scratch_pool(device), st));
            DFA2C_CUDA_CHECK(cudaMemsetAsync(layer_buf[layer], 0, layer_bytes(), st));
            DFA2C_CUDA_CHECK(cudaEventCreateWithFlags(&layer_ready[layer], cudaEventDisableTiming));
            DFA2C_CUDA_CHECK(cudaEventRecord(layer_ready[layer], st));
        } else {
            order_after_ready(layer, st);
        }
        return layer_buf[layer];
    }
    // Under CUDA-graph capture: the buffer must exist and be initialised
    // (no stream ordering can be captured against its allocation).
    void* layer_ptr_captured(int64_t layer, cudaStream_t st) {
        if (!layer_buf[layer])
            fail(DFA2C_UNSUPPORTED, "CUDA-graph capture: the cache layer is not allocated yet (run the layer "
                                    "once without capture first)");
        if (layer_ready[layer])  // an external event-wait node in the graph
            DFA2C_CUDA_CHECK(cudaStreamWaitEvent(st, layer_ready[layer], cudaEventWaitExternal));
        return layer_buf[layer];
    }
    void order_after_ready(int64_t layer, cudaStream_t st) const {
        if (layer >= 0 && layer < L && layer_ready[layer])
            DFA2C_CUDA_CHECK(cudaStreamWaitEvent(st, layer_ready[layer], 0));
    }
};

namespace {

struct ForwardSpec {
    const void *q, *k, *v;
    void* out;
    int64_t batch;
    const dfa2c_dims* dims;
    int64_t block;
    std::vector<std::vector<uint8_t>> masks;  // distinct masks (explicit, or built from mask_windows on a plan miss)
    std::vector<int64_t> mask_windows;        // per distinct mask: -1 = all active, else arrow window
    std::vector<HeadJob> jobs;                // per head (JOB_SKIP: not part of this launch)
    std::vector<int> ref_jobs;                // per head, the layer plan's job before any skipping
    std::string mask_key;                     // identifies the masks in the plan cache
    dfa2c_cache* cache;                       // slots read (copy) / written (commit)
    int64_t layer;
    int64_t scale_d = 0;                      // head dim of the softmax scale (0: dims->head_dim)
    int32_t n_parts = 0;                      // sharded launch: the layer cut into n_parts ranges...
    int32_t part = 0;                         // ...of which this launch runs `part`
    std::vector<int64_t>* shard_rows = nullptr;  // out: [n_parts + 1] flattened row bounds
    std::vector<void*> peer_outs;                // sharded P2P: the other ranks' out buffers (this process's mappings)
};

// The kernel instantiations: D = 64 serves head dims 1..64, D = 128 serves 65..128.
int kernel_dim(int64_t d) { return d <= 64 ? 64 : 128; }
// TMA maps over the caller's own [.., d] layout need a 16-byte row pitch and
// a full first 64-column box; other head dims run through zero-padded copies.
bool direct_layout(int64_t d) { return d == 64 || (d % 8 == 0 && d >= 64 && d <= 128); }

void launch_forward(const ForwardSpec& s, cudaStream_t stream);

// Head dims without a direct TMA layout (d % 8 != 0 or d < 64): q/k/v are
// copied into zero-padded [rows, D] scratch (zero columns change neither
// Q K^T nor the first d columns of P V; the softmax scale keeps the true d),
// the kernel runs with no cache binding, and the outputs, cache commits and
// cached-head copies are done as strided copies on the same stream.
void run_padded(const ForwardSpec& s, cudaStream_t st) {
    const int64_t n = seq_len(s.dims), d = s.dims->head_dim, H = s.dims->n_heads;
    const int64_t D = kernel_dim(d);
    if (s.batch < 1)
        fail(DFA2C_SHAPE, "batch must be >= 1");
    for (const void* x : {s.q, s.k, s.v, static_cast<const void*>(s.out)})
        if (!x)
            fail(DFA2C_SHAPE, "q, k, v and out must not be NULL");
    const size_t rows = static_cast<size_t>(s.batch * H * n);
    const size_t pbytes = rows * static_cast<size_t>(D) * 2;
    void *qp = nullptr, *kp = nullptr, *vp = nullptr, *op = nullptr;
    scratch_alloc(&qp, pbytes, st);
    scratch_alloc(&kp, pbytes, st);
    scratch_alloc(&vp, pbytes, st);
    scratch_alloc(&op, pbytes, st);
    const std::pair<const void*, void*> ins[3] = {{s.q, qp}, {s.k, kp}, {s.v, vp}};
    for (const auto& [src, dst] : ins) {
        DFA2C_CUDA_CHECK(cudaMemsetAsync(dst, 0, pbytes, st));
        DFA2C_CUDA_CHECK(cudaMemcpy2DAsync(dst, D * 2, src, d * 2, d * 2, rows, cudaMemcpyDeviceToDevice, st));
    }
    dfa2c_dims pd = *s.dims;
    pd.head_dim = D;
    ForwardSpec p = s;
    p.q = qp;
    p.k = kp;
    p.v = vp;
    p.out = op;
    p.dims = &pd;
    p.cache = nullptr;
    p.scale_d = d;
    bool any = false;
    for (HeadJob& j : p.jobs) {
        if (j.mask_id == JOB_COPY)
            j.mask_id = JOB_SKIP;
        j.commit = false;
        any |= j.mask_id >= 0;
    }
    if (any) {
        launch_forward(p, st);
        // every row back to the caller's layout; rows of heads the kernel
        // skipped are rewritten below or belong to other launches' heads
        // (host-path groups), so copy computed heads only
        const size_t head_rows = static_cast<size_t>(n);
        for (int64_t b = 0; b < s.batch; ++b)
            for (int64_t h = 0; h < H; ++h)
                if (p.jobs[h].mask_id >= 0) {
                    const size_t r0 = static_cast<size_t>(b * H + h) * head_rows;
                    DFA2C_CUDA_CHECK(cudaMemcpy2DAsync(static_cast<char*>(s.out) + r0 * d * 2, d * 2,
                                                       static_cast<const char*>(op) + r0 * D * 2, D * 2, d * 2,
                                                       head_rows, cudaMemcpyDeviceToDevice, st));
                }
    }
    void* cache_layer = nullptr;
    for (const HeadJob& j : s.jobs)
        if ((j.mask_id == JOB_COPY || j.commit) && !cache_layer) {
            if (!s.cache)
                fail(DFA2C_CACHE_MISS, "cached heads need a cache");
            s.cache->ensure(s.layer);
            cache_layer = s.cache->layer_ptr(s.layer, st);
        }
    const size_t head_bytes = static_cast<size_t>(n * d) * 2;
    for (int64_t h = 0; h < H; ++h) {
        const HeadJob& j = s.jobs[h];
        if (j.mask_id != JOB_COPY && !j.commit)
            continue;
        // per head, one strided copy over the samples ([batch, H, n, d] layout on both sides)
        char* slot = static_cast<char*>(cache_layer) + h * head_bytes;
        char* o = static_cast<char*>(s.out) + h * head_bytes;
        if (j.mask_id == JOB_COPY)
            DFA2C_CUDA_CHECK(cudaMemcpy2DAsync(o, H * head_bytes, slot, H * head_bytes, head_bytes, s.batch,
                                               cudaMemcpyDeviceToDevice, st));
        else
            DFA2C_CUDA_CHECK(cudaMemcpy2DAsync(slot, H * head_bytes, o, H * head_bytes, head_bytes, s.batch,
                                               cudaMemcpyDeviceToDevice, st));
    }
    for (void* x : {qp, kp, vp, op})
        DFA2C_CUDA_CHECK(cudaFreeAsync(x, st));
}

// Head dims above 128 (the reference accepts any d >= 1, src/tensor.cpp:
// 225-230): the tcgen05 kernel's TMEM budget (two lanes of S + O) holds
// d <= 128, so wider heads run through the SIMT attention kernel
// (reference_sm100.cu, one warp per query row) in f32 on the bf16 inputs,
// head by head with the head's own block mask, and the result is rounded to
// bf16 like the fused path's. Cached heads and cache commits are copies on
// the same stream. Correct for any plan; not the performance path.
void run_wide(const ForwardSpec& s, cudaStream_t st) {
    const int64_t n = seq_len(s.dims), d = s.dims->head_dim, H = s.dims->n_heads;
    if (s.batch < 1)
        fail(DFA2C_SHAPE, "batch must be >= 1");
    if (s.n_parts > 0)
        fail(DFA2C_UNSUPPORTED, "sharded launches need head_dim <= 128");
    check_ptr(s.q, "q");
    check_ptr(s.k, "k");
    check_ptr(s.v, "v");
    check_ptr(s.out, "out");
    const int64_t nb = ceil_div(n, s.block);
    const size_t head_elems = static_cast<size_t>(n * d);
    const size_t head_bytes = head_elems * 2;
    int device = 0;
    DFA2C_CUDA_CHECK(cudaGetDevice(&device));
    const int sms = num_sms(device);
    // distinct masks on the device (null: every key of every row)
    std::vector<void*> dmasks;
    const size_t n_masks = std::max(s.masks.size(), s.mask_windows.size());
    for (size_t m = 0; m < n_masks; ++m) {
        std::vector<uint8_t> bytes;
        if (!s.masks.empty())
            bytes = s.masks[m];
        else if (s.mask_windows[m] >= 0)
            bytes = arrow_mask(s.dims, s.block, s.mask_windows[m]);
        void* dm = nullptr;
        if (!bytes.empty()) {
            for (int64_t r = 0; r < nb; ++r)  // FullyMaskedRowError before any compute
                if (std::none_of(bytes.begin() + r * nb, bytes.begin() + (r + 1) * nb, [](uint8_t x) { return x; }))
                    fail(DFA2C_FULLY_MASKED, "query block " + std::to_string(r) + " has no active key blocks");
            scratch_alloc(&dm, bytes.size(), st);
            DFA2C_CUDA_CHECK(cudaMemcpyAsync(dm, bytes.data(), bytes.size(), cudaMemcpyHostToDevice, st));
        }
        dmasks.push_back(dm);
    }
    void* cache_layer = nullptr;
    for (const HeadJob& j : s.jobs)
        if ((j.mask_id == JOB_COPY || j.commit) && !cache_layer) {
            if (!s.cache)
                fail(DFA2C_CACHE_MISS, "cached heads need a cache");
            s.cache->ensure(s.layer);
            cache_layer = s.cache->layer_ptr(s.layer, st);
        }
    void *qf = nullptr, *kf = nullptr, *vf = nullptr, *of = nullptr;
    for (void** p : {&qf, &kf, &vf, &of})
        scratch_alloc(p, head_elems * 4, st);
    for (int64_t b = 0; b < s.batch; ++b)
        for (int64_t h = 0; h < H; ++h) {
            const HeadJob& j = s.jobs[h];
            const size_t off = static_cast<size_t>(b * H + h) * head_bytes;
            char* o = static_cast<char*>(s.out) + off;
            if (j.mask_id == JOB_SKIP)
                continue;
            if (j.mask_id == JOB_COPY) {
                DFA2C_CUDA_CHECK(cudaMemcpyAsync(o, static_cast<const char*>(cache_layer) + off, head_bytes,
                                                 cudaMemcpyDeviceToDevice, st));
                continue;
            }
            const std::pair<const void*, void*> ins[3] = {{s.q, qf}, {s.k, kf}, {s.v, vf}};
            for (const auto& [src, dst] : ins)
                DFA2C_CUDA_CHECK(dfa2k::launch_convert(static_cast<const char*>(src) + off, DFA2C_BF16, dst, DFA2C_F32,
                                                       static_cast<int64_t>(head_elems), sms, st));
            DFA2C_CUDA_CHECK(dfa2k::launch_attention_reference(qf, kf, vf, of, DFA2C_F32, 1, n, d,
                                                               static_cast<const uint8_t*>(dmasks[j.mask_id]),
                                                               s.block, nb, st));
            DFA2C_CUDA_CHECK(dfa2k::launch_convert(of, DFA2C_F32, o, DFA2C_BF16, static_cast<int64_t>(head_elems),
                                                   sms, st));
            if (j.commit)
                DFA2C_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(cache_layer) + off, o, head_bytes,
                                                 cudaMemcpyDeviceToDevice, st));
        }
    for (void* x : {qf, kf, vf, of})
        DFA2C_CUDA_CHECK(cudaFreeAsync(x, st));
    for (void* dm : dmasks)
        if (dm)
            DFA2C_CUDA_CHECK(cudaFreeAsync(dm, st));
    g_launches.fetch_add(1);
}

void run_forward(const ForwardSpec& s, cudaStream_t stream) {
    const int64_t d = s.dims->head_dim;
    if (d < 1 || d > dfa2k::reference_max_head_dim())
        fail(DFA2C_UNSUPPORTED, "head_dim must be in [1, " + std::to_string(dfa2k::reference_max_head_dim()) +
                                    "] (got " + std::to_string(d) + ")");
    if (d > 128)
        run_wide(s, stream);
    else if (direct_layout(d))
        launch_forward(s, stream);
    else
        run_padded(s, stream);
}

// Text rows run on both lanes when their key chains exceed this many tenths
// of the mask's average chain (0: never): d = 64 from 5x.
#ifndef DFA2_HALVES64_DEFAULT
#define DFA2_HALVES64_DEFAULT 50
#endif
#ifndef DFA2_HALVES128_DEFAULT
#define DFA2_HALVES128_DEFAULT 0
#endif
int64_t halve_ratio(int64_t d) {
    static const int64_t r128 = [] {
        const char* e = std::getenv("DFA2_HALVES128");
        return e ? 10 * std::atoll(e) : DFA2_HALVES128_DEFAULT;
    }();
    return kernel_dim(d) == 64 ? DFA2_HALVES64_DEFAULT : r128;
}

void launch_forward(const ForwardSpec& s, cudaStream_t stream) {
    const int64_t n = seq_len(s.dims), d = s.dims->head_dim, H = s.dims->n_heads;
    if (s.batch < 1)
        fail(DFA2C_SHAPE, "batch must be >= 1");
    if (s.batch * H > std::numeric_limits<int32_t>::max() / 2 || n > (1 << 24))
        fail(DFA2C_UNSUPPORTED, "problem too large for the 32-bit tile coordinates");
    check_ptr(s.q, "q");
    check_ptr(s.k, "k");
    check_ptr(s.v, "v");
    check_ptr(s.out, "out");
    int device = 0;
    DFA2C_CUDA_CHECK(cudaGetDevice(&device));

    std::string key;
    put(key, device);
    put(key, s.batch);
    put(key, H);
    put(key, n);
    put(key, d);
    put(key, s.block);
    for (const HeadJob& j : s.jobs) {
        put(key, j.mask_id);
        put(key, j.commit);
    }
    put(key, split_kv_enabled());
    if (split_kv_enabled())
        for (int rj : s.ref_jobs)
            put(key, rj);
    put(key, s.n_parts);
    put(key, s.part);
    key += s.mask_key;

    // CUDA-graph capture: a launch on a capturing stream must not touch
    // uncaptured work (no waits on the plan's upload or on other streams),
    // so it needs a work list a plain call already built and uploaded; that
    // plan is pinned for the life of the process, since the graph holds its
    // device memory.
    const bool capturing = stream_capturing(stream);
    std::shared_ptr<DevPlan> plan;
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        auto it = g_plans.find(key);
        if (it != g_plans.end()) {
            plan = it->second;
        } else if (capturing) {
            fail(DFA2C_UNSUPPORTED, "CUDA-graph capture of a layer needs one plain call with the same plan and "
                                    "shapes first (it builds and uploads the work list)");
        } else {
            // masks are only materialised when the work list has to be built
            std::vector<std::vector<uint8_t>> built;
            const std::vector<std::vector<uint8_t>>* masks = &s.masks;
            if (s.masks.empty() && !s.mask_windows.empty()) {
                const int64_t nb = ceil_div(n, s.block);
                for (int64_t w : s.mask_windows)
                    built.push_back(w < 0 ? std::vector<uint8_t>(static_cast<size_t>(nb * nb), uint8_t{1})
                                          : arrow_mask(s.dims, s.block, w));
                masks = &built;
            }
            plan = plan_insert(key, build_dev_plan(device, s.batch, H, n, s.block, *masks, s.jobs, s.ref_jobs,
                                                   text_begin(s.dims), text_end(s.dims), halve_ratio(d),
                                                   stream, s.n_parts, s.part));
        }
    }
    if (s.shard_rows)
        *s.shard_rows = plan->shard_rows;

    void* cache_layer = nullptr;
    bool need_cache = false;
    for (const HeadJob& j : s.jobs)
        need_cache |= (j.mask_id == JOB_COPY) || j.commit;
    if (need_cache) {
        if (!s.cache)
            fail(DFA2C_CACHE_MISS, "cached heads need a cache");
        s.cache->ensure(s.layer);
        cache_layer = capturing ? s.cache->layer_ptr_captured(s.layer, stream) : s.cache->layer_ptr(s.layer, stream);
    }

    const int64_t bh = s.batch * H;
    const CUtensorMap tq = make_map(s.q, bh, n, d, dfa2k::TILE_M);
    const CUtensorMap tk = make_map(s.k, bh, n, d, dfa2k::TILE_N);
    const CUtensorMap tv = make_map(s.v, bh, n, d, dfa2k::TILE_N);
    const CUtensorMap to = make_map(s.out, bh, n, d, dfa2k::TILE_M);
    const CUtensorMap tc = cache_layer ? make_map(cache_layer, bh, n, d, dfa2k::TILE_M) : to;
    dfa2k::AttnArgs a{};
    a.items = plan->items;
    a.cta_begin = plan->cta_begin;
    a.tiles = plan->tiles;
    a.masks = plan->masks;
    a.out = static_cast<__nv_bfloat16*>(s.out);
    a.cache = static_cast<__nv_bfloat16*>(cache_layer);
    a.n = static_cast<int32_t>(n);
    a.copies_last = plan->copies_last && copy_tail_enabled() ? 1 : 0;
    a.n_copy_tiles = plan->n_copy_tiles;
    a.copy_tiles = plan->copy_tiles;
    a.row_bytes = static_cast<int32_t>(d * 2);
    a.copy_ctr = plan->n_copy_tiles > 0 ? copy_counter_slot(device) : nullptr;
    a.block = static_cast<int32_t>(std::min<int64_t>(s.block, int64_t{1} << 30));
    a.nb = static_cast<int32_t>(ceil_div(n, s.block));
    a.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(s.scale_d ? s.scale_d : d)));
    a.trace = g_trace;
    if (plan->grid == 0)
        return;  // nothing to launch (every head skipped)
    // split-KV scratch: stream-ordered from the library pool, counters zeroed
    // per launch, released after the launch on the same stream
    if (plan->n_groups > 0) {
        const int D = kernel_dim(d);
        scratch_alloc(&a.part_o, static_cast<size_t>(plan->n_slots) * 2 * D * dfa2k::TILE_M * sizeof(float), stream);
        scratch_alloc(&a.part_ml, static_cast<size_t>(plan->n_slots) * 2 * 2 * dfa2k::TILE_M * sizeof(float), stream);
        scratch_alloc(&a.counters, static_cast<size_t>(plan->n_groups) * 2 * sizeof(int), stream);
        DFA2C_CUDA_CHECK(cudaMemsetAsync(a.counters, 0, static_cast<size_t>(plan->n_groups) * 2 * sizeof(int), stream));
    }
    if (capturing)
        pin_for_capture(plan, stream);
    else
        plan->acquire(stream);
    dfa2k::PeerMaps peers;
    std::memset(&peers, 0, sizeof peers);
    if (s.peer_outs.size() > static_cast<size_t>(dfa2k::MAX_PEERS))
        fail(DFA2C_UNSUPPORTED, "at most " + std::to_string(dfa2k::MAX_PEERS) + " peer outputs");
    for (size_t i = 0; i < s.peer_outs.size(); ++i) {
        check_ptr(s.peer_outs[i], "peer out");
        peers.m[i] = make_map(s.peer_outs[i], bh, n, d, dfa2k::TILE_M);
        peers.ptr[i] = s.peer_outs[i];
    }
    a.n_peers = static_cast<int32_t>(s.peer_outs.size());
    DFA2C_CUDA_CHECK(dfa2k::launch_attn(kernel_dim(d), tq, tk, tv, to, tc, a, peers, plan->grid, stream));
    if (!capturing)
        plan->release(stream);
    if (plan->n_groups > 0) {
        DFA2C_CUDA_CHECK(cudaFreeAsync(a.part_o, stream));
        DFA2C_CUDA_CHECK(cudaFreeAsync(a.part_ml, stream));
        DFA2C_CUDA_CHECK(cudaFreeAsync(a.counters, stream));
    }
    g_launches.fetch_add(1);
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// ------------------------------------------------- fused calibration pass
// influence_for_layer (src/calibrate.cpp:193-253) evaluates the original
// (all heads Full) and one all-heads Arrow(w) output per candidate window:
// 1 + |windows| attention passes. Arrow masks are nested in w, so one pass
// that folds every query tile's key tiles band by band — band 0 = the
// narrowest candidate's keys, band i = the keys the i-th window adds, the
// last band = the rest of the row — holds each candidate's exact key set
// after its band, and a snapshot of O / l there IS that candidate's output
// (SURVEY.md §8f-1). The kernel writes it to the candidate's output and
// carries on; one launch computes the original plus every Arrow candidate
// for the cost of the original. Results agree with the per-candidate passes
// up to the fold order of the key tiles (bf16 rounding of the outputs);
// dfa2c_set_influence_fused(0) selects the per-candidate passes, whose
// outputs are bitwise those of dfa2c_mha_forward.
std::atomic<int> g_influence_fused{-1};
bool influence_fused_enabled() {
    int v = g_influence_fused.load();
    if (v < 0) {
        const char* e = std::getenv("DFA2_INFLUENCE_FUSED");
        v = (e && e[0] == '0') ? 0 : 1;
        int expect = -1;
        g_influence_fused.compare_exchange_strong(expect, v);
        v = g_influence_fused.load();
    }
    return v == 1;
}

// Mask blocks must be the kernel's 128-key tiles (bands are whole tiles) and
// the head dim one the kernel reads in place.
bool influence_fused_eligible(const dfa2c_dims* dims, int64_t block, int64_t n_windows) {
    return influence_fused_enabled() && block == dfa2k::TILE_N && direct_layout(dims->head_dim) &&
           n_windows >= 1 && n_windows < dfa2k::MAX_SNAPS;
}

// One item per pair of query tiles (2p, 2p+1). Each lane folds every key
// tile of its row, band by band; a tile both lanes take in the same band is
// one shared K/V load, a tile in different bands of the two lanes is loaded
// once per lane. A lane's last tile of band i (i < last band) carries its
// SNAP bit unless it is the lane's last tile overall (the item end emits
// every remaining snapshot from the final state).
std::unique_ptr<DevPlan> build_multi_plan(int device, int64_t H, int64_t n,
                                          const std::vector<std::vector<uint8_t>>& bands, cudaStream_t stream) {
    const int64_t nt = ceil_div(n, dfa2k::TILE_N);  // key tiles == mask blocks (block == 128)
    const int64_t np = (nt + 1) / 2;
    const int S = static_cast<int>(bands.size());
    const bool ragged = n % dfa2k::TILE_N != 0;
    std::vector<uint32_t> tiles;
    struct PairWords {
        int64_t begin, len;
    };
    std::vector<PairWords> pw(static_cast<size_t>(np));
    std::vector<int> ba(static_cast<size_t>(nt)), bb(static_cast<size_t>(nt));
    auto band_of = [&](int64_t q, int64_t t) {
        for (int s = 0; s < S; ++s)
            if (bands[s][q * nt + t])
                return s;
        return S;
    };
    for (int64_t p = 0; p < np; ++p) {
        const int64_t qa = 2 * p, qb = 2 * p + 1;
        const bool has_b = qb < nt;
        for (int64_t t = 0; t < nt; ++t) {
            ba[t] = band_of(qa, t);
            bb[t] = has_b ? band_of(qb, t) : -1;
        }
        const int64_t begin = static_cast<int64_t>(tiles.size());
        std::vector<int64_t> snap_a, snap_b;  // per band: index of the lane's last tile in it
        int64_t last_a = -1, last_b = -1;
        for (int s = 0; s <= S; ++s) {
            int64_t ra = -1, rb = -1;
            auto push = [&](int64_t t, bool a, bool b) {
                uint32_t wd = static_cast<uint32_t>(t);
                const bool part = ragged && t == nt - 1;
                if (a)
                    wd |= dfa2k::TILE_NEED_A | (part ? dfa2k::TILE_PART_A : 0u);
                if (b)
                    wd |= dfa2k::TILE_NEED_B | (part ? dfa2k::TILE_PART_B : 0u);
                tiles.push_back(wd);
                const int64_t idx = static_cast<int64_t>(tiles.size()) - 1;
                if (a)
                    ra = last_a = idx;
                if (b)
                    rb = last_b = idx;
            };
            for (int64_t t = 0; t < nt; ++t)  // shared loads first
                if (ba[t] == s && bb[t] == s)
                    push(t, true, true);
            // single-lane loads alternate lanes, so one lane's MMAs still
            // overlap the other lane's softmax
            std::vector<int64_t> only_a, only_b;
            for (int64_t t = 0; t < nt; ++t) {
                if (ba[t] == s && bb[t] != s)
                    only_a.push_back(t);
                if (bb[t] == s && ba[t] != s)
                    only_b.push_back(t);
            }
            for (size_t i = 0; i < std::max(only_a.size(), only_b.size()); ++i) {
                if (i < only_a.size())
                    push(only_a[i], true, false);
                if (i < only_b.size())
                    push(only_b[i], false, true);
            }
            if (s < S) {
                snap_a.push_back(ra);
                snap_b.push_back(rb);
            }
        }
        for (int64_t i : snap_a)
            if (i >= 0 && i != last_a)
                tiles[i] |= dfa2k::TILE_SNAP_A;
        for (int64_t i : snap_b)
            if (i >= 0 && i != last_b)
                tiles[i] |= dfa2k::TILE_SNAP_B;
        pw[p] = {begin, static_cast<int64_t>(tiles.size()) - begin};
    }
    if (tiles.size() > static_cast<size_t>(std::numeric_limits<int32_t>::max()) || nt > (1 << 24))
        fail(DFA2C_UNSUPPORTED, "work list too large");
    // element masking of the ragged last key tile reads an all-active mask
    const std::vector<uint8_t> mask_bytes(static_cast<size_t>(nt * nt), uint8_t{1});
    std::vector<Cand> cands;
    for (int64_t h = 0; h < H; ++h)
        for (int64_t p = 0; p < np; ++p) {
            WorkItem w{};
            w.bh = static_cast<int32_t>(h);
            w.qtile_a = static_cast<int32_t>(2 * p);
            w.qtile_b = 2 * p + 1 < nt ? static_cast<int32_t>(2 * p + 1) : -1;
            w.tile_begin = static_cast<int32_t>(pw[p].begin);
            w.n_tiles = static_cast<int32_t>(pw[p].len);
            w.mask_off = 0;
            w.flags = dfa2k::ITEM_MULTI;
            cands.push_back({w, static_cast<double>(nt * (w.qtile_b >= 0 ? 2 : 1)) + 1.0 + 0.25 * S});
        }
    return schedule_items(device, cands, tiles, mask_bytes, 0, 0, stream);
}

// The fused pass: `orig` <- all-Full output, `cand` + m * layer <- Arrow(windows[m])
// output, every head, batch 1.
void run_influence_fused(const void* q, const void* k, const void* v, const dfa2c_dims* dims,
                         const int64_t* windows, int64_t n_windows, void* orig, void* cand, cudaStream_t stream) {
    const int64_t n = seq_len(dims), d = dims->head_dim, H = dims->n_heads;
    const int64_t B = dfa2k::TILE_N;
    if (H * n_windows > std::numeric_limits<int32_t>::max() / 2 || n > (1 << 24))
        fail(DFA2C_UNSUPPORTED, "problem too large for the 32-bit tile coordinates");
    check_ptr(q, "q");
    check_ptr(k, "k");
    check_ptr(v, "v");
    check_ptr(orig, "original");
    check_ptr(cand, "method outputs");
    int device = 0;
    DFA2C_CUDA_CHECK(cudaGetDevice(&device));
    std::string key = "influence";
    put(key, device);
    put(key, H);
    put(key, n);
    put(key, d);
    put(key, dims->n_visual);
    put(key, dims->order);
    for (int64_t m = 0; m < n_windows; ++m)
        put(key, windows[m]);
    std::shared_ptr<DevPlan> plan;
    {
        std::lock_guard<std::mutex> lk(g_plan_mu);
        auto it = g_plans.find(key);
        if (it != g_plans.end()) {
            plan = it->second;
        } else {
            // distinct effective windows (the clamp of src/arrow.cpp:135-137),
            // narrowest first: their masks are nested; a window whose mask is
            // all-active is the original's full row
            const int64_t nvb = ceil_div(dims->n_visual, B);
            std::map<int64_t, uint32_t> by_window;
            for (int64_t m = 0; m < n_windows; ++m)
                by_window[std::min(windows[m], std::max<int64_t>(0, nvb - 1))] |= 1u << m;
            uint32_t full_slots = dfa2k::SNAP_ORIGINAL;
            std::vector<std::vector<uint8_t>> bands;
            std::vector<uint32_t> band_slots;
            for (const auto& [w, bits] : by_window) {
                std::vector<uint8_t> mk = arrow_mask(dims, B, w);
                if (std::all_of(mk.begin(), mk.end(), [](uint8_t x) { return x != 0; })) {
                    full_slots |= bits;
                } else {
                    bands.push_back(std::move(mk));
                    band_slots.push_back(bits);
                }
            }
            auto p = build_multi_plan(device, H, n, bands, stream);
            p->n_snap = static_cast<int32_t>(bands.size()) + 1;
            for (size_t i = 0; i < bands.size(); ++i)
                p->snap_slots[i] = static_cast<uint16_t>(band_slots[i]);
            p->snap_slots[bands.size()] = static_cast<uint16_t>(full_slots);
            plan = plan_insert(key, std::move(p));
        }
    }
    const CUtensorMap tq = make_map(q, H, n, d, dfa2k::TILE_M);
    const CUtensorMap tk = make_map(k, H, n, d, dfa2k::TILE_N);
    const CUtensorMap tv = make_map(v, H, n, d, dfa2k::TILE_N);
    const CUtensorMap to = make_map(cand, H * n_windows, n, d, dfa2k::TILE_M);
    const CUtensorMap tc = make_map(orig, H, n, d, dfa2k::TILE_M);
    dfa2k::AttnArgs a{};
    a.items = plan->items;
    a.cta_begin = plan->cta_begin;
    a.tiles = plan->tiles;
    a.masks = plan->masks;
    a.out = static_cast<__nv_bfloat16*>(cand);
    a.cache = nullptr;
    a.n = static_cast<int32_t>(n);
    a.block = static_cast<int32_t>(B);
    a.nb = static_cast<int32_t>(ceil_div(n, B));
    a.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(d)));
    a.trace = g_trace;
    a.snap_stride = static_cast<int32_t>(H);
    a.n_snap = plan->n_snap;
    if (plan->n_copy_tiles)
        fail(DFA2C_UNSUPPORTED, "calibration plans have no cached heads");
    std::copy(plan->snap_slots, plan->snap_slots + dfa2k::MAX_SNAPS, a.snap_slots);
    plan->acquire(stream);
    dfa2k::PeerMaps no_peers;
    std::memset(&no_peers, 0, sizeof no_peers);
    DFA2C_CUDA_CHECK(dfa2k::launch_attn(kernel_dim(d), tq, tk, tv, to, tc, a, no_peers, plan->grid, stream));
    plan->release(stream);
    g_launches.fetch_add(1);
}

// Standard per-call mask bookkeeping for a LayerPlan: one mask per distinct
// window (src/dispatch.cpp:38-54) plus the all-active mask for Full heads.
void plan_jobs(const dfa2c_dims* dims, int64_t /*block*/, const int32_t* kinds, const int64_t* windows,
               bool commit, ForwardSpec& s) {
    std::map<int64_t, int> ids;  // -1 = full, else window
    for (int64_t h = 0; h < dims->n_heads; ++h) {
        const int32_t k = kind_of(kinds[h]);
        if (k == DFA2C_CACHED) {
            s.ref_jobs.push_back(JOB_COPY);
            s.jobs.push_back({skipped(kinds[h]) ? JOB_SKIP : JOB_COPY, false});
            continue;
        }
        const int64_t key = k == DFA2C_FULL ? -1 : windows[h];
        auto it = ids.find(key);
        if (it == ids.end()) {
            it = ids.emplace(key, static_cast<int>(s.mask_windows.size())).first;
            s.mask_windows.push_back(key);  // built lazily, on a plan-cache miss
            put(s.mask_key, key);
        }
        s.ref_jobs.push_back(it->second);
        s.jobs.push_back({skipped(kinds[h]) ? JOB_SKIP : it->second, commit});
    }
    put(s.mask_key, dims->n_visual);
    put(s.mask_key, dims->n_text);
    put(s.mask_key, dims->order);
}

// validate_plan_inputs + cached-head checks (src/dispatch.cpp:11-54), all
// before any device work or cache mutation.
void validate_forward(int64_t batch, const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                      const int64_t* windows, const dfa2c_cache* cache, int64_t layer) {
    validate_dims(dims);
    if (block < 1)
        fail(DFA2C_SHAPE, "block_size must be >= 1");
    if (batch < 1)
        fail(DFA2C_SHAPE, "batch must be >= 1");
    validate_plan(dims, kinds, windows);
    const int64_t H = dims->n_heads;
    if (cache) {
        if (cache->H != H || cache->n != seq_len(dims) || cache->d != dims->head_dim || cache->batch != batch)
            fail(DFA2C_SHAPE, "cache geometry disagrees with dims/batch");
        if (layer < 0)
            fail(DFA2C_SHAPE, "layer index must be >= 0");
    }
    for (int64_t h = 0; h < H; ++h)
        if (kinds[h] == DFA2C_CACHED && (!cache || !cache->has(layer, h)))  // skipped heads are not read
            fail(DFA2C_CACHE_MISS, "plan marks head " + std::to_string(h) + " Cached before it ever computed");
}

// phase 2 bookkeeping: computed heads now hold output produced at t
// (src/dispatch.cpp:85-88); cached heads keep their produced_at.
void commit_produced(const dfa2c_dims* dims, const int32_t* kinds, dfa2c_cache* cache, int64_t layer, int64_t t) {
    if (!cache)
        return;
    const int64_t H = dims->n_heads;
    for (int64_t h = 0; h < H; ++h)
        if (!skipped(kinds[h]) && kinds[h] != DFA2C_CACHED)
            cache->produced[static_cast<size_t>(layer * H + h)] = t;
}

// Per-device copy engine state of dfa2c_mha_forward_host: an upload and a
// download stream plus two device staging slots used alternately, so one
// call's uploads overlap the previous call's downloads.
struct HostPipe {
    static constexpr int kMaxGroups = 8;
    struct Slot {
        void *q = nullptr, *k = nullptr, *v = nullptr, *out = nullptr;
        size_t cap = 0;
        cudaEvent_t ev_start{}, ev_done{}, ev_free{};
        cudaEvent_t ev_in[kMaxGroups]{}, ev_out[kMaxGroups]{};
    };
    std::mutex mu;
    cudaStream_t h2d{}, d2h{};
    Slot slots[2];
    int turn = 0;

    void init() {
        DFA2C_CUDA_CHECK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
        DFA2C_CUDA_CHECK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
        for (Slot& s : slots) {
            for (cudaEvent_t* e : {&s.ev_start, &s.ev_done, &s.ev_free})
                DFA2C_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
            for (int g = 0; g < kMaxGroups; ++g) {
                DFA2C_CUDA_CHECK(cudaEventCreateWithFlags(&s.ev_in[g], cudaEventDisableTiming));
                DFA2C_CUDA_CHECK(cudaEventCreateWithFlags(&s.ev_out[g], cudaEventDisableTiming));
            }
            DFA2C_CUDA_CHECK(cudaEventRecord(s.ev_free, h2d));  // initially free
        }
    }
    Slot& next(size_t bytes) {
        Slot& s = slots[turn];
        turn ^= 1;
        if (s.cap < bytes) {
            // the slot's previous user must finish before its buffers go
            DFA2C_CUDA_CHECK(cudaEventSynchronize(s.ev_free));
            for (void** p : {&s.q, &s.k, &s.v, &s.out}) {
                if (*p)
                    DFA2C_CUDA_CHECK(cudaFree(*p));
                *p = nullptr;
                DFA2C_CUDA_CHECK(cudaMalloc(p, bytes));
            }
            s.cap = bytes;
        }
        return s;
    }
};

HostPipe& host_pipe(int device) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<HostPipe>> pipes;
    std::lock_guard<std::mutex> lk(mu);
    auto& p = pipes[device];
    if (!p) {
        auto fresh = std::make_unique<HostPipe>();
        fresh->init();
        p = std::move(fresh);
    }
    return *p;
}

}  // namespace

extern "C" {


const char* dfa2c_last_error(void) { return g_err.c_str(); }
const char* dfa2c_version(void) { return "dfa2c 0.1 (sm_100a tcgen05/TMA fused head-wise attention)"; }
int64_t dfa2c_launch_count(void) { return g_launches.load(); }
void dfa2c_debug_set_trace(void* dev_buffer) { g_trace = static_cast<long long*>(dev_buffer); }

int dfa2c_debug_schedule(const double* costs, int64_t n, int32_t n_ctas, int32_t refine, int32_t* cta_of,
                         double* max_load) {
    return guard([&] {
        if (n < 0 || n_ctas < 1 || (n > 0 && (!costs || !cta_of)) || !max_load)
            fail(DFA2C_SHAPE, "need n >= 0, n_ctas >= 1 and non-NULL buffers");
        std::vector<Cand> cands(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            if (!(costs[i] >= 0.0))
                fail(DFA2C_SHAPE, "costs must be >= 0");
            cands[i].w = WorkItem{};
            cands[i].w.bh = static_cast<int32_t>(i);
            cands[i].cost = costs[i];
        }
        std::stable_sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) { return a.cost > b.cost; });
        const int grid = static_cast<int>(std::min<int64_t>(n_ctas, std::max<int64_t>(n, 1)));
        const auto bins = assign_ctas(cands, grid, refine != 0);
        double mx = 0.0;
        for (int c = 0; c < grid; ++c) {
            double l = 0.0;
            for (const Cand* x : bins[c]) {
                cta_of[x->w.bh] = c;
                l += x->cost;
            }
            mx = std::max(mx, l);
        }
        *max_load = mx;
    });
}

int dfa2c_arrow_mask(const dfa2c_dims* dims, int64_t block, int64_t window, uint8_t* active, int64_t* nb) {
    return guard([&] {
        const auto m = arrow_mask(dims, block, window);
        if (nb)
            *nb = ceil_div(seq_len(dims), block);
        if (active)
            std::memcpy(active, m.data(), m.size());
    });
}

int dfa2c_mask_stats(const uint8_t* active, int64_t n, int64_t block, int64_t head_dim, int64_t* ap,
                     int64_t* flops, double* sparsity) {
    return guard([&] {
        if (!active || n < 1 || block < 1)
            fail(DFA2C_SHAPE, "mask stats need a mask, seq_len >= 1 and block >= 1");
        const int64_t a = active_positions(active, n, block);
        if (ap)
            *ap = a;
        if (flops) {
            if (head_dim < 1)
                fail(DFA2C_SHAPE, "head_dim must be >= 1");
            *flops = 4 * head_dim * a;
        }
        if (sparsity)
            *sparsity = 1.0 - static_cast<double>(a) / (static_cast<double>(n) * static_cast<double>(n));
    });
}

int64_t dfa2c_dense_flops(int64_t n, int64_t d) { return 4 * d * n * n; }
int64_t dfa2c_kv_tile_keys(void) { return dfa2k::TILE_N; }

int dfa2c_plan_flops(const dfa2c_dims* dims, int64_t block, const int32_t* kinds, const int64_t* windows,
                     int64_t* flops) {
    return guard([&] {
        if (block < 1)
            fail(DFA2C_SHAPE, "block_size must be >= 1");
        const int64_t f = plan_flops(dims, block, kinds, windows);
        if (flops)
            *flops = f;
    });
}

int dfa2c_plan_aggregate(const dfa2c_dims* dims, int64_t T, int64_t L, int64_t block, const int32_t* kinds,
                         const int64_t* windows, int64_t* flops_total, int64_t* flops_dense, double* sparsity) {
    return guard([&] {
        // CompressionPlan::validate (src/plan.cpp:33-56)
        validate_dims(dims);
        if (T < 1 || L < 1 || block < 1)
            fail(DFA2C_PLAN, "plan needs T >= 1, L >= 1, block >= 1");
        if (!kinds)
            fail(DFA2C_PLAN, "plan must cover every (t, layer) exactly once");
        const int64_t H = dims->n_heads;
        for (int64_t t = 0; t < T; ++t)
            for (int64_t l = 0; l < L; ++l)
                for (int64_t h = 0; h < H; ++h) {
                    const int64_t i = (t * L + l) * H + h;
                    if (kinds[i] < DFA2C_FULL || kinds[i] > DFA2C_CACHED)
                        fail(DFA2C_PLAN, "unknown strategy kind");
                    if (kinds[i] == DFA2C_ARROW && (!windows || windows[i] < 0))
                        fail(DFA2C_PLAN, "arrow window must be >= 0");
                    if (kinds[i] == DFA2C_CACHED && t == 0)
                        fail(DFA2C_PLAN, "cached must not appear at the first timestep");
                }
        int64_t total = 0;
        for (int64_t s = 0; s < T * L; ++s)
            total += plan_flops(dims, block, kinds + s * H, windows ? windows + s * H : nullptr);
        const int64_t n = seq_len(dims);
        const int64_t dense = T * L * H * (4 * dims->head_dim * n * n);
        if (flops_total)
            *flops_total = total;
        if (flops_dense)
            *flops_dense = dense;
        if (sparsity)
            *sparsity = 1.0 - static_cast<double>(total) / static_cast<double>(dense);
    });
}

int dfa2c_tile_set(const dfa2c_dims* dims, int64_t block, int32_t kind, int64_t window, int64_t* row_ptr,
                   uint32_t* cols, int64_t* n_tiles) {
    return guard([&] {
        validate_dims(dims);
        if (block < 1)
            fail(DFA2C_SHAPE, "block_size must be >= 1");
        const int64_t n = seq_len(dims);
        std::vector<uint8_t> m;
        if (kind == DFA2C_FULL)
            m.assign(static_cast<size_t>(ceil_div(n, block) * ceil_div(n, block)), 1);
        else if (kind == DFA2C_ARROW)
            m = arrow_mask(dims, block, window);
        else
            fail(DFA2C_SHAPE, "tile sets exist for Full and Arrow heads only");
        const TileSet ts = build_tile_set(m.data(), n, block);
        if (n_tiles)
            *n_tiles = static_cast<int64_t>(ts.cols.size());
        if (row_ptr)
            std::memcpy(row_ptr, ts.row_ptr.data(), ts.row_ptr.size() * sizeof(int64_t));
        if (cols)
            std::memcpy(cols, ts.cols.data(), ts.cols.size() * sizeof(uint32_t));
    });
}

int dfa2c_cache_create(int64_t L, int64_t H, int64_t batch, int64_t n, int64_t d, dfa2c_cache** out) {
    return guard([&] {
        if (!out || L < 1 || H < 1 || batch < 1 || n < 1 || d < 1)
            fail(DFA2C_SHAPE, "cache needs layers, heads, batch, seq_len, head_dim >= 1");
        auto c = std::make_unique<dfa2c_cache>();
        c->L = L;
        c->H = H;
        c->batch = batch;
        c->n = n;
        c->d = d;
        DFA2C_CUDA_CHECK(cudaGetDevice(&c->device));
        c->layer_buf.assign(static_cast<size_t>(L), nullptr);
        c->layer_ready.assign(static_cast<size_t>(L), nullptr);
        c->produced.assign(static_cast<size_t>(L * H), std::numeric_limits<int64_t>::min());
        *out = c.release();
    });
}

int dfa2c_cache_destroy(dfa2c_cache* c) {
    return guard([&] { delete c; });
}

int dfa2c_cache_has(const dfa2c_cache* c, int64_t layer, int64_t head, int32_t* has) {
    return guard([&] {
        if (!c || !has)
            fail(DFA2C_SHAPE, "NULL cache");
        *has = (layer >= 0 && layer < c->L && head >= 0 && head < c->H && c->has(layer, head)) ? 1 : 0;
    });
}

int dfa2c_cache_produced_at(const dfa2c_cache* c, int64_t layer, int64_t head, int64_t* t) {
    return guard([&] {
        if (!c || !t)
            fail(DFA2C_SHAPE, "NULL cache");
        if (layer < 0 || layer >= c->L || head < 0 || head >= c->H || !c->has(layer, head))
            fail(DFA2C_CACHE_MISS, "no cached output for layer " + std::to_string(layer) + ", head " +
                                       std::to_string(head));
        *t = c->produced[static_cast<size_t>(layer * c->H + head)];
    });
}

int dfa2c_cache_staleness(const dfa2c_cache* c, int64_t layer, int64_t head, int64_t t, int64_t* st) {
    int64_t p = 0;
    const int rc = dfa2c_cache_produced_at(c, layer, head, &p);
    if (rc == DFA2C_OK && st)
        *st = t - p;
    return rc;
}

int dfa2c_cache_store(dfa2c_cache* c, int64_t layer, int64_t head, const void* src, int64_t t, void* stream) {
    return guard([&] {
        if (!c || !src)
            fail(DFA2C_SHAPE, "NULL cache or source");
        c->check(layer, head);
        char* dst = static_cast<char*>(c->layer_ptr(layer, as_stream(stream))) +
                    static_cast<size_t>(head) * c->slot_elems() * 2;
        const size_t row = c->slot_elems() * 2;
        DFA2C_CUDA_CHECK(cudaMemcpy2DAsync(dst, row * c->H, src, row, row, static_cast<size_t>(c->batch),
                                           cudaMemcpyDeviceToDevice, as_stream(stream)));
        c->produced[static_cast<size_t>(layer * c->H + head)] = t;
    });
}

int dfa2c_cache_fetch(const dfa2c_cache* c, int64_t layer, int64_t head, void* dst, void* stream) {
    return guard([&] {
        if (!c || !dst)
            fail(DFA2C_SHAPE, "NULL cache or destination");
        if (!c->has(layer, head))
            fail(DFA2C_CACHE_MISS, "no cached output for layer " + std::to_string(layer) + ", head " +
                                       std::to_string(head));
        c->order_after_ready(layer, as_stream(stream));
        const char* src =
            static_cast<const char*>(c->layer_buf[layer]) + static_cast<size_t>(head) * c->slot_elems() * 2;
        const size_t row = c->slot_elems() * 2;
        DFA2C_CUDA_CHECK(cudaMemcpy2DAsync(dst, row, src, row * c->H, row, static_cast<size_t>(c->batch),
                                           cudaMemcpyDeviceToDevice, as_stream(stream)));
    });
}

int dfa2c_cache_clear(dfa2c_cache* c) {
    return guard([&] {
        if (!c)
            fail(DFA2C_SHAPE, "NULL cache");
        std::fill(c->produced.begin(), c->produced.end(), std::numeric_limits<int64_t>::min());
    });
}

int dfa2c_cache_size(const dfa2c_cache* c, int64_t* n) {
    return guard([&] {
        if (!c || !n)
            fail(DFA2C_SHAPE, "NULL cache");
        *n = 0;
        for (int64_t l = 0; l < c->L; ++l)
            for (int64_t h = 0; h < c->H; ++h)
                *n += c->has(l, h) ? 1 : 0;
    });
}

int dfa2c_cache_bytes(const dfa2c_cache* c, int64_t* bytes) {
    return guard([&] {
        if (!c || !bytes)
            fail(DFA2C_SHAPE, "NULL cache");
        *bytes = 0;
        for (void* p : c->layer_buf)
            if (p)
                *bytes += static_cast<int64_t>(c->layer_bytes());
    });
}

int dfa2c_mha_forward(const void* q, const void* k, const void* v, int64_t batch, const dfa2c_dims* dims,
                      int64_t block, const int32_t* kinds, const int64_t* windows, dfa2c_cache* cache,
                      int64_t layer, int64_t t, void* out, void* stream) {
    return guard([&] {
        validate_forward(batch, dims, block, kinds, windows, cache, layer);
        ForwardSpec s{};
        s.q = q;
        s.k = k;
        s.v = v;
        s.out = out;
        s.batch = batch;
        s.dims = dims;
        s.block = block;
        s.cache = cache;
        s.layer = layer;
        plan_jobs(dims, block, kinds, windows, cache != nullptr, s);
        run_forward(s, as_stream(stream));
        commit_produced(dims, kinds, cache, layer, t);
    });
}

int dfa2c_mha_forward_host(const void* q, const void* k, const void* v, int64_t batch, const dfa2c_dims* dims,
                           int64_t block, const int32_t* kinds, const int64_t* windows, dfa2c_cache* cache,
                           int64_t layer, int64_t t, void* out, void* stream) {
    return guard([&] {
        validate_forward(batch, dims, block, kinds, windows, cache, layer);
        if (!q || !k || !v || !out)
            fail(DFA2C_SHAPE, "q, k, v and out must not be NULL");
        const int64_t H = dims->n_heads, n = seq_len(dims), d = dims->head_dim;
        const size_t head_bytes = static_cast<size_t>(n * d) * 2;
        const size_t row_pitch = static_cast<size_t>(H) * head_bytes;  // one sample
        const size_t bytes = static_cast<size_t>(batch) * row_pitch;
        int device = 0;
        DFA2C_CUDA_CHECK(cudaGetDevice(&device));
        const cudaStream_t user = as_stream(stream);

        // Computed heads in index order, split into up to kGroups groups of
        // near-equal head count; each group is copied in as maximal runs of
        // consecutive heads (one 2-D copy per run and tensor: width = run
        // bytes, height = batch, pitch = one sample).
        static const int kGroups = [] {  // DFA2_HOST_GROUPS (1..8; A/B knob)
            const char* e = std::getenv("DFA2_HOST_GROUPS");
            const int g = e ? std::atoi(e) : 6;
            return std::max(1, std::min(g, HostPipe::kMaxGroups));
        }();
        std::vector<int64_t> computed;
        for (int64_t h = 0; h < H; ++h)
            if (!skipped(kinds[h]) && kinds[h] != DFA2C_CACHED)
                computed.push_back(h);
        const int G = static_cast<int>(std::min<size_t>(kGroups, computed.size()));

        HostPipe& hp = host_pipe(device);
        std::lock_guard<std::mutex> lk(hp.mu);
        HostPipe::Slot& ws = hp.next(bytes);
        // Uploads wait only for this staging slot to be free (its use two
        // calls ago), so they overlap the previous call's download tail; the
        // download stream (which reads cache slots written by earlier work on
        // `stream`) and every launch stay ordered after `stream`.
        DFA2C_CUDA_CHECK(cudaEventRecord(ws.ev_start, user));
        DFA2C_CUDA_CHECK(cudaStreamWaitEvent(hp.h2d, ws.ev_free, 0));
        DFA2C_CUDA_CHECK(cudaStreamWaitEvent(hp.d2h, ws.ev_start, 0));
        DFA2C_CUDA_CHECK(cudaStreamWaitEvent(hp.d2h, ws.ev_free, 0));
        auto copy_runs = [&](const std::vector<int64_t>& heads, const void* src, void* dst, cudaMemcpyKind kind,
                             cudaStream_t st) {
            for (size_t i = 0; i < heads.size();) {
                size_t j = i + 1;
                while (j < heads.size() && heads[j] == heads[j - 1] + 1)
                    ++j;
                const size_t off = static_cast<size_t>(heads[i]) * head_bytes;
                DFA2C_CUDA_CHECK(cudaMemcpy2DAsync(static_cast<char*>(dst) + off, row_pitch,
                                                   static_cast<const char*>(src) + off, row_pitch,
                                                   (j - i) * head_bytes, static_cast<size_t>(batch), kind, st));
                i = j;
            }
        };
        // Cached heads: their output IS the pre-call slot; it goes straight
        // from the cache to the host (no q/k/v upload, no kernel work).
        std::vector<int64_t> cached;
        for (int64_t h = 0; h < H; ++h)
            if (kinds[h] == DFA2C_CACHED)  // a skipped cached head is neither read nor written
                cached.push_back(h);
        if (!cached.empty())
            copy_runs(cached, cache->layer_ptr(layer, hp.d2h), out, cudaMemcpyDeviceToHost, hp.d2h);

        ForwardSpec base{};
        base.q = ws.q;
        base.k = ws.k;
        base.v = ws.v;
        base.out = ws.out;
        base.batch = batch;
        base.dims = dims;
        base.block = block;
        base.cache = cache;
        base.layer = layer;
        plan_jobs(dims, block, kinds, windows, cache != nullptr, base);
        for (int g = 0; g < G; ++g) {
            const size_t lo = computed.size() * g / G, hi = computed.size() * (g + 1) / G;
            const std::vector<int64_t> heads(computed.begin() + lo, computed.begin() + hi);
            copy_runs(heads, q, ws.q, cudaMemcpyHostToDevice, hp.h2d);
            copy_runs(heads, k, ws.k, cudaMemcpyHostToDevice, hp.h2d);
            copy_runs(heads, v, ws.v, cudaMemcpyHostToDevice, hp.h2d);
            DFA2C_CUDA_CHECK(cudaEventRecord(ws.ev_in[g], hp.h2d));
            DFA2C_CUDA_CHECK(cudaStreamWaitEvent(user, ws.ev_in[g], 0));
            ForwardSpec s = base;
            std::vector<bool> in_group(static_cast<size_t>(H), false);
            for (int64_t h : heads)
                in_group[h] = true;
            for (int64_t h = 0; h < H; ++h)
                if (!in_group[h])
                    s.jobs[h].mask_id = JOB_SKIP;
            run_forward(s, user);
            DFA2C_CUDA_CHECK(cudaEventRecord(ws.ev_out[g], user));
            DFA2C_CUDA_CHECK(cudaStreamWaitEvent(hp.d2h, ws.ev_out[g], 0));
            copy_runs(heads, ws.out, out, cudaMemcpyDeviceToHost, hp.d2h);
        }
        // the call completes on the caller's stream: host `out` is final once
        // `stream` reaches this point
        DFA2C_CUDA_CHECK(cudaEventRecord(ws.ev_done, hp.d2h));
        DFA2C_CUDA_CHECK(cudaStreamWaitEvent(user, ws.ev_done, 0));
        DFA2C_CUDA_CHECK(cudaEventRecord(ws.ev_free, user));
        commit_produced(dims, kinds, cache, layer, t);
    });
}

// ---------------------------------------------------------------- multi-GPU
namespace {

void head_bits(const dfa2c_dims* dims, const int32_t* kinds, uint32_t* bits) {
    for (int i = 0; i < 32; ++i)
        bits[i] = 0;
    for (int64_t h = 0; h < dims->n_heads; ++h)
        if (kind_of(kinds[h]) != DFA2C_CACHED)
            bits[h >> 5] |= 1u << (h & 31);
}

void commit_others(int64_t batch, const dfa2c_dims* dims, const int32_t* kinds, dfa2c_cache* cache, int64_t layer,
                   int64_t r0, int64_t r1, const void* out, cudaStream_t st) {
    const int64_t H = dims->n_heads, n = seq_len(dims), d = dims->head_dim;
    uint32_t bits[32];
    head_bits(dims, kinds, bits);
    bool any = false;
    for (uint32_t b : bits)
        any |= b != 0;
    if (!any)
        return;
    cache->ensure(layer);
    void* slots = cache->layer_ptr(layer, st);
    int device = 0;
    DFA2C_CUDA_CHECK(cudaGetDevice(&device));
    DFA2C_CUDA_CHECK(dfa2k::launch_commit_rows(out, slots, batch * H * n, r0, r1, n, H, d, bits, num_sms(device), st));
    g_launches.fetch_add(1);
}

void validate_sharded(int64_t batch, const dfa2c_dims* dims, const int32_t* kinds, int32_t rank, int32_t world) {
    if (world < 1 || rank < 0 || rank >= world)
        fail(DFA2C_SHAPE, "need 0 <= rank < world");
    if (!direct_layout(dims->head_dim))
        fail(DFA2C_UNSUPPORTED, "sharded launches need head_dim 64 or 72..128 (multiple of 8)");
    if (dims->n_heads > 1024)
        fail(DFA2C_UNSUPPORTED, "sharded launches support up to 1024 heads");
    for (int64_t h = 0; h < dims->n_heads; ++h)
        if (skipped(kinds[h]))
            fail(DFA2C_SHAPE, "sharded launches take the whole layer plan (no DFA2C_SKIP heads)");
    (void)batch;
}
}  // namespace

int dfa2c_mha_forward_sharded(const void* q, const void* k, const void* v, int64_t batch, const dfa2c_dims* dims,
                              int64_t block, const int32_t* kinds, const int64_t* windows, dfa2c_cache* cache,
                              int64_t layer, int64_t t, void* out, int32_t rank, int32_t world, void* nccl_comm,
                              int64_t* row_bounds, void* stream) {
    return guard([&] {
        validate_forward(batch, dims, block, kinds, windows, cache, layer);
        validate_sharded(batch, dims, kinds, rank, world);
        if (nccl_comm) {
            int nr = 0, r = 0;
            const std::string e = dfa2nccl::comm_shape(nccl_comm, &nr, &r);
            if (!e.empty())
                fail(DFA2C_CUDA, e);
            if (nr != world || r != rank)
                fail(DFA2C_SHAPE, "NCCL communicator (" + std::to_string(r) + " of " + std::to_string(nr) +
                                      ") disagrees with rank/world");
        }
        const cudaStream_t st = as_stream(stream);
        ForwardSpec s{};
        s.q = q;
        s.k = k;
        s.v = v;
        s.out = out;
        s.batch = batch;
        s.dims = dims;
        s.block = block;
        s.cache = cache;
        s.layer = layer;
        s.n_parts = world;
        s.part = rank;
        std::vector<int64_t> rows;
        s.shard_rows = &rows;
        plan_jobs(dims, block, kinds, windows, cache != nullptr, s);
        launch_forward(s, st);  // this rank's rows only; its computed rows are committed in-kernel
        if (rows.size() != static_cast<size_t>(world) + 1)
            fail(DFA2C_CUDA, "internal: shard bounds missing");
        if (row_bounds)
            std::copy(rows.begin(), rows.end(), row_bounds);
        if (nccl_comm && world > 1) {
            const int64_t rb = dims->head_dim * 2;
            std::vector<int64_t> off(rows.size());
            for (size_t i = 0; i < rows.size(); ++i)
                off[i] = rows[i] * rb;
            const std::string e = dfa2nccl::allgather_v(nccl_comm, out, off.data(), world, st);
            if (!e.empty())
                fail(DFA2C_CUDA, e);
            if (cache)
                commit_others(batch, dims, kinds, cache, layer, rows[rank], rows[rank + 1], out, st);
        }
        commit_produced(dims, kinds, cache, layer, t);
    });
}

int dfa2c_mha_forward_sharded_p2p(const void* q, const void* k, const void* v, int64_t batch,
                                  const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                                  const int64_t* windows, dfa2c_cache* cache, int64_t layer, int64_t t,
                                  void* const* outs, int32_t rank, int32_t world, int64_t* row_bounds,
                                  void* stream) {
    return guard([&] {
        validate_forward(batch, dims, block, kinds, windows, cache, layer);
        validate_sharded(batch, dims, kinds, rank, world);
        if (!outs)
            fail(DFA2C_SHAPE, "outs must hold every rank's output buffer");
        if (world - 1 > dfa2k::MAX_PEERS)
            fail(DFA2C_UNSUPPORTED, "peer-memory assembly supports up to " + std::to_string(dfa2k::MAX_PEERS + 1) +
                                        " ranks");
        const cudaStream_t st = as_stream(stream);
        ForwardSpec s{};
        s.q = q;
        s.k = k;
        s.v = v;
        s.out = outs[rank];
        s.batch = batch;
        s.dims = dims;
        s.block = block;
        s.cache = cache;
        s.layer = layer;
        s.n_parts = world;
        s.part = rank;
        for (int32_t r = 0; r < world; ++r)
            if (r != rank) {
                if (!outs[r] || outs[r] == outs[rank])
                    fail(DFA2C_SHAPE, "outs must be distinct non-NULL buffers");
                s.peer_outs.push_back(outs[r]);
            }
        std::vector<int64_t> rows;
        s.shard_rows = &rows;
        plan_jobs(dims, block, kinds, windows, cache != nullptr, s);
        // this rank's rows, stored to its own out and, box by box from the
        // epilogue, to every peer's out over NVLink (no collective); its
        // computed rows are committed to its cache in-kernel
        launch_forward(s, st);
        if (rows.size() != static_cast<size_t>(world) + 1)
            fail(DFA2C_CUDA, "internal: shard bounds missing");
        if (row_bounds)
            std::copy(rows.begin(), rows.end(), row_bounds);
        commit_produced(dims, kinds, cache, layer, t);
    });
}

int dfa2c_ipc_handle(const void* ptr, char* handle, int64_t* offset) {
    return guard([&] {
        if (!ptr || !handle || !offset)
            fail(DFA2C_SHAPE, "ptr, handle and offset must not be NULL");
        // the IPC handle names the whole allocation: find its base (the
        // driver entry point, as for the tensor maps: no libcuda link)
        using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static RangeFn range = [] {
            cudaDriverEntryPointQueryResult q{};
            void* p = nullptr;
            return cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
                           q == cudaDriverEntryPointSuccess
                       ? reinterpret_cast<RangeFn>(p)
                       : nullptr;
        }();
        CUdeviceptr base = 0;
        size_t size = 0;
        if (!range || range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
            fail(DFA2C_CUDA, "cuMemGetAddressRange failed (not a device allocation?)");
        cudaIpcMemHandle_t h;
        DFA2C_CUDA_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
        static_assert(sizeof h == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(handle, &h, sizeof h);
        *offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(ptr) - base);
    });
}

int dfa2c_ipc_open(const char* handle, int64_t offset, void** ptr) {
    return guard([&] {
        if (!handle || !ptr || offset < 0)
            fail(DFA2C_SHAPE, "handle and ptr must not be NULL, offset >= 0");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        void* base = nullptr;
        DFA2C_CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        *ptr = static_cast<char*>(base) + offset;
    });
}

int dfa2c_ipc_close(void* ptr, int64_t offset) {
    return guard([&] {
        if (!ptr)
            fail(DFA2C_SHAPE, "ptr must not be NULL");
        DFA2C_CUDA_CHECK(cudaIpcCloseMemHandle(static_cast<char*>(ptr) - offset));
    });
}

int dfa2c_shard_rows(int64_t batch, const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                     const int64_t* windows, int32_t world, int64_t* row_bounds) {
    return guard([&] {
        validate_dims(dims);
        if (block < 1 || batch < 1)
            fail(DFA2C_SHAPE, "block_size and batch must be >= 1");
        validate_plan(dims, kinds, windows);
        validate_sharded(batch, dims, kinds, 0, world);
        if (!row_bounds)
            fail(DFA2C_SHAPE, "row_bounds must not be NULL");
        ForwardSpec s{};
        plan_jobs(dims, block, kinds, windows, false, s);
        const int64_t n = seq_len(dims), nb = ceil_div(n, block);
        std::vector<std::vector<uint8_t>> masks;
        for (int64_t w : s.mask_windows)
            masks.push_back(w < 0 ? std::vector<uint8_t>(static_cast<size_t>(nb * nb), uint8_t{1})
                                  : arrow_mask(dims, block, w));
        const PlanGeometry g = plan_geometry(batch, dims->n_heads, n, block, masks, s.jobs, s.ref_jobs,
                                             text_begin(dims), text_end(dims), 0, world);
        std::copy(g.shard_rows.begin(), g.shard_rows.end(), row_bounds);
    });
}

int dfa2c_shard_commit(int64_t batch, const dfa2c_dims* dims, const int32_t* kinds, dfa2c_cache* cache, int64_t layer,
                       const int64_t* row_bounds, int32_t rank, int32_t world, const void* out, void* stream) {
    return guard([&] {
        validate_dims(dims);
        if (!cache || !row_bounds || !out)
            fail(DFA2C_SHAPE, "shard_commit needs a cache, the row bounds and the gathered output");
        if (world < 1 || rank < 0 || rank >= world)
            fail(DFA2C_SHAPE, "need 0 <= rank < world");
        if (cache->H != dims->n_heads || cache->n != seq_len(dims) || cache->d != dims->head_dim ||
            cache->batch != batch)
            fail(DFA2C_SHAPE, "cache geometry disagrees with dims/batch");
        if (dims->n_heads > 1024)
            fail(DFA2C_UNSUPPORTED, "sharded launches support up to 1024 heads");
        commit_others(batch, dims, kinds, cache, layer, row_bounds[rank], row_bounds[rank + 1], out,
                      as_stream(stream));
    });
}

int dfa2c_nccl_available(void) { return dfa2nccl::available(nullptr) ? 1 : 0; }

int dfa2c_nccl_unique_id(char* id) {
    return guard([&] {
        if (!id)
            fail(DFA2C_SHAPE, "id buffer must not be NULL");
        const std::string e = dfa2nccl::unique_id(id);
        if (!e.empty())
            fail(DFA2C_CUDA, e);
    });
}

int dfa2c_nccl_comm_init(const char* id, int32_t world, int32_t rank, void** comm) {
    return guard([&] {
        if (!id || !comm || world < 1 || rank < 0 || rank >= world)
            fail(DFA2C_SHAPE, "nccl_comm_init needs an id, a comm slot and 0 <= rank < world");
        const std::string e = dfa2nccl::comm_init(comm, world, id, rank);
        if (!e.empty())
            fail(DFA2C_CUDA, e);
    });
}

int dfa2c_nccl_comm_destroy(void* comm) {
    return guard([&] {
        if (!comm)
            return;
        const std::string e = dfa2nccl::comm_destroy(comm);
        if (!e.empty())
            fail(DFA2C_CUDA, e);
    });
}

int dfa2c_allgather_rows(void* comm, void* buf, const int64_t* row_bounds, int32_t world, int64_t row_bytes,
                         void* stream) {
    return guard([&] {
        if (!comm || !buf || !row_bounds || world < 1 || row_bytes < 1)
            fail(DFA2C_SHAPE, "allgather_rows needs a comm, a buffer, the bounds and row_bytes >= 1");
        std::vector<int64_t> off(static_cast<size_t>(world) + 1);
        for (int32_t i = 0; i <= world; ++i)
            off[i] = row_bounds[i] * row_bytes;
        const std::string e = dfa2nccl::allgather_v(comm, buf, off.data(), world, as_stream(stream));
        if (!e.empty())
            fail(DFA2C_CUDA, e);
    });
}

int dfa2c_sparse_attention_forward(const void* q, const void* k, const void* v, void* out, int64_t n_heads,
                                   int64_t n, int64_t d, const uint8_t* active, int64_t block, void* stream) {
    return guard([&] {
        if (n_heads < 1 || n < 1 || d < 1 || block < 1 || !active)
            fail(DFA2C_SHAPE, "sparse attention needs heads, seq_len, head_dim, block >= 1 and a mask");
        const int64_t nb = ceil_div(n, block);
        check_rows_nonempty(active, nb);
        dfa2c_dims dims{n_heads, d, n, 0, DFA2C_VISUAL_FIRST};
        ForwardSpec s{};
        s.q = q;
        s.k = k;
        s.v = v;
        s.out = out;
        s.batch = 1;
        s.dims = &dims;
        s.block = block;
        s.cache = nullptr;
        s.masks.emplace_back(active, active + nb * nb);
        // key the plan cache on the mask bytes themselves
        s.mask_key.assign(reinterpret_cast<const char*>(active), static_cast<size_t>(nb * nb));
        s.jobs.assign(static_cast<size_t>(n_heads), HeadJob{0, false});
        run_forward(s, as_stream(stream));
    });
}

int dfa2c_dense_attention_forward(const void* q, const void* k, const void* v, void* out, int64_t n_heads,
                                  int64_t n, int64_t d, void* stream) {
    return guard([&] {
        if (n_heads < 1 || n < 1 || d < 1)
            fail(DFA2C_SHAPE, "dense attention needs heads, seq_len, head_dim >= 1");
        dfa2c_dims dims{n_heads, d, n, 0, DFA2C_VISUAL_FIRST};
        std::vector<int32_t> kinds(static_cast<size_t>(n_heads), DFA2C_FULL);
        ForwardSpec s{};
        s.q = q;
        s.k = k;
        s.v = v;
        s.out = out;
        s.batch = 1;
        s.dims = &dims;
        s.block = 128;
        s.cache = nullptr;
        plan_jobs(&dims, 128, kinds.data(), nullptr, false, s);
        run_forward(s, as_stream(stream));
    });
}

int dfa2c_attention_reference(const void* q, const void* k, const void* v, void* out, int32_t dtype,
                              int64_t n_heads, int64_t n, int64_t d, const uint8_t* active, int64_t block,
                              void* stream) {
    return guard([&] {
        if (!q || !k || !v || !out)
            fail(DFA2C_SHAPE, "attention_reference operands must not be NULL");
        if (dtype != DFA2C_F32 && dtype != DFA2C_F64)
            fail(DFA2C_SHAPE, "attention_reference computes in f32 or f64");
        if (n_heads < 1 || n < 1 || d < 1)
            fail(DFA2C_SHAPE, "attention needs heads, seq_len, head_dim >= 1");
        if (d > dfa2k::reference_max_head_dim())
            fail(DFA2C_UNSUPPORTED, "attention_reference supports head_dim <= " +
                                        std::to_string(dfa2k::reference_max_head_dim()));
        if (n_heads > 65535 || n > (int64_t{1} << 30))
            fail(DFA2C_UNSUPPORTED, "attention_reference problem too large");
        const cudaStream_t st = as_stream(stream);
        uint8_t* dmask = nullptr;
        int64_t nb = 1;
        if (active) {
            if (block < 1)
                fail(DFA2C_SHAPE, "block_size must be >= 1");
            nb = ceil_div(n, block);
            check_rows_nonempty(active, nb);  // FullyMaskedRowError before any compute (tensor.cpp:97-99)
            scratch_alloc(&dmask, static_cast<size_t>(nb * nb), st);
            DFA2C_CUDA_CHECK(cudaMemcpyAsync(dmask, active, static_cast<size_t>(nb * nb), cudaMemcpyHostToDevice, st));
        }
        DFA2C_CUDA_CHECK(dfa2k::launch_attention_reference(q, k, v, out, dtype, n_heads, n, d, dmask,
                                                           active ? block : n, nb, st));
        g_launches.fetch_add(1);
        if (dmask) {
            DFA2C_CUDA_CHECK(cudaFreeAsync(dmask, st));
            DFA2C_CUDA_CHECK(cudaStreamSynchronize(st));  // the host mask bytes may be freed on return
        }
    });
}

int dfa2c_rse_async(const void* y_m, const void* y_o, int32_t dtype, int64_t n_heads, int64_t numel, int32_t mode,
                    double* out_dev, void* stream) {
    return guard([&] {
        if (!y_m || !y_o || !out_dev)
            fail(DFA2C_SHAPE, "rse operands must not be NULL");
        if (dtype != DFA2C_BF16 && dtype != DFA2C_F32 && dtype != DFA2C_F64)
            fail(DFA2C_SHAPE, "rse operands must be bf16, f32 or f64");
        if (n_heads < 1 || numel < 1)
            fail(DFA2C_SHAPE, "rse needs at least one element");
        if (mode != DFA2C_RSE_STANDARD && mode != DFA2C_RSE_LITERAL)
            fail(DFA2C_SHAPE, "unknown rse mode");
        if (n_heads > 65535)
            fail(DFA2C_UNSUPPORTED, "too many heads for one rse launch");
        const cudaStream_t st = as_stream(stream);
        int device = 0;
        DFA2C_CUDA_CHECK(cudaGetDevice(&device));
        // one wave: nblk CTAs per head so that nblk * H fills the resident
        // slots (rse_ctas_per_sm per SM), each CTA streaming >= 8 K elements
        const int64_t target = std::max<int64_t>(1, dfa2k::rse_ctas_per_sm() * num_sms(device) / n_heads);
        const int nblk = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(target, ceil_div(numel, 8192))));
        double* scratch = nullptr;
        scratch_alloc(&scratch, static_cast<size_t>(n_heads * nblk * 5) * sizeof(double), st);
        DFA2C_CUDA_CHECK(dfa2k::launch_rse(y_m, y_o, dtype, n_heads, numel, mode, out_dev, scratch, nblk, st));
        g_launches.fetch_add(2);
        DFA2C_CUDA_CHECK(cudaFreeAsync(scratch, st));
    });
}

int dfa2c_rse(const void* y_m, const void* y_o, int32_t dtype, int64_t n_heads, int64_t numel, int32_t mode,
              double* out, void* stream) {
    return guard([&] {
        if (!out)
            fail(DFA2C_SHAPE, "rse output must not be NULL");
        const cudaStream_t st = as_stream(stream);
        double* dev = nullptr;
        scratch_alloc(&dev, static_cast<size_t>(n_heads) * sizeof(double), st);
        const int rc = dfa2c_rse_async(y_m, y_o, dtype, n_heads, numel, mode, dev, stream);
        if (rc != DFA2C_OK) {
            cudaFreeAsync(dev, st);
            fail(rc, g_err);
        }
        DFA2C_CUDA_CHECK(cudaMemcpyAsync(out, dev, static_cast<size_t>(n_heads) * sizeof(double),
                                         cudaMemcpyDeviceToHost, st));
        DFA2C_CUDA_CHECK(cudaFreeAsync(dev, st));
        DFA2C_CUDA_CHECK(cudaStreamSynchronize(st));
        for (int64_t h = 0; h < n_heads; ++h)
            if (std::isnan(out[h]))
                fail(DFA2C_DEGENERATE, "reference output has zero variance (head " + std::to_string(h) + ")");
    });
}

namespace {
// influence_for_layer up to the RSE results: every launch enqueued on
// `stream`, the per-(m, h) RSE values copied (asynchronously) to
// influence_host[m * H + h] and the eligibility of each entry returned;
// nothing is synchronised.
std::vector<uint8_t> influence_enqueue(const void* q, const void* k, const void* v, const dfa2c_dims* dims,
                                       int64_t block, const int64_t* windows, int64_t n_windows,
                                       int32_t include_cached, const dfa2c_cache* cache, int64_t layer, int64_t t,
                                       int32_t mode, double* influence_host, void* original, void* method_outputs,
                                       void* stream) {
    validate_dims(dims);
    if (block < 1)
        fail(DFA2C_SHAPE, "block_size must be >= 1");
    if (n_windows < 0 || (n_windows > 0 && !windows))
        fail(DFA2C_SHAPE, "bad candidate windows");
    for (int64_t i = 0; i < n_windows; ++i)
        if (windows[i] < 0)
            fail(DFA2C_SHAPE, "window radii must be >= 0");
    const int64_t M = n_windows + (include_cached ? 1 : 0);
    if (M == 0)
        fail(DFA2C_SHAPE, "candidate set must be nonempty");
    if (!influence_host)
        fail(DFA2C_SHAPE, "influence output must not be NULL");
    const int64_t H = dims->n_heads, n = seq_len(dims), d = dims->head_dim;
    const size_t head_elems = static_cast<size_t>(n * d);
    const size_t layer_bytes = static_cast<size_t>(H) * head_elems * 2;
    if (include_cached && cache &&
        (cache->H != H || cache->n != n || cache->d != d || cache->batch != 1))
        fail(DFA2C_SHAPE, "cache geometry disagrees with dims");
    const cudaStream_t st = as_stream(stream);

    void* orig = original;
    void* scratch_orig = nullptr;
    if (!orig) {
        scratch_alloc(&scratch_orig, layer_bytes, st);
        orig = scratch_orig;
    }
    // fused: one launch writes the original and every Arrow candidate
    // (all candidates resident at once); otherwise one pass per candidate
    const bool fused = influence_fused_eligible(dims, block, n_windows);
    void* scratch_cand = nullptr;
    if (!method_outputs)
        scratch_alloc(&scratch_cand, layer_bytes * static_cast<size_t>(fused ? n_windows : 1), st);
    double* rse_dev = nullptr;
    scratch_alloc(&rse_dev, static_cast<size_t>(M * H) * sizeof(double), st);
    std::vector<uint8_t> eligible(static_cast<size_t>(M * H), 0);
    std::vector<const void*> rse_ym(static_cast<size_t>(M), nullptr);  // measured candidates' outputs
    if (mode != DFA2C_RSE_STANDARD && mode != DFA2C_RSE_LITERAL)
        fail(DFA2C_SHAPE, "unknown rse mode");

    std::vector<int32_t> kinds(static_cast<size_t>(H), DFA2C_FULL);
    std::vector<int64_t> wins(static_cast<size_t>(H), 0);
    if (fused) {
        run_influence_fused(q, k, v, dims, windows, n_windows, orig,
                            method_outputs ? method_outputs : scratch_cand, st);
    } else {
        // 1 original evaluation: all heads Full (src/calibrate.cpp:206).
        ForwardSpec s{};
        s.q = q; s.k = k; s.v = v; s.out = orig; s.batch = 1; s.dims = dims; s.block = block;
        plan_jobs(dims, block, kinds.data(), wins.data(), false, s);
        run_forward(s, st);
    }
    for (int64_t m = 0; m < M; ++m) {
        void* cand = method_outputs ? static_cast<char*>(method_outputs) + m * layer_bytes
                                    : static_cast<char*>(scratch_cand) + (fused ? m * layer_bytes : 0);
        if (m < n_windows) {
            // Arrow(w) over every head, then per-head RSE (src/calibrate.cpp:238-250).
            if (!fused) {
                std::fill(kinds.begin(), kinds.end(), DFA2C_ARROW);
                std::fill(wins.begin(), wins.end(), windows[m]);
                ForwardSpec s{};
                s.q = q; s.k = k; s.v = v; s.out = cand; s.batch = 1; s.dims = dims; s.block = block;
                plan_jobs(dims, block, kinds.data(), wins.data(), false, s);
                run_forward(s, st);
            }
            rse_ym[m] = cand;
            for (int64_t h = 0; h < H; ++h)
                eligible[m * H + h] = 1;
        } else if (t > 0 && cache && layer >= 0 && layer < cache->L && cache->layer_buf[layer]) {
            // Cached: slot vs original for heads with a slot (src/calibrate.cpp:222-235),
            // one RSE launch over the layer's contiguous [H, N, d] slot array; heads
            // without a slot stay ineligible (+inf).
            cache->order_after_ready(layer, st);
            const void* slots = cache->layer_buf[layer];
            if (method_outputs)  // the slot where there is one, zeros (unset) elsewhere
                for (int64_t h = 0; h < H; ++h) {
                    char* dst = static_cast<char*>(cand) + h * head_elems * 2;
                    if (cache->has(layer, h))
                        DFA2C_CUDA_CHECK(cudaMemcpyAsync(dst, static_cast<const char*>(slots) + h * head_elems * 2,
                                                         head_elems * 2, cudaMemcpyDeviceToDevice, st));
                    else
                        DFA2C_CUDA_CHECK(cudaMemsetAsync(dst, 0, head_elems * 2, st));
                }
            rse_ym[m] = slots;
            for (int64_t h = 0; h < H; ++h)
                eligible[m * H + h] = cache->has(layer, h) ? 1 : 0;
        }
    }
    // the layer's RSE grid: runs of consecutive measured candidates share one
    // launch that streams the original once (rse_multi_partial)
    if (H > 65535)
        fail(DFA2C_UNSUPPORTED, "too many heads for one rse launch");
    int device = 0;
    DFA2C_CUDA_CHECK(cudaGetDevice(&device));
    for (int64_t m0 = 0; m0 < M;) {
        if (!rse_ym[m0]) {
            ++m0;
            continue;
        }
        int64_t m1 = m0;
        while (m1 < M && rse_ym[m1] && m1 - m0 < dfa2k::rse_multi_max())
            ++m1;
        const int g = static_cast<int>(m1 - m0);
        // one wave of (2 stages x (g + 1) operands x 8 KB)-smem CTAs
        const int64_t per_sm = std::max<int64_t>(1, (227 * 1024) / (2 * (g + 1) * 8 * 1024 + 64));
        const int64_t target = std::max<int64_t>(1, per_sm * num_sms(device) / H);
        const int nblk =
            static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(target, ceil_div(static_cast<int64_t>(head_elems), 8192))));
        double* scratch = nullptr;
        scratch_alloc(&scratch, static_cast<size_t>(g * H * nblk * 5) * sizeof(double), st);
        DFA2C_CUDA_CHECK(dfa2k::launch_rse_multi(rse_ym.data() + m0, g, orig, DFA2C_BF16, H,
                                                 static_cast<int64_t>(head_elems), mode, rse_dev + m0 * H, scratch,
                                                 nblk, st));
        g_launches.fetch_add(2);
        DFA2C_CUDA_CHECK(cudaFreeAsync(scratch, st));
        m0 = m1;
    }
    DFA2C_CUDA_CHECK(cudaMemcpyAsync(influence_host, rse_dev, static_cast<size_t>(M * H) * sizeof(double),
                                     cudaMemcpyDeviceToHost, st));
    DFA2C_CUDA_CHECK(cudaFreeAsync(rse_dev, st));
    if (scratch_orig)
        DFA2C_CUDA_CHECK(cudaFreeAsync(scratch_orig, st));
    if (scratch_cand)
        DFA2C_CUDA_CHECK(cudaFreeAsync(scratch_cand, st));
    return eligible;
}

// host[m * H + h] (RSE, NaN = degenerate) + eligibility -> influence[h * M + m]
void influence_finalize(const double* host, const uint8_t* eligible, int64_t H, int64_t M, double* influence) {
    for (int64_t h = 0; h < H; ++h)
        for (int64_t m = 0; m < M; ++m) {
            double val = std::numeric_limits<double>::infinity();
            if (eligible[m * H + h]) {
                val = host[m * H + h];
                if (std::isnan(val))
                    fail(DFA2C_DEGENERATE, "reference output has zero variance (head " + std::to_string(h) + ")");
            }
            influence[h * M + m] = val;
        }
}
}  // namespace

int dfa2c_influence_for_layer(const void* q, const void* k, const void* v, const dfa2c_dims* dims, int64_t block,
                              const int64_t* windows, int64_t n_windows, int32_t include_cached,
                              const dfa2c_cache* cache, int64_t layer, int64_t t, int32_t mode, double* influence,
                              void* original, void* method_outputs, int64_t* evals, void* stream) {
    return guard([&] {
        if (!influence)
            fail(DFA2C_SHAPE, "influence output must not be NULL");
        validate_dims(dims);
        const int64_t M = n_windows + (include_cached ? 1 : 0);
        std::vector<double> host(static_cast<size_t>(std::max<int64_t>(M, 1) * dims->n_heads));
        const std::vector<uint8_t> eligible =
            influence_enqueue(q, k, v, dims, block, windows, n_windows, include_cached, cache, layer, t, mode,
                              host.data(), original, method_outputs, stream);
        DFA2C_CUDA_CHECK(cudaStreamSynchronize(as_stream(stream)));
        influence_finalize(host.data(), eligible.data(), dims->n_heads, M, influence);
        if (evals)
            *evals += 1 + M;
    });
}

int dfa2c_influence_for_layer_async(const void* q, const void* k, const void* v, const dfa2c_dims* dims,
                                    int64_t block, const int64_t* windows, int64_t n_windows,
                                    int32_t include_cached, const dfa2c_cache* cache, int64_t layer, int64_t t,
                                    int32_t mode, double* rse_host, uint8_t* eligible, void* original,
                                    void* method_outputs, int64_t* evals, void* stream) {
    return guard([&] {
        if (!rse_host || !eligible)
            fail(DFA2C_SHAPE, "rse_host and eligible must not be NULL");
        const std::vector<uint8_t> el =
            influence_enqueue(q, k, v, dims, block, windows, n_windows, include_cached, cache, layer, t, mode,
                              rse_host, original, method_outputs, stream);
        std::copy(el.begin(), el.end(), eligible);
        if (evals)
            *evals += 1 + n_windows + (include_cached ? 1 : 0);
    });
}

int dfa2c_influence_finalize(const double* rse_host, const uint8_t* eligible, int64_t n_heads, int64_t n_methods,
                             double* influence) {
    return guard([&] {
        if (!rse_host || !eligible || !influence || n_heads < 1 || n_methods < 1)
            fail(DFA2C_SHAPE, "bad influence_finalize arguments");
        influence_finalize(rse_host, eligible, n_heads, n_methods, influence);
    });
}

int dfa2c_release_cached_memory(void) {
    return guard([&] {
        {
            std::lock_guard<std::mutex> lk(g_plan_mu);
            g_plans.clear();  // blocks are released after their last launch (event-ordered)
            g_plan_order.clear();
            g_plan_bytes = 0;
        }
        int cur = 0;
        DFA2C_CUDA_CHECK(cudaGetDevice(&cur));
        DFA2C_CUDA_CHECK(cudaDeviceSynchronize());  // the releases above have run
        DFA2C_CUDA_CHECK(cudaMemPoolTrimTo(scratch_pool(cur), 0));
    });
}

int dfa2c_set_influence_fused(int32_t on) {
    g_influence_fused.store(on ? 1 : 0);
    return DFA2C_OK;
}

int32_t dfa2c_influence_fused_enabled(void) { return influence_fused_enabled() ? 1 : 0; }

int dfa2c_set_split_kv(int32_t on) {
    g_split_kv.store(on ? 1 : 0);
    return DFA2C_OK;
}

int dfa2c_convert(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, int64_t n, void* stream) {
    return guard([&] {
        for (int32_t dt : {src_dtype, dst_dtype})
            if (dt != DFA2C_BF16 && dt != DFA2C_F32 && dt != DFA2C_F64)
                fail(DFA2C_SHAPE, "dtype must be DFA2C_BF16, DFA2C_F32 or DFA2C_F64");
        if (n < 0 || (n > 0 && (!src || !dst)))
            fail(DFA2C_SHAPE, "convert needs device buffers and n >= 0");
        int device = 0;
        DFA2C_CUDA_CHECK(cudaGetDevice(&device));
        DFA2C_CUDA_CHECK(dfa2k::launch_convert(src, src_dtype, dst, dst_dtype, n, num_sms(device), as_stream(stream)));
        if (n > 0)
            g_launches.fetch_add(1);
    });
}

// analytic_costs (reference: src/plansolver.cpp, CostModel in
// inc/plansolver.hpp:12-23): full_cost = 1; Arrow(w) = flops_count of its
// mask / dense_flops; Cached = 0; Full = 1.
int dfa2c_analytic_costs(const dfa2c_dims* dims, int64_t block, const int32_t* kinds, const int64_t* windows,
                         int64_t n_methods, double* full_cost, double* method_cost) {
    return guard([&] {
        validate_dims(dims);
        if (block < 1)
            fail(DFA2C_SHAPE, "block_size must be >= 1");
        if (n_methods < 0 || (n_methods > 0 && (!kinds || !method_cost)))
            fail(DFA2C_SHAPE, "bad method list");
        const int64_t n = seq_len(dims), d = dims->head_dim;
        const double dense = static_cast<double>(4 * d * n * n);
        for (int64_t m = 0; m < n_methods; ++m) {
            switch (kinds[m]) {
            case DFA2C_FULL: method_cost[m] = 1.0; break;
            case DFA2C_CACHED: method_cost[m] = 0.0; break;
            case DFA2C_ARROW: {
                if (!windows || windows[m] < 0)
                    fail(DFA2C_SHAPE, "window_blocks must be >= 0");
                const std::vector<uint8_t> mk = arrow_mask(dims, block, windows[m]);
                method_cost[m] = static_cast<double>(4 * d * active_positions(mk.data(), n, block)) / dense;
                break;
            }
            default: fail(DFA2C_SHAPE, "unknown strategy kind");
            }
        }
        if (full_cost)
            *full_cost = 1.0;
    });
}

// ------------------------------------------------------------ plan files
// The reference's plan file (JSON version 1; inc/plan.hpp:44-52,
// src/plan.cpp:109-228): same schema, same validation, same text.

int dfa2c_fnv1a_hex(const void* bytes, int64_t n, char* out) {
    return guard([&] {
        if (!out || n < 0 || (n > 0 && !bytes))
            fail(DFA2C_SHAPE, "fnv1a_hex needs bytes and a 17-byte output");
        uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a 64 offset basis / prime
        const auto* p = static_cast<const unsigned char*>(bytes);
        for (int64_t i = 0; i < n; ++i) {
            h ^= p[i];
            h *= 0x100000001b3ull;
        }
        std::snprintf(out, 17, "%016llx", static_cast<unsigned long long>(h));
    });
}

int dfa2c_plan_to_json(const dfa2c_plan_header* hdr, const int32_t* kinds, const int64_t* windows,
                       const int64_t* window_set, const char* influence_digest, char* buf, int64_t cap,
                       int64_t* len) {
    return guard([&] {
        using json_lite::Value;
        if (!hdr || hdr->n_timesteps < 0 || hdr->n_layers < 0 || hdr->n_heads < 0 || hdr->n_window_set < 0)
            fail(DFA2C_SHAPE, "bad plan header");
        const int64_t T = hdr->n_timesteps, L = hdr->n_layers, H = hdr->n_heads;
        if (T * L * H > 0 && !kinds)
            fail(DFA2C_SHAPE, "plan arrays must not be NULL");
        Value j = Value::object();
        j.set("version", Value::integer(1));
        Value dims = Value::object();
        dims.set("T", Value::integer(T));
        dims.set("L", Value::integer(L));
        dims.set("H", Value::integer(H));
        dims.set("d", Value::integer(hdr->head_dim));
        dims.set("n_visual", Value::integer(hdr->n_visual));
        dims.set("n_text", Value::integer(hdr->n_text));
        dims.set("block", Value::integer(hdr->block_size));
        j.set("dims", std::move(dims));
        j.set("delta", Value::real(hdr->delta));
        j.set("coeff", Value::real(hdr->coeff));
        Value ws = Value::array();
        for (int64_t i = 0; i < hdr->n_window_set; ++i)
            ws.push(Value::integer(window_set[i]));
        j.set("window_set", std::move(ws));
        Value entries = Value::array();
        for (int64_t t = 0; t < T; ++t)
            for (int64_t l = 0; l < L; ++l) {
                Value heads = Value::array();
                for (int64_t h = 0; h < H; ++h) {
                    const int64_t i = (t * L + l) * H + h;
                    Value e = Value::object();
                    switch (kinds[i]) {
                    case DFA2C_FULL: e.set("kind", Value::str("full")); break;
                    case DFA2C_ARROW:
                        e.set("kind", Value::str("arrow"));
                        e.set("window_blocks", Value::integer(windows ? windows[i] : 0));
                        break;
                    case DFA2C_CACHED: e.set("kind", Value::str("cached")); break;
                    default: fail(DFA2C_PLAN, "unknown strategy kind");
                    }
                    heads.push(std::move(e));
                }
                Value entry = Value::object();
                entry.set("t", Value::integer(t));
                entry.set("layer", Value::integer(l));
                entry.set("heads", std::move(heads));
                entries.push(std::move(entry));
            }
        j.set("plan", std::move(entries));
        j.set("influence_digest", Value::str(influence_digest ? influence_digest : ""));
        const std::string text = j.dump(2) + "\n";
        if (len)
            *len = static_cast<int64_t>(text.size());
        if (buf) {
            if (cap < static_cast<int64_t>(text.size()) + 1)
                fail(DFA2C_SHAPE, "output buffer too small");
            std::memcpy(buf, text.c_str(), text.size() + 1);
        }
    });
}

int dfa2c_plan_from_json(const char* text, int64_t text_len, dfa2c_plan_header* hdr, int32_t* kinds,
                         int64_t* windows, int64_t* window_set, char* digest, int64_t digest_cap) {
    return guard([&] {
        using json_lite::Value;
        if (!text || !hdr)
            fail(DFA2C_SHAPE, "plan text and header must not be NULL");
        const std::string src = text_len >= 0 ? std::string(text, static_cast<size_t>(text_len)) : std::string(text);
        Value j;
        try {
            j = json_lite::parse(src);
        } catch (const json_lite::ParseError& e) {
            fail(DFA2C_PLAN, std::string("malformed plan JSON: ") + e.what());
        }
        try {
            if (j.at("version").as_int() != 1)
                fail(DFA2C_PLAN, "unsupported plan version");
            const Value& d = j.at("dims");
            dfa2c_plan_header h{};
            h.n_timesteps = d.at("T").as_int();
            h.n_layers = d.at("L").as_int();
            h.n_heads = d.at("H").as_int();
            h.head_dim = d.at("d").as_int();
            h.n_visual = d.at("n_visual").as_int();
            h.n_text = d.at("n_text").as_int();
            h.block_size = d.at("block").as_int();
            h.delta = j.at("delta").as_double();
            h.coeff = j.at("coeff").as_double();
            const auto& wsv = j.at("window_set").items();
            h.n_window_set = static_cast<int64_t>(wsv.size());
            const std::string& dig = j.at("influence_digest").as_string();
            h.digest_len = static_cast<int64_t>(dig.size());
            if (h.n_timesteps < 1 || h.n_layers < 1)
                fail(DFA2C_PLAN, "plan needs T >= 1 and L >= 1");
            const int64_t T = h.n_timesteps, L = h.n_layers, H = h.n_heads;
            const dfa2c_dims dims{H, h.head_dim, h.n_visual, h.n_text, DFA2C_VISUAL_FIRST};
            validate_dims(&dims);  // AttentionDims::validate -> ShapeError
            std::vector<int32_t> k(static_cast<size_t>(T * L * H), -1);
            std::vector<int64_t> w(static_cast<size_t>(T * L * H), 0);
            std::vector<uint8_t> seen(static_cast<size_t>(T * L), 0);
            for (const Value& e : j.at("plan").items()) {
                const int64_t t = e.at("t").as_int();
                const int64_t l = e.at("layer").as_int();
                if (t < 0 || t >= T || l < 0 || l >= L)
                    fail(DFA2C_PLAN, "plan entry out of range");
                const size_t idx = static_cast<size_t>(t * L + l);
                if (seen[idx])
                    fail(DFA2C_PLAN, "duplicate plan entry");
                seen[idx] = 1;
                const auto& heads = e.at("heads").items();
                if (static_cast<int64_t>(heads.size()) != H)
                    fail(DFA2C_PLAN, "head array length must equal H");
                for (int64_t hh = 0; hh < H; ++hh) {
                    const Value& hv = heads[static_cast<size_t>(hh)];
                    const std::string& kind = hv.at("kind").as_string();
                    const size_t i = idx * static_cast<size_t>(H) + static_cast<size_t>(hh);
                    if (kind == "full") {
                        k[i] = DFA2C_FULL;
                    } else if (kind == "arrow") {
                        k[i] = DFA2C_ARROW;
                        w[i] = hv.at("window_blocks").as_int();
                    } else if (kind == "cached") {
                        k[i] = DFA2C_CACHED;
                    } else {
                        fail(DFA2C_PLAN, "unknown strategy kind: " + kind);
                    }
                }
            }
            for (uint8_t sflag : seen)
                if (!sflag)
                    fail(DFA2C_PLAN, "plan must cover every (t, layer)");
            // CompressionPlan::validate (src/plan.cpp:33-56): dims (ShapeError),
            // then T/L/block, delta, coeff, coverage, per-head rules
            if (h.block_size < 1)
                fail(DFA2C_PLAN, "plan needs T >= 1, L >= 1, block >= 1");
            if (!(h.delta >= 0.0))
                fail(DFA2C_PLAN, "delta must be >= 0");
            if (!(h.coeff >= 1.0))
                fail(DFA2C_PLAN, "coeff must be >= 1");
            const int rc = dfa2c_plan_aggregate(&dims, T, L, h.block_size, k.data(), w.data(), nullptr, nullptr,
                                                nullptr);
            if (rc != DFA2C_OK)
                fail(rc, g_err);
            *hdr = h;
            if (kinds) {
                std::copy(k.begin(), k.end(), kinds);
                if (windows)
                    std::copy(w.begin(), w.end(), windows);
                if (window_set)
                    for (size_t i = 0; i < wsv.size(); ++i)
                        window_set[i] = wsv[i].as_int();
                if (digest) {
                    if (digest_cap < h.digest_len + 1)
                        fail(DFA2C_SHAPE, "digest buffer too small");
                    std::memcpy(digest, dig.c_str(), dig.size() + 1);
                }
            }
        } catch (const json_lite::TypeError& e) {
            fail(DFA2C_PLAN, std::string("plan schema violation: ") + e.what());
        }
    });
}

}  // extern "C"
