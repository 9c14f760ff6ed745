// C++ drop-in API tests: the reference's operator API (include/dfa2/*.hpp)
// exercised exactly the way /root/reference/proj/tests/test_{arrow,cache,
// dispatch,calibrate}.cpp do, against libdfa2_b200.so. Numeric checks use the
// stated bf16 tolerance: max-abs / max|ref| <= 1e-2 against an
// f64 two-pass attention written here from scratch.
//   ./test_dfa2_api host   -> host-only cases (no GPU needed)
//   ./test_dfa2_api gpu    -> everything
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "dfa2/arrow.hpp"
#include "dfa2/cache.hpp"
#include "dfa2/calibrate.hpp"
#include "dfa2/dispatch.hpp"
#include "dfa2/plan.hpp"
#include "dfa2/workload.hpp"

using namespace dfa2;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                               \
    do {                                                                       \
        ++g_checks;                                                            \
        if (!(c)) {                                                            \
            ++g_fail;                                                          \
            std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);         \
        }                                                                      \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                               \
    do {                                                                       \
        ++g_checks;                                                            \
        bool ok_ = false;                                                      \
        try {                                                                  \
            (void)(expr);                                                      \
        } catch (const T&) {                                                   \
            ok_ = true;                                                        \
        } catch (...) {                                                        \
        }                                                                      \
        if (!ok_) {                                                            \
            ++g_fail;                                                          \
            std::printf("  FAIL %s:%d: %s did not throw %s\n", __FILE__, __LINE__, #expr, #T); \
        }                                                                      \
    } while (0)

struct Case {
    const char* name;
    bool gpu;
    std::function<void()> fn;
};
static std::vector<Case>& cases() {
    static std::vector<Case> c;
    return c;
}
struct Reg {
    Reg(const char* n, bool g, std::function<void()> f) { cases().push_back({n, g, std::move(f)}); }
};
#define TEST(name, gpu) static void name(); static Reg reg_##name(#name, gpu, name); static void name()

static AttentionDims dims_of(int64_t h, int64_t d, int64_t nv, int64_t nt, TokenOrder o = TokenOrder::visual_first) {
    AttentionDims a;
    a.n_heads = h;
    a.head_dim = d;
    a.n_visual = nv;
    a.n_text = nt;
    a.order = o;
    return a;
}

static float bf16r(float f) {  // round to bf16 and back
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    std::memcpy(&f, &u, 4);
    return f;
}

static Tensor gaussian(std::vector<int64_t> shape, uint64_t seed) {
    std::mt19937_64 eng(seed);
    std::normal_distribution<float> nd(0.f, 1.f);
    Tensor t = Tensor::zeros(std::move(shape));
    for (int64_t i = 0; i < t.numel(); ++i)
        t.f32()[i] = bf16r(nd(eng));
    return t;
}

// f64 masked two-pass attention on one head (independent restatement).
static std::vector<double> oracle_head(const float* q, const float* k, const float* v, int64_t n, int64_t d,
                                       const BlockMask* m) {
    std::vector<double> out(static_cast<size_t>(n * d), 0.0), w(static_cast<size_t>(n));
    const double sc = 1.0 / std::sqrt(static_cast<double>(d));
    for (int64_t i = 0; i < n; ++i) {
        double mx = -INFINITY;
        for (int64_t j = 0; j < n; ++j) {
            if (m && !m->is_active(i / m->block_size, j / m->block_size)) {
                w[j] = -INFINITY;
                continue;
            }
            double s = 0;
            for (int64_t x = 0; x < d; ++x)
                s += static_cast<double>(q[i * d + x]) * k[j * d + x];
            w[j] = s * sc;
            mx = std::max(mx, w[j]);
        }
        double den = 0;
        for (int64_t j = 0; j < n; ++j) {
            w[j] = std::isinf(w[j]) ? 0.0 : std::exp(w[j] - mx);
            den += w[j];
        }
        for (int64_t j = 0; j < n; ++j)
            for (int64_t x = 0; x < d; ++x)
                out[i * d + x] += w[j] / den * v[j * d + x];
    }
    return out;
}

static double max_rel(const float* got, const std::vector<double>& want) {
    double ma = 0, mr = 0;
    for (size_t i = 0; i < want.size(); ++i) {
        ma = std::max(ma, std::abs(got[i] - want[i]));
        mr = std::max(mr, std::abs(want[i]));
    }
    return ma / mr;
}

// ---------------------------------------------------------------- host-only
TEST(large_tensor_storage_is_reused_and_zeros_still_zero, false) {
    // freed large buffers are kept for reuse (no per-call page faults of
    // fresh outputs); zeros() must still zero a recycled buffer
    const int64_t n = int64_t{3} << 20;  // 12 MB of f32
    const float* first = nullptr;
    {
        Tensor t = Tensor::zeros({n});
        float* p = t.f32();
        for (int64_t i = 0; i < n; i += 4099)
            p[i] = 7.0f;  // garbage left behind
        first = p;
    }
    Tensor z = Tensor::zeros({n});
    CHECK(z.f32() == first);  // the same storage came back
    bool all_zero = true;
    for (int64_t i = 0; i < n; ++i)
        all_zero = all_zero && z.f32()[i] == 0.0f;
    CHECK(all_zero);
}

TEST(arrow_mask_known_answers, false) {  // test_arrow.cpp:53-92
    const BlockMask m = build_arrow_mask({dims_of(1, 16, 512, 128), 128, 0});
    CHECK(m.n_query_blocks == 5 && m.n_key_blocks == 5);
    int64_t c = 0;
    for (uint8_t a : m.active)
        c += a;
    CHECK(c == 13);
    CHECK(std::abs(sparsity_ratio(m) - 0.48) < 1e-12);
    for (int64_t j = 0; j < 5; ++j)
        CHECK(m.is_active(4, j) && m.is_active(j, 4));
    CHECK(!m.is_active(0, 2));
    for (int64_t w : {3, 4, 100})
        CHECK(sparsity_ratio(build_arrow_mask({dims_of(1, 16, 512, 128), 128, w})) == 0.0);
    const BlockMask t = build_arrow_mask({dims_of(1, 16, 512, 128, TokenOrder::text_first), 128, 0});
    CHECK(t.is_active(0, 3) && t.is_active(3, 0) && !t.is_active(1, 3));
    CHECK_THROWS_AS(build_arrow_mask({dims_of(1, 16, 64, 8), 0, 0}), ShapeError);
}

TEST(flops_and_plan_flops, false) {  // test_arrow.cpp:112-152, test_dispatch.cpp:133-162
    BlockMask m = BlockMask::all_active(5, 2);
    CHECK(m.active_positions() == 25);
    m.set(2, 2, false);
    CHECK(m.active_positions() == 24);
    CHECK(flops_count(BlockMask::all_active(64, 16), 8) == dense_flops(64, 8));
    const AttentionDims d = dims_of(4, 8, 56, 8);
    LayerPlan plan{{HeadStrategy::Full(), HeadStrategy::Arrow(0), HeadStrategy::Arrow(2), HeadStrategy::Cached()}};
    const int64_t by_head = dense_flops(64, 8) + flops_count(build_arrow_mask({d, 8, 0}), 8) +
                            flops_count(build_arrow_mask({d, 8, 2}), 8);
    CHECK(plan_flops(plan, d, 8) == by_head);
    CHECK_THROWS_AS(plan_flops(LayerPlan{{HeadStrategy::Full()}}, d, 8), ShapeError);
}

TEST(compression_plan_validation, false) {  // plan.cpp:33-73
    const AttentionDims d = dims_of(2, 64, 500, 12);
    CompressionPlan p = CompressionPlan::all_full(d, 2, 3, 64);
    CHECK(p.aggregate_sparsity() == 0.0);
    p.at(1, 2) = LayerPlan{{HeadStrategy::Cached(), HeadStrategy::Arrow(1)}};
    p.validate();
    CHECK(p.flops_total() < p.flops_dense_total());
    p.at(0, 0) = LayerPlan{{HeadStrategy::Cached(), HeadStrategy::Full()}};
    CHECK_THROWS_AS(p.validate(), PlanValidationError);
}

TEST(cache_host_semantics, false) {  // test_cache.cpp
    HeadCache c;
    CHECK(!c.has(0, 0));
    CHECK_THROWS_AS(c.fetch(0, 0), CacheMissError);
    CHECK_THROWS_AS(c.staleness(0, 0, 1), CacheMissError);
    const Tensor a = gaussian({6, 4}, 1);
    c.store(1, 1, a, 3);
    CHECK(c.produced_at(1, 1) == 3 && c.staleness(1, 1, 5) == 2);
    CHECK(c.fetch(1, 1) == a);  // pending host copy (not yet bound to a device)
    CHECK_THROWS_AS(c.store(0, 0, Tensor::zeros({2, 2, 2}), 0), ShapeError);
    CHECK(make_candidates({0, 2}).size() == 3 && make_candidates({0, 2})[2].id == "cached");
    CHECK_THROWS_AS(make_candidates({}, false), ShapeError);
}

TEST(cache_is_a_copyable_value_type, false) {  // reference cache.hpp:15-32 (implicit copy)
    HeadCache c;
    const Tensor a = gaussian({6, 4}, 2);
    c.store(0, 1, a, 4);
    HeadCache copy = c;  // deep copy
    CHECK(copy.has(0, 1) && copy.produced_at(0, 1) == 4 && copy.fetch(0, 1) == a);
    c.store(0, 1, gaussian({6, 4}, 3), 5);  // the copy does not alias the original
    CHECK(copy.fetch(0, 1) == a && copy.produced_at(0, 1) == 4 && c.produced_at(0, 1) == 5);
    HeadCache assigned;
    assigned = copy;
    CHECK(assigned.size() == 1 && assigned.fetch(0, 1) == a);
    HeadCache moved = std::move(assigned);
    CHECK(moved.size() == 1 && moved.fetch(0, 1) == a);
}

// ---------------------------------------------------------------- GPU
TEST(mixed_plan_matches_per_head_oracles, true) {  // test_dispatch.cpp:63-88
    const AttentionDims d = dims_of(3, 64, 256, 44);
    const int64_t n = d.seq_len(), B = 32;
    const Tensor q = gaussian({3, n, 64}, 11), k = gaussian({3, n, 64}, 12), v = gaussian({3, n, 64}, 13);
    HeadCache cache;
    const Tensor stored = gaussian({n, 64}, 99);
    cache.store(0, 2, stored, 0);
    LayerPlan plan{{HeadStrategy::Full(), HeadStrategy::Arrow(0), HeadStrategy::Cached()}};
    const Tensor out = multi_strategy_attention(q, k, v, plan, cache, 0, 1, d, B);
    const Tensor h0 = head_slice(out, 0), h1 = head_slice(out, 1), h2 = head_slice(out, 2);
    CHECK(max_rel(h0.f32(), oracle_head(head_slice(q, 0).f32(), head_slice(k, 0).f32(), head_slice(v, 0).f32(), n, 64,
                                        nullptr)) < 1e-2);
    const BlockMask m = build_arrow_mask({d, B, 0});
    CHECK(max_rel(h1.f32(), oracle_head(head_slice(q, 1).f32(), head_slice(k, 1).f32(), head_slice(v, 1).f32(), n, 64,
                                        &m)) < 1e-2);
    CHECK(h2 == stored);  // bf16-representable slot: spliced bit-exactly
    CHECK(cache.produced_at(0, 2) == 0 && cache.produced_at(0, 0) == 1 && cache.produced_at(0, 1) == 1);
    CHECK(cache.fetch(0, 0) == h0 && cache.fetch(0, 1) == h1);  // commit == output
}

TEST(cache_miss_and_shape_errors_before_compute, true) {  // test_dispatch.cpp:90-131
    const AttentionDims d = dims_of(3, 64, 100, 28);
    const Tensor q = gaussian({3, 128, 64}, 1);
    HeadCache cache;
    LayerPlan plan{{HeadStrategy::Full(), HeadStrategy::Cached(), HeadStrategy::Full()}};
    CHECK_THROWS_AS(multi_strategy_attention(q, q, q, plan, cache, 0, 0, d, 32), CacheMissError);
    CHECK(cache.size() == 0);
    CHECK_THROWS_AS(multi_strategy_attention(q, q, q, LayerPlan{{HeadStrategy::Full()}}, cache, 0, 0, d, 32),
                    ShapeError);
}

TEST(full_plan_equals_max_window_and_is_deterministic, true) {
    const AttentionDims d = dims_of(2, 128, 600, 40);
    const int64_t n = d.seq_len();
    const Tensor q = gaussian({2, n, 128}, 5), k = gaussian({2, n, 128}, 6), v = gaussian({2, n, 128}, 7);
    HeadCache c1, c2, c3;
    const Tensor a = multi_strategy_attention(q, k, v, LayerPlan::all_full(2), c1, 0, 0, d, 128);
    const Tensor b = multi_strategy_attention(q, k, v, LayerPlan{{HeadStrategy::Arrow(99), HeadStrategy::Arrow(99)}},
                                              c2, 0, 0, d, 128);
    const Tensor c = multi_strategy_attention(q, k, v, LayerPlan::all_full(2), c3, 0, 0, d, 128);
    CHECK(a == b && a == c);
}

TEST(sparse_forward_and_fully_masked_rows, true) {  // test_arrow.cpp:154-301
    const AttentionDims d = dims_of(1, 64, 256, 32);
    const Tensor q = gaussian({288, 64}, 15), k = gaussian({288, 64}, 16), v = gaussian({288, 64}, 17);
    for (int64_t w : {0, 1, 2, 7}) {
        const BlockMask m = build_arrow_mask({d, 32, w});
        const Tensor got = sparse_attention_forward(q, k, v, m);
        CHECK(max_rel(got.f32(), oracle_head(q.f32(), k.f32(), v.f32(), 288, 64, &m)) < 1e-2);
    }
    BlockMask bad = BlockMask::all_active(64, 16);
    for (int64_t j = 0; j < 4; ++j)
        bad.set(2, j, false);
    const Tensor x = gaussian({64, 64}, 20);
    CHECK_THROWS_AS(sparse_attention_forward(x, x, x, bad), FullyMaskedRowError);
}

TEST(rse_semantics, true) {  // test_calibrate.cpp:48-72
    const Tensor y = gaussian({4, 4}, 1);
    CHECK(rse(y, y) == 0.0);
    const Tensor y_o = Tensor::from_f32({2}, {1, 3}), y_m = Tensor::from_f32({2}, {2, 2});
    CHECK(std::abs(rse(y_m, y_o) - 1.0) < 1e-12);
    CHECK(std::abs(rse(y_o, y_o, RseMode::literal) - 1.0) < 1e-12);
    CHECK_THROWS_AS(rse(Tensor::from_f32({2}, {5, 6}), Tensor::from_f32({2}, {5, 5})), DegenerateReferenceError);
    const Tensor a64 = gaussian({1000}, 3).to_f64(), b64 = gaussian({1000}, 4).to_f64();
    double mean = 0, den = 0, num = 0;  // from-scratch (test_calibrate.cpp:31-44)
    for (int64_t i = 0; i < 1000; ++i)
        mean += a64.f64()[i];
    mean /= 1000;
    for (int64_t i = 0; i < 1000; ++i) {
        den += (a64.f64()[i] - mean) * (a64.f64()[i] - mean);
        num += (b64.f64()[i] - a64.f64()[i]) * (b64.f64()[i] - a64.f64()[i]);
    }
    CHECK(std::abs(rse(b64, a64) - num / den) <= 1e-12 * (num / den));
}

TEST(influence_for_layer_semantics, true) {  // test_calibrate.cpp:85-146
    const AttentionDims d = dims_of(3, 64, 300, 20);
    const int64_t n = d.seq_len();
    const Tensor q = gaussian({3, n, 64}, 31), k = gaussian({3, n, 64}, 32), v = gaussian({3, n, 64}, 33);
    HeadCache cache;
    CalibrationStats st;
    const auto methods = make_candidates({0, 100}, true);
    const LayerInfluence li = influence_for_layer(q, k, v, methods, cache, 0, 0, d, 64, RseMode::standard, &st);
    CHECK(st.attention_evals == 4);
    for (int64_t h = 0; h < 3; ++h) {
        CHECK(std::isinf(li.influence[h * 3 + 2]));  // Cached ineligible at t = 0
        CHECK(li.influence[h * 3 + 1] == 0.0);      // max window == Full bitwise
        CHECK(li.influence[h * 3 + 0] > 0.0);
    }
}

TEST(influence_takes_const_cache_and_copies_carry_device_slots, true) {  // calibrate.hpp:80-86
    const AttentionDims d = dims_of(2, 64, 256, 32);
    const int64_t n = d.seq_len();
    const Tensor q = gaussian({2, n, 64}, 41), k = gaussian({2, n, 64}, 42), v = gaussian({2, n, 64}, 43);
    HeadCache cache;
    const Tensor out0 = multi_strategy_attention(q, k, v, LayerPlan::all_full(2), cache, 0, 0, d, 64);
    const HeadCache& cref = cache;  // a const caller, as in the reference
    const LayerInfluence li = influence_for_layer(q, k, v, make_candidates({0}, true), cref, 0, 1, d, 64,
                                                  RseMode::standard, nullptr);
    CHECK(std::isfinite(li.influence[1]) && std::isfinite(li.influence[3]));
    HeadCache copy = cache;  // device-resident slots deep-copied through the host
    CHECK(copy.fetch(0, 0) == head_slice(out0, 0) && copy.produced_at(0, 1) == 0);
    const Tensor again = multi_strategy_attention(q, k, v, LayerPlan{{HeadStrategy::Cached(), HeadStrategy::Cached()}},
                                                  copy, 0, 1, d, 64);
    CHECK(again == out0);  // the copy's re-uploaded slots splice bit-exactly
}

TEST(attention_reference_is_f32_and_f64_accurate, true) {  // tensor.cpp:73-114, 268-295
    const AttentionDims d = dims_of(2, 64, 200, 40);
    const int64_t n = d.seq_len();
    const Tensor q = gaussian({2, n, 64}, 51), k = gaussian({2, n, 64}, 52), v = gaussian({2, n, 64}, 53);
    const BlockMask m = build_arrow_mask({d, 32, 1});
    const Tensor r32 = attention_reference(q, k, v, &m);
    const Tensor r64 = attention_reference(q.to_f64(), k.to_f64(), v.to_f64(), &m);
    CHECK(r32.dtype() == Dtype::f32 && r64.dtype() == Dtype::f64);
    for (int64_t h = 0; h < 2; ++h) {
        const std::vector<double> want = oracle_head(head_slice(q, h).f32(), head_slice(k, h).f32(),
                                                    head_slice(v, h).f32(), n, 64, &m);
        const Tensor g32 = head_slice(r32, h), g64 = head_slice(r64, h);
        double e32 = 0, e64 = 0, mx = 0;
        for (size_t i = 0; i < want.size(); ++i) {
            e32 = std::max(e32, std::abs(static_cast<double>(g32.f32()[i]) - want[i]));
            e64 = std::max(e64, std::abs(g64.f64()[i] - want[i]));
            mx = std::max(mx, std::abs(static_cast<double>(want[i])));
        }
        CHECK(e32 <= 1e-5 * mx);  // f32 precision, not bf16 (bf16 would be ~1e-3)
        CHECK(e64 <= 1e-12 * mx);  // f64 to rounding
    }
    BlockMask bad = BlockMask::all_active(n, 32);
    for (int64_t j = 0; j < bad.n_key_blocks; ++j)
        bad.set(1, j, false);
    CHECK_THROWS_AS(attention_reference(q, k, v, &bad), FullyMaskedRowError);
}

// dump-workload H d nv nt order L T B seed path: raw f32 q|k|v of every
// (t, layer) slot of generate(), t-major, for the bit-exactness check
// against the reference generator (tests/test_cpp_api.py).
static int dump_workload(char** a) {
    WorkloadConfig cfg;
    cfg.dims.n_heads = std::atoll(a[0]);
    cfg.dims.head_dim = std::atoll(a[1]);
    cfg.dims.n_visual = std::atoll(a[2]);
    cfg.dims.n_text = std::atoll(a[3]);
    cfg.dims.order = std::atoi(a[4]) ? TokenOrder::text_first : TokenOrder::visual_first;
    cfg.n_layers = std::atoll(a[5]);
    cfg.n_timesteps = std::atoll(a[6]);
    cfg.block_size = std::atoll(a[7]);
    cfg.seed = std::strtoull(a[8], nullptr, 10);
    const Workload w = generate(cfg);
    FILE* f = std::fopen(a[9], "wb");
    if (!f)
        return 2;
    for (int64_t t = 0; t < cfg.n_timesteps; ++t)
        for (int64_t l = 0; l < cfg.n_layers; ++l)
            for (const Tensor* x : {&w.q(t, l), &w.k(t, l), &w.v(t, l)})
                std::fwrite(x->f32(), sizeof(float), static_cast<size_t>(x->numel()), f);
    return std::fclose(f) == 0 ? 0 : 2;
}

int main(int argc, char** argv) {
    if (argc == 12 && std::string(argv[1]) == "dump-workload")
        return dump_workload(argv + 2);
    const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
    int ran = 0;
    for (const Case& c : cases()) {
        if (c.gpu && !gpu)
            continue;
        const int before = g_fail;
        try {
            c.fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("  FAIL %s: uncaught %s\n", c.name, e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", c.name);
        ++ran;
    }
    std::printf("%d cases, %d checks, %d failures\n", ran, g_checks, g_fail);
    return g_fail ? 1 : 0;
}
