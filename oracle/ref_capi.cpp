// TEST INFRASTRUCTURE ONLY — extern "C" shim over the UNMODIFIED reference
// library (compiled in place from /root/reference/proj/src by oracle/Makefile).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load the resulting oracle/_ref/libdfa2ref.so.
//
// Every entry point forwards to the reference's own C++ operator API
// (/root/reference/proj/include/dfa2/*.hpp) and maps its exception taxonomy
// (/root/reference/proj/include/dfa2/errors.hpp:8-45) onto integer status
// codes identical to include/dfa2c.h.

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "dfa2/arrow.hpp"
#include "dfa2/cache.hpp"
#include "dfa2/calibrate.hpp"
#include "dfa2/dispatch.hpp"
#include "dfa2/plan.hpp"
#include "dfa2/plansolver.hpp"
#include "dfa2/tensor.hpp"
#include "dfa2/workload.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

enum Status {
    OK = 0, SHAPE = 1, NONFINITE = 2, FULLY_MASKED = 3, CACHE_MISS = 4,
    DEGENERATE = 5, PLAN = 6, IO = 7, ORACLE = 8, OTHER = 9
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return OK;
    } catch (const dfa2::ShapeError& e) { g_err = e.what(); return SHAPE; }
    catch (const dfa2::NonFiniteError& e) { g_err = e.what(); return NONFINITE; }
    catch (const dfa2::FullyMaskedRowError& e) { g_err = e.what(); return FULLY_MASKED; }
    catch (const dfa2::CacheMissError& e) { g_err = e.what(); return CACHE_MISS; }
    catch (const dfa2::DegenerateReferenceError& e) { g_err = e.what(); return DEGENERATE; }
    catch (const dfa2::PlanValidationError& e) { g_err = e.what(); return PLAN; }
    catch (const dfa2::IoError& e) { g_err = e.what(); return IO; }
    catch (const dfa2::OracleError& e) { g_err = e.what(); return ORACLE; }
    catch (const std::exception& e) { g_err = e.what(); return OTHER; }
}

dfa2::AttentionDims make_dims(int64_t H, int64_t d, int64_t nv, int64_t nt, int order) {
    dfa2::AttentionDims dims;
    dims.n_heads = H;
    dims.head_dim = d;
    dims.n_visual = nv;
    dims.n_text = nt;
    dims.order = order ? dfa2::TokenOrder::text_first : dfa2::TokenOrder::visual_first;
    return dims;
}

dfa2::HeadStrategy make_strategy(int32_t kind, int64_t w) {
    switch (kind) {
    case 0: return dfa2::HeadStrategy::Full();
    case 1: return dfa2::HeadStrategy::Arrow(w);
    case 2: return dfa2::HeadStrategy::Cached();
    default: throw dfa2::ShapeError("unknown strategy kind");
    }
}

dfa2::LayerPlan make_plan(int64_t H, const int32_t* kinds, const int64_t* windows) {
    dfa2::LayerPlan lp;
    for (int64_t h = 0; h < H; ++h)
        lp.strategies.push_back(make_strategy(kinds[h], windows ? windows[h] : 0));
    return lp;
}

dfa2::BlockMask mask_from_bytes(const uint8_t* active, int64_t n, int64_t B) {
    dfa2::BlockMask m = dfa2::BlockMask::all_active(n, B);
    std::memcpy(m.active.data(), active, m.active.size());
    return m;
}

dfa2::Tensor tensor_f32(std::vector<int64_t> shape, const float* p) {
    int64_t n = 1;
    for (int64_t s : shape) n *= s;
    return dfa2::Tensor::from_f32(std::move(shape), std::vector<float>(p, p + n));
}

} // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// build_arrow_mask (/root/reference/proj/src/arrow.cpp:113-153).
REF_API int ref_arrow_mask(int64_t H, int64_t d, int64_t nv, int64_t nt, int order,
                           int64_t B, int64_t w, uint8_t* active, int64_t* nb) {
    return guard([&] {
        const dfa2::BlockMask m = dfa2::build_arrow_mask({make_dims(H, d, nv, nt, order), B, w});
        if (nb) *nb = m.n_query_blocks;
        if (active) std::memcpy(active, m.active.data(), m.active.size());
    });
}

// active_positions / flops_count / sparsity_ratio (arrow.cpp:95-104, 155-169)
// of an arbitrary byte mask.
REF_API int ref_mask_stats(const uint8_t* active, int64_t n, int64_t B, int64_t d,
                           int64_t* active_positions, int64_t* flops, double* sparsity) {
    return guard([&] {
        const dfa2::BlockMask m = mask_from_bytes(active, n, B);
        if (active_positions) *active_positions = m.active_positions();
        if (flops) *flops = dfa2::flops_count(m, d);
        if (sparsity) *sparsity = dfa2::sparsity_ratio(m);
    });
}

REF_API int64_t ref_dense_flops(int64_t n, int64_t d) { return dfa2::dense_flops(n, d); }

// plan_flops (dispatch.cpp:93-120).
REF_API int ref_plan_flops(int64_t H, int64_t d, int64_t nv, int64_t nt, int order,
                           int64_t B, const int32_t* kinds, const int64_t* windows,
                           int64_t* out) {
    return guard([&] {
        *out = dfa2::plan_flops(make_plan(H, kinds, windows), make_dims(H, d, nv, nt, order), B);
    });
}

// sparse_attention_forward pointer overload (arrow.cpp:171-194).
REF_API int ref_sparse_attention_forward(const float* q, const float* k, const float* v,
                                         float* out, int64_t n, int64_t d,
                                         const uint8_t* active, int64_t B, int parallel) {
    return guard([&] {
        dfa2::sparse_attention_forward(q, k, v, out, n, d, mask_from_bytes(active, n, B),
                                       parallel != 0);
    });
}

// dense_tiled_attention (arrow.cpp:210-228).
REF_API int ref_dense_tiled_attention(const float* q, const float* k, const float* v,
                                      float* out, int64_t n, int64_t d, int64_t B,
                                      int parallel) {
    return guard([&] { dfa2::dense_tiled_attention(q, k, v, out, n, d, B, parallel != 0); });
}

// attention_reference, f64 (tensor.cpp:268-295); mask may be NULL.
REF_API int ref_attention_reference_f64(const double* q, const double* k, const double* v,
                                        double* out, int64_t H, int64_t n, int64_t d,
                                        const uint8_t* active, int64_t B) {
    return guard([&] {
        const int64_t numel = H * n * d;
        auto mk = [&](const double* p) {
            return dfa2::Tensor::from_f64({H, n, d}, std::vector<double>(p, p + numel));
        };
        dfa2::BlockMask mask;
        if (active) mask = mask_from_bytes(active, n, B);
        const dfa2::Tensor o = dfa2::attention_reference(mk(q), mk(k), mk(v), active ? &mask : nullptr);
        std::memcpy(out, o.f64(), sizeof(double) * numel);
    });
}

// attention_reference, f32 (tensor.cpp:268-295).
REF_API int ref_attention_reference_f32(const float* q, const float* k, const float* v,
                                        float* out, int64_t H, int64_t n, int64_t d,
                                        const uint8_t* active, int64_t B) {
    return guard([&] {
        dfa2::BlockMask mask;
        if (active) mask = mask_from_bytes(active, n, B);
        const dfa2::Tensor o = dfa2::attention_reference(
            tensor_f32({H, n, d}, q), tensor_f32({H, n, d}, k), tensor_f32({H, n, d}, v),
            active ? &mask : nullptr);
        std::memcpy(out, o.f32(), sizeof(float) * H * n * d);
    });
}

// HeadCache (cache.cpp:7-41).
REF_API void* ref_cache_create() { return new dfa2::HeadCache(); }
REF_API void ref_cache_destroy(void* c) { delete static_cast<dfa2::HeadCache*>(c); }
REF_API int ref_cache_store(void* c, int64_t layer, int64_t head, const float* data,
                            int64_t n, int64_t d, int64_t t) {
    return guard([&] {
        static_cast<dfa2::HeadCache*>(c)->store(layer, head, tensor_f32({n, d}, data), t);
    });
}
REF_API int ref_cache_has(void* c, int64_t layer, int64_t head) {
    return static_cast<dfa2::HeadCache*>(c)->has(layer, head) ? 1 : 0;
}
REF_API int ref_cache_produced_at(void* c, int64_t layer, int64_t head, int64_t* t) {
    return guard([&] { *t = static_cast<dfa2::HeadCache*>(c)->produced_at(layer, head); });
}
REF_API int ref_cache_fetch(void* c, int64_t layer, int64_t head, float* out, int64_t numel) {
    return guard([&] {
        const dfa2::Tensor& x = static_cast<dfa2::HeadCache*>(c)->fetch(layer, head);
        if (x.numel() != numel) throw dfa2::ShapeError("fetch size mismatch");
        std::memcpy(out, x.f32(), sizeof(float) * numel);
    });
}

// multi_strategy_attention (dispatch.cpp:30-91).
REF_API int ref_multi_strategy_attention(const float* q, const float* k, const float* v,
                                         int64_t H, int64_t d, int64_t nv, int64_t nt,
                                         int order, const int32_t* kinds,
                                         const int64_t* windows, void* cache,
                                         int64_t layer, int64_t t, int64_t B, float* out) {
    return guard([&] {
        const dfa2::AttentionDims dims = make_dims(H, d, nv, nt, order);
        const int64_t n = dims.seq_len();
        const dfa2::Tensor o = dfa2::multi_strategy_attention(
            tensor_f32({H, n, d}, q), tensor_f32({H, n, d}, k), tensor_f32({H, n, d}, v),
            make_plan(H, kinds, windows), *static_cast<dfa2::HeadCache*>(cache), layer, t,
            dims, B);
        std::memcpy(out, o.f32(), sizeof(float) * H * n * d);
    });
}

// rse (calibrate.cpp:75-87) on flat f32 buffers of `numel` elements.
REF_API int ref_rse(const float* y_m, const float* y_o, int64_t numel, int mode, double* out) {
    return guard([&] {
        *out = dfa2::rse(tensor_f32({numel}, y_m), tensor_f32({numel}, y_o),
                         mode ? dfa2::RseMode::literal : dfa2::RseMode::standard);
    });
}

// influence_for_layer (calibrate.cpp:193-253). Candidates are Arrow(w) for
// each window, then Cached when include_cached != 0 (make_candidates,
// calibrate.cpp:89-103). influence is [H*M]; original [H,N,d];
// method_outputs [M,H,N,d] (may be NULL; ineligible entries left untouched).
REF_API int ref_influence_for_layer(const float* q, const float* k, const float* v,
                                    int64_t H, int64_t d, int64_t nv, int64_t nt, int order,
                                    const int64_t* windows, int64_t n_windows,
                                    int include_cached, void* cache, int64_t layer,
                                    int64_t t, int64_t B, int mode, double* influence,
                                    float* original, float* method_outputs, int64_t* evals) {
    return guard([&] {
        const dfa2::AttentionDims dims = make_dims(H, d, nv, nt, order);
        const int64_t n = dims.seq_len();
        const auto methods = dfa2::make_candidates(
            std::vector<int64_t>(windows, windows + n_windows), include_cached != 0);
        dfa2::CalibrationStats stats;
        const dfa2::LayerInfluence li = dfa2::influence_for_layer(
            tensor_f32({H, n, d}, q), tensor_f32({H, n, d}, k), tensor_f32({H, n, d}, v),
            methods, *static_cast<dfa2::HeadCache*>(cache), layer, t, dims, B,
            mode ? dfa2::RseMode::literal : dfa2::RseMode::standard, &stats);
        const int64_t M = static_cast<int64_t>(methods.size());
        std::memcpy(influence, li.influence.data(), sizeof(double) * H * M);
        if (original) std::memcpy(original, li.original.f32(), sizeof(float) * H * n * d);
        if (method_outputs)
            for (int64_t m = 0; m < M; ++m)
                if (li.method_outputs[m].numel() == H * n * d)
                    std::memcpy(method_outputs + m * H * n * d, li.method_outputs[m].f32(),
                                sizeof(float) * H * n * d);
        if (evals) *evals = stats.attention_evals;
    });
}

// Workload generator (workload.cpp:120-228): q/k/v are [T*L, H, N, d].
REF_API int ref_generate(int64_t H, int64_t d, int64_t nv, int64_t nt, int order,
                         int64_t L, int64_t T, int64_t B, uint64_t seed, float* q, float* k,
                         float* v) {
    return guard([&] {
        dfa2::WorkloadConfig cfg;
        cfg.dims = make_dims(H, d, nv, nt, order);
        cfg.n_layers = L;
        cfg.n_timesteps = T;
        cfg.block_size = B;
        cfg.seed = seed;
        const dfa2::Workload w = dfa2::generate(cfg);
        const int64_t per = H * cfg.dims.seq_len() * d;
        for (int64_t t = 0; t < T; ++t)
            for (int64_t l = 0; l < L; ++l) {
                const int64_t s = t * L + l;
                std::memcpy(q + s * per, w.q(t, l).f32(), sizeof(float) * per);
                std::memcpy(k + s * per, w.k(t, l).f32(), sizeof(float) * per);
                std::memcpy(v + s * per, w.v(t, l).f32(), sizeof(float) * per);
            }
    });
}

// calibrate_model (calibrate.cpp:255-348) on the reference's own generated
// workload (workload.cpp:120-228): the selected plan [T*L*H] (kinds,
// windows) and the per-(t, layer) solver objective and budget spent.
REF_API int ref_calibrate_model(int64_t H, int64_t d, int64_t nv, int64_t nt, int order,
                                int64_t L, int64_t T, int64_t B, uint64_t seed,
                                const int64_t* windows, int64_t n_windows, int include_cached,
                                double delta, double coeff, int32_t* kinds, int64_t* wins,
                                double* objective, double* budget) {
    return guard([&] {
        dfa2::WorkloadConfig cfg;
        cfg.dims = make_dims(H, d, nv, nt, order);
        cfg.n_layers = L;
        cfg.n_timesteps = T;
        cfg.block_size = B;
        cfg.seed = seed;
        const dfa2::Workload w = dfa2::generate(cfg);
        dfa2::CalibrationConfig cc;
        cc.methods = dfa2::make_candidates(std::vector<int64_t>(windows, windows + n_windows),
                                           include_cached != 0);
        cc.delta = delta;
        cc.coeff = coeff;
        const dfa2::CalibrationResult r = dfa2::calibrate_model(w, cc);
        for (int64_t s = 0; s < T * L; ++s) {
            const dfa2::LayerPlan& lp = r.plan.layers[static_cast<size_t>(s)];
            for (int64_t h = 0; h < H; ++h) {
                const dfa2::HeadStrategy& st = lp.strategies[static_cast<size_t>(h)];
                kinds[s * H + h] = st.kind == dfa2::StrategyKind::full ? 0
                                   : st.kind == dfa2::StrategyKind::arrow ? 1 : 2;
                wins[s * H + h] = st.kind == dfa2::StrategyKind::arrow ? st.window_blocks : 0;
            }
            if (objective) objective[s] = r.stats.objective[static_cast<size_t>(s)];
            if (budget) budget[s] = r.stats.budget_spent[static_cast<size_t>(s)];
        }
    });
}

// CompressionPlan::aggregate_sparsity (plan.cpp:58-73) over a [T*L*H] plan.
REF_API int ref_plan_aggregate(int64_t H, int64_t d, int64_t nv, int64_t nt, int order,
                               int64_t T, int64_t L, int64_t B, const int32_t* kinds,
                               const int64_t* windows, int64_t* flops_total,
                               int64_t* flops_dense, double* sparsity) {
    return guard([&] {
        dfa2::CompressionPlan p = dfa2::CompressionPlan::all_full(make_dims(H, d, nv, nt, order), T, L, B);
        for (int64_t s = 0; s < T * L; ++s)
            p.layers[s] = make_plan(H, kinds + s * H, windows + s * H);
        p.validate();
        if (flops_total) *flops_total = p.flops_total();
        if (flops_dense) *flops_dense = p.flops_dense_total();
        if (sparsity) *sparsity = p.aggregate_sparsity();
    });
}

// Bounded CPU sample of one joint-attention layer for the benchmark's
// reference arm: each listed head runs through the reference's own
// multi-threaded kernels (DFA2_THREADS): Full -> dense_tiled_attention
// (arrow.cpp:210-228, the reference bench's dense path), Arrow(w) ->
// sparse_attention_forward with build_arrow_mask (arrow.cpp:113-194), Cached
// -> copy of the stored slot (dispatch.cpp:77-81). q/k/v/out/slots [H,N,d].
REF_API int ref_layer_sample(const float* q, const float* k, const float* v,
                             const float* slots, float* out, int64_t H, int64_t d,
                             int64_t nv, int64_t nt, int order, int64_t B,
                             const int32_t* kinds, const int64_t* windows,
                             const int64_t* heads, int64_t n_heads) {
    return guard([&] {
        const dfa2::AttentionDims dims = make_dims(H, d, nv, nt, order);
        const int64_t n = dims.seq_len();
        for (int64_t i = 0; i < n_heads; ++i) {
            const int64_t h = heads[i];
            const int64_t off = h * n * d;
            switch (kinds[h]) {
            case 0:
                dfa2::dense_tiled_attention(q + off, k + off, v + off, out + off, n, d, B, true);
                break;
            case 1:
                dfa2::sparse_attention_forward(
                    q + off, k + off, v + off, out + off, n, d,
                    dfa2::build_arrow_mask({dims, B, windows[h]}), true);
                break;
            default:
                std::memcpy(out + off, slots + off, sizeof(float) * n * d);
            }
        }
    });
}

// plan_to_json (src/plan.cpp:109-143) of a plan given as flat timestep-major
// arrays; *len receives the text size, buf (cap bytes) the NUL-terminated
// text when large enough.
REF_API int ref_plan_to_json(int64_t H, int64_t d, int64_t nv, int64_t nt, int64_t T, int64_t L,
                             int64_t B, double delta, double coeff, const int64_t* window_set,
                             int64_t n_ws, const int32_t* kinds, const int64_t* windows,
                             const char* digest, char* buf, int64_t cap, int64_t* len) {
    return guard([&] {
        dfa2::CompressionPlan p = dfa2::CompressionPlan::all_full(make_dims(H, d, nv, nt, 0), T, L, B);
        p.delta = delta;
        p.coeff = coeff;
        p.window_set.assign(window_set, window_set + n_ws);
        for (int64_t i = 0; i < T * L; ++i)
            p.layers[static_cast<size_t>(i)] = make_plan(H, kinds + i * H, windows + i * H);
        p.influence_digest = digest ? digest : "";
        const std::string s = dfa2::plan_to_json(p);
        *len = static_cast<int64_t>(s.size());
        if (buf && cap > *len)
            std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}

// plan_from_json (src/plan.cpp:145-209) -> status (PLAN on any schema or
// validation failure) and, on success, the flat kinds/windows arrays.
REF_API int ref_plan_from_json(const char* text, int64_t cap_entries, int32_t* kinds, int64_t* windows,
                               int64_t* n_entries) {
    return guard([&] {
        const dfa2::CompressionPlan p = dfa2::plan_from_json(text);
        const int64_t H = p.dims.n_heads;
        *n_entries = p.n_timesteps * p.n_layers * H;
        if (*n_entries > cap_entries)
            return;
        for (int64_t i = 0; i < p.n_timesteps * p.n_layers; ++i)
            for (int64_t h = 0; h < H; ++h) {
                const dfa2::HeadStrategy& s = p.layers[static_cast<size_t>(i)].strategies[static_cast<size_t>(h)];
                kinds[i * H + h] = static_cast<int32_t>(s.kind);
                windows[i * H + h] = s.window_blocks;
            }
    });
}

// solve / brute_force / lp_relaxation_bound (src/plansolver.cpp) of one
// selection problem; choice[H] gets -1 (Full) or a method index.
REF_API int ref_plan_solve(int64_t H, int64_t M, const double* infl, double full_cost,
                           const double* method_cost, double delta, double coeff, int brute,
                           int64_t* choice, double* objective, double* total_influence,
                           double* lp_bound) {
    return guard([&] {
        dfa2::PlanProblem p;
        p.n_heads = H;
        p.n_methods = M;
        p.influence.assign(infl, infl + H * M);
        p.costs.full_cost = full_cost;
        p.costs.method_cost.assign(method_cost, method_cost + M);
        p.delta = delta;
        p.coeff = coeff;
        const dfa2::PlanSolution s = brute ? dfa2::brute_force(p) : dfa2::solve(p);
        for (int64_t h = 0; h < H; ++h)
            choice[h] = s.choice[static_cast<size_t>(h)];
        *objective = s.objective;
        *total_influence = s.total_influence;
        if (lp_bound)
            *lp_bound = dfa2::lp_relaxation_bound(p);
    });
}
