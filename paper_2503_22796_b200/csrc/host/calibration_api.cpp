// calibration_api.cpp — the reference's calibration driver, plan-selection,
// workload and DFA2-dump API (include/dfa2/{plansolver,workload,io,
// calibrate}.hpp) on top of the C-ABI (include/dfa2c.h) and the
// multi_strategy_attention / influence_for_layer entry points of
// dfa2_api.cpp.
//
//   solve / brute_force / lp_relaxation_bound -> dfa2c_plan_solve / _lp_bound
//   analytic_costs                            -> dfa2c_analytic_costs
//   generate                                  -> host C++, bit-identical to
//       /root/reference/proj/src/workload.cpp:120-228 (per-(layer, head)
//       seeded mt19937_64 streams, run on one std::thread per stream)
//   run_pipeline                              -> t-major loop of fused launches
//   calibrate_model                           -> src/calibrate.cpp:255-348
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <istream>
#include <limits>
#include <map>
#include <ostream>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "dfa2/calibrate.hpp"
#include "dfa2/errors.hpp"
#include "dfa2/io.hpp"
#include "dfa2/plan.hpp"
#include "dfa2/plansolver.hpp"
#include "dfa2/workload.hpp"
#include "dfa2c.h"

#define DFA2_API __attribute__((visibility("default")))

namespace dfa2 {

void throw_status(int status);  // dfa2_api.cpp

namespace {

dfa2c_dims to_cdims(const AttentionDims& d) {
    return {d.n_heads, d.head_dim, d.n_visual, d.n_text,
            d.order == TokenOrder::visual_first ? DFA2C_VISUAL_FIRST : DFA2C_TEXT_FIRST};
}

int32_t kind_code(StrategyKind k) {
    return k == StrategyKind::full ? DFA2C_FULL : k == StrategyKind::arrow ? DFA2C_ARROW : DFA2C_CACHED;
}

// invalid problems surface as ShapeError (std::invalid_argument), as the
// reference's solver throws std::invalid_argument
PlanSolution run_solver(const PlanProblem& p, bool exhaustive) {
    if (static_cast<int64_t>(p.influence.size()) != p.n_heads * p.n_methods)
        throw ShapeError("influence grid does not match H x M");
    if (static_cast<int64_t>(p.costs.method_cost.size()) != p.n_methods)
        throw ShapeError("cost model does not match method count");
    PlanSolution s;
    s.choice.assign(static_cast<size_t>(std::max<int64_t>(p.n_heads, 1)), kFullChoice);
    throw_status(dfa2c_plan_solve(p.n_heads, p.n_methods, p.influence.data(), p.costs.full_cost,
                                  p.costs.method_cost.data(), p.delta, p.coeff, exhaustive ? 1 : 0, s.choice.data(),
                                  &s.objective, &s.total_influence, &s.nodes));
    s.choice.resize(static_cast<size_t>(p.n_heads));
    return s;
}

}  // namespace

// ---------------------------------------------------------------- plansolver
DFA2_API double selection_cap(double coeff, int64_t n_heads, double delta) {
    return dfa2c_selection_cap(coeff, n_heads, delta);
}

DFA2_API CostModel analytic_costs(const AttentionDims& dims, int64_t block_size,
                                  const std::vector<HeadStrategy>& methods) {
    dims.validate();
    std::vector<int32_t> kinds;
    std::vector<int64_t> wins;
    for (const HeadStrategy& s : methods) {
        kinds.push_back(kind_code(s.kind));
        wins.push_back(s.window_blocks);
    }
    CostModel cm;
    cm.method_cost.assign(methods.size(), 0.0);
    const dfa2c_dims cd = to_cdims(dims);
    throw_status(dfa2c_analytic_costs(&cd, block_size, kinds.data(), wins.data(),
                                      static_cast<int64_t>(methods.size()), &cm.full_cost, cm.method_cost.data()));
    return cm;
}

DFA2_API PlanSolution solve(const PlanProblem& problem) { return run_solver(problem, false); }
DFA2_API PlanSolution brute_force(const PlanProblem& problem) { return run_solver(problem, true); }

DFA2_API double lp_relaxation_bound(const PlanProblem& p) {
    if (static_cast<int64_t>(p.influence.size()) != p.n_heads * p.n_methods ||
        static_cast<int64_t>(p.costs.method_cost.size()) != p.n_methods)
        throw ShapeError("plan problem arrays do not match H x M");
    double b = 0.0;
    throw_status(dfa2c_plan_lp_bound(p.n_heads, p.n_methods, p.influence.data(), p.costs.full_cost,
                                     p.costs.method_cost.data(), p.delta, p.coeff, &b));
    return b;
}

DFA2_API LayerPlan to_layer_plan(const PlanSolution& solution, const std::vector<HeadStrategy>& methods) {
    LayerPlan plan;
    for (int64_t c : solution.choice)
        plan.strategies.push_back(c == kFullChoice ? HeadStrategy::Full() : methods.at(static_cast<size_t>(c)));
    return plan;
}

// ---------------------------------------------------------------- DFA2 dumps
namespace {
constexpr char kMagic[4] = {'D', 'F', 'A', '2'};
template <class T>
void put_le(std::ostream& out, T v) {
    unsigned char b[sizeof(T)];
    for (size_t i = 0; i < sizeof(T); ++i)
        b[i] = static_cast<unsigned char>((static_cast<uint64_t>(v) >> (8 * i)) & 0xFF);
    out.write(reinterpret_cast<const char*>(b), sizeof(T));
}
template <class T>
T get_le(std::istream& in) {
    unsigned char b[sizeof(T)];
    if (!in.read(reinterpret_cast<char*>(b), sizeof(T)))
        throw IoError("truncated DFA2 header");
    uint64_t v = 0;
    for (size_t i = 0; i < sizeof(T); ++i)
        v |= static_cast<uint64_t>(b[i]) << (8 * i);
    return static_cast<T>(v);
}
}  // namespace

DFA2_API void write_dfa2(std::ostream& out, const Tensor& t) {
    out.write(kMagic, 4);
    put_le<uint32_t>(out, 1u);
    put_le<uint32_t>(out, t.dtype() == Dtype::f32 ? 0u : 1u);
    put_le<uint32_t>(out, static_cast<uint32_t>(t.ndim()));
    for (int64_t dim : t.shape())
        put_le<uint64_t>(out, static_cast<uint64_t>(dim));
    // payload: little-endian scalars (the host is little-endian x86_64/aarch64)
    if (t.dtype() == Dtype::f32)
        out.write(reinterpret_cast<const char*>(t.f32()), static_cast<std::streamsize>(t.numel() * 4));
    else
        out.write(reinterpret_cast<const char*>(t.f64()), static_cast<std::streamsize>(t.numel() * 8));
    if (!out)
        throw IoError("failed writing DFA2 tensor");
}

DFA2_API Tensor read_dfa2(std::istream& in) {
    char magic[4];
    if (!in.read(magic, 4) || std::memcmp(magic, kMagic, 4) != 0)
        throw IoError("bad DFA2 magic");
    if (get_le<uint32_t>(in) != 1u)
        throw IoError("unsupported DFA2 version");
    const uint32_t dtype = get_le<uint32_t>(in);
    if (dtype > 1u)
        throw IoError("unknown DFA2 dtype");
    const uint32_t ndim = get_le<uint32_t>(in);
    if (ndim > 16)
        throw IoError("implausible DFA2 rank");
    std::vector<int64_t> shape;
    int64_t numel = 1;
    for (uint32_t i = 0; i < ndim; ++i) {
        const uint64_t d = get_le<uint64_t>(in);
        if (d > (uint64_t{1} << 40))
            throw IoError("implausible DFA2 dimension");
        shape.push_back(static_cast<int64_t>(d));
        numel *= static_cast<int64_t>(d);
    }
    Tensor t = Tensor::zeros(shape, dtype == 0 ? Dtype::f32 : Dtype::f64);
    const std::streamsize bytes = static_cast<std::streamsize>(numel * (dtype == 0 ? 4 : 8));
    char* dst = dtype == 0 ? reinterpret_cast<char*>(t.f32()) : reinterpret_cast<char*>(t.f64());
    if (bytes > 0 && !in.read(dst, bytes))
        throw IoError("truncated DFA2 payload");
    return t;
}

DFA2_API void save_dfa2(const Tensor& tensor, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out)
        throw IoError("cannot open " + path + " for writing");
    write_dfa2(out, tensor);
}

DFA2_API Tensor load_dfa2(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in)
        throw IoError("cannot open " + path);
    return read_dfa2(in);
}

// ---------------------------------------------------------------- workload
namespace {

constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
// signal scales of the reference generator (src/workload.cpp:67-72)
constexpr double kPosGain = 6.0, kVisNoise = 0.3, kTextGain = 3.0;

uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// independent stream per (seed, layer, head, timestep, tag)
uint64_t stream_seed(uint64_t base, uint64_t l, uint64_t h, uint64_t t, uint64_t tag) {
    uint64_t s = mix64(base ^ 0x9e3779b97f4a7c15ull);
    s = mix64(s ^ (l * 0xff51afd7ed558ccdull));
    s = mix64(s ^ (h * 0xc4ceb9fe1a85ec53ull));
    s = mix64(s ^ (t * 0xd6e8feb86659fd93ull));
    return mix64(s ^ tag);
}

// mt19937_64 uniforms on [0, 1) with 53 bits, Box-Muller pairs (cosine
// first, the sine kept for the next draw)
class Gauss {
public:
    explicit Gauss(uint64_t seed) : eng_(seed) {}
    double uniform() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    double next() {
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        double u1;
        do
            u1 = uniform();
        while (u1 <= 0.0);
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        spare_ = r * std::sin(kTwoPi * u2);
        spare_ok_ = true;
        return r * std::cos(kTwoPi * u2);
    }

private:
    std::mt19937_64 eng_;
    bool spare_ok_ = false;
    double spare_ = 0.0;
};

}  // namespace

DFA2_API std::vector<HeadProfile> default_profiles(const AttentionDims& dims, int64_t n_layers, int64_t block_size) {
    const double b = static_cast<double>(block_size);
    const double inf = std::numeric_limits<double>::infinity();
    const double locality[6] = {b / 2, b, 2 * b, 4 * b, 8 * b, inf};
    const double drift[7] = {0.01, 0.02, 0.04, 0.07, 0.11, 0.16, 0.22};
    std::vector<HeadProfile> out;
    for (int64_t l = 0; l < n_layers; ++l)
        for (int64_t h = 0; h < dims.n_heads; ++h) {
            HeadProfile p;
            p.locality = h == 0 ? inf : h == 1 ? b / 4 : locality[(h - 2 + l) % 6];
            p.drift = h == dims.n_heads - 1 ? 0.0 : drift[(h + l) % 7];  // last head frozen
            out.push_back(p);
        }
    return out;
}

DFA2_API Workload::Workload(WorkloadConfig config, std::vector<Tensor> q, std::vector<Tensor> k,
                            std::vector<Tensor> v)
    : config_(std::move(config)), q_(std::move(q)), k_(std::move(k)), v_(std::move(v)) {}

DFA2_API const HeadProfile& Workload::profile(int64_t layer, int64_t head) const {
    return config_.profiles.at(static_cast<size_t>(layer * config_.dims.n_heads + head));
}

DFA2_API size_t Workload::index(int64_t t, int64_t layer) const {
    if (t < 0 || t >= config_.n_timesteps || layer < 0 || layer >= config_.n_layers)
        throw ShapeError("timestep or layer out of range");
    return static_cast<size_t>(t * config_.n_layers + layer);
}

DFA2_API Workload generate(const WorkloadConfig& config) {
    WorkloadConfig cfg = config;
    cfg.dims.validate();
    if (cfg.n_layers < 1 || cfg.n_timesteps < 1 || cfg.block_size < 1)
        throw ShapeError("need n_layers >= 1, n_timesteps >= 1, block >= 1");
    if (cfg.profiles.empty())
        cfg.profiles = default_profiles(cfg.dims, cfg.n_layers, cfg.block_size);
    if (static_cast<int64_t>(cfg.profiles.size()) != cfg.n_layers * cfg.dims.n_heads)
        throw ShapeError("profiles must cover every (layer, head)");
    const int64_t d = cfg.dims.head_dim, n = cfg.dims.seq_len(), H = cfg.dims.n_heads;
    const int64_t L = cfg.n_layers, T = cfg.n_timesteps;
    const int64_t tlo = cfg.dims.text_begin(), thi = cfg.dims.text_end();
    std::vector<Tensor> qs, ks, vs;
    for (int64_t i = 0; i < T * L; ++i) {
        qs.push_back(Tensor::zeros({H, n, d}));
        ks.push_back(Tensor::zeros({H, n, d}));
        vs.push_back(Tensor::zeros({H, n, d}));
    }
    // one (layer, head) stream: t = 0 from positional features + noise, then
    // a seeded random walk per timestep (drift 0 copies bit for bit)
    auto one_stream = [&](int64_t l, int64_t h) {
        const HeadProfile& prof = cfg.profiles[static_cast<size_t>(l * H + h)];
        const double feat = std::sqrt(2.0 / static_cast<double>(d));
        std::vector<double> omega(static_cast<size_t>(d)), phase(static_cast<size_t>(d));
        Gauss pos(stream_seed(cfg.seed, l, h, 0, 1));
        for (int64_t f = 0; f < d; ++f) {
            omega[f] = std::isinf(prof.locality) ? 0.0 : pos.next() / prof.locality;
            phase[f] = pos.uniform() * kTwoPi;
        }
        Gauss gq(stream_seed(cfg.seed, l, h, 0, 2)), gk(stream_seed(cfg.seed, l, h, 0, 3)),
            gv(stream_seed(cfg.seed, l, h, 0, 4));
        const size_t off = static_cast<size_t>(h * n * d);
        float* q0 = qs[static_cast<size_t>(l)].f32() + off;
        float* k0 = ks[static_cast<size_t>(l)].f32() + off;
        float* v0 = vs[static_cast<size_t>(l)].f32() + off;
        const double text_scale = kTextGain / std::sqrt(static_cast<double>(d));
        for (int64_t i = 0; i < n; ++i) {
            const bool text = i >= tlo && i < thi;
            for (int64_t f = 0; f < d; ++f) {
                double qv, kv;
                if (text) {
                    qv = text_scale * gq.next();
                    kv = text_scale * gk.next();
                } else {
                    const double u = feat * std::cos(omega[f] * static_cast<double>(i) + phase[f]);
                    qv = kPosGain * u + kVisNoise * gq.next();
                    kv = kPosGain * u + kVisNoise * gk.next();
                }
                q0[i * d + f] = static_cast<float>(qv);
                k0[i * d + f] = static_cast<float>(kv);
                v0[i * d + f] = static_cast<float>(gv.next());
            }
        }
        for (int64_t t = 1; t < T; ++t) {
            const size_t pi = static_cast<size_t>((t - 1) * L + l), ci = static_cast<size_t>(t * L + l);
            const float* src[3] = {qs[pi].f32() + off, ks[pi].f32() + off, vs[pi].f32() + off};
            float* dst[3] = {qs[ci].f32() + off, ks[ci].f32() + off, vs[ci].f32() + off};
            if (prof.drift == 0.0) {
                for (int j = 0; j < 3; ++j)
                    std::copy(src[j], src[j] + n * d, dst[j]);
                continue;
            }
            Gauss walk(stream_seed(cfg.seed, l, h, t, 5));
            for (int j = 0; j < 3; ++j)
                for (int64_t i = 0; i < n * d; ++i)
                    dst[j][i] = src[j][i] + static_cast<float>(prof.drift * walk.next());
        }
    };
    // streams are independent and write disjoint memory: one thread each
    // (bounded by the host's cores), same bits as a serial run
    const int64_t streams = L * H;
    const int64_t workers = std::max<int64_t>(1, std::min<int64_t>(streams, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int64_t w = 0; w < workers; ++w)
        pool.emplace_back([&, w] {
            for (int64_t s = w; s < streams; s += workers)
                one_stream(s / H, s % H);
        });
    for (std::thread& th : pool)
        th.join();
    return Workload(std::move(cfg), std::move(qs), std::move(ks), std::move(vs));
}

DFA2_API RunStats run_pipeline(const Workload& workload, const CompressionPlan& plan) {
    plan.validate();
    const WorkloadConfig& cfg = workload.config();
    if (plan.dims.n_heads != cfg.dims.n_heads || plan.dims.head_dim != cfg.dims.head_dim ||
        plan.dims.n_visual != cfg.dims.n_visual || plan.dims.n_text != cfg.dims.n_text ||
        plan.n_timesteps != cfg.n_timesteps || plan.n_layers != cfg.n_layers || plan.block_size != cfg.block_size)
        throw PlanValidationError("plan dims do not match the workload");
    const auto t0 = std::chrono::steady_clock::now();
    RunStats st;
    HeadCache cache;
    const int64_t dense = cfg.dims.n_heads * 4 * cfg.dims.head_dim * cfg.dims.seq_len() * cfg.dims.seq_len();
    for (int64_t t = 0; t < cfg.n_timesteps; ++t)
        for (int64_t l = 0; l < cfg.n_layers; ++l) {
            const LayerPlan& lp = plan.at(t, l);
            st.outputs.push_back(multi_strategy_attention(workload.q(t, l), workload.k(t, l), workload.v(t, l), lp,
                                                          cache, l, t, cfg.dims, cfg.block_size));
            st.flops_total += plan_flops(lp, cfg.dims, cfg.block_size);
            st.flops_dense += dense;
        }
    st.sparsity = 1.0 - static_cast<double>(st.flops_total) / static_cast<double>(st.flops_dense);
    st.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return st;
}

// ---------------------------------------------------------------- influence table
DFA2_API InfluenceTable::InfluenceTable(int64_t t, int64_t layers, int64_t heads, std::vector<std::string> ids)
    : t_(t), layers_(layers), heads_(heads), method_ids_(std::move(ids)) {
    values_.assign(static_cast<size_t>(t_ * layers_ * heads_ * n_methods()), std::nan(""));
}

DFA2_API size_t InfluenceTable::index(int64_t t, int64_t layer, int64_t head, int64_t m) const {
    if (t < 0 || t >= t_ || layer < 0 || layer >= layers_ || head < 0 || head >= heads_ || m < 0 || m >= n_methods())
        throw ShapeError("influence index out of range");
    return static_cast<size_t>(((t * layers_ + layer) * heads_ + head) * n_methods() + m);
}

DFA2_API double InfluenceTable::get(int64_t t, int64_t layer, int64_t head, int64_t m) const {
    return values_[index(t, layer, head, m)];
}
DFA2_API void InfluenceTable::set(int64_t t, int64_t layer, int64_t head, int64_t m, double v) {
    values_[index(t, layer, head, m)] = v;
}
DFA2_API bool InfluenceTable::measured(int64_t t, int64_t layer, int64_t head, int64_t m) const {
    return !std::isnan(values_[index(t, layer, head, m)]);
}

DFA2_API void InfluenceTable::write_csv(std::ostream& out) const {
    out << "t,layer,head,method,influence\n";
    char num[40];
    for (int64_t t = 0; t < t_; ++t)
        for (int64_t l = 0; l < layers_; ++l)
            for (int64_t h = 0; h < heads_; ++h)
                for (int64_t m = 0; m < n_methods(); ++m) {
                    const double v = get(t, l, h, m);
                    if (std::isnan(v))
                        continue;
                    std::snprintf(num, sizeof num, "%.17g", v);  // round-trips exactly
                    out << t << ',' << l << ',' << h << ',' << method_ids_[static_cast<size_t>(m)] << ',' << num
                        << '\n';
                }
}

DFA2_API std::string InfluenceTable::to_csv() const {
    std::ostringstream ss;
    write_csv(ss);
    return ss.str();
}

DFA2_API InfluenceTable parse_influence_csv(std::istream& in, int64_t t, int64_t layers, int64_t heads,
                                            const std::vector<std::string>& method_ids) {
    InfluenceTable table(t, layers, heads, method_ids);
    std::map<std::string, int64_t> col;
    for (size_t m = 0; m < method_ids.size(); ++m)
        col[method_ids[m]] = static_cast<int64_t>(m);
    std::string line;
    if (!std::getline(in, line) || line != "t,layer,head,method,influence")
        throw IoError("influence CSV header mismatch");
    while (std::getline(in, line)) {
        if (line.empty())
            continue;
        std::vector<std::string> f;
        std::stringstream ls(line);
        std::string tok;
        while (std::getline(ls, tok, ','))
            f.push_back(tok);
        if (f.size() != 5)
            throw IoError("malformed influence CSV row: " + line);
        const auto it = col.find(f[3]);
        if (it == col.end())
            throw IoError("unknown method id in influence CSV: " + f[3]);
        try {
            table.set(std::stoll(f[0]), std::stoll(f[1]), std::stoll(f[2]), it->second, std::stod(f[4]));
        } catch (const std::logic_error&) {
            throw IoError("malformed influence CSV row: " + line);
        }
    }
    return table;
}

// ---------------------------------------------------------------- calibration
DFA2_API CalibrationResult calibrate_model(const Workload& workload, const CalibrationConfig& config) {
    if (config.methods.empty())
        throw ShapeError("candidate set must be nonempty");
    if (!(config.delta >= 0.0))
        throw ShapeError("delta must be >= 0");
    if (!(config.coeff >= 1.0))
        throw ShapeError("coeff must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    const WorkloadConfig& cfg = workload.config();
    const int64_t T = cfg.n_timesteps, L = cfg.n_layers, H = cfg.dims.n_heads;
    const int64_t M = static_cast<int64_t>(config.methods.size());
    std::vector<HeadStrategy> strategies;
    std::vector<std::string> ids;
    std::vector<int64_t> windows;
    for (const MethodCandidate& c : config.methods) {
        strategies.push_back(c.strategy);
        ids.push_back(c.id);
        if (c.strategy.kind == StrategyKind::arrow)
            windows.push_back(c.strategy.window_blocks);
    }
    const CostModel costs = analytic_costs(cfg.dims, cfg.block_size, strategies);

    CalibrationResult r;
    r.plan.dims = cfg.dims;
    r.plan.n_timesteps = T;
    r.plan.n_layers = L;
    r.plan.block_size = cfg.block_size;
    r.plan.delta = config.delta;
    r.plan.coeff = config.coeff;
    r.plan.window_set = windows;
    r.plan.layers.assign(static_cast<size_t>(T * L), LayerPlan{});
    r.influences = InfluenceTable(T, L, H, ids);
    r.stats.budget_spent.assign(static_cast<size_t>(T * L), 0.0);
    r.stats.objective.assign(static_cast<size_t>(T * L), 0.0);

    HeadCache cache;
    for (int64_t t = 0; t < T; ++t)
        for (int64_t l = 0; l < L; ++l) {
            const LayerInfluence li = influence_for_layer(workload.q(t, l), workload.k(t, l), workload.v(t, l),
                                                          config.methods, cache, l, t, cfg.dims, cfg.block_size,
                                                          config.rse_mode, &r.stats);
            for (int64_t h = 0; h < H; ++h)
                for (int64_t m = 0; m < M; ++m) {
                    const double v = li.influence[static_cast<size_t>(h * M + m)];
                    if (std::isfinite(v))
                        r.influences.set(t, l, h, m, v);
                }
            PlanProblem prob;
            prob.n_heads = H;
            prob.n_methods = M;
            prob.influence = li.influence;
            prob.costs = costs;
            prob.delta = config.delta;
            prob.coeff = config.coeff;
            const PlanSolution sol = solve(prob);
            const size_t slot = static_cast<size_t>(t * L + l);
            r.stats.budget_spent[slot] = sol.total_influence;
            r.stats.objective[slot] = sol.objective;
            r.plan.layers[slot] = to_layer_plan(sol, strategies);
            // splice: computed heads commit the output of their chosen
            // measurement pass (no extra attention evaluation); Cached heads
            // keep their slot
            for (int64_t h = 0; h < H; ++h) {
                const int64_t c = sol.choice[static_cast<size_t>(h)];
                if (c == kFullChoice)
                    cache.store(l, h, head_slice(li.original, h), t);
                else if (strategies[static_cast<size_t>(c)].kind == StrategyKind::arrow)
                    cache.store(l, h, head_slice(li.method_outputs[static_cast<size_t>(c)], h), t);
            }
        }
    r.stats.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return r;
}

DFA2_API int64_t audit_plan_constraints(const CompressionPlan& plan, const InfluenceTable& influences) {
    plan.validate();
    std::map<std::string, int64_t> col;
    for (size_t m = 0; m < influences.method_ids().size(); ++m)
        col[influences.method_ids()[m]] = static_cast<int64_t>(m);
    const double cap = selection_cap(plan.coeff, plan.dims.n_heads, plan.delta);
    int64_t bad = 0;
    for (int64_t t = 0; t < plan.n_timesteps; ++t)
        for (int64_t l = 0; l < plan.n_layers; ++l) {
            double spent = 0.0;
            for (int64_t h = 0; h < plan.dims.n_heads; ++h) {
                const HeadStrategy& s = plan.at(t, l).strategies[static_cast<size_t>(h)];
                if (s.kind == StrategyKind::full)
                    continue;
                const auto it = col.find(method_id(s));
                if (it == col.end() || !influences.measured(t, l, h, it->second)) {
                    ++bad;  // a selection without a measured influence
                    continue;
                }
                const double v = influences.get(t, l, h, it->second);
                spent += v;
                if (v > cap)
                    ++bad;
            }
            if (spent > plan.delta)
                ++bad;
        }
    return bad;
}

}  // namespace dfa2
