// dfa2 — command-line front end of the B200 path with the reference CLI's
// subcommands, flags, outputs and exit codes (/root/reference/proj/tools/
// dfa2_main.cpp:28-613): calibrate | run | verify | bench | workload.
// Exit codes: 0 success, 2 validation error, 3 oracle failure.
//
// Everything runs through the drop-in C++ API (include/dfa2/*.hpp) over
// libdfa2_b200.so, i.e. on the sm_100a kernels. The only host arithmetic on
// attention values is the f64 checker of `verify`, which is what that
// subcommand is for.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "dfa2/bench.hpp"
#include "dfa2/calibrate.hpp"
#include "dfa2/io.hpp"
#include "dfa2/plan.hpp"
#include "dfa2/plansolver.hpp"
#include "dfa2/workload.hpp"
#include "json_lite.h"

namespace {

constexpr int kExitOk = 0, kExitValidation = 2, kExitOracle = 3;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------ flag parsing
// --name value / --name=value options and --name switches; unknown flags
// and missing values are usage errors (exit 2). Repeated options: last wins.
class Flags {
public:
    Flags(int argc, char** argv, int first, std::map<std::string, std::string> defaults,
          std::vector<std::string> switches)
        : values_(std::move(defaults)) {
        for (const std::string& s : switches)
            switches_[s] = false;
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0)
                throw UsageError("unexpected argument '" + a + "'");
            std::string name = a.substr(2), value;
            const size_t eq = name.find('=');
            const bool inline_value = eq != std::string::npos;
            if (inline_value) {
                value = name.substr(eq + 1);
                name = name.substr(0, eq);
            }
            if (switches_.count(name)) {
                if (inline_value)
                    throw UsageError("--" + name + " takes no value");
                switches_[name] = true;
                continue;
            }
            if (!values_.count(name))
                throw UsageError("unknown flag --" + name);
            if (!inline_value) {
                if (i + 1 >= argc)
                    throw UsageError("--" + name + " needs a value");
                value = argv[++i];
            }
            values_[name] = value;
            given_[name] = true;
        }
    }
    std::string str(const std::string& n) const { return values_.at(n); }
    bool given(const std::string& n) const { return given_.count(n) != 0; }
    bool on(const std::string& n) const { return switches_.at(n); }
    int64_t i64(const std::string& n) const {
        try {
            size_t used = 0;
            const long long v = std::stoll(values_.at(n), &used);
            if (used != values_.at(n).size())
                throw std::invalid_argument("trailing");
            return v;
        } catch (const std::exception&) {
            throw UsageError("--" + n + " expects an integer");
        }
    }
    double f64(const std::string& n) const {
        try {
            size_t used = 0;
            const double v = std::stod(values_.at(n), &used);
            if (used != values_.at(n).size())
                throw std::invalid_argument("trailing");
            return v;
        } catch (const std::exception&) {
            throw UsageError("--" + n + " expects a number");
        }
    }

private:
    std::map<std::string, std::string> values_;
    std::map<std::string, bool> switches_, given_;
};

std::map<std::string, std::string> workload_defaults() {
    return {{"timesteps", "8"}, {"layers", "4"},  {"heads", "8"},  {"head-dim", "32"},
            {"visual-tokens", "256"}, {"text-tokens", "32"}, {"block", "32"}, {"seed", "1234"},
            {"token-order", "visual-first"}};
}

dfa2::WorkloadConfig workload_config(const Flags& f) {
    dfa2::WorkloadConfig cfg;
    cfg.dims.n_heads = f.i64("heads");
    cfg.dims.head_dim = f.i64("head-dim");
    cfg.dims.n_visual = f.i64("visual-tokens");
    cfg.dims.n_text = f.i64("text-tokens");
    const std::string order = f.str("token-order");
    if (order == "visual-first")
        cfg.dims.order = dfa2::TokenOrder::visual_first;
    else if (order == "text-first")
        cfg.dims.order = dfa2::TokenOrder::text_first;
    else
        throw dfa2::ShapeError("token order must be visual-first or text-first");
    cfg.n_layers = f.i64("layers");
    cfg.n_timesteps = f.i64("timesteps");
    cfg.block_size = f.i64("block");
    cfg.seed = static_cast<uint64_t>(f.i64("seed"));
    return cfg;
}

template <class T>
std::vector<T> parse_list(const std::string& text) {
    std::vector<T> out;
    std::stringstream ss(text);
    std::string tok;
    while (std::getline(ss, tok, ','))
        if (!tok.empty()) {
            try {
                out.push_back(static_cast<T>(std::is_integral_v<T> ? std::stoll(tok) : std::stod(tok)));
            } catch (const std::exception&) {
                throw UsageError("bad list element '" + tok + "'");
            }
        }
    return out;
}

void write_text(const std::string& path, const std::string& text) {
    std::ofstream out(path, std::ios::binary);
    if (!out)
        throw dfa2::IoError("cannot open " + path + " for writing");
    out << text;
    if (!out)
        throw dfa2::IoError("failed writing " + path);
}

// ---------------------------------------------------------------- calibrate
int cmd_calibrate(const Flags& f) {
    const std::string out_path = f.str("out");
    std::string csv_path = f.str("influence-csv");
    if (csv_path.empty())
        csv_path = out_path + ".influence.csv";
    const dfa2::Workload workload = dfa2::generate(workload_config(f));
    dfa2::CalibrationConfig cc;
    cc.methods = dfa2::make_candidates(parse_list<int64_t>(f.str("windows")), !f.on("no-cache-method"));
    cc.delta = f.f64("delta");
    cc.coeff = f.f64("coeff");
    cc.rse_mode = f.on("rse-literal") ? dfa2::RseMode::literal : dfa2::RseMode::standard;
    dfa2::CalibrationResult r = dfa2::calibrate_model(workload, cc);
    const std::string csv = r.influences.to_csv();
    write_text(csv_path, csv);
    r.plan.influence_digest = dfa2::fnv1a_hex(csv);
    dfa2::save_plan(r.plan, out_path);
    std::printf("plan:               %s\n", out_path.c_str());
    std::printf("influence csv:      %s\n", csv_path.c_str());
    std::printf("aggregate sparsity: %.6f\n", r.plan.aggregate_sparsity());
    std::printf("attention evals:    %lld\n", static_cast<long long>(r.stats.attention_evals));
    std::printf("wall time:          %.3f s\n", r.stats.wall_seconds);
    return kExitOk;
}

// --------------------------------------------------------------------- run
int cmd_run(const Flags& f) {
    if (!f.given("plan"))
        throw UsageError("--plan is required");
    const dfa2::CompressionPlan plan = dfa2::load_plan(f.str("plan"));
    const dfa2::WorkloadConfig cfg = workload_config(f);
    if (plan.dims.n_heads != cfg.dims.n_heads || plan.dims.head_dim != cfg.dims.head_dim ||
        plan.dims.n_visual != cfg.dims.n_visual || plan.dims.n_text != cfg.dims.n_text ||
        plan.n_timesteps != cfg.n_timesteps || plan.n_layers != cfg.n_layers || plan.block_size != cfg.block_size)
        throw dfa2::PlanValidationError("plan dims do not match workload flags");
    plan.validate();  // before any work: a tampered plan never starts a run
    const dfa2::Workload workload = dfa2::generate(cfg);
    const dfa2::RunStats run = dfa2::run_pipeline(workload, plan);
    const dfa2::RunStats base = dfa2::run_pipeline(
        workload, dfa2::CompressionPlan::all_full(cfg.dims, cfg.n_timesteps, cfg.n_layers, cfg.block_size));
    double mean = 0.0, worst = 0.0;
    for (size_t i = 0; i < run.outputs.size(); ++i) {
        const double r = run.outputs[i] == base.outputs[i] ? 0.0 : dfa2::rse(run.outputs[i], base.outputs[i]);
        mean += r;
        worst = std::max(worst, r);
    }
    mean /= static_cast<double>(run.outputs.size());
    if (!f.str("report").empty()) {
        json_lite::Value rep = json_lite::Value::object();
        rep.set("sparsity", json_lite::Value::real(run.sparsity));
        rep.set("flops_reduction", json_lite::Value::real(run.sparsity));
        rep.set("mean_layer_rse", json_lite::Value::real(mean));
        rep.set("max_layer_rse", json_lite::Value::real(worst));
        rep.set("wall_time", json_lite::Value::real(run.wall_seconds));
        write_text(f.str("report"), rep.dump(2) + "\n");
    }
    std::printf("sparsity:        %.6f\n", run.sparsity);
    std::printf("flops reduction: %.6f\n", run.sparsity);
    std::printf("mean layer rse:  %.6g\n", mean);
    std::printf("max layer rse:   %.6g\n", worst);
    std::printf("wall time:       %.3f s\n", run.wall_seconds);
    return kExitOk;
}

// ------------------------------------------------------------------ verify
// f64 two-pass masked attention of one [n, d] head (the checker).
std::vector<double> masked_attention_f64(const dfa2::Tensor& q, const dfa2::Tensor& k, const dfa2::Tensor& v,
                                         const dfa2::BlockMask& m) {
    const int64_t n = q.dim(0), d = q.dim(1);
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    std::vector<double> out(static_cast<size_t>(n * d), 0.0), w(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        double mx = -INFINITY;
        for (int64_t j = 0; j < n; ++j) {
            if (!m.is_active(i / m.block_size, j / m.block_size)) {
                w[j] = -INFINITY;
                continue;
            }
            double s = 0.0;
            for (int64_t c = 0; c < d; ++c)
                s += static_cast<double>(q.f32()[i * d + c]) * static_cast<double>(k.f32()[j * d + c]);
            w[j] = s * scale;
            mx = std::max(mx, w[j]);
        }
        double den = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            w[j] = std::isinf(w[j]) ? 0.0 : std::exp(w[j] - mx);
            den += w[j];
        }
        for (int64_t j = 0; j < n; ++j)
            if (w[j] != 0.0)
                for (int64_t c = 0; c < d; ++c)
                    out[i * d + c] += w[j] / den * static_cast<double>(v.f32()[j * d + c]);
    }
    return out;
}

// the reference's self-test fault: the visual band shifted one block right
dfa2::BlockMask corrupt_mask_off_by_one(const dfa2::BlockMask& mask, const dfa2::AttentionDims& dims) {
    dfa2::BlockMask bad = mask;
    auto text_block = [&](int64_t i) {
        const int64_t lo = i * mask.block_size, hi = std::min(lo + mask.block_size, mask.seq_len);
        return lo < dims.text_end() && hi > dims.text_begin();
    };
    for (int64_t i = 0; i < mask.n_query_blocks; ++i)
        for (int64_t j = 0; j < mask.n_key_blocks; ++j)
            if (!text_block(i) && !text_block(j))
                bad.set(i, j, j > 0 ? mask.is_active(i, j - 1) : false);
    return bad;
}

struct Section {
    std::string name;
    bool pass = true;
    int64_t checks = 0;
    std::string detail;
};

int cmd_verify(const Flags& f) {
    const std::vector<int64_t> sizes = parse_list<int64_t>(f.str("sizes"));
    const std::string fault = f.str("fault");
    if (fault != "none" && fault != "mask-off-by-one")
        throw UsageError("--fault must be none or mask-off-by-one");
    std::mt19937_64 eng(static_cast<uint64_t>(f.i64("seed")));
    auto uniform = [&] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
    auto gaussian = [&] {
        double u1;
        do
            u1 = uniform();
        while (u1 <= 0.0);
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * uniform());
    };
    auto head = [&](int64_t n, int64_t d) {
        dfa2::Tensor t = dfa2::Tensor::zeros({n, d});
        for (int64_t i = 0; i < n * d; ++i)  // bf16-representable, so the checker sees the kernel's inputs
            t.f32()[i] = static_cast<float>(std::ldexp(std::round(std::ldexp(gaussian(), 6)), -6));
        return t;
    };
    std::vector<Section> sections;

    // 1. masked-dense oracle: the sm_100a sparse pass vs the f64 checker
    //    (stated bf16 tolerance: max |err| / max |ref| <= 1e-2)
    {
        Section s{"masked-dense-oracle"};
        double worst = 0.0;
        for (int64_t n : sizes)
            for (int64_t b : {int64_t{16}, int64_t{32}}) {
                dfa2::AttentionDims dims;
                dims.n_heads = 1;
                dims.head_dim = 16;
                dims.n_text = std::max<int64_t>(1, n / 5);
                dims.n_visual = n - dims.n_text;
                if (dims.n_visual < 1)
                    continue;
                const int64_t max_w = (dims.n_visual + b - 1) / b - 1;
                for (int64_t w : {int64_t{0}, int64_t{1}, max_w}) {
                    const dfa2::BlockMask mask = dfa2::build_arrow_mask({dims, b, w});
                    const dfa2::BlockMask used = fault == "mask-off-by-one" ? corrupt_mask_off_by_one(mask, dims) : mask;
                    const dfa2::Tensor q = head(n, 16), k = head(n, 16), v = head(n, 16);
                    const dfa2::Tensor got = dfa2::sparse_attention_forward(q, k, v, used);
                    const std::vector<double> want = masked_attention_f64(q, k, v, mask);
                    double err = 0.0, ref = 0.0;
                    for (size_t i = 0; i < want.size(); ++i) {
                        err = std::max(err, std::fabs(got.f32()[i] - want[i]));
                        ref = std::max(ref, std::fabs(want[i]));
                    }
                    worst = std::max(worst, err / (ref + 1e-300));
                    ++s.checks;
                    if (err / (ref + 1e-300) > 1e-2)
                        s.pass = false;
                }
            }
        char buf[64];
        std::snprintf(buf, sizeof buf, "max rel err %.3g", worst);
        s.detail = buf;
        sections.push_back(s);
    }
    // 2. exact solver vs exhaustive enumeration
    {
        Section s{"solver-brute-force"};
        const double deltas[] = {0.0, 0.2, 0.6, 1.0}, coeffs[] = {1.0, 1.5, 2.0};
        for (int inst = 0; inst < 200; ++inst) {
            dfa2::PlanProblem p;
            p.n_heads = 2 + static_cast<int64_t>(eng() % 7);
            p.n_methods = 1 + static_cast<int64_t>(eng() % 3);
            p.delta = deltas[eng() % 4];
            p.coeff = coeffs[eng() % 3];
            for (int64_t m = 0; m < p.n_methods; ++m)
                p.costs.method_cost.push_back(uniform());
            for (int64_t i = 0; i < p.n_heads * p.n_methods; ++i)
                p.influence.push_back(uniform());
            const dfa2::PlanSolution a = dfa2::solve(p), b = dfa2::brute_force(p);
            ++s.checks;
            if (a.objective != b.objective || a.choice != b.choice) {
                s.pass = false;
                s.detail = "instance " + std::to_string(inst) + " diverged";
                break;
            }
        }
        sections.push_back(s);
    }
    // 3. streaming-softmax parity: the tile loop folds the same key tiles in
    //    the same order whatever the mask, so Arrow(max window) and Full
    //    agree bit for bit
    {
        Section s{"streaming-softmax-parity"};
        for (int64_t n : sizes) {
            dfa2::AttentionDims dims;
            dims.n_heads = 1;
            dims.head_dim = 16;
            dims.n_text = std::max<int64_t>(1, n / 6);
            dims.n_visual = n - dims.n_text;
            if (dims.n_visual < 1)
                continue;
            const dfa2::Tensor q = head(n, 16), k = head(n, 16), v = head(n, 16);
            const dfa2::Tensor dense = dfa2::sparse_attention_forward(q, k, v, dfa2::BlockMask::all_active(n, 16));
            const dfa2::Tensor arrow = dfa2::sparse_attention_forward(q, k, v, dfa2::build_arrow_mask({dims, 16, 1 << 20}));
            ++s.checks;
            if (!(dense == arrow))
                s.pass = false;
        }
        sections.push_back(s);
    }
    // 4. cache semantics
    {
        Section s{"cache-semantics"};
        dfa2::HeadCache cache;
        dfa2::Tensor a = dfa2::Tensor::zeros({4, 2});
        for (int64_t i = 0; i < 8; ++i)
            a.f32()[i] = static_cast<float>(gaussian());
        bool ok = true;
        try {
            cache.fetch(0, 0);
            ok = false;
        } catch (const dfa2::CacheMissError&) {
        }
        cache.store(0, 0, a, 3);
        ok = ok && cache.fetch(0, 0) == a && cache.staleness(0, 0, 5) == 2;
        dfa2::Tensor b = a;
        b.f32()[0] += 1.0f;
        cache.store(0, 1, b, 4);
        ok = ok && cache.fetch(0, 0) == a && cache.fetch(0, 1) == b;
        cache.store(0, 0, b, 6);
        ok = ok && cache.fetch(0, 0) == b && cache.produced_at(0, 0) == 6;
        s.checks = 5;
        s.pass = ok;
        sections.push_back(s);
    }
    bool all = true;
    for (const Section& s : sections) {
        std::printf("%-28s %s  (%lld checks%s%s)\n", s.name.c_str(), s.pass ? "PASS" : "FAIL",
                    static_cast<long long>(s.checks), s.detail.empty() ? "" : ", ", s.detail.c_str());
        all = all && s.pass;
    }
    return all ? kExitOk : kExitOracle;
}

// ------------------------------------------------------------------- bench
int cmd_bench(const Flags& f) {
    dfa2::BenchConfig cfg;
    cfg.n_visual = f.i64("visual-tokens");
    cfg.n_text = f.i64("text-tokens");
    cfg.head_dim = f.i64("head-dim");
    cfg.block = f.i64("block");
    cfg.targets = parse_list<double>(f.str("targets"));
    cfg.iters = static_cast<int>(f.i64("iters"));
    cfg.warmup = static_cast<int>(f.i64("warmup"));
    cfg.parallel = f.on("parallel");
    cfg.check_outputs = !f.on("no-check");
    std::ostringstream csv;
    dfa2::write_bench_csv(csv, dfa2::run_bench(cfg));
    if (!f.str("out").empty())
        write_text(f.str("out"), csv.str());
    std::fputs(csv.str().c_str(), stdout);
    return kExitOk;
}

// ---------------------------------------------------------------- workload
int cmd_workload(const Flags& f) {
    namespace fs = std::filesystem;
    const dfa2::WorkloadConfig cfg = workload_config(f);
    const dfa2::Workload w = dfa2::generate(cfg);
    const std::string dir = f.str("out-dir");
    fs::create_directories(dir);
    const int64_t T = cfg.n_timesteps, L = cfg.n_layers, H = cfg.dims.n_heads, n = cfg.dims.seq_len(),
                  d = cfg.dims.head_dim, slice = H * n * d;
    const char* names[3] = {"q.dfa2", "k.dfa2", "v.dfa2"};
    for (int which = 0; which < 3; ++which) {
        dfa2::Tensor big = dfa2::Tensor::zeros({T, L, H, n, d});  // [T, L, H, N, d]
        for (int64_t t = 0; t < T; ++t)
            for (int64_t l = 0; l < L; ++l) {
                const dfa2::Tensor& src = which == 0 ? w.q(t, l) : which == 1 ? w.k(t, l) : w.v(t, l);
                std::copy(src.f32(), src.f32() + slice, big.f32() + (t * L + l) * slice);
            }
        const std::string path = (fs::path(dir) / names[which]).string();
        dfa2::save_dfa2(big, path);
        if (!(dfa2::load_dfa2(path) == big))
            throw dfa2::IoError("DFA2 round trip mismatch");
    }
    json_lite::Value side = json_lite::Value::object();
    side.set("T", json_lite::Value::integer(T));
    side.set("L", json_lite::Value::integer(L));
    side.set("H", json_lite::Value::integer(H));
    side.set("d", json_lite::Value::integer(d));
    side.set("n_visual", json_lite::Value::integer(cfg.dims.n_visual));
    side.set("n_text", json_lite::Value::integer(cfg.dims.n_text));
    side.set("block", json_lite::Value::integer(cfg.block_size));
    side.set("seed", json_lite::Value::integer(static_cast<int64_t>(cfg.seed)));
    side.set("token_order", json_lite::Value::str(cfg.dims.order == dfa2::TokenOrder::visual_first ? "visual-first"
                                                                                                   : "text-first"));
    json_lite::Value profiles = json_lite::Value::array();
    for (int64_t l = 0; l < L; ++l)
        for (int64_t h = 0; h < H; ++h) {
            const dfa2::HeadProfile& p = w.profile(l, h);
            json_lite::Value e = json_lite::Value::object();
            e.set("layer", json_lite::Value::integer(l));
            e.set("head", json_lite::Value::integer(h));
            e.set("locality", std::isinf(p.locality) ? json_lite::Value::str("inf") : json_lite::Value::real(p.locality));
            e.set("drift", json_lite::Value::real(p.drift));
            profiles.push(std::move(e));
        }
    side.set("profiles", std::move(profiles));
    write_text((fs::path(dir) / "workload.json").string(), side.dump(2) + "\n");
    std::printf("wrote %s/{q,k,v}.dfa2 and workload.json (round trip verified)\n", dir.c_str());
    return kExitOk;
}

void usage() {
    std::fprintf(stderr,
                 "usage: dfa2 <calibrate|run|verify|bench|workload> [flags]\n"
                 "  workload flags: --timesteps --layers --heads --head-dim --visual-tokens --text-tokens\n"
                 "                  --block --seed --token-order\n"
                 "  calibrate: --delta --coeff --windows --out --influence-csv --rse-literal --no-cache-method\n"
                 "  run:       --plan (required) --report\n"
                 "  verify:    --sizes --fault none|mask-off-by-one --seed\n"
                 "  bench:     --visual-tokens --text-tokens --head-dim --block --targets --iters --warmup\n"
                 "             --parallel --no-check --out\n"
                 "  workload:  --out-dir\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return kExitValidation;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "calibrate") {
            auto def = workload_defaults();
            def.insert({{"delta", "0.4"}, {"coeff", "1.5"}, {"windows", "0,2"}, {"out", "plan.json"},
                        {"influence-csv", ""}});
            return cmd_calibrate(Flags(argc, argv, 2, def, {"rse-literal", "no-cache-method"}));
        }
        if (cmd == "run") {
            auto def = workload_defaults();
            def.insert({{"plan", ""}, {"report", ""}});
            return cmd_run(Flags(argc, argv, 2, def, {}));
        }
        if (cmd == "verify")
            return cmd_verify(Flags(argc, argv, 2, {{"sizes", "17,64,130"}, {"fault", "none"}, {"seed", "99"}}, {}));
        if (cmd == "bench")
            return cmd_bench(Flags(argc, argv, 2,
                                   {{"visual-tokens", "4096"}, {"text-tokens", "512"}, {"head-dim", "64"},
                                    {"block", "128"}, {"targets", "0.25,0.5,0.75"}, {"iters", "20"},
                                    {"warmup", "3"}, {"out", ""}},
                                   {"parallel", "no-check"}));
        if (cmd == "workload") {
            auto def = workload_defaults();
            def.insert({"out-dir", "workload_out"});
            return cmd_workload(Flags(argc, argv, 2, def, {}));
        }
        usage();
        return kExitValidation;
    } catch (const UsageError& e) {
        std::fprintf(stderr, "usage error: %s\n", e.what());
        return kExitValidation;
    } catch (const dfa2::OracleError& e) {
        std::fprintf(stderr, "oracle failure: %s\n", e.what());
        return kExitOracle;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return kExitValidation;
    }
}
