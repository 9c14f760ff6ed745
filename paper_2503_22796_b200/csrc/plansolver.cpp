// plansolver.cpp — the per-layer head-plan selection problem behind the
// calibration driver (reference contract: /root/reference/proj/include/dfa2/
// plansolver.hpp:19-75; used by calibrate_model, src/calibrate.cpp:314-320).
//
// Problem: H heads, M candidate methods; per head pick Full (cost full_cost,
// influence 0) or one eligible method m (finite influence I[h][m] <= cap,
// cap = coeff / H * delta) so that the summed influence stays <= delta and
// the summed cost is minimal. Ties: lower summed influence, then the
// lexicographically smaller code vector (code = method index, Full = M).
// delta == 0 admits no selection (all Full). Sums accumulate in head order.
//
// Exact solver: depth-first search over heads in index order, options in
// code order (so equal plans are met in lexicographic order and the first
// one found is kept), pruned by the LP relaxation of the remaining heads
// (fractional multiple-choice knapsack: each head starts at its cheapest
// option and buys influence reductions along its lower convex hull; the
// cheapest reductions across heads are taken first). Host-only C++.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <vector>

#include "capi_status.h"
#include "dfa2c.h"

using dfa2c_detail::fail;
using dfa2c_detail::guard;

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct Problem {
    int64_t H = 0, M = 0;
    const double* infl = nullptr;  // [H*M]
    double full_cost = 1.0;
    const double* method_cost = nullptr;  // [M]
    double delta = 0.0, coeff = 1.5;
};

struct Option {
    int64_t code;
    double cost;
    double infl;
};

double cap_of(double coeff, int64_t H, double delta) { return coeff / static_cast<double>(H) * delta; }

void check_problem(const Problem& p) {
    if (p.H < 1)
        fail(DFA2C_SHAPE, "plan problem needs at least one head");
    if (p.M < 0 || (p.M > 0 && (!p.infl || !p.method_cost)))
        fail(DFA2C_SHAPE, "cost model does not match method count");
    if (!(p.delta >= 0.0))
        fail(DFA2C_SHAPE, "delta must be >= 0");
    if (!(p.coeff >= 1.0))
        fail(DFA2C_SHAPE, "coeff must be >= 1");
    for (int64_t m = 0; m < p.M; ++m)
        if (!(p.method_cost[m] >= 0.0) || p.method_cost[m] > p.full_cost)
            fail(DFA2C_SHAPE, "method costs must lie in [0, full_cost]");
    for (int64_t i = 0; i < p.H * p.M; ++i)
        if (p.infl[i] < 0.0)
            fail(DFA2C_SHAPE, "influences must be >= 0");
}

// Eligible options of every head in code order, Full last.
std::vector<std::vector<Option>> options_of(const Problem& p) {
    const double cap = cap_of(p.coeff, p.H, p.delta);
    std::vector<std::vector<Option>> out(static_cast<size_t>(p.H));
    for (int64_t h = 0; h < p.H; ++h) {
        for (int64_t m = 0; m < p.M; ++m) {
            const double w = p.infl[h * p.M + m];
            if (std::isfinite(w) && w <= cap)
                out[h].push_back({m, p.method_cost[m], w});
        }
        out[h].push_back({p.M, p.full_cost, 0.0});
    }
    return out;
}

// Drops methods no tie-break optimum uses: b is dominated when another
// method a is no costlier and no more influential and is strictly better
// in one of them or has the lower code. Full always stays.
void prune_dominated(std::vector<std::vector<Option>>& heads, int64_t M) {
    for (auto& opts : heads) {
        std::vector<Option> keep;
        for (const Option& b : opts) {
            bool dominated = false;
            if (b.code != M)
                for (const Option& a : opts)
                    if (a.code != M && a.code != b.code && a.cost <= b.cost && a.infl <= b.infl &&
                        (a.cost < b.cost || a.infl < b.infl || a.code < b.code)) {
                        dominated = true;
                        break;
                    }
            if (!dominated)
                keep.push_back(b);
        }
        opts.swap(keep);
    }
}

// LP bound tables: per suffix [h, H) the summed cheapest-option cost/influence
// and the reduction steps of all suffix heads sorted by marginal cost.
struct Step {
    double rate, dw, dc;
};
struct Suffix {
    double c0 = 0.0, w0 = 0.0;
    std::vector<double> rate, cum_w, cum_c;  // sorted by rate; cumulative sums
};

// One head's reduction steps: from its cheapest option (lowest influence
// among the cheapest) along the lower convex hull of (influence, cost)
// toward influence 0, as (rate, dw, dc) with non-decreasing rate.
void head_steps(const std::vector<Option>& opts, double& c0, double& w0, std::vector<Step>& steps) {
    const Option* s = &opts[0];
    for (const Option& o : opts)
        if (o.cost < s->cost || (o.cost == s->cost && o.infl < s->infl))
            s = &o;
    c0 = s->cost;
    w0 = s->infl;
    if (w0 <= 0.0)
        return;
    // Pareto points below the start: influence ascending, each kept only
    // if cheaper than every point of lower influence (the cheapest of a
    // level comes first after the sort)
    std::vector<std::pair<double, double>> pts;  // (influence, cost)
    for (const Option& o : opts)
        if (o.infl < w0 && o.cost > c0)
            pts.emplace_back(o.infl, o.cost);
    std::sort(pts.begin(), pts.end());
    std::vector<std::pair<double, double>> useful;
    double cheapest = kInf;
    for (const auto& pt : pts) {
        if (!useful.empty() && useful.back().first == pt.first)
            continue;
        if (pt.second < cheapest) {
            useful.push_back(pt);
            cheapest = pt.second;
        }
    }
    // lower convex chain from (w0, c0) toward influence 0
    std::vector<std::pair<double, double>> chain{{w0, c0}};
    for (auto it = useful.rbegin(); it != useful.rend(); ++it) {  // influence descending
        while (chain.size() >= 2) {
            const auto& a = chain[chain.size() - 2];
            const auto& b = chain.back();
            // drop b when the step a->b is no cheaper per unit than b->it
            if ((b.second - a.second) * (b.first - it->first) >= (it->second - b.second) * (a.first - b.first))
                chain.pop_back();
            else
                break;
        }
        chain.push_back(*it);
    }
    for (size_t i = 1; i < chain.size(); ++i) {
        const double dw = chain[i - 1].first - chain[i].first;
        const double dc = chain[i].second - chain[i - 1].second;
        steps.push_back({dc / dw, dw, dc});
    }
}

std::vector<Suffix> suffix_tables(const std::vector<std::vector<Option>>& heads) {
    const size_t H = heads.size();
    std::vector<Suffix> t(H + 1);
    std::vector<Step> pool;
    for (size_t h = H; h-- > 0;) {
        double c0 = 0, w0 = 0;
        head_steps(heads[h], c0, w0, pool);
        t[h].c0 = t[h + 1].c0 + c0;
        t[h].w0 = t[h + 1].w0 + w0;
        std::vector<Step> sorted = pool;
        std::stable_sort(sorted.begin(), sorted.end(), [](const Step& a, const Step& b) { return a.rate < b.rate; });
        double cw = 0, cc = 0;
        for (const Step& s : sorted) {
            cw += s.dw;
            cc += s.dc;
            t[h].rate.push_back(s.rate);
            t[h].cum_w.push_back(cw);
            t[h].cum_c.push_back(cc);
        }
    }
    return t;
}

// Least fractional cost of heads [h, H) with `budget` influence left.
double lp_bound(const Suffix& s, double budget) {
    const double need = s.w0 - budget;
    if (need <= 0.0)
        return s.c0;
    const size_t i = static_cast<size_t>(std::lower_bound(s.cum_w.begin(), s.cum_w.end(), need) - s.cum_w.begin());
    if (i >= s.cum_w.size())  // cannot happen: Full (influence 0) ends every chain
        return s.c0 + (s.cum_c.empty() ? 0.0 : s.cum_c.back());
    const double w_prev = i ? s.cum_w[i - 1] : 0.0, c_prev = i ? s.cum_c[i - 1] : 0.0;
    return s.c0 + c_prev + (need - w_prev) * s.rate[i];
}

struct Best {
    bool valid = false;
    double obj = kInf, infl = kInf;
    std::vector<int64_t> codes;
    bool improved_by(double o, double w, const std::vector<int64_t>& c) const {
        if (!valid)
            return true;
        if (o != obj)
            return o < obj;
        if (w != infl)
            return w < infl;
        return c < codes;
    }
};

struct Search {
    const Problem& p;
    std::vector<std::vector<Option>> heads;
    std::vector<Suffix> tabs;
    std::vector<int64_t> codes;
    Best best;
    int64_t nodes = 0;

    void run(size_t h, double cost, double infl) {
        ++nodes;
        if (h == heads.size()) {
            if (best.improved_by(cost, infl, codes))
                best = {true, cost, infl, codes};
            return;
        }
        for (const Option& o : heads[h]) {
            const double w = infl + o.infl;
            if (w > p.delta)
                continue;
            const double c = cost + o.cost;
            // the bound is a float evaluation of a real lower bound; a hair of
            // slack keeps rounding from pruning a branch that ties the incumbent
            const double lb = c + lp_bound(tabs[h + 1], p.delta - w);
            if (best.valid && lb - 1e-12 * (1.0 + std::fabs(lb)) > best.obj)
                continue;
            codes[h] = o.code;
            run(h + 1, c, w);
        }
    }
};

void emit(const Problem& p, const Best& b, int64_t nodes, int64_t* choice, double* objective, double* total,
          int64_t* n_nodes) {
    if (!b.valid)
        fail(DFA2C_CUDA, "no feasible plan (all-Full is always feasible)");
    for (int64_t h = 0; h < p.H; ++h)
        choice[h] = b.codes[h] == p.M ? -1 : b.codes[h];
    if (objective)
        *objective = b.obj;
    if (total)
        *total = b.infl;
    if (n_nodes)
        *n_nodes = nodes;
}

Best all_full(const Problem& p) {
    Best b;
    b.valid = true;
    b.obj = 0.0;
    for (int64_t h = 0; h < p.H; ++h)
        b.obj += p.full_cost;
    b.infl = 0.0;
    b.codes.assign(static_cast<size_t>(p.H), p.M);
    return b;
}

}  // namespace

extern "C" {

double dfa2c_selection_cap(double coeff, int64_t n_heads, double delta) { return cap_of(coeff, n_heads, delta); }

int dfa2c_plan_solve(int64_t n_heads, int64_t n_methods, const double* influence, double full_cost,
                     const double* method_cost, double delta, double coeff, int32_t exhaustive, int64_t* choice,
                     double* objective, double* total_influence, int64_t* nodes) {
    return guard([&] {
        const Problem p{n_heads, n_methods, influence, full_cost, method_cost, delta, coeff};
        check_problem(p);
        if (!choice)
            fail(DFA2C_SHAPE, "choice output must not be NULL");
        if (p.delta == 0.0) {
            emit(p, all_full(p), 0, choice, objective, total_influence, nodes);
            return;
        }
        if (!exhaustive) {
            Search s{p, options_of(p), {}, std::vector<int64_t>(static_cast<size_t>(p.H), 0), {}, 0};
            prune_dominated(s.heads, p.M);
            s.tabs = suffix_tables(s.heads);
            s.run(0, 0.0, 0.0);
            emit(p, s.best, s.nodes, choice, objective, total_influence, nodes);
            return;
        }
        // exhaustive enumeration of every eligible assignment in lexicographic
        // code order (the test oracle of the search)
        if (std::pow(static_cast<double>(p.M + 1), static_cast<double>(p.H)) > 1e7)
            fail(DFA2C_SHAPE, "instance too large for brute force");
        const auto heads = options_of(p);
        std::vector<size_t> pos(static_cast<size_t>(p.H), 0);
        std::vector<int64_t> codes(static_cast<size_t>(p.H), 0);
        Best best;
        for (;;) {
            double c = 0.0, w = 0.0;
            bool ok = true;
            for (int64_t h = 0; h < p.H && ok; ++h) {
                const Option& o = heads[h][pos[h]];
                codes[h] = o.code;
                c += o.cost;
                w += o.infl;
                ok = w <= p.delta;
            }
            if (ok && best.improved_by(c, w, codes))
                best = {true, c, w, codes};
            int64_t h = p.H - 1;
            for (; h >= 0; --h) {
                if (++pos[h] < heads[h].size())
                    break;
                pos[h] = 0;
            }
            if (h < 0)
                break;
        }
        emit(p, best, 0, choice, objective, total_influence, nodes);
    });
}

int dfa2c_plan_lp_bound(int64_t n_heads, int64_t n_methods, const double* influence, double full_cost,
                        const double* method_cost, double delta, double coeff, double* bound) {
    return guard([&] {
        const Problem p{n_heads, n_methods, influence, full_cost, method_cost, delta, coeff};
        check_problem(p);
        if (!bound)
            fail(DFA2C_SHAPE, "bound output must not be NULL");
        if (p.delta == 0.0) {
            *bound = all_full(p).obj;
            return;
        }
        auto heads = options_of(p);
        prune_dominated(heads, p.M);
        *bound = lp_bound(suffix_tables(heads)[0], p.delta);
    });
}

}  // extern "C"
