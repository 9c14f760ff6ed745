// Times the C++ drop-in dfa2::multi_strategy_attention (host f32 tensors in
// and out, the reference's calling convention) on one FLUX 2K FLUX68 layer.
//   g++ -std=c++20 -O2 -Iinclude tools/cpp_api_bench.cpp -Lpaper_2503_22796_b200 -ldfa2_b200 \
//       -Wl,-rpath,paper_2503_22796_b200 -o /tmp/cpp_api_bench && /tmp/cpp_api_bench
#include <chrono>
#include <cstdio>
#include <random>

#include "dfa2/dispatch.hpp"

int main() {
    using namespace dfa2;
    AttentionDims dims;
    dims.n_heads = 24;
    dims.head_dim = 128;
    dims.n_visual = 16384;
    dims.n_text = 512;
    const int64_t n = dims.seq_len(), numel = dims.n_heads * n * dims.head_dim;
    std::mt19937 rng(1);
    std::normal_distribution<float> g;
    std::vector<float> buf(static_cast<size_t>(numel));
    auto fill = [&] {
        for (auto& x : buf)
            x = g(rng);
        return Tensor::from_f32({dims.n_heads, n, dims.head_dim}, buf);
    };
    const Tensor q = fill(), k = fill(), v = fill();
    LayerPlan plan;
    const char* pat = "FACa";  // F A8 C A0 repeated (FLUX68 head pattern)
    for (int h = 0; h < 24; ++h) {
        const int g4 = h / 4, r = h % 4;
        plan.strategies.push_back(r == 0 ? HeadStrategy::Full()
                                  : r == 1 ? HeadStrategy::Arrow(8)
                                  : r == 2 ? HeadStrategy::Cached()
                                           : HeadStrategy::Arrow(g4 % 3 != 1 ? 0 : 8));
    }
    (void)pat;
    HeadCache cache;
    multi_strategy_attention(q, k, v, LayerPlan::all_full(24), cache, 0, 0, dims, 128);  // t = 0 fills the cache
    for (int i = 0; i < 2; ++i)
        multi_strategy_attention(q, k, v, plan, cache, 0, 1, dims, 128);
    const auto t0 = std::chrono::steady_clock::now();
    const int reps = 5;
    for (int i = 0; i < reps; ++i)
        multi_strategy_attention(q, k, v, plan, cache, 0, 1, dims, 128);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() / reps;
    std::printf("{\"api\": \"dfa2::multi_strategy_attention (host f32 Tensors)\", \"layer\": \"FLUX 2K FLUX68\", "
                "\"ms_per_call\": %.2f}\n", ms);
    return 0;
}
