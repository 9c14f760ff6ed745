// Host cost vs device time of ONE C-ABI call at the single-head shape of the
// reference's run_bench (4096 + 512 tokens, d = 64, acceptance criterion 7):
// dense and Arrow(w) for the 25/50/75% windows, split-KV on and off.
//   host us/call   = wall time of N back-to-back calls / N (no sync inside)
//   device us/call = CUDA events around the same N calls / N
//   kernel us      = CUDA events around ONE call after a sync (queue empty)
// g++ -std=c++20 -O2 -I include tools/capi_latency.cpp -o build/capi_latency \
//     -L paper_2503_22796_b200 -ldfa2_b200 -lcudart -Wl,-rpath,$PWD/paper_2503_22796_b200
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "dfa2c.h"

int main() {
    const int64_t nv = 4096, nt = 512, n = nv + nt, d = 64, B = 128;
    void *q, *k, *v, *o;
    const size_t bytes = static_cast<size_t>(n * d) * 2;
    for (void** p : {&q, &k, &v, &o}) {
        cudaMalloc(p, bytes);
        cudaMemset(*p, 0, bytes);
    }
    dfa2c_dims dims{1, d, nv, nt, 0};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int N = 200;
    for (int split : {1, 0}) {
        dfa2c_set_split_kv(split);
        for (int64_t w : {-1L, 13L, 6L, 0L}) {
            std::vector<uint8_t> mask(static_cast<size_t>((n + B - 1) / B * ((n + B - 1) / B)), 1);
            int64_t nb = 0;
            if (w >= 0)
                dfa2c_arrow_mask(&dims, B, w, mask.data(), &nb);
            auto call = [&] {
                return w < 0 ? dfa2c_dense_attention_forward(q, k, v, o, 1, n, d, nullptr)
                             : dfa2c_sparse_attention_forward(q, k, v, o, 1, n, d, mask.data(), B, nullptr);
            };
            for (int i = 0; i < 10; ++i)
                call();
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            if (call() != 0)
                return 1;
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float one = 0.f;
            cudaEventElapsedTime(&one, e0, e1);
            const auto h0 = std::chrono::steady_clock::now();
            cudaEventRecord(e0);
            for (int i = 0; i < N; ++i)
                call();
            cudaEventRecord(e1);
            const auto h1 = std::chrono::steady_clock::now();
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            const double host_us = std::chrono::duration<double, std::micro>(h1 - h0).count() / N;
            std::printf("split %d %-6s host %6.1f us/call  device %6.1f us/call  single call %6.1f us\n", split,
                        w < 0 ? "dense" : (w == 13 ? "A13" : (w == 6 ? "A6" : "A0")), host_us, ms * 1e3 / N,
                        one * 1e3);
        }
    }
    return 0;
}
