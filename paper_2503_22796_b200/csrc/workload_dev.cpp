// workload_dev.cpp — host side of the device workload generator
// (dfa2c_workload_*; kernels in workload_sm100.cu).
//
// The stream model is the reference's generate() (src/workload.cpp:120-228):
// default_profiles' locality / drift ladders (src/workload.cpp:76-103),
// positional features omega/phase drawn from the reference's own seeded
// mt19937_64 streams (bit-identical to the reference's draws), and per
// element gaussians from a counter-based Philox stream keyed by the
// reference's derive_seed(seed, layer, head, t, tag) — so a FLUX-scale
// 28 x 57 drifting schedule is produced on the GPU at HBM speed instead of
// ~10^11 sequential mt19937 draws on the host. Each layer keeps its walk
// state in HBM (fp32 [3, H, N, d]); slots are emitted as bf16 q/k/v.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "capi_status.h"
#include "dfa2c.h"
#include "gen_types.h"

using dfa2c_detail::fail;
using dfa2c_detail::guard;

namespace dfa2k {
cudaError_t launch_gen_init(float* state, void* q, void* k, void* v, const GenHead* heads, const double* features,
                            int H, int n, int d, int text_lo, int text_hi, float feat_scale, float text_scale, int sms,
                            cudaStream_t st);
cudaError_t launch_gen_step(float* state, void* q, void* k, void* v, const GenHead* heads, int H, int n, int d,
                            int emit_only, int sms, cudaStream_t st);
}  // namespace dfa2k

namespace {

constexpr double kPi = 3.14159265358979323846;

uint64_t splitmix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// the reference's per-stream seed (src/workload.cpp:26-33)
uint64_t derive_seed(uint64_t base, uint64_t l, uint64_t h, uint64_t t, uint64_t tag) {
    uint64_t s = splitmix(base ^ 0x9e3779b97f4a7c15ull);
    s = splitmix(s ^ (l * 0xff51afd7ed558ccdull));
    s = splitmix(s ^ (h * 0xc4ceb9fe1a85ec53ull));
    s = splitmix(s ^ (t * 0xd6e8feb86659fd93ull));
    return splitmix(s ^ tag);
}

// the reference's Rng (src/workload.cpp:38-63): mt19937_64, 53-bit
// uniforms, Box-Muller pairs
struct Rng {
    std::mt19937_64 eng;
    bool spare_ok = false;
    double spare = 0.0;
    explicit Rng(uint64_t s) : eng(s) {}
    double uniform() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
    double gaussian() {
        if (spare_ok) {
            spare_ok = false;
            return spare;
        }
        double u1 = uniform();
        while (u1 <= 0.0)
            u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        spare = r * std::sin(2.0 * kPi * u2);
        spare_ok = true;
        return r * std::cos(2.0 * kPi * u2);
    }
};

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(DFA2C_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

struct dfa2c_workload {
    dfa2c_dims dims{};
    int64_t L = 0, block = 0;
    uint64_t seed = 0;
    int device = 0;
    std::vector<double> locality, drift;  // [L * H] (default_profiles)
    std::vector<float*> state;            // [L] device fp32 [3, H, N, d] (lazy)
    std::vector<double*> features;        // [L] device [H][2d] omega | phase (lazy)
    std::vector<int64_t> cur_t;           // [L] timestep the state holds, -1 = none
    dfa2k::GenHead* heads = nullptr;      // device [H] (per call)
    ~dfa2c_workload() {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(device);
        cudaDeviceSynchronize();
        for (float* p : state)
            cudaFree(p);
        for (double* p : features)
            cudaFree(p);
        cudaFree(heads);
        cudaSetDevice(cur);
    }
};

namespace {

int64_t seq_len(const dfa2c_dims& d) { return d.n_visual + d.n_text; }

void default_profiles(dfa2c_workload& w) {
    const double b = static_cast<double>(w.block), inf = std::numeric_limits<double>::infinity();
    const double ladder[6] = {b / 2, b, 2 * b, 4 * b, 8 * b, inf};
    const double drift[7] = {0.01, 0.02, 0.04, 0.07, 0.11, 0.16, 0.22};
    const int64_t H = w.dims.n_heads;
    for (int64_t l = 0; l < w.L; ++l)
        for (int64_t h = 0; h < H; ++h) {
            w.locality.push_back(h == 0 ? inf : h == 1 ? b / 4 : ladder[(h - 2 + l) % 6]);
            w.drift.push_back(h == H - 1 ? 0.0 : drift[(h + l) % 7]);
        }
}

void set_key(dfa2k::GenHead& g, int i, uint64_t s) {
    g.key[i][0] = static_cast<uint32_t>(s);
    g.key[i][1] = static_cast<uint32_t>(s >> 32);
}

void upload_heads(dfa2c_workload& w, const std::vector<dfa2k::GenHead>& hs, cudaStream_t st) {
    // pageable source: the copy is staged before cudaMemcpyAsync returns
    cuda_ok(cudaMemcpyAsync(w.heads, hs.data(), hs.size() * sizeof(dfa2k::GenHead), cudaMemcpyHostToDevice, st),
            "generator upload");
}

int sm_count(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v > 0 ? v : 148;
}

// t = 0 of layer l: positional features (the reference's draws) + noise
void init_layer(dfa2c_workload& w, int64_t l, void* q, void* k, void* v, cudaStream_t st) {
    const int64_t H = w.dims.n_heads, d = w.dims.head_dim, n = seq_len(w.dims);
    if (!w.state[l])
        cuda_ok(cudaMalloc(&w.state[l], static_cast<size_t>(3 * H * n * d) * sizeof(float)), "generator state");
    if (!w.features[l]) {
        std::vector<double> f(static_cast<size_t>(H * 2 * d));
        for (int64_t h = 0; h < H; ++h) {
            Rng pos(derive_seed(w.seed, l, h, 0, 1));  // src/workload.cpp:155-162
            const double loc = w.locality[l * H + h];
            for (int64_t x = 0; x < d; ++x) {
                f[h * 2 * d + x] = std::isinf(loc) ? 0.0 : pos.gaussian() / loc;
                f[h * 2 * d + d + x] = pos.uniform() * 2.0 * kPi;
            }
        }
        cuda_ok(cudaMalloc(&w.features[l], f.size() * sizeof(double)), "generator features");
        cuda_ok(cudaMemcpy(w.features[l], f.data(), f.size() * sizeof(double), cudaMemcpyHostToDevice),
                "generator features");
    }
    std::vector<dfa2k::GenHead> hs(static_cast<size_t>(H));
    for (int64_t h = 0; h < H; ++h) {
        for (int i = 0; i < 3; ++i)
            set_key(hs[h], i, derive_seed(w.seed, l, h, 0, 2 + i));  // tags 2, 3, 4: q, k, v
        hs[h].drift = 0.f;
        hs[h].omega_off = static_cast<int32_t>(h * 2 * d);
    }
    upload_heads(w, hs, st);
    const int64_t tlo = w.dims.order == DFA2C_VISUAL_FIRST ? w.dims.n_visual : 0;
    const int64_t thi = w.dims.order == DFA2C_VISUAL_FIRST ? n : w.dims.n_text;
    cuda_ok(dfa2k::launch_gen_init(w.state[l], q, k, v, w.heads, w.features[l], static_cast<int>(H),
                                   static_cast<int>(n), static_cast<int>(d), static_cast<int>(tlo),
                                   static_cast<int>(thi), static_cast<float>(std::sqrt(2.0 / static_cast<double>(d))),
                                   static_cast<float>(3.0 / std::sqrt(static_cast<double>(d))), sm_count(w.device),
                                   st),
            "generator init");
    w.cur_t[l] = 0;
}

// state of layer l from timestep t-1 to t (tag 5: the drift stream)
void step_layer(dfa2c_workload& w, int64_t l, int64_t t, void* q, void* k, void* v, bool emit_only,
                cudaStream_t st) {
    const int64_t H = w.dims.n_heads, d = w.dims.head_dim, n = seq_len(w.dims);
    std::vector<dfa2k::GenHead> hs(static_cast<size_t>(H));
    for (int64_t h = 0; h < H; ++h) {
        set_key(hs[h], 0, derive_seed(w.seed, l, h, t, 5));
        hs[h].drift = static_cast<float>(w.drift[l * H + h]);
    }
    upload_heads(w, hs, st);
    cuda_ok(dfa2k::launch_gen_step(w.state[l], q, k, v, w.heads, static_cast<int>(H), static_cast<int>(n),
                                   static_cast<int>(d), emit_only ? 1 : 0, sm_count(w.device), st),
            "generator step");
    if (!emit_only)
        w.cur_t[l] = t;
}

}  // namespace

extern "C" {

int dfa2c_workload_create(const dfa2c_dims* dims, int64_t n_layers, int64_t block, uint64_t seed,
                          dfa2c_workload** out) {
    return guard([&] {
        if (!dims || !out)
            fail(DFA2C_SHAPE, "dims and out must not be NULL");
        if (dims->n_heads < 1 || dims->head_dim < 1 || dims->n_visual < 1 || dims->n_text < 0)
            fail(DFA2C_SHAPE, "invalid attention dims");
        if (n_layers < 1 || block < 1)
            fail(DFA2C_SHAPE, "need n_layers >= 1 and block >= 1");
        if (dims->head_dim % 4 != 0)
            fail(DFA2C_UNSUPPORTED, "the device generator needs head_dim % 4 == 0");
        if (seq_len(*dims) * dims->head_dim > (int64_t{1} << 31))
            fail(DFA2C_UNSUPPORTED, "head too large for the device generator");
        auto w = new dfa2c_workload();
        w->dims = *dims;
        w->L = n_layers;
        w->block = block;
        w->seed = seed;
        cudaGetDevice(&w->device);
        default_profiles(*w);
        w->state.assign(static_cast<size_t>(n_layers), nullptr);
        w->features.assign(static_cast<size_t>(n_layers), nullptr);
        w->cur_t.assign(static_cast<size_t>(n_layers), -1);
        if (cudaMalloc(&w->heads, static_cast<size_t>(dims->n_heads) * sizeof(dfa2k::GenHead)) != cudaSuccess) {
            delete w;
            fail(DFA2C_CUDA, "generator allocation failed");
        }
        *out = w;
    });
}

int dfa2c_workload_destroy(dfa2c_workload* w) {
    return guard([&] { delete w; });
}

int dfa2c_workload_profile(const dfa2c_workload* w, int64_t layer, int64_t head, double* locality, double* drift) {
    return guard([&] {
        if (!w || layer < 0 || layer >= w->L || head < 0 || head >= w->dims.n_heads)
            fail(DFA2C_SHAPE, "profile index out of range");
        const size_t i = static_cast<size_t>(layer * w->dims.n_heads + head);
        if (locality)
            *locality = w->locality[i];
        if (drift)
            *drift = w->drift[i];
    });
}

int dfa2c_workload_slot(dfa2c_workload* w, int64_t t, int64_t layer, void* q, void* k, void* v, void* stream) {
    return guard([&] {
        if (!w || !q || !k || !v)
            fail(DFA2C_SHAPE, "workload and q/k/v must not be NULL");
        if (t < 0 || layer < 0 || layer >= w->L)
            fail(DFA2C_SHAPE, "timestep or layer out of range");
        for (void* p : {q, k, v})
            if (reinterpret_cast<uintptr_t>(p) % 16)
                fail(DFA2C_SHAPE, "q/k/v must be 16-byte aligned");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        int64_t& cur = w->cur_t[layer];
        if (cur < 0 || t < cur) {  // (re)start the walk: slots are a pure function of (seed, t, layer)
            init_layer(*w, layer, q, k, v, st);
            if (t == 0)
                return;
        }
        if (t == cur) {
            step_layer(*w, layer, t, q, k, v, true, st);  // re-emit
            return;
        }
        while (cur < t)
            step_layer(*w, layer, cur + 1, q, k, v, false, st);
    });
}

}  // extern "C"
