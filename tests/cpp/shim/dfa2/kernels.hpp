// dfa2/kernels.hpp — TEST-ONLY stub of the reference's CPU ISA table
// (/root/reference/proj/include/dfa2/kernels.hpp:13-30), present only so the
// reference's test_arrow.cpp compiles unchanged against this repo's drop-in
// headers. The product has no such table: on B200 the dot/axpy/scale inner
// loops are the tcgen05 MMAs (DESIGN.md §0 row a9) and the north star
// forbids multi-backend dispatch. avx2_supported() is false, so the
// reference's SIMD-agreement case skips; force_isa() is a no-op.
#pragma once
#include <cstdint>

namespace dfa2::kern {

enum class Isa { scalar, avx2 };

struct Ops {
    float (*dot)(const float* a, const float* b, int64_t n);
    void (*axpy)(float alpha, const float* x, float* y, int64_t n);
    void (*scale)(float* x, float s, int64_t n);
    const char* name;
};

namespace stub {
inline float dot(const float* a, const float* b, int64_t n) {
    float s = 0.f;
    for (int64_t i = 0; i < n; ++i)
        s += a[i] * b[i];
    return s;
}
inline void axpy(float alpha, const float* x, float* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        y[i] += alpha * x[i];
}
inline void scale(float* x, float s, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        x[i] *= s;
}
}  // namespace stub

inline const Ops& scalar_ops() {
    static const Ops o{stub::dot, stub::axpy, stub::scale, "scalar (test stub)"};
    return o;
}
inline bool avx2_supported() { return false; }
inline const Ops& avx2_ops() { return scalar_ops(); }
inline const Ops& ops() { return scalar_ops(); }
inline Isa active_isa() { return Isa::scalar; }
inline void force_isa(Isa) {}

}  // namespace dfa2::kern
