// gen_types.h — per-head parameters of the device workload generator
// (workload_sm100.cu), filled by the host (workload_dev.cpp).
#pragma once
#include <cstdint>

namespace dfa2k {

struct GenHead {
    uint32_t key[3][2];  // Philox keys: q, k, v noise at t = 0; key[0] = the drift stream at t > 0
    float drift;         // t > 0: random-walk scale (0: frozen head)
    int32_t omega_off;   // offset of this head's omega[d], phase[d] in the feature table
};

}  // namespace dfa2k
