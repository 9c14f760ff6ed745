// dfa2/cache.hpp — HeadCache (names and semantics of
// /root/reference/proj/include/dfa2/cache.hpp:15-32). Slots live on the GPU
// as bf16 (a dfa2c_cache); fetch() downloads a host f32 copy.
#pragma once

#include <cstdint>
#include <map>
#include <utility>

#include "dfa2/tensor.hpp"

struct dfa2c_cache;

namespace dfa2 {

class HeadCache {
public:
    HeadCache() = default;
    // A value type like the reference's (cache.hpp:15-32): a copy is a deep
    // copy of every entry (device-resident slots are read back into the
    // copy's host entries and re-uploaded when the copy is first used on the
    // GPU); a move transfers the device slots.
    HeadCache(const HeadCache& other);
    HeadCache& operator=(const HeadCache& other);
    HeadCache(HeadCache&& other) noexcept;
    HeadCache& operator=(HeadCache&& other) noexcept;
    ~HeadCache();

    void store(int64_t layer, int64_t head, Tensor output, int64_t t);
    const Tensor& fetch(int64_t layer, int64_t head) const;  // CacheMissError
    bool has(int64_t layer, int64_t head) const;
    int64_t produced_at(int64_t layer, int64_t head) const;  // CacheMissError
    int64_t staleness(int64_t layer, int64_t head, int64_t t) const;
    void clear();
    int64_t size() const;

    // Device binding used by multi_strategy_attention / influence_for_layer:
    // creates (or checks) the device slot array for H heads of [n, d] and
    // uploads pending slots. Logically const (the entries do not change; only
    // where they live), so influence_for_layer keeps the reference's
    // `const HeadCache&` signature (calibrate.hpp:80-86).
    dfa2c_cache* bind(int64_t n_heads, int64_t seq_len, int64_t head_dim) const;

private:
    struct Slot {
        int64_t produced_at = 0;
        bool on_device = false;
        bool host_fresh = false;
        Tensor host;  // [n, d] f32 (pending upload, or downloaded copy)
    };
    Slot& slot(int64_t layer, int64_t head) const;  // slots_ is mutable (device residency)
    void release_device();
    mutable std::map<std::pair<int64_t, int64_t>, Slot> slots_;
    mutable dfa2c_cache* dev_ = nullptr;
    mutable int64_t heads_ = 0, n_ = 0, d_ = 0, layers_ = 0;
    friend class CacheAccess;
};

}  // namespace dfa2
