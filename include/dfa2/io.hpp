// dfa2/io.hpp — the reference's "DFA2" binary tensor dump (names and format
// of /root/reference/proj/include/dfa2/io.hpp:9-19): magic "DFA2", u32
// version 1, u32 dtype (0 f32, 1 f64), u32 ndim, ndim x u64 dims, raw
// little-endian row-major scalars. Bit-exact round trip; IoError on bad
// magic, version, dtype or truncation.
#pragma once

#include <iosfwd>
#include <string>

#include "dfa2/tensor.hpp"

namespace dfa2 {

void write_dfa2(std::ostream& out, const Tensor& tensor);
Tensor read_dfa2(std::istream& in);

void save_dfa2(const Tensor& tensor, const std::string& path);
Tensor load_dfa2(const std::string& path);

}  // namespace dfa2
