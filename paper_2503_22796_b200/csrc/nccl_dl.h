// nccl_dl.h — run-time bound NCCL calls used by the sharded layer (nccl_dl.cpp).
// Every function returns an empty string on success, else the error text.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace dfa2nccl {

constexpr int kUniqueIdBytes = 128;

bool available(std::string* why);
std::string unique_id(char* out /* kUniqueIdBytes */);
std::string comm_init(void** comm, int nranks, const char* id /* kUniqueIdBytes */, int rank);
std::string comm_destroy(void* comm);
std::string comm_shape(void* comm, int* nranks, int* rank);
// in-place all-gather of unequal contiguous byte ranges [off[r], off[r+1]) of buf
std::string allgather_v(void* comm, void* buf, const int64_t* off, int world, cudaStream_t stream);

}  // namespace dfa2nccl
