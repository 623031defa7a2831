// Internal host helpers shared by the translation units of libtpf.so.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "../../include/tpf.h"

namespace tpf {
int set_error(int code, const char* msg);
int set_cuda_error(const char* where, cudaError_t err);
size_t dense_smem_bytes(int b);
}  // namespace tpf
