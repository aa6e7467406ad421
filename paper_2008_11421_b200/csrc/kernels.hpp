#pragma once
#include <cuda_runtime.h>

#include "optim.hpp"

namespace krt {
// All pointers 16-byte aligned (the runtime's regions are 256-byte aligned).
cudaError_t launch_update(float* master, float* m, float* v, const float* grad, void* weights, int weight_dtype,
                          size_t n, const OptimScalars& s, cudaStream_t stream);
cudaError_t launch_reduce_cast(const float* const* in, int n_in, void* out, int out_dtype, size_t n, float scale,
                               cudaStream_t stream);
cudaError_t launch_unpack_bf16(const void* in, float* out, size_t n, float scale, cudaStream_t stream);
}  // namespace krt
