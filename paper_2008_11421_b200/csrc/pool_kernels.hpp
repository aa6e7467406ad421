#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace krt {
// ResNet stem max-pool fused with the BN + ReLU that feeds it (pool_kernels.cu)
cudaError_t bn_relu_maxpool(const void* x, const float* mean, const float* invstd, const void* g, const void* b,
                            void* y, int n, int h, int w, int c, int k, int s, int p, cudaStream_t st);
size_t bn_relu_maxpool_bwd_workspace(int n, int h, int w, int c, int k, int s, int p);
cudaError_t bn_relu_maxpool_bwd(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                                const void* b, void* dx, void* ws, int n, int h, int w, int c, int k, int s, int p,
                                cudaStream_t st);
}  // namespace krt
