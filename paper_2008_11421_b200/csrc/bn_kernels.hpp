#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace krt {
// NHWC bf16 batch-norm kernels (bn_kernels.cu); gamma/beta bf16, stats fp32.
size_t bn_workspace_bytes(int C);
cudaError_t bn_stats(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd, void* ws,
                     cudaStream_t s);
cudaError_t bn_stats_apply(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd,
                           const void* g, const void* b, const void* res, int relu, void* y, void* ws,
                           cudaStream_t s);
cudaError_t bn_apply(const void* x, const float* mean, const float* invstd, const void* g, const void* b,
                     const void* res, const float* rmean, const float* rinvstd, const void* rg, const void* rb,
                     int relu, void* y, int64_t rows, int C, cudaStream_t s);
cudaError_t bn_add_relu_bwd(const void* dy, const void* dy2, const void* x, const float* mean, const float* invstd, const void* g,
                            const void* b, const void* res, const float* rmean, const float* rinvstd,
                            const void* rg, const void* rb, void* dz, int64_t rows, int C, cudaStream_t s);
cudaError_t bn_backward(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                        const void* b, int relu, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
                        void* ws, const void* addend, cudaStream_t s);
cudaError_t bn_add_relu_backward(const void* dy, const void* dy2, const void* x, const float* mean,
                                 const float* invstd, const void* g, const void* b, const void* res, void* dz,
                                 void* dx, float* dgamma, float* dbeta, int64_t rows, int C, void* ws,
                                 cudaStream_t s);
// the elementwise half of bn_backward with coefficients from elsewhere
// (coef [3][C] = A, B, D: dx = A*gm + B*x + D [+ addend], gm = dy*mask)
cudaError_t bn_backward_elemt(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                              const void* b, const float* coef, const void* addend, int relu, void* dx, int64_t rows,
                              int C, cudaStream_t s);
}  // namespace krt
