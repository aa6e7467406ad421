#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace krt {
// GPT-layer kernels (ln_kernels.cu)
cudaError_t ln_fwd(const void* x, const void* r, void* x2, const void* g, const void* b, void* h, float* mean,
                   float* rstd, int64_t T, int H, float eps, cudaStream_t s);
size_t ln_bwd_workspace(int64_t T, int H);
cudaError_t ln_bwd(const void* dy, const void* x, const void* g, const float* mean, const float* rstd,
                   const void* addend, void* dx, float* dgamma, float* dbeta, void* ws, int64_t T, int H,
                   cudaStream_t s);
size_t gelu_bwd_colsum_workspace(int64_t T, int N);
cudaError_t gelu_bwd_colsum(const void* dy, const void* f, void* dx, float* colsum, void* ws, int64_t T, int N,
                            cudaStream_t s);
cudaError_t lm_xent(const void* z, const int64_t* y, void* dz, float* row_loss, int64_t T, int V, float scale,
                    cudaStream_t s);
cudaError_t attn_softmax_bwd(const float* S, const float* dP, const float* lse, const float* D, void* P, void* dS,
                             int64_t rows, int s, float scale, cudaStream_t st);
}  // namespace krt
