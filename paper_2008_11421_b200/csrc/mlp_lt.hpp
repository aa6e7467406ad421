#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace krt {
// GPT MLP GEMMs with the bias / GELU work in the cuBLASLt epilogue (mlp_lt.cpp).
// Row-major bf16: x [M, K], w1 [N, K], b1 [N] -> f1 [M, N] (GELU input) and
// g = gelu_tanh(f1) [M, N]
void mlp_fc1_gelu(const void* x, const void* w1, const void* b1, void* f1, void* g, int64_t M, int64_t N, int64_t K,
                  cudaStream_t s);
// dy [M, K], w2 [K, N] (fc2's weight, out x in), f1 [M, N] -> df1 = (dy . w2) *
// gelu_tanh'(f1) [M, N] bf16
void mlp_fc2_dgelu(const void* dy, const void* w2, const void* f1, void* df1, int64_t M, int64_t N, int64_t K,
                   cudaStream_t s);
// g [M, K], w2 [N, K], b2 [N], x2 [M, N] -> y = x2 + g . w2^T + b2 [M, N]
// (y may alias x2)
void mlp_fc2_residual(const void* g, const void* w2, const void* b2, const void* x2, void* y, int64_t M, int64_t N,
                      int64_t K, cudaStream_t s);
// a linear layer's weight and bias gradients in one GEMM (cuBLASLt BGRADB
// epilogue): dy [M, N], x [M, K] bf16 -> dw = dy^T . x [N, K] and db = the
// column sums of dy [N], both fp32
void linear_wgrad_bgrad(const void* dy, const void* x, float* dw, float* db, int64_t M, int64_t N, int64_t K,
                        cudaStream_t s);
}  // namespace krt
