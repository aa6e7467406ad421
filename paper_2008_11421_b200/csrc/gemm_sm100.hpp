#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace krt {
// tcgen05 1x1-convolution GEMM with fused BN prologue / statistics epilogue (gemm_sm100.cu)
bool conv1x1_supported(int64_t M, int N, int K);
size_t conv1x1_partials_bytes(int N);
cudaError_t conv1x1_bn_fprop(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                             const float* pinvstd, const void* pg, const void* pb, float* part, int* part_rows,
                             cudaStream_t s);
// RGB NHWC bf16 [pixels, 3] -> [pixels, 4] (4th channel 0)
cudaError_t pad_rgb4(const void* x, void* y, int64_t pixels, cudaStream_t s);
// implicit-GEMM convolution (the ResNet stem): C[n*ho*wo, N] = im2col(x) .
// wk^T with x NHWC [n, h, w, cin], wk [N, K] (K = (kh*k + kw)*cin + c, zero
// padded to K), the im2col rows gathered in shared memory, never written;
// part/part_rows: BN statistics partials as conv1x1_bn_fprop.  N = 64.
cudaError_t conv_gather_fprop(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int ho, int wo,
                              int k, int stride, int pad, int N, int K, float* part, int* part_rows, cudaStream_t s);
// as conv1x1_bn_fprop, plus a residual: C = f(A) . B^T + res (res [M, N] bf16)
cudaError_t conv1x1_bn_res_fprop(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                                 const float* pinvstd, const void* pg, const void* pb, const void* res, float* part,
                                 int* part_rows, cudaStream_t s);
// dX[M,N] = dY[M,K] . Wt[N,K]^T (1x1 dgrad, Wt = the weights transposed) with
// the backward reduce of the BN (+ReLU) whose input is x fused in the epilogue
cudaError_t conv1x1_bn_dgrad(const void* dY, const void* Wt, void* dX, int64_t M, int N, int K, const void* x,
                             const float* mean, const float* invstd, const void* g, const void* b, float* part,
                             int* part_rows, cudaStream_t s);
// implicit-GEMM convolution with im2col TMA A tiles (k x k, stride, pad; cin %
// 64 == 0): C[n*ho*wo, N] = f(im2col(x)) . wk^T, wk [N, k*k*cin] (OHWI
// flattened), f = relu(bn(.)) per input channel when pmean (padding stays
// zero); part: BN statistics of C (EPI 1) or, with bx, the BN-backward reduce
// of (C, bx) (EPI 2, the dgrad form)
cudaError_t conv_im2col_fprop(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int ho, int wo,
                              int k, int stride, int pad, int N, const float* pmean, const float* pinvstd,
                              const void* pg, const void* pb, float* part, int* part_rows, const void* bx,
                              const float* bmean, const float* binvstd, const void* bg, const void* bb,
                              cudaStream_t s);
cudaError_t bn_partials_bwd_finalize(const float* part, int part_rows, int N, int64_t M, const float* mean,
                                     const float* invstd, const void* g, float* dgamma, float* dbeta, float* coef,
                                     cudaStream_t s);
cudaError_t bn_partials_finalize(const float* part, int part_rows, int N, int64_t M, float eps, float* mean,
                                 float* invstd, cudaStream_t s);
}  // namespace krt
