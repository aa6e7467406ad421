#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace krt {
// 3x3 / stride-1 / pad-1 convolution with halo windows (halo_sm100.cu):
// C[n*h*w, N] = f(x) (*) wk, x NHWC bf16 [n, h, w, cin] (cin % 64 == 0), wk
// [N][3][3][cin] bf16 (OHWI), N in {64, 128}; f = relu(bn(.)) per input channel
// when pmean is non-NULL (the zero padding stays zero); part/part_rows: BN
// statistics partials of C as conv1x1_bn_fprop (bn_partials_finalize).
// KRT_CONV_HALO=0 disables it (conv3x3_halo_supported then returns false).
bool conv3x3_halo_supported(int h, int w, int cin, int N, bool pro);
cudaError_t conv3x3_halo_fprop(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int N,
                               const float* pmean, const float* pinvstd, const void* pg, const void* pb, float* part,
                               int* part_rows, cudaStream_t s);
// Weight gradient of a 3x3 / stride-1 / pad-1 convolution with C = cin = cout
// in {16, 32, 64} from halo windows (wgrad_halo_sm100.cu): dw [C][3][3][C] fp32
// (OHWI, written) = sum over pixels of dy (x) f(x), f = relu(bn(.)) when pmean;
// ws: wgrad3x3_halo_workspace(C) bytes (per-CTA partial accumulators).
bool wgrad3x3_halo_supported(int h, int w, int C);
size_t wgrad3x3_halo_workspace(int C);
cudaError_t wgrad3x3_halo(const void* x, const void* dy, float* dw, int n, int h, int w, int C, const float* pmean,
                          const float* pinvstd, const void* pg, const void* pb, void* ws, size_t ws_bytes,
                          cudaStream_t s);
// Weight gradient of a 1x1 convolution with few channels (one side 64 / 128 /
// 256, the other 16 / 32 / 64): dw [co][ci] fp32 (written) = sum over the M
// pixels of dy [M, co] (x) f(x [M, ci]), f = relu(bn(.)) when pmean
bool wgrad1x1_narrow_supported(int ci, int co);
size_t wgrad1x1_narrow_workspace(int ci, int co);
cudaError_t wgrad1x1_narrow(const void* x, const void* dy, float* dw, int64_t M, int ci, int co, const float* pmean,
                            const float* pinvstd, const void* pg, const void* pb, void* ws, size_t ws_bytes,
                            cudaStream_t s);
// The ResNet stem's weight gradient (7x7 / stride 2 / pad 3, 64 output
// channels): x4 [n, h, w, 4] bf16 (RGB padded to 4 channels, krt_pad_rgb4),
// dc [n, ho, wo, 64] bf16 -> dw [64][7][7][3] fp32 (OHWI, written)
size_t stem_wgrad_workspace();
cudaError_t stem_wgrad(const void* x4, const void* dc, float* dw, int n, int h, int w, void* ws, size_t ws_bytes,
                       cudaStream_t s);
}  // namespace krt
