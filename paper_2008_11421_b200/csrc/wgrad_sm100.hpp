#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace krt {
// Weight gradient of an NHWC bf16 convolution on tcgen05 (wgrad_sm100.cu):
// dw[cout][k][k][cin] (fp32, OHWI) = sum over output pixels of dy (x) f(x),
// f = relu(bn(.)) per input channel when pmean is non-NULL (else identity).
// dy [n, ho, wo, cout], x [n, h, w, cin]; cout % 128 == 0, cin % 64 == 0,
// k in {1, 3}, stride in {1, 2}; ws: conv_wgrad_workspace_bytes.
bool conv_wgrad_supported(int cout, int cin, int k, int stride);
size_t conv_wgrad_workspace_bytes(int n, int ho, int wo, int cout, int cin, int k);
cudaError_t conv_wgrad(const void* dy, const void* x, float* dw, int n, int h, int w, int cin, int ho, int wo,
                       int cout, int k, int stride, int pad, const float* pmean, const float* pinvstd, const void* pg,
                       const void* pb, void* ws, size_t ws_bytes, cudaStream_t s);
}  // namespace krt
