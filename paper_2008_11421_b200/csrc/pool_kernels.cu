// ResNet stem: y = maxpool_kxk/s(relu(bn(c))) and its backward, NHWC bf16 (sm_100a).
//
// The stem's post-BN activation a = relu(bn(c)) is never materialised: the
// forward reads c once and writes only the pooled output, and the backward
// recomputes each window's argmax from c instead of storing indices (aten's
// NHWC max_pool2d_with_indices keeps an int64 index per output element and
// moved ~10x the algorithmic bytes; profiles/round1_s2_launches_b512_summary.md).
//
// Semantics follow aten exactly, so results are bitwise those of
// apply -> max_pool2d_with_indices -> max_pool2d_with_indices_backward:
//   * a = bf16(max(fma(c, scale, shift), 0)), rounded before the max
//   * window scan h-major then w, "val > max || isnan(val)" takes the element
//     (first maximum wins), padding excluded
//   * the gradient of an input sums, in fp32 and in (oh, ow) scan order, the
//     output gradients of the windows whose argmax it is, then rounds to bf16
// Thread mapping: one thread per (pixel, 8-channel octet): 16-byte vectors,
// consecutive threads = consecutive octets of one pixel (coalesced).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "pool_kernels.hpp"

namespace krt {
namespace {

constexpr int kThreads = 256;

struct Pool {
  int n, h, w, c, oh, ow, k, s, p;
};

__device__ __forceinline__ void load_bf8(const __nv_bfloat16* p, float* f) {
  uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 t = __bfloat1622float2(h[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}

// per-channel affine of the BN: a = relu(c*sc + sh), rounded to bf16
__device__ __forceinline__ void coeffs(const float* mean, const float* invstd, const __nv_bfloat16* g,
                                       const __nv_bfloat16* b, int c0, float* sc, float* sh) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float s = invstd[c0 + k] * __bfloat162float(g[c0 + k]);
    sc[k] = s;
    sh[k] = __bfloat162float(b[c0 + k]) - mean[c0 + k] * s;
  }
}

__device__ __forceinline__ float act(float v, float sc, float sh) {
  return __bfloat162float(__float2bfloat16_rn(fmaxf(__fmaf_rn(v, sc, sh), 0.0f)));
}

// scan one window; returns max values and argmax offsets (kh*k + kw).
// K > 0: compile-time window, all K*K loads issued before the compares (the
// pass is latency-bound otherwise); K == 0: runtime P.k.
template <int K>
__device__ __forceinline__ void window_max(const __nv_bfloat16* __restrict__ x, const Pool& P, int n, int oh, int ow,
                                           int c0, const float* sc, const float* sh, float* mx, int* arg) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    mx[j] = -INFINITY;
    arg[j] = -1;
  }
  const int h0 = oh * P.s - P.p, w0 = ow * P.s - P.p;
  const __nv_bfloat16* base = x + (int64_t)n * P.h * P.w * P.c + c0;
  if constexpr (K > 0) {
    uint4 raw[K * K];
    bool ok[K * K];
#pragma unroll
    for (int kh = 0; kh < K; ++kh) {
#pragma unroll
      for (int kw = 0; kw < K; ++kw) {
        const int ih = h0 + kh, iw = w0 + kw;
        ok[kh * K + kw] = ih >= 0 && ih < P.h && iw >= 0 && iw < P.w;
        if (ok[kh * K + kw])
          raw[kh * K + kw] = __ldg(reinterpret_cast<const uint4*>(base + ((int64_t)ih * P.w + iw) * P.c));
      }
    }
#pragma unroll
    for (int q = 0; q < K * K; ++q) {
      if (!ok[q]) continue;
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&raw[q]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float2 t = __bfloat1622float2(hv[j / 2]);
        float a = act(j & 1 ? t.y : t.x, sc[j], sh[j]);
        if (a > mx[j] || isnan(a)) {
          mx[j] = a;
          arg[j] = q;
        }
      }
    }
  } else {
    for (int kh = 0; kh < P.k; ++kh) {
      const int ih = h0 + kh;
      if (ih < 0 || ih >= P.h) continue;
      for (int kw = 0; kw < P.k; ++kw) {
        const int iw = w0 + kw;
        if (iw < 0 || iw >= P.w) continue;
        float v[8];
        load_bf8(base + ((int64_t)ih * P.w + iw) * P.c, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float a = act(v[j], sc[j], sh[j]);
          if (a > mx[j] || isnan(a)) {
            mx[j] = a;
            arg[j] = kh * P.k + kw;
          }
        }
      }
    }
  }
}

template <int K>
__global__ void __launch_bounds__(kThreads) bn_relu_maxpool_kernel(
    const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ invstd,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ y,
    Pool P) {
  const int oc = P.c / 8;
  const int64_t total = (int64_t)P.n * P.oh * P.ow * oc;
  for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < total; t += (int64_t)gridDim.x * kThreads) {
    const int c0 = (int)(t % oc) * 8;
    int64_t pix = t / oc;
    const int ow = (int)(pix % P.ow);
    pix /= P.ow;
    const int oh = (int)(pix % P.oh);
    const int n = (int)(pix / P.oh);
    float sc[8], sh[8], mx[8];
    int arg[8];
    coeffs(mean, invstd, g, b, c0, sc, sh);
    window_max<K>(x, P, n, oh, ow, c0, sc, sh, mx, arg);
    uint4 u;
    __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) hv[k] = __floats2bfloat162_rn(mx[2 * k], mx[2 * k + 1]);
    *reinterpret_cast<uint4*>(y + t * 8) = u;
  }
}

// phase 1 of the backward: argmax offset of every (window, channel), one byte each
template <int K>
__global__ void __launch_bounds__(kThreads) maxpool_argmax_kernel(
    const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ invstd,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, uint8_t* __restrict__ arg_out,
    Pool P) {
  const int oc = P.c / 8;
  const int64_t total = (int64_t)P.n * P.oh * P.ow * oc;
  for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < total; t += (int64_t)gridDim.x * kThreads) {
    const int c0 = (int)(t % oc) * 8;
    int64_t pix = t / oc;
    const int ow = (int)(pix % P.ow);
    pix /= P.ow;
    const int oh = (int)(pix % P.oh);
    const int n = (int)(pix / P.oh);
    float sc[8], sh[8], mx[8];
    int arg[8];
    coeffs(mean, invstd, g, b, c0, sc, sh);
    window_max<K>(x, P, n, oh, ow, c0, sc, sh, mx, arg);
    uint2 packed;
    packed.x = (uint32_t)(arg[0] & 0xff) | ((uint32_t)(arg[1] & 0xff) << 8) | ((uint32_t)(arg[2] & 0xff) << 16) |
               ((uint32_t)(arg[3] & 0xff) << 24);
    packed.y = (uint32_t)(arg[4] & 0xff) | ((uint32_t)(arg[5] & 0xff) << 8) | ((uint32_t)(arg[6] & 0xff) << 16) |
               ((uint32_t)(arg[7] & 0xff) << 24);
    *reinterpret_cast<uint2*>(arg_out + t * 8) = packed;
  }
}

// Shared-memory tiled variant for the ResNet stem (k 3, s 2, p 1, C 64): a CTA
// owns an 8 x 8 block of output pixels of one image; the 17 x 17 input patch
// is loaded once with coalesced 16-byte loads, activated once (the windows
// overlap 2.25x) and kept in shared memory with a padded pixel stride; padding
// positions hold -inf, which never wins the scan (the window centre is always
// inside the image and relu output is >= 0), so argmax offsets are unchanged.
constexpr int kTile = 8, kPatch = 2 * kTile + 1, kTC = 64, kPixStride = kTC + 8;  // bf16 elements

template <bool ARGMAX>
__global__ void __launch_bounds__(kThreads) stem_pool_tiled_kernel(
    const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ invstd,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ y,
    uint8_t* __restrict__ arg_out, Pool P) {
  __shared__ alignas(16) __nv_bfloat16 patch[kPatch * kPatch * kPixStride];
  const int tiles_w = (P.ow + kTile - 1) / kTile, tiles_h = (P.oh + kTile - 1) / kTile;
  const int tw = blockIdx.x % tiles_w, th = (blockIdx.x / tiles_w) % tiles_h, n = blockIdx.x / (tiles_w * tiles_h);
  const int oh0 = th * kTile, ow0 = tw * kTile;
  const int ih0 = oh0 * 2 - 1, iw0 = ow0 * 2 - 1;
  // phase 1: patch load + activation (octet = threadIdx & 7 is fixed per thread)
  const int oct = threadIdx.x & 7;
  float sc[8], sh[8];
  coeffs(mean, invstd, g, b, oct * 8, sc, sh);
  const __nv_bfloat16* xb = x + (int64_t)n * P.h * P.w * kTC;
  constexpr int kPer = (kPatch * kPatch + kThreads / 8 - 1) / (kThreads / 8);  // patch pixels per thread
  uint4 raw[kPer];
  bool ok[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {  // all loads in flight before any use
    const int q = (threadIdx.x >> 3) + i * (kThreads / 8);
    const int pr = q / kPatch, pc = q % kPatch;
    const int ih = ih0 + pr, iw = iw0 + pc;
    ok[i] = q < kPatch * kPatch && ih >= 0 && ih < P.h && iw >= 0 && iw < P.w;
    if (ok[i]) raw[i] = __ldg(reinterpret_cast<const uint4*>(xb + ((int64_t)ih * P.w + iw) * kTC + oct * 8));
  }
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int q = (threadIdx.x >> 3) + i * (kThreads / 8);
    if (q >= kPatch * kPatch) break;
    uint4 u;
    __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&u);
    if (ok[i]) {
      const __nv_bfloat162* rv = reinterpret_cast<const __nv_bfloat162*>(&raw[i]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(rv[e]);
        hv[e] = __floats2bfloat162_rn(act(f.x, sc[2 * e], sh[2 * e]), act(f.y, sc[2 * e + 1], sh[2 * e + 1]));
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) hv[e] = __floats2bfloat162_rn(-INFINITY, -INFINITY);
    }
    *reinterpret_cast<uint4*>(patch + q * kPixStride + oct * 8) = u;
  }
  __syncthreads();
  // phase 2: one output octet per thread and pass (8 x 8 pixels x 8 octets = 2 passes)
  for (int t = threadIdx.x; t < kTile * kTile * 8; t += kThreads) {
    const int o8 = t & 7, op = t >> 3;
    const int lr = op / kTile, lc = op % kTile;
    const int oh = oh0 + lr, ow = ow0 + lc;
    if (oh >= P.oh || ow >= P.ow) continue;
    if constexpr (!ARGMAX) {
      // forward: packed bf16x2 max over the window (NaN-propagating like aten's
      // max_pool; the max of bf16 values is one of them, so no rounding)
      const __nv_bfloat16* pp = patch + (2 * lr * kPatch + 2 * lc) * kPixStride + o8 * 8;
      uint4 m = *reinterpret_cast<const uint4*>(pp);
      __nv_bfloat162* mh = reinterpret_cast<__nv_bfloat162*>(&m);
#pragma unroll
      for (int kk = 1; kk < 9; ++kk) {
        const uint4 u = *reinterpret_cast<const uint4*>(pp + ((kk / 3) * kPatch + kk % 3) * kPixStride);
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) mh[e] = __hmax2_nan(mh[e], hv[e]);
      }
      *reinterpret_cast<uint4*>(y + (((int64_t)n * P.oh + oh) * P.ow + ow) * kTC + o8 * 8) = m;
      continue;
    }
    float mx[8];
    int am[8];
    // argmax (backward): the packed max first; without a NaN, the index is the
    // first window position equal to it (aten's strict '>' keeps the first of
    // ties), found scanning backwards so the last match written is the first
    const __nv_bfloat16* pp = patch + (2 * lr * kPatch + 2 * lc) * kPixStride + o8 * 8;
    uint4 m = *reinterpret_cast<const uint4*>(pp);
    __nv_bfloat162* mh = reinterpret_cast<__nv_bfloat162*>(&m);
#pragma unroll
    for (int kk = 1; kk < 9; ++kk) {
      const uint4 u = *reinterpret_cast<const uint4*>(pp + ((kk / 3) * kPatch + kk % 3) * kPixStride);
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) mh[e] = __hmax2_nan(mh[e], hv[e]);
    }
    bool nan_seen = false;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(mh[e]);
      mx[2 * e] = f.x;
      mx[2 * e + 1] = f.y;
      nan_seen |= isnan(f.x) || isnan(f.y);
    }
    if (!nan_seen) {
#pragma unroll
      for (int j = 0; j < 8; ++j) am[j] = 0;
#pragma unroll
      for (int kk = 8; kk > 0; --kk) {
        const uint4 u = *reinterpret_cast<const uint4*>(pp + ((kk / 3) * kPatch + kk % 3) * kPixStride);
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(hv[e]);
          am[2 * e] = f.x == mx[2 * e] ? kk : am[2 * e];
          am[2 * e + 1] = f.y == mx[2 * e + 1] ? kk : am[2 * e + 1];
        }
      }
      // position 0 wins whenever it equals the max: am stays 0 unless a later match was the first
      {
        const uint4 u = *reinterpret_cast<const uint4*>(pp);
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(hv[e]);
          am[2 * e] = f.x == mx[2 * e] ? 0 : am[2 * e];
          am[2 * e + 1] = f.y == mx[2 * e + 1] ? 0 : am[2 * e + 1];
        }
      }
    } else
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      mx[j] = -INFINITY;
      am[j] = -1;
    }
    if (nan_seen)
#pragma unroll
    for (int kh = 0; kh < 3; ++kh) {
#pragma unroll
      for (int kw = 0; kw < 3; ++kw) {
        const uint4 u = *reinterpret_cast<const uint4*>(patch + ((2 * lr + kh) * kPatch + 2 * lc + kw) * kPixStride + o8 * 8);
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float2 f = __bfloat1622float2(hv[j / 2]);
          float a = j & 1 ? f.y : f.x;
          if (a > mx[j] || isnan(a)) {
            mx[j] = a;
            am[j] = kh * 3 + kw;
          }
        }
      }
    }
    const int64_t o = (((int64_t)n * P.oh + oh) * P.ow + ow) * kTC + o8 * 8;
    if (ARGMAX) {
      uint2 packed;
      packed.x = (uint32_t)am[0] | ((uint32_t)am[1] << 8) | ((uint32_t)am[2] << 16) | ((uint32_t)am[3] << 24);
      packed.y = (uint32_t)am[4] | ((uint32_t)am[5] << 8) | ((uint32_t)am[6] << 16) | ((uint32_t)am[7] << 24);
      *reinterpret_cast<uint2*>(arg_out + o) = packed;
    } else {
      uint4 u;
      __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int e = 0; e < 4; ++e) hv[e] = __floats2bfloat162_rn(mx[2 * e], mx[2 * e + 1]);
      *reinterpret_cast<uint4*>(y + o) = u;
    }
  }
}

bool stem_tiled(const Pool& P) { return P.k == 3 && P.s == 2 && P.p == 1 && P.c == kTC; }

int stem_tiles(const Pool& P) {
  return P.n * ((P.oh + kTile - 1) / kTile) * ((P.ow + kTile - 1) / kTile);
}

// phase 2: gather, per input pixel, the output gradients of the windows whose
// argmax it is (aten's max_pool_backward_nhwc order and fp32 accumulation)
__global__ void __launch_bounds__(kThreads) maxpool_bwd_gather_kernel(const __nv_bfloat16* __restrict__ dy,
                                                                      const uint8_t* __restrict__ arg,
                                                                      __nv_bfloat16* __restrict__ dx, Pool P) {
  const int oc = P.c / 8;
  const int64_t total = (int64_t)P.n * P.h * P.w * oc;
  for (int64_t t = (int64_t)blockIdx.x * kThreads + threadIdx.x; t < total; t += (int64_t)gridDim.x * kThreads) {
    const int c0 = (int)(t % oc) * 8;
    int64_t pix = t / oc;
    const int iw = (int)(pix % P.w);
    pix /= P.w;
    const int ih = (int)(pix % P.h);
    const int n = (int)(pix / P.h);
    // windows oh with oh*s - p <= ih <= oh*s - p + k - 1
    const int phs = (ih + P.p < P.k) ? 0 : (ih + P.p - P.k) / P.s + 1;
    const int phe = min((ih + P.p) / P.s + 1, P.oh);
    const int pws = (iw + P.p < P.k) ? 0 : (iw + P.p - P.k) / P.s + 1;
    const int pwe = min((iw + P.p) / P.s + 1, P.ow);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const bool small = (phe - phs) <= 2 && (pwe - pws) <= 2;
    if (small) {  // k <= 2s (the 3x3/s2 stem): at most 2x2 windows, loads issued together
      uint2 a[4];
      uint4 d[4];
      bool ok[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int oh = phs + (q >> 1), ow = pws + (q & 1);
        ok[q] = oh < phe && ow < pwe;
        if (ok[q]) {
          const int64_t o = (((int64_t)n * P.oh + oh) * P.ow + ow) * P.c + c0;
          a[q] = __ldg(reinterpret_cast<const uint2*>(arg + o));
          d[q] = __ldg(reinterpret_cast<const uint4*>(dy + o));
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // (oh, ow) scan order, as aten
        if (!ok[q]) continue;
        const int oh = phs + (q >> 1), ow = pws + (q & 1);
        const int me = (ih - (oh * P.s - P.p)) * P.k + (iw - (ow * P.s - P.p));
        const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&d[q]);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t word = j < 4 ? a[q].x : a[q].y;
          const int sel = (int)((word >> (8 * (j & 3))) & 0xff);
          float2 tv = __bfloat1622float2(hv[j / 2]);
          if (sel == me) acc[j] += j & 1 ? tv.y : tv.x;
        }
      }
    } else {
      for (int oh = phs; oh < phe; ++oh) {
        for (int ow = pws; ow < pwe; ++ow) {
          const int me = (ih - (oh * P.s - P.p)) * P.k + (iw - (ow * P.s - P.p));
          const int64_t o = (((int64_t)n * P.oh + oh) * P.ow + ow) * P.c + c0;
          const uint2 a = __ldg(reinterpret_cast<const uint2*>(arg + o));
          float d[8];
          load_bf8(dy + o, d);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t word = j < 4 ? a.x : a.y;
            const int sel = (int)((word >> (8 * (j & 3))) & 0xff);
            if (sel == me) acc[j] += d[j];
          }
        }
      }
    }
    uint4 u;
    __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) hv[k] = __floats2bfloat162_rn(acc[2 * k], acc[2 * k + 1]);
    *reinterpret_cast<uint4*>(dx + t * 8) = u;
  }
}

// the stem's gather (k 3, s 2, p 1, C 64; fewer than 2^31 threads): 32-bit
// index math with constant divisors, the same (oh, ow) scan order and fp32 sums
__global__ void __launch_bounds__(kThreads) stem_gather_kernel(const __nv_bfloat16* __restrict__ dy,
                                                               const uint8_t* __restrict__ arg,
                                                               __nv_bfloat16* __restrict__ dx, Pool P) {
  const uint32_t total = (uint32_t)P.n * P.h * P.w * 8;
  for (uint32_t t = blockIdx.x * kThreads + threadIdx.x; t < total; t += gridDim.x * kThreads) {
    const uint32_t oct = t & 7, pix = t >> 3;
    const int iw = (int)(pix % (uint32_t)P.w);
    const uint32_t rest = pix / (uint32_t)P.w;
    const int ih = (int)(rest % (uint32_t)P.h);
    const uint32_t n = rest / (uint32_t)P.h;
    const int phs = ih >= 2 ? ih >> 1 : 0, phe = min(((ih + 1) >> 1) + 1, P.oh);
    const int pws = iw >= 2 ? iw >> 1 : 0, pwe = min(((iw + 1) >> 1) + 1, P.ow);
    uint2 a[4];
    uint4 d[4];
    bool ok[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int oh = phs + (q >> 1), ow = pws + (q & 1);
      ok[q] = oh < phe && ow < pwe;
      if (ok[q]) {
        const uint32_t o = ((n * P.oh + oh) * P.ow + ow) * 64 + oct * 8;
        a[q] = __ldg(reinterpret_cast<const uint2*>(arg + o));
        d[q] = __ldg(reinterpret_cast<const uint4*>(dy + o));
      }
    }
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!ok[q]) continue;
      const int oh = phs + (q >> 1), ow = pws + (q & 1);
      const int me = (ih - 2 * oh + 1) * 3 + (iw - 2 * ow + 1);
      const __nv_bfloat162* hv = reinterpret_cast<const __nv_bfloat162*>(&d[q]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t word = j < 4 ? a[q].x : a[q].y;
        const int sel = (int)((word >> (8 * (j & 3))) & 0xff);
        float2 tv = __bfloat1622float2(hv[j / 2]);
        if (sel == me) acc[j] += j & 1 ? tv.y : tv.x;
      }
    }
    uint4 u;
    __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) hv[k] = __floats2bfloat162_rn(acc[2 * k], acc[2 * k + 1]);
    *reinterpret_cast<uint4*>(dx + (size_t)t * 8) = u;
  }
}

int grid_for(int64_t total) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = (total + kThreads - 1) / kThreads;
  int64_t cap = (int64_t)sms * 8;  // 8 resident 256-thread CTAs per SM
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

bool pool_ok(const Pool& P) {
  return P.n > 0 && P.h > 0 && P.w > 0 && P.c >= 8 && P.c % 8 == 0 && P.k >= 1 && P.k <= 16 && P.s >= 1 &&
         P.p >= 0 && P.p < P.k && P.oh == (P.h + 2 * P.p - P.k) / P.s + 1 && P.ow == (P.w + 2 * P.p - P.k) / P.s + 1;
}

}  // namespace

cudaError_t bn_relu_maxpool(const void* x, const float* mean, const float* invstd, const void* g, const void* b,
                            void* y, int n, int h, int w, int c, int k, int s, int p, cudaStream_t st) {
  Pool P{n, h, w, c, (h + 2 * p - k) / s + 1, (w + 2 * p - k) / s + 1, k, s, p};
  if (!pool_ok(P)) return cudaErrorInvalidValue;
  const int64_t total = (int64_t)n * P.oh * P.ow * (c / 8);
  if (stem_tiled(P)) {
    stem_pool_tiled_kernel<false><<<stem_tiles(P), kThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), mean, invstd, static_cast<const __nv_bfloat16*>(g),
        static_cast<const __nv_bfloat16*>(b), static_cast<__nv_bfloat16*>(y), nullptr, P);
    return cudaGetLastError();
  }
  auto go = [&](auto kernel) {
    kernel<<<grid_for(total), kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(x), mean, invstd,
                                                  static_cast<const __nv_bfloat16*>(g),
                                                  static_cast<const __nv_bfloat16*>(b),
                                                  static_cast<__nv_bfloat16*>(y), P);
  };
  if (k == 3) go(bn_relu_maxpool_kernel<3>);
  else go(bn_relu_maxpool_kernel<0>);
  return cudaGetLastError();
}

size_t bn_relu_maxpool_bwd_workspace(int n, int h, int w, int c, int k, int s, int p) {
  const int64_t oh = (h + 2 * p - k) / s + 1, ow = (w + 2 * p - k) / s + 1;
  return (size_t)(n * oh * ow * c);
}

cudaError_t bn_relu_maxpool_bwd(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                                const void* b, void* dx, void* ws, int n, int h, int w, int c, int k, int s, int p,
                                cudaStream_t st) {
  Pool P{n, h, w, c, (h + 2 * p - k) / s + 1, (w + 2 * p - k) / s + 1, k, s, p};
  if (!pool_ok(P) || P.k * P.k > 255) return cudaErrorInvalidValue;
  auto* arg = static_cast<uint8_t*>(ws);
  const int64_t outs = (int64_t)n * P.oh * P.ow * (c / 8);
  auto go = [&](auto kernel) {
    kernel<<<grid_for(outs), kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(x), mean, invstd,
                                                 static_cast<const __nv_bfloat16*>(g),
                                                 static_cast<const __nv_bfloat16*>(b), arg, P);
  };
  if (stem_tiled(P))
    stem_pool_tiled_kernel<true><<<stem_tiles(P), kThreads, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), mean, invstd, static_cast<const __nv_bfloat16*>(g),
        static_cast<const __nv_bfloat16*>(b), nullptr, arg, P);
  else if (k == 3) go(maxpool_argmax_kernel<3>);
  else go(maxpool_argmax_kernel<0>);
  const int64_t ins = (int64_t)n * h * w * (c / 8);
  if (stem_tiled(P) && ins < (int64_t(1) << 31))
    stem_gather_kernel<<<grid_for(ins), kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(dy), arg,
                                                           static_cast<__nv_bfloat16*>(dx), P);
  else
    maxpool_bwd_gather_kernel<<<grid_for(ins), kThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(dy), arg,
                                                                   static_cast<__nv_bfloat16*>(dx), P);
  return cudaGetLastError();
}

}  // namespace krt
