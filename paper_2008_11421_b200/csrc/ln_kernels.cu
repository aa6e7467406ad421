// Transformer-layer elementwise work for the GPT units (sm_100a), bf16 rows
// [T, H] with H % 8 == 0:
//
//   ln_fwd          : h = LayerNorm(x [+ r]) with the sum x2 = x + r stored
//                     (the residual add fused in front of the norm), and
//                     the row mean / rstd (fp32) the backward needs.  Used for
//                     the forward and for the backward's recompute, so the
//                     recomputed h is bitwise the forward's.
//   ln_bwd          : LayerNorm backward in one pass over dy and x: dx (+ an
//                     addend: the residual branch's gradient) and the
//                     gamma / beta gradients, deterministic (fixed row ->
//                     CTA mapping, fixed-order shared-memory column sums,
//                     a double-precision finalize over the CTA partials).
//   gelu_bwd_colsum : df = gelu'(f) * dg (tanh GELU) and, in the same pass,
//                     the column sums of df (fc1's bias gradient): no second
//                     read of the widest activation of the layer.
//
// LayerNorm: one warp per row, 16-byte vectors; mean from the rounded x2,
// variance by a second pass over x2 (L2-resident re-read), both in fp32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ln_kernels.hpp"

namespace krt {
namespace {

constexpr int kRowsPerCta = 8;  // one warp per row

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 t = __bfloat1622float2(h[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
  return u;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <bool RES>
__global__ void __launch_bounds__(32 * kRowsPerCta) ln_fwd_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ r, __nv_bfloat16* __restrict__ x2,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ h,
    float* __restrict__ mean, float* __restrict__ rstd, int64_t T, int H, float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kRowsPerCta + (threadIdx.x >> 5);
  if (row >= T) return;
  const int oct = H / 8;
  const __nv_bfloat16* xr = x + row * H;
  const __nv_bfloat16* src = RES ? x2 + row * H : xr;  // what the norm reads back
  // pass 1: (x + r) rounded to bf16, stored; row sum
  float s = 0.f;
  for (int j = lane; j < oct; j += 32) {
    float a[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(xr) + j), a);
    if (RES) {
      float c[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(r + row * H) + j), c);
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = __fadd_rn(a[k], c[k]);
      const uint4 u = pack8(a);
      reinterpret_cast<uint4*>(x2 + row * H)[j] = u;
      unpack8(u, a);  // the stored, rounded values
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
  }
  const float mu = warp_sum(s) / (float)H;
  // pass 2: variance about the mean (re-read, L1/L2 resident)
  float q = 0.f;
  for (int j = lane; j < oct; j += 32) {
    float a[8];
    unpack8(reinterpret_cast<const uint4*>(src)[j], a);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float d = a[k] - mu;
      q = __fmaf_rn(d, d, q);
    }
  }
  const float rs = rsqrtf(warp_sum(q) / (float)H + eps);
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
  // pass 3: normalise
  for (int j = lane; j < oct; j += 32) {
    float a[8], gg[8], bb[8];
    unpack8(reinterpret_cast<const uint4*>(src)[j], a);
    unpack8(__ldg(reinterpret_cast<const uint4*>(g) + j), gg);
    unpack8(__ldg(reinterpret_cast<const uint4*>(b) + j), bb);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __fmaf_rn((a[k] - mu) * rs, gg[k], bb[k]);
    reinterpret_cast<uint4*>(h + row * H)[j] = pack8(a);
  }
}

// H <= 32 * 8 * J: the row lives in registers (J octets per lane), one read of
// x (and r), all loads in flight before the reductions; same arithmetic as
// ln_fwd_kernel (mean of the rounded sum, variance about it, fp32)
template <bool RES, int J>
__global__ void __launch_bounds__(32 * kRowsPerCta) ln_fwd_reg_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ r, __nv_bfloat16* __restrict__ x2,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ h,
    float* __restrict__ mean, float* __restrict__ rstd, int64_t T, int H, float eps) {
  const int lane = threadIdx.x & 31;
  const int oct = H / 8;
  // persistent: warps stride the rows.  The row stays packed (bf16, 4
  // registers per octet) and is unpacked per pass: half the registers of an
  // fp32 copy, so twice the warps (rows in flight) per SM.
  for (int64_t row = (int64_t)blockIdx.x * kRowsPerCta + (threadIdx.x >> 5); row < T;
       row += (int64_t)gridDim.x * kRowsPerCta) {
    uint4 ux[J];
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = lane + 32 * i;
      if (j < oct) ux[i] = __ldcs(reinterpret_cast<const uint4*>(x + row * H) + j);
    }
    if (RES) {
      uint4 ur[J];
#pragma unroll
      for (int i = 0; i < J; ++i) {
        const int j = lane + 32 * i;
        if (j < oct) ur[i] = __ldcs(reinterpret_cast<const uint4*>(r + row * H) + j);
      }
#pragma unroll
      for (int i = 0; i < J; ++i) {
        const int j = lane + 32 * i;
        if (j < oct) {
          float a[8], c[8];
          unpack8(ux[i], a);
          unpack8(ur[i], c);
#pragma unroll
          for (int k = 0; k < 8; ++k) a[k] = __fadd_rn(a[k], c[k]);
          ux[i] = pack8(a);  // the stored, rounded sum
          reinterpret_cast<uint4*>(x2 + row * H)[j] = ux[i];
        }
      }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < J; ++i) {
      if (lane + 32 * i < oct) {
        float a[8];
        unpack8(ux[i], a);
#pragma unroll
        for (int k = 0; k < 8; ++k) s += a[k];
      }
    }
    const float mu = warp_sum(s) / (float)H;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < J; ++i) {
      if (lane + 32 * i < oct) {
        float a[8];
        unpack8(ux[i], a);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float d = a[k] - mu;
          q = __fmaf_rn(d, d, q);
        }
      }
    }
    const float rs = rsqrtf(warp_sum(q) / (float)H + eps);
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = lane + 32 * i;
      if (j < oct) {
        float a[8], gg[8], bb[8];
        unpack8(ux[i], a);
        unpack8(__ldg(reinterpret_cast<const uint4*>(g) + j), gg);
        unpack8(__ldg(reinterpret_cast<const uint4*>(b) + j), bb);
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __fmaf_rn((a[k] - mu) * rs, gg[k], bb[k]);
        reinterpret_cast<uint4*>(h + row * H)[j] = pack8(a);
      }
    }
  }
}

// tanh-GELU derivative, the formula of aten's GeluBackward (tanh), in fp32
// (the hardware tanh keeps the pass memory-bound: with tanhf it was ALU-bound)
__device__ __forceinline__ float gelu_tanh_grad(float dy, float x) {
  constexpr float kBeta = 0.7978845608028654f;  // sqrt(2 / pi)
  constexpr float kKappa = 0.044715f;
  const float x_sq = x * x;
  const float x_cube = x_sq * x;
  const float inner = kBeta * (x + kKappa * x_cube);
  float t;  // MUFU tanh: ~2^-11 relative error, far below the bf16 rounding of the result
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(inner));
  const float left = 0.5f * x;
  const float right = 1.f + t;
  const float left_d = 0.5f * right;
  const float tanh_d = 1.f - t * t;
  const float inner_d = kBeta * (1.f + 3.f * kKappa * x_sq);
  const float right_d = left * tanh_d * inner_d;
  return dy * (left_d + right_d);
}

constexpr int kColThreads = 256;   // 8 columns each: 2048 columns per CTA
constexpr int kColRows = 256;      // rows per CTA (one partial row)

__global__ void __launch_bounds__(kColThreads) gelu_bwd_colsum_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ f, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ part, int64_t T, int N) {
  const int col = (blockIdx.x * kColThreads + threadIdx.x) * 8;
  const int64_t r0 = (int64_t)blockIdx.y * kColRows;
  if (col >= N) return;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t r1 = r0 + kColRows < T ? r0 + kColRows : T;
  for (int64_t r = r0; r < r1; r += 4) {  // four rows in flight
    uint4 ud[4], uf[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (r + u < r1) {
        ud[u] = __ldcs(reinterpret_cast<const uint4*>(dy + (r + u) * N + col));
        uf[u] = __ldcs(reinterpret_cast<const uint4*>(f + (r + u) * N + col));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (r + u < r1) {
        float d[8], xv[8], o[8];
        unpack8(ud[u], d);
        unpack8(uf[u], xv);
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = gelu_tanh_grad(d[k], xv[k]);
        const uint4 p = pack8(o);
        *reinterpret_cast<uint4*>(dx + (r + u) * N + col) = p;
        unpack8(p, o);  // the bias gradient sums the stored (rounded) values
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] += o[k];
      }
    }
  }
  float* out = part + (int64_t)blockIdx.y * N + col;
  *reinterpret_cast<float4*>(out) = make_float4(acc[0], acc[1], acc[2], acc[3]);
  *reinterpret_cast<float4*>(out + 4) = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

// column sums of the partial rows: CTA = 32 columns x 32 warps striding the
// rows, then a fixed-order pass over the warps in double (deterministic)
__global__ void __launch_bounds__(1024) colsum_finalize_kernel(const float* __restrict__ part, int rows, int N,
                                                               float* __restrict__ out) {
  __shared__ double sh[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double s = 0;
  if (c < N)
    for (int r = w; r < rows; r += 32) s += (double)part[(size_t)r * N + c];
  sh[w][lane] = s;
  __syncthreads();
  if (w != 0 || c >= N) return;
  s = 0;
  for (int k = 0; k < 32; ++k) s += sh[k][lane];
  out[c] = (float)s;
}

// LayerNorm backward.  One warp per row, rows strided over a persistent grid;
// the row (dy, x and the addend) is loaded packed into registers with every
// load in flight at once (J octets per lane), the two row sums reduced by
// shuffles, dx stored.  Each warp adds its rows' dy*xhat and dy into its own
// fp32 column accumulators in shared memory ([2][8][H/8]: lane j owns the
// columns of octets j, j+32, ..., so no two lanes touch a word and no
// barrier is needed per row); at the end the CTA sums its warps in warp order
// into one partial row pair.  Deterministic for a given grid.
constexpr int kBwdWarps = 4;

template <bool ADD, int J>
__global__ void __launch_bounds__(32 * kBwdWarps) ln_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
    const float* __restrict__ mean, const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ addend,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ part, int64_t T, int H) {
  extern __shared__ float stage[];  // [kBwdWarps][2][8][H / 8]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int oct = H / 8;
  float* ag = stage + (size_t)w * 2 * H;  // this warp's sum of dy*xhat, [8][oct]
  float* ab = ag + H;                     // and of dy
  for (int c = lane; c < H; c += 32) ag[c] = ab[c] = 0.f;
  const float inv_h = 1.f / (float)H;
  for (int64_t row = (int64_t)blockIdx.x * kBwdWarps + w; row < T; row += (int64_t)gridDim.x * kBwdWarps) {
    uint4 ud[J], ux[J], ua[ADD ? J : 1];
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = lane + 32 * i;
      if (j < oct) {
        ud[i] = __ldcs(reinterpret_cast<const uint4*>(dy + row * H) + j);
        ux[i] = __ldcs(reinterpret_cast<const uint4*>(x + row * H) + j);
        if (ADD) ua[i] = __ldcs(reinterpret_cast<const uint4*>(addend + row * H) + j);
      }
    }
    const float mu = __ldg(mean + row), rs = __ldg(rstd + row);
    float s1 = 0.f, s2 = 0.f;  // sum g*dy, sum g*dy*xhat
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = lane + 32 * i;
      if (j < oct) {
        float d[8], xv[8], gg[8];
        unpack8(ud[i], d);
        unpack8(ux[i], xv);
        unpack8(__ldg(reinterpret_cast<const uint4*>(g) + j), gg);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (xv[k] - mu) * rs;
          const float gd = d[k] * gg[k];
          s1 += gd;
          s2 = __fmaf_rn(gd, xh, s2);
          ag[k * oct + j] += d[k] * xh;
          ab[k * oct + j] += d[k];
        }
      }
    }
    const float c1 = warp_sum(s1) * inv_h, c2 = warp_sum(s2) * inv_h;
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = lane + 32 * i;
      if (j < oct) {
        float d[8], xv[8], gg[8], o[8];
        unpack8(ud[i], d);
        unpack8(ux[i], xv);
        unpack8(__ldg(reinterpret_cast<const uint4*>(g) + j), gg);
        if (ADD) unpack8(ua[i], o);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (xv[k] - mu) * rs;
          const float v = rs * (d[k] * gg[k] - c1 - xh * c2);
          o[k] = ADD ? __fadd_rn(v, o[k]) : v;
        }
        __stcs(reinterpret_cast<uint4*>(dx + row * H) + j, pack8(o));
      }
    }
  }
  __syncthreads();
  // this CTA's partial row pair: its warps' accumulators added in warp order
  for (int c = threadIdx.x; c < 2 * H; c += 32 * kBwdWarps) {
    float s = 0.f;
#pragma unroll
    for (int r = 0; r < kBwdWarps; ++r) s += stage[(size_t)r * 2 * H + c];
    // [2][8][oct] -> [2][H] column order
    const int half = c / H, rem = c - half * H, k = rem / oct, j = rem - k * oct;
    part[(size_t)blockIdx.x * 2 * H + half * H + 8 * j + k] = s;
  }
}

// dgamma / dbeta from the CTA partial rows: part [rows][2][H] -> out_g, out_b
__global__ void __launch_bounds__(1024) ln_bwd_finalize_kernel(const float* __restrict__ part, int rows, int H,
                                                               float* __restrict__ out_g, float* __restrict__ out_b) {
  __shared__ double sh[2][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double sgm = 0, sbt = 0;
  if (c < H)
    for (int r = w; r < rows; r += 32) {
      sgm += (double)part[(size_t)r * 2 * H + c];
      sbt += (double)part[(size_t)r * 2 * H + H + c];
    }
  sh[0][w][lane] = sgm;
  sh[1][w][lane] = sbt;
  __syncthreads();
  if (w != 0 || c >= H) return;
  sgm = sbt = 0;
  for (int k = 0; k < 32; ++k) {
    sgm += sh[0][k][lane];
    sbt += sh[1][k][lane];
  }
  out_g[c] = (float)sgm;
  out_b[c] = (float)sbt;
}

int ln_bwd_grid(int64_t T) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (T + kBwdWarps - 1) / kBwdWarps, cap = (int64_t)sms * 4;
  return (int)(want < cap ? want : cap);
}

template <bool ADD, int J>
cudaError_t launch_ln_bwd(const void* dy, const void* x, const void* g, const float* mean, const float* rstd,
                          const void* addend, void* dx, float* part, int grid, int64_t T, int H, cudaStream_t s) {
  const size_t smem = (size_t)kBwdWarps * 2 * H * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(ln_bwd_kernel<ADD, J>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ln_bwd_kernel<ADD, J><<<grid, 32 * kBwdWarps, smem, s>>>(
      static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x),
      static_cast<const __nv_bfloat16*>(g), mean, rstd, static_cast<const __nv_bfloat16*>(addend),
      static_cast<__nv_bfloat16*>(dx), part, T, H);
  return cudaGetLastError();
}

template <bool ADD>
cudaError_t ln_bwd_dispatch(const void* dy, const void* x, const void* g, const float* mean, const float* rstd,
                            const void* addend, void* dx, float* part, int grid, int64_t T, int H, cudaStream_t s) {
  const int oct = H / 8;
  if (oct <= 32 * 2) return launch_ln_bwd<ADD, 2>(dy, x, g, mean, rstd, addend, dx, part, grid, T, H, s);
  if (oct <= 32 * 4) return launch_ln_bwd<ADD, 4>(dy, x, g, mean, rstd, addend, dx, part, grid, T, H, s);
  if (oct <= 32 * 8) return launch_ln_bwd<ADD, 8>(dy, x, g, mean, rstd, addend, dx, part, grid, T, H, s);
  if (oct <= 32 * 12) return launch_ln_bwd<ADD, 12>(dy, x, g, mean, rstd, addend, dx, part, grid, T, H, s);
  return launch_ln_bwd<ADD, 17>(dy, x, g, mean, rstd, addend, dx, part, grid, T, H, s);
}

}  // namespace

size_t ln_bwd_workspace(int64_t T, int H) { return (size_t)ln_bwd_grid(T) * 2 * H * sizeof(float); }

cudaError_t ln_bwd(const void* dy, const void* x, const void* g, const float* mean, const float* rstd,
                   const void* addend, void* dx, float* dgamma, float* dbeta, void* ws, int64_t T, int H,
                   cudaStream_t s) {
  if (T <= 0 || H <= 0 || H % 8 != 0 || H > 32 * 17 * 8) return cudaErrorInvalidValue;
  const int grid = ln_bwd_grid(T);
  float* part = static_cast<float*>(ws);
  cudaError_t e = addend ? ln_bwd_dispatch<true>(dy, x, g, mean, rstd, addend, dx, part, grid, T, H, s)
                         : ln_bwd_dispatch<false>(dy, x, g, mean, rstd, addend, dx, part, grid, T, H, s);
  if (e != cudaSuccess) return e;
  ln_bwd_finalize_kernel<<<(H + 31) / 32, 1024, 0, s>>>(part, grid, H, dgamma, dbeta);
  return cudaGetLastError();
}

cudaError_t ln_fwd(const void* x, const void* r, void* x2, const void* g, const void* b, void* h, float* mean,
                   float* rstd, int64_t T, int H, float eps, cudaStream_t s) {
  if (T <= 0 || H <= 0 || H % 8 != 0 || (r != nullptr && x2 == nullptr)) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)((T + kRowsPerCta - 1) / kRowsPerCta));
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto R = static_cast<const __nv_bfloat16*>(r);
  auto X2 = static_cast<__nv_bfloat16*>(x2);
  auto G = static_cast<const __nv_bfloat16*>(g);
  auto B = static_cast<const __nv_bfloat16*>(b);
  auto Hh = static_cast<__nv_bfloat16*>(h);
  const int oct = H / 8;
  if (oct <= 32 * 8) {  // row in registers, persistent grid
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (T + kRowsPerCta - 1) / kRowsPerCta, cap = (int64_t)sms * 8;
    const dim3 pgrid((unsigned)(want < cap ? want : cap));
    if (r) ln_fwd_reg_kernel<true, 8><<<pgrid, 32 * kRowsPerCta, 0, s>>>(X, R, X2, G, B, Hh, mean, rstd, T, H, eps);
    else ln_fwd_reg_kernel<false, 8><<<pgrid, 32 * kRowsPerCta, 0, s>>>(X, R, X2, G, B, Hh, mean, rstd, T, H, eps);
  } else if (r) {
    ln_fwd_kernel<true><<<grid, 32 * kRowsPerCta, 0, s>>>(X, R, X2, G, B, Hh, mean, rstd, T, H, eps);
  } else {
    ln_fwd_kernel<false><<<grid, 32 * kRowsPerCta, 0, s>>>(X, R, X2, G, B, Hh, mean, rstd, T, H, eps);
  }
  return cudaGetLastError();
}

size_t gelu_bwd_colsum_workspace(int64_t T, int N) {
  return (size_t)((T + kColRows - 1) / kColRows) * N * sizeof(float);
}

cudaError_t gelu_bwd_colsum(const void* dy, const void* f, void* dx, float* colsum, void* ws, int64_t T, int N,
                            cudaStream_t s) {
  if (T <= 0 || N <= 0 || N % 8 != 0) return cudaErrorInvalidValue;
  const int rb = (int)((T + kColRows - 1) / kColRows);
  const dim3 grid((unsigned)((N / 8 + kColThreads - 1) / kColThreads), (unsigned)rb);
  float* part = static_cast<float*>(ws);
  gelu_bwd_colsum_kernel<<<grid, kColThreads, 0, s>>>(static_cast<const __nv_bfloat16*>(dy),
                                                      static_cast<const __nv_bfloat16*>(f),
                                                      static_cast<__nv_bfloat16*>(dx), part, T, N);
  colsum_finalize_kernel<<<(N + 31) / 32, 1024, 0, s>>>(part, rb, N, colsum);
  return cudaGetLastError();
}

}  // namespace krt
