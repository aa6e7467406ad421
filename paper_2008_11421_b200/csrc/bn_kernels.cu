// Fused batch-norm kernels for NHWC bf16 activations (sm_100a).
//
// The ResNet units' hot elementwise work ("warp-level fused
// elementwise/norm kernels elsewhere").  All are HBM-bound streaming kernels
// over a [rows, C] matrix (rows = N*H*W, C contiguous, C % 8 == 0):
//
//   stats     : per-channel mean / invstd (batch statistics)       1R
//   apply     : y = relu?(bn(x) [+ res | + bn'(res)])               1-2R + 1W
//   add_relu_bwd_mask : dz = dy * (bn(x) + (res | bn'(res)) > 0)    2-3R + 1W
//   bwd       : dgamma, dbeta (reduce) and dx (elementwise), with the
//               ReLU mask recomputed from x when the BN feeds a ReLU   2R + 2R+1W
//
// Thread mapping: a thread owns 8 consecutive channels (one 16-byte vector)
// for its whole life, so per-channel scale/shift stay in registers; the rows
// are grid-strided.  Reductions: per-thread fp32 partials -> shared-memory
// tree over the rows of a CTA -> one fp32 partial per CTA and channel ->
// a finalize kernel sums the CTA partials in double (fixed order:
// deterministic, so in-core and out-of-core runs stay bitwise equal).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "bn_kernels.hpp"

namespace krt {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxGrid = 148 * 4;

struct Vec8 {
  float v[8];
};

__device__ __forceinline__ Vec8 load8(const __nv_bfloat16* p) {
  uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  Vec8 r;
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float2 f = __bfloat1622float2(h[k]);
    r.v[2 * k] = f.x;
    r.v[2 * k + 1] = f.y;
  }
  return r;
}

__device__ __forceinline__ void store8(__nv_bfloat16* p, const Vec8& x) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(x.v[2 * k], x.v[2 * k + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

__device__ __forceinline__ float bf(const __nv_bfloat16* p, int i) { return __bfloat162float(p[i]); }

// threads of a CTA: tx = channel group (C/8 of them), ty = row lane
struct Map {
  int tc, rb, tx, ty;
  __device__ Map(int C) {
    tc = C / 8;
    rb = kThreads / tc;  // rows per CTA sweep (>= 1 since C <= 2048)
    tx = threadIdx.x % tc;
    ty = threadIdx.x / tc;
  }
};

// per-channel (scale, shift) of y = x*scale + shift
__device__ __forceinline__ void bn_coeffs(const float* mean, const float* invstd, const __nv_bfloat16* g,
                                          const __nv_bfloat16* b, int c0, float* sc, float* sh) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float s = invstd[c0 + k] * bf(g, c0 + k);
    sc[k] = s;
    sh[k] = bf(b, c0 + k) - mean[c0 + k] * s;
  }
}

// reduce two 8-vectors over the ty dimension of the CTA; result in ty == 0
__device__ __forceinline__ void cta_reduce2(float* a, float* b, float* smem, const Map& m) {
  // smem: [rb][tc][16]
  float* mine = smem + ((size_t)m.ty * m.tc + m.tx) * 16;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    mine[k] = a[k];
    mine[8 + k] = b[k];
  }
  __syncthreads();
  for (int s = 1; s < m.rb; s <<= 1) {
    if ((m.ty % (2 * s)) == 0 && m.ty + s < m.rb) {
      float* other = smem + ((size_t)(m.ty + s) * m.tc + m.tx) * 16;
#pragma unroll
      for (int k = 0; k < 16; ++k) mine[k] += other[k];
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    a[k] = mine[k];
    b[k] = mine[8 + k];
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) stats_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows, int C,
                                                         float* __restrict__ part) {
  extern __shared__ float smem[];
  Map m(C);
  int c0 = m.tx * 8;
  float s[8] = {0}, q[8] = {0};
  const int64_t step = (int64_t)gridDim.x * m.rb;
  int64_t r = (int64_t)blockIdx.x * m.rb + m.ty;
  for (; r + step < rows; r += 2 * step) {
    Vec8 v0 = load8(x + r * C + c0), v1 = load8(x + (r + step) * C + c0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s[k] += v0.v[k] + v1.v[k];
      q[k] += v0.v[k] * v0.v[k] + v1.v[k] * v1.v[k];
    }
  }
  if (r < rows) {
    Vec8 v = load8(x + r * C + c0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s[k] += v.v[k];
      q[k] += v.v[k] * v.v[k];
    }
  }
  cta_reduce2(s, q, smem, m);
  if (m.ty == 0) {
    float* out = part + (size_t)blockIdx.x * 2 * C;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      out[c0 + k] = s[k];
      out[C + c0 + k] = q[k];
    }
  }
}

// Sum CTA partials for 32 channels per block: lane = channel, the 32 warps
// stride over the partial rows, then a fixed-order pass over the warps
// (deterministic).  Returns the two double sums in lane c of warp 0.
constexpr int kFinWarps = 32;
__device__ __forceinline__ bool sum_partials(const float* __restrict__ part, int nblk, int C, double& s1,
                                             double& s2) {
  __shared__ double sh[2][kFinWarps][33];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int c = blockIdx.x * 32 + lane;
  double a = 0, q = 0;
  if (c < C)
    for (int b = w; b < nblk; b += kFinWarps) {
      a += part[(size_t)b * 2 * C + c];
      q += part[(size_t)b * 2 * C + C + c];
    }
  sh[0][w][lane] = a;
  sh[1][w][lane] = q;
  __syncthreads();
  if (w != 0 || c >= C) return false;
  s1 = 0;
  s2 = 0;
  for (int k = 0; k < kFinWarps; ++k) {
    s1 += sh[0][k][lane];
    s2 += sh[1][k][lane];
  }
  return true;
}

__global__ void __launch_bounds__(1024) stats_finalize(const float* __restrict__ part, int nblk, int64_t rows, int C,
                                                      float eps, float* __restrict__ mean, float* __restrict__ invstd) {
  double s, q;
  if (!sum_partials(part, nblk, C, s, q)) return;
  int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double mu = s / (double)rows;
  double var = q / (double)rows - mu * mu;
  if (var < 0) var = 0;
  mean[c] = (float)mu;
  invstd[c] = (float)(1.0 / sqrt(var + (double)eps));
}

// ---------------------------------------------------------------------------
// mode: 0 none, 1 identity residual, 2 bn(residual).  Two rows in flight
// per thread (all loads issued before the math) for memory-level parallelism.
template <int MODE, bool RELU>
__device__ __forceinline__ Vec8 apply_row(const Vec8& v, const Vec8& rv, const float* sc, const float* sh,
                                          const float* rsc, const float* rsh) {
  Vec8 o;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    o.v[k] = __fmaf_rn(v.v[k], sc[k], sh[k]);
    if (MODE == 2) o.v[k] = __fadd_rn(o.v[k], __fmaf_rn(rv.v[k], rsc[k], rsh[k]));
    if (MODE == 1) o.v[k] = __fadd_rn(o.v[k], rv.v[k]);
    if (RELU) o.v[k] = fmaxf(o.v[k], 0.0f);
  }
  return o;
}

template <int MODE, bool RELU>
__global__ void __launch_bounds__(kThreads) apply_kernel(
    const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ invstd,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, const __nv_bfloat16* __restrict__ res,
    const float* __restrict__ rmean, const float* __restrict__ rinvstd, const __nv_bfloat16* __restrict__ rg,
    const __nv_bfloat16* __restrict__ rb_, __nv_bfloat16* __restrict__ y, int64_t rows, int C) {
  Map m(C);
  int c0 = m.tx * 8;
  float sc[8], sh[8], rsc[8], rsh[8];
  bn_coeffs(mean, invstd, g, b, c0, sc, sh);
  if (MODE == 2) bn_coeffs(rmean, rinvstd, rg, rb_, c0, rsc, rsh);
  const int64_t step = (int64_t)gridDim.x * m.rb;
  int64_t r = (int64_t)blockIdx.x * m.rb + m.ty;
  Vec8 z{};
  for (; r + step < rows; r += 2 * step) {
    const int64_t o0 = r * C + c0, o1 = (r + step) * C + c0;
    Vec8 v0 = load8(x + o0), v1 = load8(x + o1);
    Vec8 q0 = z, q1 = z;
    if (MODE != 0) {
      q0 = load8(res + o0);
      q1 = load8(res + o1);
    }
    store8(y + o0, apply_row<MODE, RELU>(v0, q0, sc, sh, rsc, rsh));
    store8(y + o1, apply_row<MODE, RELU>(v1, q1, sc, sh, rsc, rsh));
  }
  if (r < rows) {
    const int64_t o0 = r * C + c0;
    Vec8 v0 = load8(x + o0), q0 = z;
    if (MODE != 0) q0 = load8(res + o0);
    store8(y + o0, apply_row<MODE, RELU>(v0, q0, sc, sh, rsc, rsh));
  }
}

// dz = dy * ( bn(x) [+ res | + bn'(res)] > 0 )   (backward of the add + ReLU);
// the forward sum is re-rounded to bf16 exactly as apply_kernel stored it
template <int MODE>
__device__ __forceinline__ Vec8 add_relu_row(const Vec8& v, const Vec8& rv, const Vec8& d, const float* sc,
                                             const float* sh, const float* rsc, const float* rsh) {
  Vec8 o;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float pre = __fadd_rn(__fmaf_rn(v.v[k], sc[k], sh[k]), MODE == 2 ? __fmaf_rn(rv.v[k], rsc[k], rsh[k]) : rv.v[k]);
    float yk = __bfloat162float(__float2bfloat16_rn(pre));
    o.v[k] = yk > 0.0f ? d.v[k] : 0.0f;
  }
  return o;
}

// dy = bf16(dy + dy2): the residual-gradient sum the next unit handed over
// unmaterialised, rounded exactly like a separate bf16 add would
__device__ __forceinline__ Vec8 add_grad(const Vec8& a, const Vec8& b) {
  Vec8 o;
#pragma unroll
  for (int k = 0; k < 8; ++k) o.v[k] = __bfloat162float(__float2bfloat16_rn(__fadd_rn(a.v[k], b.v[k])));
  return o;
}

template <int MODE, bool DY2>
__global__ void __launch_bounds__(kThreads) add_relu_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ dy2, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ mean,
    const float* __restrict__ invstd, const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b,
    const __nv_bfloat16* __restrict__ res, const float* __restrict__ rmean, const float* __restrict__ rinvstd,
    const __nv_bfloat16* __restrict__ rg, const __nv_bfloat16* __restrict__ rb_, __nv_bfloat16* __restrict__ dz,
    int64_t rows, int C) {
  Map m(C);
  int c0 = m.tx * 8;
  float sc[8], sh[8], rsc[8], rsh[8];
  bn_coeffs(mean, invstd, g, b, c0, sc, sh);
  if (MODE == 2) bn_coeffs(rmean, rinvstd, rg, rb_, c0, rsc, rsh);
  const int64_t step = (int64_t)gridDim.x * m.rb;
  int64_t r = (int64_t)blockIdx.x * m.rb + m.ty;
  for (; r + step < rows; r += 2 * step) {
    const int64_t o0 = r * C + c0, o1 = (r + step) * C + c0;
    Vec8 v0 = load8(x + o0), v1 = load8(x + o1);
    Vec8 q0 = load8(res + o0), q1 = load8(res + o1);
    Vec8 d0 = load8(dy + o0), d1 = load8(dy + o1);
    if (DY2) {
      Vec8 e0 = load8(dy2 + o0), e1 = load8(dy2 + o1);
      d0 = add_grad(d0, e0);
      d1 = add_grad(d1, e1);
    }
    store8(dz + o0, add_relu_row<MODE>(v0, q0, d0, sc, sh, rsc, rsh));
    store8(dz + o1, add_relu_row<MODE>(v1, q1, d1, sc, sh, rsc, rsh));
  }
  if (r < rows) {
    const int64_t o0 = r * C + c0;
    Vec8 v0 = load8(x + o0), q0 = load8(res + o0), d0 = load8(dy + o0);
    if (DY2) d0 = add_grad(d0, load8(dy2 + o0));
    store8(dz + o0, add_relu_row<MODE>(v0, q0, d0, sc, sh, rsc, rsh));
  }
}

// backward reduce: sum(gm) and sum(gm * xhat) with gm = dy * mask
template <bool RELU>
__device__ __forceinline__ void bwd_acc(const Vec8& v, const Vec8& d, const float* sc, const float* sh,
                                        const float* mu, const float* is, float* s1, float* s2) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float gm = d.v[k];
    if (RELU) {
      float yk = __bfloat162float(__float2bfloat16_rn(__fmaf_rn(v.v[k], sc[k], sh[k])));
      gm = yk > 0.0f ? gm : 0.0f;
    }
    s1[k] += gm;
    s2[k] += gm * ((v.v[k] - mu[k]) * is[k]);
  }
}

template <bool RELU>
__global__ void __launch_bounds__(kThreads) bwd_reduce_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ invstd, const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b,
    int64_t rows, int C, float* __restrict__ part) {
  extern __shared__ float smem[];
  Map m(C);
  int c0 = m.tx * 8;
  float sc[8], sh[8], mu[8], is[8];
  bn_coeffs(mean, invstd, g, b, c0, sc, sh);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    mu[k] = mean[c0 + k];
    is[k] = invstd[c0 + k];
  }
  float s1[8] = {0}, s2[8] = {0};
  const int64_t step = (int64_t)gridDim.x * m.rb;
  int64_t r = (int64_t)blockIdx.x * m.rb + m.ty;
  for (; r + step < rows; r += 2 * step) {
    const int64_t o0 = r * C + c0, o1 = (r + step) * C + c0;
    Vec8 v0 = load8(x + o0), v1 = load8(x + o1);
    Vec8 d0 = load8(dy + o0), d1 = load8(dy + o1);
    bwd_acc<RELU>(v0, d0, sc, sh, mu, is, s1, s2);
    bwd_acc<RELU>(v1, d1, sc, sh, mu, is, s1, s2);
  }
  if (r < rows) {
    const int64_t o0 = r * C + c0;
    Vec8 v0 = load8(x + o0), d0 = load8(dy + o0);
    bwd_acc<RELU>(v0, d0, sc, sh, mu, is, s1, s2);
  }
  cta_reduce2(s1, s2, smem, m);
  if (m.ty == 0) {
    float* out = part + (size_t)blockIdx.x * 2 * C;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      out[c0 + k] = s1[k];
      out[C + c0 + k] = s2[k];
    }
  }
}

__global__ void __launch_bounds__(1024) bwd_finalize(const float* __restrict__ part, int nblk, int64_t rows, int C,
                                                    float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                    float* __restrict__ coef) {
  double s1, s2;
  if (!sum_partials(part, nblk, C, s1, s2)) return;
  int c = blockIdx.x * 32 + (threadIdx.x & 31);
  if (dbeta) dbeta[c] = (float)s1;
  if (dgamma) dgamma[c] = (float)s2;
  coef[c] = (float)(s1 / (double)rows);
  coef[C + c] = (float)(s2 / (double)rows);
}

// dx = gamma*invstd * (gm - mean(gm) - xhat * mean(gm*xhat))
template <bool RELU>
__device__ __forceinline__ Vec8 bwd_row(const Vec8& v, const Vec8& d, const float* sc, const float* sh,
                                        const float* mu, const float* is, const float* k1, const float* k2,
                                        const float* gs) {
  Vec8 o;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float gm = d.v[k];
    if (RELU) {
      float yk = __bfloat162float(__float2bfloat16_rn(__fmaf_rn(v.v[k], sc[k], sh[k])));
      gm = yk > 0.0f ? gm : 0.0f;
    }
    float xh = (v.v[k] - mu[k]) * is[k];
    o.v[k] = gs[k] * (gm - k1[k] - xh * k2[k]);
  }
  return o;
}

template <bool RELU>
__global__ void __launch_bounds__(kThreads) bwd_elemt_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ invstd, const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b,
    const float* __restrict__ coef, __nv_bfloat16* __restrict__ dx, int64_t rows, int C) {
  Map m(C);
  int c0 = m.tx * 8;
  float sc[8], sh[8], mu[8], is[8], k1[8], k2[8], gs[8];
  bn_coeffs(mean, invstd, g, b, c0, sc, sh);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    mu[k] = mean[c0 + k];
    is[k] = invstd[c0 + k];
    k1[k] = coef[c0 + k];
    k2[k] = coef[C + c0 + k];
    gs[k] = bf(g, c0 + k) * is[k];
  }
  const int64_t step = (int64_t)gridDim.x * m.rb;
  int64_t r = (int64_t)blockIdx.x * m.rb + m.ty;
  for (; r + step < rows; r += 2 * step) {
    const int64_t o0 = r * C + c0, o1 = (r + step) * C + c0;
    Vec8 v0 = load8(x + o0), v1 = load8(x + o1);
    Vec8 d0 = load8(dy + o0), d1 = load8(dy + o1);
    store8(dx + o0, bwd_row<RELU>(v0, d0, sc, sh, mu, is, k1, k2, gs));
    store8(dx + o1, bwd_row<RELU>(v1, d1, sc, sh, mu, is, k1, k2, gs));
  }
  if (r < rows) {
    const int64_t o0 = r * C + c0;
    Vec8 v0 = load8(x + o0), d0 = load8(dy + o0);
    store8(dx + o0, bwd_row<RELU>(v0, d0, sc, sh, mu, is, k1, k2, gs));
  }
}

size_t reduce_smem(int C);

// persistent grid: one full wave of resident CTAs (148 SMs x occupancy),
// capped at kMaxGrid so the reduction partials fit the workspace
template <class K>
int grid_rows(K kernel, size_t smem, int64_t rows, int C) {
  static int resident = 0;  // per kernel instantiation
  if (resident == 0) {
    int per_sm = 0, sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
    resident = sms * (per_sm < 1 ? 1 : per_sm);
  }
  int rb = kThreads / (C / 8);
  int64_t want = (rows + rb - 1) / rb;
  int cap = resident < kMaxGrid ? resident : kMaxGrid;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

size_t reduce_smem(int C) {
  int tc = C / 8, rb = kThreads / tc;
  return (size_t)rb * tc * 16 * sizeof(float);
}

bool shape_ok(int64_t rows, int C) { return rows > 0 && C >= 8 && C % 8 == 0 && C <= 8 * kThreads && (kThreads % (C / 8)) == 0; }

}  // namespace

size_t bn_workspace_bytes(int C) { return (size_t)kMaxGrid * 2 * C * sizeof(float) + 2 * C * sizeof(float); }

cudaError_t bn_stats(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd, void* ws,
                     cudaStream_t s) {
  if (!shape_ok(rows, C)) return cudaErrorInvalidValue;
  int grid = grid_rows(stats_kernel, reduce_smem(C), rows, C);
  float* part = static_cast<float*>(ws);
  stats_kernel<<<grid, kThreads, reduce_smem(C), s>>>(static_cast<const __nv_bfloat16*>(x), rows, C, part);
  stats_finalize<<<(C + 31) / 32, 32 * kFinWarps, 0, s>>>(part, grid, rows, C, eps, mean, invstd);
  return cudaGetLastError();
}

cudaError_t bn_apply(const void* x, const float* mean, const float* invstd, const void* g, const void* b,
                     const void* res, const float* rmean, const float* rinvstd, const void* rg, const void* rb,
                     int relu, void* y, int64_t rows, int C, cudaStream_t s) {
  if (!shape_ok(rows, C)) return cudaErrorInvalidValue;
  int mode = res == nullptr ? 0 : (rmean == nullptr ? 1 : 2);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto G = static_cast<const __nv_bfloat16*>(g);
  auto B = static_cast<const __nv_bfloat16*>(b);
  auto R = static_cast<const __nv_bfloat16*>(res);
  auto RG = static_cast<const __nv_bfloat16*>(rg);
  auto RB = static_cast<const __nv_bfloat16*>(rb);
  auto Y = static_cast<__nv_bfloat16*>(y);
#define KRT_APPLY(M, RL)                                                                              \
  apply_kernel<M, RL><<<grid_rows(apply_kernel<M, RL>, 0, rows, C), kThreads, 0, s>>>(X, mean, invstd, G, B, R, \
                                                                                      rmean, rinvstd, RG, RB, Y, rows, C)
  if (mode == 0) { if (relu) KRT_APPLY(0, true); else KRT_APPLY(0, false); }
  else if (mode == 1) { if (relu) KRT_APPLY(1, true); else KRT_APPLY(1, false); }
  else { if (relu) KRT_APPLY(2, true); else KRT_APPLY(2, false); }
#undef KRT_APPLY
  return cudaGetLastError();
}

cudaError_t bn_add_relu_bwd(const void* dy, const void* dy2, const void* x, const float* mean, const float* invstd,
                            const void* g, const void* b, const void* res, const float* rmean, const float* rinvstd,
                            const void* rg, const void* rb, void* dz, int64_t rows, int C, cudaStream_t s) {
  if (!shape_ok(rows, C) || res == nullptr) return cudaErrorInvalidValue;
  auto args = [&](auto kernel) {
    kernel<<<grid_rows(kernel, 0, rows, C), kThreads, 0, s>>>(
        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(dy2),
        static_cast<const __nv_bfloat16*>(x), mean, invstd, static_cast<const __nv_bfloat16*>(g),
        static_cast<const __nv_bfloat16*>(b), static_cast<const __nv_bfloat16*>(res), rmean, rinvstd,
        static_cast<const __nv_bfloat16*>(rg), static_cast<const __nv_bfloat16*>(rb),
        static_cast<__nv_bfloat16*>(dz), rows, C);
  };
  if (rmean == nullptr) {
    if (dy2) args(add_relu_bwd_kernel<1, true>);
    else args(add_relu_bwd_kernel<1, false>);
  } else {
    if (dy2) args(add_relu_bwd_kernel<2, true>);
    else args(add_relu_bwd_kernel<2, false>);
  }
  return cudaGetLastError();
}

cudaError_t bn_backward(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                        const void* b, int relu, void* dx, float* dgamma, float* dbeta, int64_t rows, int C,
                        void* ws, cudaStream_t s) {
  if (!shape_ok(rows, C)) return cudaErrorInvalidValue;
  int grid = relu ? grid_rows(bwd_reduce_kernel<true>, reduce_smem(C), rows, C)
                  : grid_rows(bwd_reduce_kernel<false>, reduce_smem(C), rows, C);
  float* part = static_cast<float*>(ws);
  float* coef = part + (size_t)kMaxGrid * 2 * C;
  auto red = [&](auto kernel) {
    kernel<<<grid, kThreads, reduce_smem(C), s>>>(
        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), mean, invstd,
        static_cast<const __nv_bfloat16*>(g), static_cast<const __nv_bfloat16*>(b), rows, C, part);
  };
  if (relu) red(bwd_reduce_kernel<true>);
  else red(bwd_reduce_kernel<false>);
  bwd_finalize<<<(C + 31) / 32, 32 * kFinWarps, 0, s>>>(part, grid, rows, C, dgamma, dbeta, coef);
  if (dx) {
    auto launch = [&](auto kernel) {
      kernel<<<grid_rows(kernel, 0, rows, C), kThreads, 0, s>>>(
          static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), mean, invstd,
          static_cast<const __nv_bfloat16*>(g), static_cast<const __nv_bfloat16*>(b), coef,
          static_cast<__nv_bfloat16*>(dx), rows, C);
    };
    if (relu) launch(bwd_elemt_kernel<true>);
    else launch(bwd_elemt_kernel<false>);
  }
  return cudaGetLastError();
}

}  // namespace krt
