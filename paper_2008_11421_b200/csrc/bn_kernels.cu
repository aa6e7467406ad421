// Fused batch-norm kernels for NHWC bf16 activations (sm_100a).
//
// The ResNet units' hot elementwise work ("warp-level fused
// elementwise/norm kernels elsewhere").  All are HBM-bound streaming kernels
// over a [rows, C] matrix (rows = N*H*W, C contiguous, C % 8 == 0):
//
//   stats        : per-channel mean / invstd (batch statistics)          1R
//   stats_apply  : stats, then y = relu?(bn(x) [+ res])                  1R | 1R + 1W (+1R)
//   apply        : y = relu?(bn(x) [+ res | + bn'(res)])                  1-2R + 1W
//   add_relu_bwd : dz = dy * (bn(x) + (res | bn'(res)) > 0)               2-3R + 1W
//   backward     : dgamma, dbeta (reduce) and dx (elementwise), with the
//                  ReLU mask recomputed from x when the BN feeds a ReLU   2R + 2R+1W
//   add_relu_backward : add_relu_bwd and backward of the same BN; the
//                  reduce runs on dz while it is produced                 3R+1W | 2R+1W
//
// Thread mapping: a thread owns 8 consecutive channels (one 16-byte vector)
// for its whole life, so per-channel coefficients stay in registers; rows are
// grid-strided with kU rows in flight per thread and tensor (the bytes in
// flight per SM, not the instruction count, set the achieved HBM rate).
//
// Reductions are one cooperative kernel (grid = one wave of resident CTAs):
//   pass   per-thread fp32 partials -> CTA fixed-order sum -> one partial per CTA
//   sync   grid barrier
//   final  CTA k sums the partials of channel octets k, k+grid, ... in double
//          (fixed order: deterministic, so in-core and out-of-core runs stay
//          bitwise equal) with coalesced 32-byte sector reads, and writes the
//          per-channel results (mean/invstd, or dgamma/dbeta + dx coefficients)
// so the separate finalize launch and its latency are gone.  The elementwise
// pass that follows a reduction is its own kernel: measured on B200, a second
// streaming pass inside the cooperative kernel after the barrier ran at 4.5
// TB/s against 5.8 TB/s as a fresh launch (scripts/bench_bn.py, round 1).
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "bn_kernels.hpp"

namespace cg = cooperative_groups;

namespace krt {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxGrid = 148 * 8;  // partial rows the workspace holds
constexpr int kU = 4;              // rows in flight per thread and tensor

struct Vec8 {
  float v[8];
};

__device__ __forceinline__ uint4 ld16(const __nv_bfloat16* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

// streaming load: the data is touched once more at most (evict-first in L1)
__device__ __forceinline__ uint4 ld16s(const __nv_bfloat16* p) { return __ldcs(reinterpret_cast<const uint4*>(p)); }

__device__ __forceinline__ Vec8 unpack(const uint4& u) {
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

__device__ __forceinline__ uint4 pack(const Vec8& x) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(x.v[2 * k], x.v[2 * k + 1]);
  return u;
}

__device__ __forceinline__ void st16(__nv_bfloat16* p, const Vec8& x) { *reinterpret_cast<uint4*>(p) = pack(x); }

__device__ __forceinline__ float bf(const __nv_bfloat16* p, int i) { return __bfloat162float(p[i]); }

// threads of a CTA: tx = channel octet (C/8 of them), ty = row lane
struct Map {
  int tc, rb, tx, ty;
  __device__ Map(int C) {
    tc = C / 8;
    rb = kThreads / tc;  // rows per CTA sweep (>= 1 since C <= 2048)
    tx = threadIdx.x % tc;
    ty = threadIdx.x / tc;
  }
};

// Row iteration: thread rows are r0 + k*step; one "group" is kU of them.
struct Rows {
  int64_t first, step, rows;
  __device__ Rows(const Map& m, int64_t rows_) : rows(rows_) {
    first = (int64_t)blockIdx.x * m.rb + m.ty;
    step = (int64_t)gridDim.x * m.rb;
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

// Reduce the per-thread partials (a: sum, b: second sum; 8 channels each)
// over the CTA's rows and write one partial row [2][C] for this CTA:
//   1) butterfly shuffles over the rows one warp holds (C < 256: 32/tc rows)
//   2) the remaining row groups (warps, or rows of tc >= 32 threads) are added
//      in fixed group order through a C-float shared buffer, sum then second
// Deterministic, and at most C floats of shared memory: the streaming passes
// need the L1 the shared-memory carve-out would otherwise take.
__device__ __forceinline__ void cta_partial(float* a, float* b, float* smem, const Map& m, float* part, int C,
                                            int c0) {
  const int lane = threadIdx.x & 31;
  int groups, gid;
  bool leader;
  if (m.tc < 32) {
    for (int off = m.tc; off < 32; off <<= 1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        a[k] += __shfl_xor_sync(0xffffffffu, a[k], off);
        b[k] += __shfl_xor_sync(0xffffffffu, b[k], off);
      }
    }
    groups = kThreads / 32;
    gid = threadIdx.x >> 5;
    leader = lane < m.tc;
  } else {
    groups = m.rb;
    gid = m.ty;
    leader = true;
  }
  float* out = part + (size_t)blockIdx.x * 2 * C;
  for (int half = 0; half < 2; ++half) {
    const float* v = half ? b : a;
    for (int g = 0; g < groups; ++g) {
      if (leader && gid == g) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float t = g == 0 ? v[k] : smem[c0 + k] + v[k];
          if (g == groups - 1) out[half * C + c0 + k] = t;
          else smem[c0 + k] = t;
        }
      }
      if (groups > 1) __syncthreads();
    }
  }
}

// Sum the gridDim.x CTA partials of channel octet `oct`: thread = (row lane
// 0..31, channel 0..7), so a warp reads four full 32-byte sectors per step
// (eight loads in flight per thread); then butterfly shuffles over the four
// row lanes of a warp and a fixed-order pass over the eight warps.  Threads
// 0..7 return the sums of channel oct*8+threadIdx.x.
__device__ __forceinline__ bool sum_octet(const float* part, int nblk, int C, int oct, double* sh, double& s1,
                                          double& s2) {
  const int lr = threadIdx.x >> 3, ch = threadIdx.x & 7;
  const int c = oct * 8 + ch;
  constexpr int L = kThreads / 8;  // row lanes
  double a[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
  int b = lr;
  for (; b + 3 * L < nblk; b += 4 * L) {
    float x[4], y[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = __ldcg(part + (size_t)(b + u * L) * 2 * C + c);
      y[u] = __ldcg(part + (size_t)(b + u * L) * 2 * C + C + c);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] += (double)x[u];
      q[u] += (double)y[u];
    }
  }
#pragma unroll
  for (int u = 0; u < 3; ++u) {
    if (b + u * L < nblk) {
      a[u] += (double)__ldcg(part + (size_t)(b + u * L) * 2 * C + c);
      q[u] += (double)__ldcg(part + (size_t)(b + u * L) * 2 * C + C + c);
    }
  }
  double sa = (a[0] + a[1]) + (a[2] + a[3]);
  double sq = (q[0] + q[1]) + (q[2] + q[3]);
  sa += __shfl_xor_sync(0xffffffffu, sa, 8);
  sq += __shfl_xor_sync(0xffffffffu, sq, 8);
  sa += __shfl_xor_sync(0xffffffffu, sa, 16);
  sq += __shfl_xor_sync(0xffffffffu, sq, 16);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane < 8) {
    sh[w * 16 + lane] = sa;
    sh[w * 16 + 8 + lane] = sq;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    s1 = 0;
    s2 = 0;
    for (int k = 0; k < kThreads / 32; ++k) {
      s1 += sh[k * 16 + threadIdx.x];
      s2 += sh[k * 16 + 8 + threadIdx.x];
    }
  }
  __syncthreads();  // sh reused by the next octet
  return threadIdx.x < 8;
}

// ---------------------------------------------------------------------------
// forward: stats [+ apply]
//   MODE: 0 none, 1 identity residual, 2 bn(residual)
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

// the apply pass over one group of U rows (rows >= rows_ skipped)
template <int MODE, bool RELU, int U>
__device__ __forceinline__ void apply_group(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ res,
                                            __nv_bfloat16* __restrict__ y, int64_t r0, int64_t step, int64_t rows,
                                            int C, int c0, const float* sc, const float* sh, const float* rsc,
                                            const float* rsh) {
  uint4 v[U], q[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t r = r0 + u * step;
    if (r < rows) {
      v[u] = ld16s(x + r * C + c0);
      if (MODE != 0) q[u] = ld16s(res + r * C + c0);
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t r = r0 + u * step;
    if (r < rows) {
      Vec8 rv{};
      if (MODE != 0) rv = unpack(q[u]);
      st16(y + r * C + c0, apply_row<MODE, RELU>(unpack(v[u]), rv, sc, sh, rsc, rsh));
    }
  }
}

// stats pass-1 accumulation of one group
template <int U>
__device__ __forceinline__ void stats_group(const __nv_bfloat16* __restrict__ x, int64_t r0, int64_t step,
                                            int64_t rows, int C, int c0, float* s, float* q) {
  uint4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t r = r0 + u * step;
    v[u] = r < rows ? ld16(x + r * C + c0) : make_uint4(0, 0, 0, 0);  // bf16 zero bits
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    Vec8 f = unpack(v[u]);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s[k] += f.v[k];
      q[k] += f.v[k] * f.v[k];
    }
  }
}

template <int U>
__global__ void __launch_bounds__(kThreads) stats_kernel(const __nv_bfloat16* __restrict__ x, int64_t rows, int C,
                                                         float eps, float* __restrict__ part,
                                                         float* __restrict__ mean, float* __restrict__ invstd) {
  extern __shared__ float smem[];
  Map m(C);
  Rows rw(m, rows);
  const int c0 = m.tx * 8;
  float s[8] = {0}, q[8] = {0};
  for (int64_t r0 = rw.first; r0 < rows; r0 += rw.step * U) stats_group<U>(x, r0, rw.step, rows, C, c0, s, q);
  cta_partial(s, q, smem, m, part, C, c0);
  cg::this_grid().sync();
  double* shd = reinterpret_cast<double*>(smem);
  for (int oct = blockIdx.x; oct < C / 8; oct += gridDim.x) {
    double s1, s2;
    if (sum_octet(part, gridDim.x, C, oct, shd, s1, s2)) {
      const int c = oct * 8 + threadIdx.x;
      double mu = s1 / (double)rows;
      double var = s2 / (double)rows - mu * mu;
      if (var < 0) var = 0;
      mean[c] = (float)mu;
      invstd[c] = (float)(1.0 / sqrt(var + (double)eps));
    }
  }
}

template <int MODE, bool RELU, int U>
__global__ void __launch_bounds__(kThreads) apply_kernel(
    const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ invstd,
    const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b, const __nv_bfloat16* __restrict__ res,
    const float* __restrict__ rmean, const float* __restrict__ rinvstd, const __nv_bfloat16* __restrict__ rg,
    const __nv_bfloat16* __restrict__ rb_, __nv_bfloat16* __restrict__ y, int64_t rows, int C) {
  Map m(C);
  Rows rw(m, rows);
  const int c0 = m.tx * 8;
  float sc[8], sh[8], rsc[8], rsh[8];
  bn_coeffs(mean, invstd, g, b, c0, sc, sh);
  if (MODE == 2) bn_coeffs(rmean, rinvstd, rg, rb_, c0, rsc, rsh);
  for (int64_t r0 = rw.first; r0 < rows; r0 += rw.step * U)
    apply_group<MODE, RELU, U>(x, res, y, r0, rw.step, rows, C, c0, sc, sh, rsc, rsh);
}

// ---------------------------------------------------------------------------
// backward
//
// dz = dy * ( bn(x) [+ res | + bn'(res)] > 0 )   (backward of the add + ReLU);
// the forward sum is re-rounded to bf16 exactly as apply_kernel stored it
template <int MODE>
__device__ __forceinline__ Vec8 add_relu_row(const Vec8& v, const Vec8& rv, const Vec8& d, const float* sc,
                                             const float* sh, const float* rsc, const float* rsh) {
  Vec8 o;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float pre = __fadd_rn(__fmaf_rn(v.v[k], sc[k], sh[k]), MODE == 2 ? __fmaf_rn(rv.v[k], rsc[k], rsh[k]) : rv.v[k]);
    o.v[k] = pre > 0x1p-134f ? d.v[k] : 0.0f;  // == (bf16(pre) > 0), see relu_mask
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
    const float* __restrict__ mean, const float* __restrict__ invstd, const __nv_bfloat16* __restrict__ g,
    const __nv_bfloat16* __restrict__ b, const __nv_bfloat16* __restrict__ res, const float* __restrict__ rmean,
    const float* __restrict__ rinvstd, const __nv_bfloat16* __restrict__ rg, const __nv_bfloat16* __restrict__ rb_,
    __nv_bfloat16* __restrict__ dz, int64_t rows, int C) {
  Map m(C);
  Rows rw(m, rows);
  const int c0 = m.tx * 8;
  float sc[8], sh[8], rsc[8], rsh[8];
  bn_coeffs(mean, invstd, g, b, c0, sc, sh);
  if (MODE == 2) bn_coeffs(rmean, rinvstd, rg, rb_, c0, rsc, rsh);
  constexpr int U = 2;  // 3-4 tensors per row: two rows already saturate HBM
  for (int64_t r0 = rw.first; r0 < rows; r0 += rw.step * U) {
    uint4 v[U], q[U], d[U], e[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * rw.step;
      if (r < rows) {
        const int64_t o = r * C + c0;
        v[u] = ld16s(x + o);
        q[u] = ld16s(res + o);
        d[u] = ld16s(dy + o);
        if (DY2) e[u] = ld16s(dy2 + o);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * rw.step;
      if (r < rows) {
        Vec8 dd = unpack(d[u]);
        if (DY2) dd = add_grad(dd, unpack(e[u]));
        st16(dz + r * C + c0, add_relu_row<MODE>(unpack(v[u]), unpack(q[u]), dd, sc, sh, rsc, rsh));
      }
    }
  }
}

// Backward coefficients.  With gm = dy * mask, xhat = (x - mean) * invstd:
//   dbeta = sum gm, dgamma = sum gm * xhat
//   dx = gamma*invstd * (gm - dbeta/n - xhat * dgamma/n)  =  A*gm + B*x + D
struct BwdCoef {
  float sc[8], sh[8];  // forward affine (ReLU mask)
  float a[8], bx[8], d[8];
};

template <bool RELU>
__device__ __forceinline__ float relu_mask(float v, float sc, float sh, float gm) {
  if (!RELU) return gm;
  // bf16(fma) > 0  <=>  fma > 2^-134 (round-to-nearest-even sends (0, 2^-134]
  // to +0 and everything above to a positive bf16): the forward's exact mask
  // without the convert round trip
  return __fmaf_rn(v, sc, sh) > 0x1p-134f ? gm : 0.0f;
}

// pass-1 accumulation: s1 += gm, s2 += gm * (x - mu); the finalize applies
// invstd (sum gm * xhat = invstd * s2), one multiply per channel instead of
// one per element
template <bool RELU>
__device__ __forceinline__ void bwd_acc(const Vec8& v, const Vec8& d, const float* sc, const float* sh,
                                        const float* mu, float* s1, float* s2) {
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    float gm = relu_mask<RELU>(v.v[k], sc[k], sh[k], d.v[k]);
    s1[k] += gm;
    s2[k] = __fmaf_rn(gm, v.v[k] - mu[k], s2[k]);
  }
}

template <bool RELU>
__device__ __forceinline__ Vec8 bwd_row(const Vec8& v, const Vec8& d, const BwdCoef& k) {
  Vec8 o;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float gm = relu_mask<RELU>(v.v[j], k.sc[j], k.sh[j], d.v[j]);
    o.v[j] = __fmaf_rn(k.a[j], gm, __fmaf_rn(k.bx[j], v.v[j], k.d[j]));
  }
  return o;
}

// finalize: dgamma/dbeta and the dx coefficients (coef: [3][C] = A, B, D)
__device__ __forceinline__ void bwd_finalize(const float* part, int64_t rows, int C, const float* mean,
                                             const float* invstd, const __nv_bfloat16* g, float* dgamma,
                                             float* dbeta, float* coef, double* shd) {
  for (int oct = blockIdx.x; oct < C / 8; oct += gridDim.x) {
    double s1, s2;
    if (sum_octet(part, gridDim.x, C, oct, shd, s1, s2)) {
      const int c = oct * 8 + threadIdx.x;
      const double is = invstd[c], mu = mean[c];
      s2 *= is;  // sum gm * (x - mu) -> sum gm * xhat
      if (dbeta) dbeta[c] = (float)s1;
      if (dgamma) dgamma[c] = (float)s2;
      const double gs = (double)bf(g, c) * is;
      const double k1 = s1 / (double)rows, k2 = s2 / (double)rows;
      // dx = gs*(gm - k1 - (x - mu)*is*k2)
      coef[c] = (float)gs;
      coef[C + c] = (float)(-gs * is * k2);
      coef[2 * C + c] = (float)(gs * (mu * is * k2 - k1));
    }
  }
}

// reduce + finalize (dgamma, dbeta, dx coefficients), one cooperative kernel
template <bool RELU, int U>
__global__ void __launch_bounds__(kThreads) bwd_reduce_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ invstd, const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b,
    int64_t rows, int C, float* __restrict__ part, float* __restrict__ coef, float* __restrict__ dgamma,
    float* __restrict__ dbeta) {
  extern __shared__ float smem[];
  Map m(C);
  Rows rw(m, rows);
  const int c0 = m.tx * 8;
  float sc[8], sh[8], mu[8];
  bn_coeffs(mean, invstd, g, b, c0, sc, sh);
#pragma unroll
  for (int j = 0; j < 8; ++j) mu[j] = mean[c0 + j];
  float s1[8] = {0}, s2[8] = {0};
  for (int64_t r0 = rw.first; r0 < rows; r0 += rw.step * U) {
    uint4 v[U], d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * rw.step;
      v[u] = r < rows ? ld16s(x + r * C + c0) : make_uint4(0, 0, 0, 0);
      d[u] = r < rows ? ld16s(dy + r * C + c0) : make_uint4(0, 0, 0, 0);  // gm = 0 on padding
    }
#pragma unroll
    for (int u = 0; u < U; ++u) bwd_acc<RELU>(unpack(v[u]), unpack(d[u]), sc, sh, mu, s1, s2);
  }
  cta_partial(s1, s2, smem, m, part, C, c0);
  cg::this_grid().sync();
  bwd_finalize(part, rows, C, mean, invstd, g, dgamma, dbeta, coef, reinterpret_cast<double*>(smem));
}

// add_relu_bwd of the residual sum and the reduce of the BN (no ReLU of its
// own) that produced x, in one pass: dz = (dy [+ dy2]) * mask(bn(x) + res) is
// written out and accumulated from registers; then the finalize
template <bool DY2, int U>
__global__ void __launch_bounds__(kThreads) add_relu_reduce_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ dy2, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ mean, const float* __restrict__ invstd, const __nv_bfloat16* __restrict__ g,
    const __nv_bfloat16* __restrict__ b, const __nv_bfloat16* __restrict__ res, __nv_bfloat16* __restrict__ dz,
    int64_t rows, int C, float* __restrict__ part, float* __restrict__ coef, float* __restrict__ dgamma,
    float* __restrict__ dbeta) {
  extern __shared__ float smem[];
  Map m(C);
  Rows rw(m, rows);
  const int c0 = m.tx * 8;
  float sc[8], sh[8], mu[8];
  bn_coeffs(mean, invstd, g, b, c0, sc, sh);
#pragma unroll
  for (int j = 0; j < 8; ++j) mu[j] = mean[c0 + j];
  float s1[8] = {0}, s2[8] = {0};
  for (int64_t r0 = rw.first; r0 < rows; r0 += rw.step * U) {  // U rows x 3-4 tensors in flight
    uint4 v[U], q[U], d[U], e[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * rw.step;
      if (r < rows) {
        const int64_t o = r * C + c0;
        v[u] = ld16s(x + o);
        q[u] = ld16s(res + o);
        d[u] = ld16s(dy + o);
        if (DY2) e[u] = ld16s(dy2 + o);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * rw.step;
      if (r < rows) {
        Vec8 dd = unpack(d[u]);
        if (DY2) dd = add_grad(dd, unpack(e[u]));
        Vec8 xv = unpack(v[u]);
        Vec8 z = add_relu_row<1>(xv, unpack(q[u]), dd, sc, sh, nullptr, nullptr);
        st16(dz + r * C + c0, z);
        bwd_acc<false>(xv, z, sc, sh, mu, s1, s2);
      }
    }
  }
  cta_partial(s1, s2, smem, m, part, C, c0);
  cg::this_grid().sync();
  bwd_finalize(part, rows, C, mean, invstd, g, dgamma, dbeta, coef, reinterpret_cast<double*>(smem));
}

// dx = A*gm + B*x + D [+ addend] with gm = dy * mask (coefficients from the
// reduce); the optional addend (a residual gradient) is summed before the one
// bf16 rounding, so no separate add pass re-reads dx
template <bool RELU, bool ADD, int U>
__global__ void __launch_bounds__(kThreads) bwd_elemt_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const float* __restrict__ mean,
    const float* __restrict__ invstd, const __nv_bfloat16* __restrict__ g, const __nv_bfloat16* __restrict__ b,
    const float* __restrict__ coef, const __nv_bfloat16* __restrict__ addend, __nv_bfloat16* __restrict__ dx,
    int64_t rows, int C) {
  Map m(C);
  Rows rw(m, rows);
  const int c0 = m.tx * 8;
  BwdCoef k;
  if (RELU) bn_coeffs(mean, invstd, g, b, c0, k.sc, k.sh);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    k.a[j] = coef[c0 + j];
    k.bx[j] = coef[C + c0 + j];
    k.d[j] = coef[2 * C + c0 + j];
  }
  for (int64_t r0 = rw.first; r0 < rows; r0 += rw.step * U) {
    uint4 v[U], d[U], e[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * rw.step;
      if (r < rows) {
        v[u] = ld16s(x + r * C + c0);
        d[u] = ld16s(dy + r * C + c0);
        if (ADD) e[u] = ld16s(addend + r * C + c0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = r0 + u * rw.step;
      if (r < rows) {
        Vec8 o = bwd_row<RELU>(unpack(v[u]), unpack(d[u]), k);
        if (ADD) {
          Vec8 a = unpack(e[u]);
#pragma unroll
          for (int j = 0; j < 8; ++j) o.v[j] = __fadd_rn(o.v[j], a.v[j]);
        }
        st16(dx + r * C + c0, o);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// launch helpers

size_t reduce_smem(int C) {
  size_t tree = C >= 8 * kThreads ? 0 : (size_t)C * sizeof(float);  // rb == 1: no cross-row step
  size_t fin = (size_t)(kThreads / 32) * 16 * sizeof(double);
  return tree > fin ? tree : fin;
}

bool shape_ok(int64_t rows, int C) {
  return rows > 0 && C >= 8 && C % 8 == 0 && C <= 8 * kThreads && (kThreads % (C / 8)) == 0;
}

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 148;
  }
  return sms;
}

// one full wave of resident CTAs (148 SMs x occupancy), capped at kMaxGrid
// so the reduction partials fit the workspace; never more CTAs than row
// sweeps.  Cooperative kernels need every CTA resident, which this grants.
// Resident CTAs per kernel instantiation and shared-memory size.  Kernels
// that use shared memory get the smallest carve-out that still holds their
// full occupancy: the rest stays L1, which is what keeps enough streaming
// loads in flight (measured: the default carve-out for 16 KB/CTA cost 30% of
// the apply pass's bandwidth).
int resident_ctas(const void* kernel, size_t smem) {
  static std::mutex mu;
  static std::unordered_map<const void*, std::unordered_map<size_t, int>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto& per = cache[kernel];
  auto it = per.find(smem);
  if (it != per.end()) return it->second;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem);
  if (per_sm < 1) per_sm = 1;
  if (smem > 0) {
    int dev = 0, max_smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    size_t need = (size_t)per_sm * (smem + 1024);  // + the per-CTA reservation
    int pct = (int)((need * 100 + max_smem - 1) / max_smem);
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct < 100 ? pct : 100);
    int again = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&again, kernel, kThreads, smem);
    if (again >= 1 && again < per_sm) per_sm = again;
  }
  int r = num_sms() * per_sm;
  per[smem] = r;
  return r;
}

template <class K>
int grid_rows(K kernel, size_t smem, int64_t rows, int C) {
  const int resident = resident_ctas(reinterpret_cast<const void*>(kernel), smem);
  int rb = kThreads / (C / 8);
  int64_t want = (rows + rb - 1) / rb;
  int cap = resident < kMaxGrid ? resident : kMaxGrid;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

template <class T>
struct Id {
  using type = T;
};

// cooperative launch; every argument converted to the kernel's exact parameter type
template <class... P>
cudaError_t coop(void (*kernel)(P...), int64_t rows, int C, cudaStream_t s, typename Id<P>::type... args) {
  size_t smem = reduce_smem(C);
  int grid = grid_rows(kernel, smem, rows, C);
  void* argv[] = {static_cast<void*>(&args)...};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(grid), dim3(kThreads), argv, smem,
                                     s);
}

// Rows in flight per thread and tensor, per kernel family and channel count:
// KRT_BN_U_<FAMILY>=2|4|8 forces a value (tuning sweeps), otherwise the
// measured table (scripts/bench_bn.py at the ResNet-200 widths).
enum Fam { kStats, kApply, kBwdReduce, kBwdElemt, kFams };

int rows_in_flight(Fam f, int C) {
  static int force[kFams] = {-1, -1, -1, -1};
  static const char* names[kFams] = {"KRT_BN_U_STATS", "KRT_BN_U_APPLY", "KRT_BN_U_BWDREDUCE", "KRT_BN_U_BWDELEMT"};
  if (force[f] < 0) {
    const char* e = getenv(names[f]);
    force[f] = e ? atoi(e) : 0;
  }
  if (force[f] == 2 || force[f] == 4 || force[f] == 8) return force[f];
  // measured at batch 1024 on the ResNet-200 widths (profiles/round1_s2_bn_rows_in_flight.md):
  // apply 2-5% faster with two rows, stats up to 25% faster with eight (four at
  // C = 1024), the backward pair best with four everywhere
  switch (f) {
    case kApply: return 2;
    case kStats: return C == 1024 ? 4 : 8;
    default: return 4;
  }
}

using bf16 = __nv_bfloat16;
inline const bf16* B(const void* p) { return static_cast<const bf16*>(p); }
inline bf16* BW_(void* p) { return static_cast<bf16*>(p); }

cudaError_t bwd_elemt(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                      const void* b, const float* coef, const void* addend, void* dx, int64_t rows, int C, int relu,
                      cudaStream_t s) {
  auto go = [&](auto kernel) {
    kernel<<<grid_rows(kernel, 0, rows, C), kThreads, 0, s>>>(B(dy), B(x), mean, invstd, B(g), B(b), coef,
                                                              B(addend), BW_(dx), rows, C);
  };
  const int u = rows_in_flight(kBwdElemt, C);
#define KRT_ELEMT(U)                                                     \
  if (addend) {                                                          \
    if (relu) go(bwd_elemt_kernel<true, true, U>);                       \
    else go(bwd_elemt_kernel<false, true, U>);                           \
  } else {                                                               \
    if (relu) go(bwd_elemt_kernel<true, false, U>);                      \
    else go(bwd_elemt_kernel<false, false, U>);                          \
  }
  if (u == 2) { KRT_ELEMT(2) } else if (u == 8) { KRT_ELEMT(8) } else { KRT_ELEMT(4) }
#undef KRT_ELEMT
  return cudaGetLastError();
}

}  // namespace

size_t bn_workspace_bytes(int C) { return (size_t)kMaxGrid * 2 * C * sizeof(float) + 3 * C * sizeof(float); }

cudaError_t bn_stats(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd, void* ws,
                     cudaStream_t s) {
  if (!shape_ok(rows, C)) return cudaErrorInvalidValue;
  const int u = rows_in_flight(kStats, C);
  float* part = static_cast<float*>(ws);
  if (u == 2) return coop(stats_kernel<2>, rows, C, s, B(x), rows, C, eps, part, mean, invstd);
  if (u == 8) return coop(stats_kernel<8>, rows, C, s, B(x), rows, C, eps, part, mean, invstd);
  return coop(stats_kernel<4>, rows, C, s, B(x), rows, C, eps, part, mean, invstd);
}

cudaError_t bn_stats_apply(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd,
                           const void* g, const void* b, const void* res, int relu, void* y, void* ws,
                           cudaStream_t s) {
  cudaError_t e = bn_stats(x, rows, C, eps, mean, invstd, ws, s);
  if (e != cudaSuccess) return e;
  return bn_apply(x, mean, invstd, g, b, res, nullptr, nullptr, nullptr, nullptr, relu, y, rows, C, s);
}

cudaError_t bn_apply(const void* x, const float* mean, const float* invstd, const void* g, const void* b,
                     const void* res, const float* rmean, const float* rinvstd, const void* rg, const void* rb,
                     int relu, void* y, int64_t rows, int C, cudaStream_t s) {
  if (!shape_ok(rows, C)) return cudaErrorInvalidValue;
  int mode = res == nullptr ? 0 : (rmean == nullptr ? 1 : 2);
  const int u = rows_in_flight(kApply, C);
#define KRT_APPLY_U(M, RL, U)                                                                                   \
  apply_kernel<M, RL, U><<<grid_rows(apply_kernel<M, RL, U>, 0, rows, C), kThreads, 0, s>>>(                    \
      B(x), mean, invstd, B(g), B(b), B(res), rmean, rinvstd, B(rg), B(rb), BW_(y), rows, C)
#define KRT_APPLY(M, RL)                                                           \
  do {                                                                             \
    if (u == 2) KRT_APPLY_U(M, RL, 2);                                             \
    else if (u == 8) KRT_APPLY_U(M, RL, 8);                                        \
    else KRT_APPLY_U(M, RL, 4);                                                    \
  } while (0)
  if (mode == 0) { if (relu) KRT_APPLY(0, true); else KRT_APPLY(0, false); }
  else if (mode == 1) { if (relu) KRT_APPLY(1, true); else KRT_APPLY(1, false); }
  else { if (relu) KRT_APPLY(2, true); else KRT_APPLY(2, false); }
#undef KRT_APPLY
#undef KRT_APPLY_U
  return cudaGetLastError();
}

cudaError_t bn_add_relu_bwd(const void* dy, const void* dy2, const void* x, const float* mean, const float* invstd,
                            const void* g, const void* b, const void* res, const float* rmean, const float* rinvstd,
                            const void* rg, const void* rb, void* dz, int64_t rows, int C, cudaStream_t s) {
  if (!shape_ok(rows, C) || res == nullptr) return cudaErrorInvalidValue;
  auto args = [&](auto kernel) {
    kernel<<<grid_rows(kernel, 0, rows, C), kThreads, 0, s>>>(B(dy), B(dy2), B(x), mean, invstd, B(g), B(b), B(res),
                                                              rmean, rinvstd, B(rg), B(rb), BW_(dz), rows, C);
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
                        void* ws, const void* addend, cudaStream_t s) {
  if (!shape_ok(rows, C)) return cudaErrorInvalidValue;
  float* part = static_cast<float*>(ws);
  float* coef = part + (size_t)kMaxGrid * 2 * C;
  auto red = [&](auto kernel) {
    return coop(kernel, rows, C, s, B(dy), B(x), mean, invstd, B(g), B(b), rows, C, part, coef, dgamma, dbeta);
  };
  const int u = rows_in_flight(kBwdReduce, C);
  cudaError_t e = u == 2 ? (relu ? red(bwd_reduce_kernel<true, 2>) : red(bwd_reduce_kernel<false, 2>))
                  : u == 8 ? (relu ? red(bwd_reduce_kernel<true, 8>) : red(bwd_reduce_kernel<false, 8>))
                           : (relu ? red(bwd_reduce_kernel<true, 4>) : red(bwd_reduce_kernel<false, 4>));
  if (e != cudaSuccess || dx == nullptr) return e;
  return bwd_elemt(dy, x, mean, invstd, g, b, coef, addend, dx, rows, C, relu, s);
}

cudaError_t bn_backward_elemt(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                              const void* b, const float* coef, const void* addend, int relu, void* dx, int64_t rows,
                              int C, cudaStream_t s) {
  if (!shape_ok(rows, C) || coef == nullptr || dx == nullptr) return cudaErrorInvalidValue;
  return bwd_elemt(dy, x, mean, invstd, g, b, coef, addend, dx, rows, C, relu, s);
}

cudaError_t bn_add_relu_backward(const void* dy, const void* dy2, const void* x, const float* mean,
                                 const float* invstd, const void* g, const void* b, const void* res, void* dz,
                                 void* dx, float* dgamma, float* dbeta, int64_t rows, int C, void* ws,
                                 cudaStream_t s) {
  if (!shape_ok(rows, C) || res == nullptr || dz == nullptr || dx == nullptr) return cudaErrorInvalidValue;
  float* part = static_cast<float*>(ws);
  float* coef = part + (size_t)kMaxGrid * 2 * C;
  auto red = [&](auto kernel) {
    return coop(kernel, rows, C, s, B(dy), B(dy2), B(x), mean, invstd, B(g), B(b), B(res), BW_(dz), rows, C, part,
                coef, dgamma, dbeta);
  };
  // two rows in flight per thread, four at C = 1024 (measured: the ResNet-200
  // stage-3 output width, 13% faster there and slower at every other width)
  static const int force_u = getenv("KRT_BN_ADDRELU_U") ? atoi(getenv("KRT_BN_ADDRELU_U")) : 0;
  const bool u4 = force_u ? force_u == 4 : C == 1024;
  cudaError_t e = u4 ? (dy2 ? red(add_relu_reduce_kernel<true, 4>) : red(add_relu_reduce_kernel<false, 4>))
                     : (dy2 ? red(add_relu_reduce_kernel<true, 2>) : red(add_relu_reduce_kernel<false, 2>));
  if (e != cudaSuccess) return e;
  return bwd_elemt(dz, x, mean, invstd, g, b, coef, nullptr, dx, rows, C, 0, s);
}

}  // namespace krt
