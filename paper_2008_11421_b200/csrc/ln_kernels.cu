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
//   lm_xent         : the LM head's next-token cross-entropy, forward and
//                     backward in one pass over the bf16 logits (the row in
//                     registers): per-row loss lse - z[y] and
//                     dz = (softmax(z) - onehot(y)) * scale, fp32 math.
//
// LayerNorm: one warp per row, 16-byte vectors; mean from the rounded x2,
// variance by a second pass over x2 (L2-resident re-read), both in fp32.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "ln_kernels.hpp"
#include "sm100_common.cuh"

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

// LayerNorm backward.  One CTA per row at a time, rows strided over a
// persistent grid; thread t owns the J octets t, t + nt, ... of every row
// (nt = blockDim.x, sized to the row), so its dgamma / dbeta column partials
// stay in registers for all the CTA's rows (no shared-memory accumulators:
// those capped the old warp-per-row kernel at 12 warps per SM, latency-bound
// at 0.33-0.55 of HBM).  The next row's dy / x / addend are loaded while the
// current row is reduced and written (one row of prefetch per CTA).  The two
// row sums: warp shuffles, then the warps' partials summed in warp order
// through a parity-double-buffered shared slot (one barrier per row).  At the
// end each thread stores its column partials: one partial row pair per CTA.
// Deterministic for a given grid.
constexpr int kBwdMaxWarps = 12;  // 384 threads: J = 2 octets per thread up to H = 6144, J = 4 up to 12288

template <bool ADD, int J>
__device__ __forceinline__ void ln_bwd_load(const __nv_bfloat16* dy, const __nv_bfloat16* x,
                                            const __nv_bfloat16* addend, int64_t row, int H, int oct, uint4* ud,
                                            uint4* ux, uint4* ua) {
#pragma unroll
  for (int i = 0; i < J; ++i) {
    const int j = threadIdx.x + blockDim.x * i;
    if (j < oct) {
      ud[i] = __ldcs(reinterpret_cast<const uint4*>(dy + row * H) + j);
      ux[i] = __ldcs(reinterpret_cast<const uint4*>(x + row * H) + j);
      if (ADD) ua[i] = __ldcs(reinterpret_cast<const uint4*>(addend + row * H) + j);
    }
  }
}

template <bool ADD, int J>
__global__ void __maxnreg__(112) ln_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
    const float* __restrict__ mean, const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ addend,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ part, int64_t T, int H) {
  __shared__ float red[2][kBwdMaxWarps][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int oct = H / 8;
  const float inv_h = 1.f / (float)H;
  float accg[J][8], accb[J][8];  // gamma is re-read per row (L1-resident): registers go to the prefetch
#pragma unroll
  for (int i = 0; i < J; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) accg[i][k] = accb[i][k] = 0.f;
  uint4 ud[J], ux[J], ua[ADD ? J : 1];
  int64_t row = blockIdx.x;
  if (row < T) ln_bwd_load<ADD, J>(dy, x, addend, row, H, oct, ud, ux, ua);
  for (int par = 0; row < T; row += gridDim.x, par ^= 1) {
    const float mu = __ldg(mean + row), rs = __ldg(rstd + row);
    // prefetch the next row
    uint4 nd[J], nx[J], na[ADD ? J : 1];
    const int64_t nrow = row + gridDim.x;
    if (nrow < T) ln_bwd_load<ADD, J>(dy, x, addend, nrow, H, oct, nd, nx, na);
    float s1 = 0.f, s2 = 0.f;  // sum g*dy, sum g*dy*xhat
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = threadIdx.x + blockDim.x * i;
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
          accg[i][k] += d[k] * xh;
          accb[i][k] += d[k];
        }
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      red[par][w][0] = s1;
      red[par][w][1] = s2;
    }
    __syncthreads();
    float t1 = 0.f, t2 = 0.f;
    for (int k = 0; k < nw; ++k) {
      t1 += red[par][k][0];
      t2 += red[par][k][1];
    }
    const float c1 = t1 * inv_h, c2 = t2 * inv_h;
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = threadIdx.x + blockDim.x * i;
      if (j < oct) {
        float d[8], xv[8], o[8], gg[8];
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
#pragma unroll
    for (int i = 0; i < J; ++i) {
      ud[i] = nd[i];
      ux[i] = nx[i];
      if (ADD) ua[i] = na[i];
    }
  }
  // this CTA's partial row pair, straight from the registers
#pragma unroll
  for (int i = 0; i < J; ++i) {
    const int j = threadIdx.x + blockDim.x * i;
    if (j < oct) {
      float4* pg = reinterpret_cast<float4*>(part + (size_t)blockIdx.x * 2 * H + 8 * j);
      float4* pb = reinterpret_cast<float4*>(part + (size_t)blockIdx.x * 2 * H + H + 8 * j);
      pg[0] = make_float4(accg[i][0], accg[i][1], accg[i][2], accg[i][3]);
      pg[1] = make_float4(accg[i][4], accg[i][5], accg[i][6], accg[i][7]);
      pb[0] = make_float4(accb[i][0], accb[i][1], accb[i][2], accb[i][3]);
      pb[1] = make_float4(accb[i][4], accb[i][5], accb[i][6], accb[i][7]);
    }
  }
}


// The same LayerNorm backward with the rows staged in shared memory by the
// bulk-copy engine: one thread issues cp.async.bulk for the dy / x / addend
// rows of the CTA's next S rows into an S-stage ring (an mbarrier per stage,
// complete_tx), so S rows per CTA are in flight while the threads work on the
// current one from shared memory (the register-prefetch kernel above holds
// one row ahead and its register budget caps it at one or two CTAs per SM).
// A stage is refilled right after the row barrier of the iteration that
// consumed it (every thread has copied its octets into registers by then).
// Same arithmetic, same column ownership, same partial rows as ln_bwd_kernel.
template <bool ADD, int J>
__global__ void __launch_bounds__(32 * kBwdMaxWarps) ln_bwd_bulk_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
    const float* __restrict__ mean, const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ addend,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ part, int64_t T, int H, int S) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ float red[2][kBwdMaxWarps][2];
  constexpr int NT = ADD ? 3 : 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);   // S mbarriers (<= 16)
  uint8_t* stages = smem_raw + 128;
  const uint32_t row_bytes = (uint32_t)H * 2;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int oct = H / 8;
  const float inv_h = 1.f / (float)H;
  auto stage = [&](int st, int t) { return stages + ((size_t)st * NT + t) * row_bytes; };
  auto issue = [&](int it) {
    const int64_t row = blockIdx.x + (int64_t)it * gridDim.x;
    if (row >= T) return;
    const int st = it % S;
    sm100::mbar_expect_tx(&full[st], NT * row_bytes);
    const __nv_bfloat16* src[3] = {dy + row * H, x + row * H, ADD ? addend + row * H : nullptr};
#pragma unroll
    for (int t = 0; t < NT; ++t)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              sm100::smem_u32(stage(st, t))),
          "l"(src[t]), "r"(row_bytes), "r"(sm100::smem_u32(&full[st]))
          : "memory");
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < S; ++st) sm100::mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int it = 0; it < S; ++it) issue(it);
  float accg[J][8], accb[J][8], gam[J][8];  // gamma held in registers for all rows
#pragma unroll
  for (int i = 0; i < J; ++i) {
    const int j = threadIdx.x + blockDim.x * i;
    if (j < oct) unpack8(__ldg(reinterpret_cast<const uint4*>(g) + j), gam[i]);
#pragma unroll
    for (int k = 0; k < 8; ++k) accg[i][k] = accb[i][k] = 0.f;
  }
  int it = 0;
  for (int64_t row = blockIdx.x; row < T; row += gridDim.x, ++it) {
    const int st = it % S, par = it & 1;
    const float mu = __ldg(mean + row), rs = __ldg(rstd + row);
    sm100::mbar_wait(&full[st], (uint32_t)((it / S) & 1));
    uint4 ud[J], ux[J], ua[ADD ? J : 1];
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = threadIdx.x + blockDim.x * i;
      if (j < oct) {
        ud[i] = reinterpret_cast<const uint4*>(stage(st, 0))[j];
        ux[i] = reinterpret_cast<const uint4*>(stage(st, 1))[j];
        if (ADD) ua[i] = reinterpret_cast<const uint4*>(stage(st, 2))[j];
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = threadIdx.x + blockDim.x * i;
      if (j < oct) {
        float d[8], xv[8];
        unpack8(ud[i], d);
        unpack8(ux[i], xv);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (xv[k] - mu) * rs;
          const float gd = d[k] * gam[i][k];
          s1 += gd;
          s2 = __fmaf_rn(gd, xh, s2);
          accg[i][k] += d[k] * xh;
          accb[i][k] += d[k];
        }
      }
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
      red[par][w][0] = s1;
      red[par][w][1] = s2;
    }
    __syncthreads();  // also: every thread holds this stage's octets in registers
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(it + S);
    }
    float t1 = 0.f, t2 = 0.f;
    for (int k = 0; k < nw; ++k) {
      t1 += red[par][k][0];
      t2 += red[par][k][1];
    }
    const float c1 = t1 * inv_h, c2 = t2 * inv_h;
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = threadIdx.x + blockDim.x * i;
      if (j < oct) {
        float d[8], xv[8], o[8];
        unpack8(ud[i], d);
        unpack8(ux[i], xv);
        if (ADD) unpack8(ua[i], o);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (xv[k] - mu) * rs;
          const float v = rs * (d[k] * gam[i][k] - c1 - xh * c2);
          o[k] = ADD ? __fadd_rn(v, o[k]) : v;
        }
        __stcs(reinterpret_cast<uint4*>(dx + row * H) + j, pack8(o));
      }
    }
  }
#pragma unroll
  for (int i = 0; i < J; ++i) {
    const int j = threadIdx.x + blockDim.x * i;
    if (j < oct) {
      float4* pg = reinterpret_cast<float4*>(part + (size_t)blockIdx.x * 2 * H + 8 * j);
      float4* pb = reinterpret_cast<float4*>(part + (size_t)blockIdx.x * 2 * H + H + 8 * j);
      pg[0] = make_float4(accg[i][0], accg[i][1], accg[i][2], accg[i][3]);
      pg[1] = make_float4(accg[i][4], accg[i][5], accg[i][6], accg[i][7]);
      pb[0] = make_float4(accb[i][0], accb[i][1], accb[i][2], accb[i][3]);
      pb[1] = make_float4(accb[i][4], accb[i][5], accb[i][6], accb[i][7]);
    }
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

// octets per thread and threads per CTA: the row's octets over J per thread, whole warps
int ln_bwd_j(int H) { return H / 8 <= 32 * kBwdMaxWarps * 2 ? 2 : 4; }

int ln_bwd_threads(int H) {
  const int oct = H / 8, J = ln_bwd_j(H);
  const int t = ((oct + J - 1) / J + 31) / 32 * 32;
  return t < 32 ? 32 : t;
}

template <int J>
int ln_bwd_grid_j(int64_t T, int H, bool add) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int nt = ln_bwd_threads(H);
  if (add) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ln_bwd_kernel<true, J>, nt, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ln_bwd_kernel<false, J>, nt, 0);
  const int64_t cap = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);  // one full wave, no tail
  return (int)(T < cap ? T : cap);
}

// KRT_LN_BWD_BULK=0: the register-prefetch kernel (A/B)
bool bulk_enabled() {
  static const bool on = [] {
    const char* e = getenv("KRT_LN_BWD_BULK");
    return !(e && e[0] == '0');
  }();
  return on;
}

// the bulk-copy kernel: S stages of NT rows, ~110 KB of ring per CTA
constexpr size_t kBulkRing = 110 * 1024;
int ln_bwd_stages(int H, bool add) {
  const size_t st = (size_t)(add ? 3 : 2) * H * 2;
  const int S = (int)(kBulkRing / st);
  return S < 2 ? 2 : (S > 8 ? 8 : S);
}
size_t ln_bwd_bulk_smem(int H, bool add) { return 128 + (size_t)ln_bwd_stages(H, add) * (add ? 3 : 2) * H * 2; }
// measured (scripts/bench_ln_bwd.py): bulk 4.8 / 3.9 TB/s vs registers 3.6 / 2.6 at H 3072 / 4256;
// at H 1920 the register kernel's 128-thread CTAs fit more rows per SM (4.2 vs 3.9 TB/s)
bool ln_bwd_bulk_ok(int H, bool add) {
  return H > 2048 && ln_bwd_j(H) == 2 && ln_bwd_bulk_smem(H, add) <= 200 * 1024;
}

int ln_bwd_grid(int64_t T, int H, bool add) {
  if (ln_bwd_bulk_ok(H, add)) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int smem = (int)ln_bwd_bulk_smem(H, add);
    auto k = add ? ln_bwd_bulk_kernel<true, 2> : ln_bwd_bulk_kernel<false, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, ln_bwd_threads(H), smem);
    const int64_t cap = (int64_t)sms * (per_sm < 1 ? 1 : per_sm);
    return (int)(T < cap ? T : cap);
  }
  return ln_bwd_j(H) == 2 ? ln_bwd_grid_j<2>(T, H, add) : ln_bwd_grid_j<4>(T, H, add);
}

template <int J>
void launch_ln_bwd(const __nv_bfloat16* dy, const __nv_bfloat16* x, const __nv_bfloat16* g, const float* mean,
                   const float* rstd, const __nv_bfloat16* addend, __nv_bfloat16* dx, float* part, int grid, int nt,
                   int64_t T, int H, cudaStream_t s) {
  if (addend) ln_bwd_kernel<true, J><<<grid, nt, 0, s>>>(dy, x, g, mean, rstd, addend, dx, part, T, H);
  else ln_bwd_kernel<false, J><<<grid, nt, 0, s>>>(dy, x, g, mean, rstd, addend, dx, part, T, H);
}


// ---------------------------------------------------------------------------
// lm_xent: one CTA per row (grid-stride), the row's V / 8 octets spread over
// the CTA's threads (J per thread, all loads in flight at once), block
// reductions for the max and the sum of exp(z - max) in a fixed order
// (deterministic), then dz written from the registers: 2 bytes read and 2
// written per logit instead of the fp32 chunk passes of an unfused softmax.
// 256 threads, two CTAs per SM (launch bounds cap the registers at 128).
// Measured at V 51200 with single max / sum chains: 0.32 of HBM in the GPT
// step, the same as one 512-thread CTA per SM (latency of the chains and the
// two exp passes per logit, not the loads)
constexpr int kXentThreads = 256;

__device__ __forceinline__ float block_reduce(float v, float* sh, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const float t = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, t) : v + t;
  }
  __syncthreads();  // sh reused across calls
  if (lane == 0) sh[w] = v;
  __syncthreads();
  float r = sh[0];
  for (int k = 1; k < kXentThreads / 32; ++k) r = is_max ? fmaxf(r, sh[k]) : r + sh[k];
  return r;
}

template <int J>
__global__ void __launch_bounds__(kXentThreads, 2) lm_xent_kernel(const __nv_bfloat16* __restrict__ z,
                                                                  const int64_t* __restrict__ y,
                                                                  __nv_bfloat16* __restrict__ dz,
                                                                  float* __restrict__ row_loss, int64_t T, int V,
                                                                  float scale) {
  __shared__ float sh[kXentThreads / 32];
  const int oct = V / 8;
  for (int64_t row = blockIdx.x; row < T; row += gridDim.x) {
    const uint4* zr = reinterpret_cast<const uint4*>(z + row * V);
    uint4 u[J];
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = threadIdx.x + kXentThreads * i;
      if (j < oct) u[i] = __ldcs(zr + j);
    }
    // four independent max / sum chains per thread (the single 8J-long
    // chains were latency-bound), combined in a fixed order
    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int i = 0; i < J; ++i) {
      if (threadIdx.x + kXentThreads * i < oct) {
        float f[8];
        unpack8(u[i], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) m4[k & 3] = fmaxf(m4[k & 3], f[k]);
      }
    }
    const float m = block_reduce(fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])), sh, true);
    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < J; ++i) {
      if (threadIdx.x + kXentThreads * i < oct) {
        float f[8];
        unpack8(u[i], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) s4[k & 3] += __expf(f[k] - m);
      }
    }
    const float se = block_reduce((s4[0] + s4[1]) + (s4[2] + s4[3]), sh, false);
    const float lse = m + __logf(se);
    const int64_t tgt = y[row];
#pragma unroll
    for (int i = 0; i < J; ++i) {
      const int j = threadIdx.x + kXentThreads * i;
      if (j < oct) {
        float f[8];
        unpack8(u[i], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int col = 8 * j + k;
          if (col == tgt) row_loss[row] = lse - f[k];
          f[k] = __fmul_rn(__expf(f[k] - lse), scale) - (col == tgt ? scale : 0.f);
        }
        __stcs(reinterpret_cast<uint4*>(dz + row * V) + j, pack8(f));
      }
    }
  }
}


// ---------------------------------------------------------------------------
// attn_softmax_bwd: the elementwise middle of an unfused causal attention
// backward (head dims cuDNN's fused backward rejects): from the fp32 score
// and score-gradient matrices S = Q K^T and dP = dO V^T of a batch of
// (sequence, head) pairs, one pass writes
//   P  = exp(scale * S - lse)          (bf16; 0 above the diagonal)
//   dS = P * (dP - D) * scale          (bf16, from the fp32 P)
// with lse the forward's natural-log logsumexp and D = rowsum(dO * O).
// 8 columns per thread; fully masked octets read nothing.
__global__ void __launch_bounds__(256) attn_softmax_bwd_kernel(const float* __restrict__ S,
                                                               const float* __restrict__ dP,
                                                               const float* __restrict__ lse,
                                                               const float* __restrict__ Dr,
                                                               __nv_bfloat16* __restrict__ P,
                                                               __nv_bfloat16* __restrict__ dS, int64_t rows, int s,
                                                               float scale) {
  const int oct = s / 8;
  const int64_t total = rows * oct;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / oct;           // (pair, query row) flattened
    const int j0 = (int)(t - r * oct) * 8;
    const int i = (int)(r % s);
    float p[8], g[8];
    if (j0 > i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) p[k] = g[k] = 0.f;
    } else {
      const float l = lse[r], d = Dr[r];
      const float4* s4 = reinterpret_cast<const float4*>(S + r * s + j0);
      const float4* d4 = reinterpret_cast<const float4*>(dP + r * s + j0);
      const float4 a0 = __ldcs(s4), a1 = __ldcs(s4 + 1), b0 = __ldcs(d4), b1 = __ldcs(d4 + 1);
      const float sv[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float dv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        p[k] = (j0 + k <= i) ? expf(__fmaf_rn(sv[k], scale, -l)) : 0.f;
        g[k] = p[k] * (dv[k] - d) * scale;
      }
    }
    __stcs(reinterpret_cast<uint4*>(P + r * s + j0), pack8(p));
    __stcs(reinterpret_cast<uint4*>(dS + r * s + j0), pack8(g));
  }
}
}  // namespace

size_t ln_bwd_workspace(int64_t T, int H) {
  const int a = ln_bwd_grid(T, H, true), b = ln_bwd_grid(T, H, false);
  return (size_t)(a > b ? a : b) * 2 * H * sizeof(float);
}

cudaError_t ln_bwd(const void* dy, const void* x, const void* g, const float* mean, const float* rstd,
                   const void* addend, void* dx, float* dgamma, float* dbeta, void* ws, int64_t T, int H,
                   cudaStream_t s) {
  if (T <= 0 || H <= 0 || H % 8 != 0 || ln_bwd_threads(H) > 32 * kBwdMaxWarps) return cudaErrorInvalidValue;
  const int grid = ln_bwd_grid(T, H, addend != nullptr), nt = ln_bwd_threads(H);
  float* part = static_cast<float*>(ws);
  auto DY = static_cast<const __nv_bfloat16*>(dy);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto G = static_cast<const __nv_bfloat16*>(g);
  auto A = static_cast<const __nv_bfloat16*>(addend);
  auto DX = static_cast<__nv_bfloat16*>(dx);
  const bool add = addend != nullptr;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(x) |
                         reinterpret_cast<uintptr_t>(addend)) & 15) == 0;
  if (aligned && bulk_enabled() && ln_bwd_bulk_ok(H, add)) {
    const int S = ln_bwd_stages(H, add);
    const size_t smem = ln_bwd_bulk_smem(H, add);
    if (add) ln_bwd_bulk_kernel<true, 2><<<grid, nt, smem, s>>>(DY, X, G, mean, rstd, A, DX, part, T, H, S);
    else ln_bwd_bulk_kernel<false, 2><<<grid, nt, smem, s>>>(DY, X, G, mean, rstd, A, DX, part, T, H, S);
  } else if (ln_bwd_j(H) == 2) {
    launch_ln_bwd<2>(DY, X, G, mean, rstd, A, DX, part, grid, nt, T, H, s);
  } else {
    launch_ln_bwd<4>(DY, X, G, mean, rstd, A, DX, part, grid, nt, T, H, s);
  }
  cudaError_t e = cudaGetLastError();
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
  if (oct <= 32 * 17) {  // row in registers, persistent grid
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (T + kRowsPerCta - 1) / kRowsPerCta, cap = (int64_t)sms * 8;
    const dim3 pgrid((unsigned)(want < cap ? want : cap));
    auto go = [&](auto k_res, auto k_plain) {
      if (r) k_res<<<pgrid, 32 * kRowsPerCta, 0, s>>>(X, R, X2, G, B, Hh, mean, rstd, T, H, eps);
      else k_plain<<<pgrid, 32 * kRowsPerCta, 0, s>>>(X, R, X2, G, B, Hh, mean, rstd, T, H, eps);
    };
    // J octets per lane: H <= 2048 / 3072 (Megatron) / 4352 (Turing-NLG 4256)
    if (oct <= 32 * 8) go(ln_fwd_reg_kernel<true, 8>, ln_fwd_reg_kernel<false, 8>);
    else if (oct <= 32 * 12) go(ln_fwd_reg_kernel<true, 12>, ln_fwd_reg_kernel<false, 12>);
    else go(ln_fwd_reg_kernel<true, 17>, ln_fwd_reg_kernel<false, 17>);
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

cudaError_t lm_xent(const void* z, const int64_t* y, void* dz, float* row_loss, int64_t T, int V, float scale,
                    cudaStream_t s) {
  if (T <= 0 || V <= 0 || V % 8 != 0 || V / 8 > kXentThreads * 32) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cap = (int64_t)sms * 2;  // one wave of two CTAs per SM
  const dim3 grid((unsigned)(T < cap ? T : cap));
  auto Z = static_cast<const __nv_bfloat16*>(z);
  auto D = static_cast<__nv_bfloat16*>(dz);
  const int oct = V / 8;
  if (oct <= kXentThreads) lm_xent_kernel<1><<<grid, kXentThreads, 0, s>>>(Z, y, D, row_loss, T, V, scale);
  else if (oct <= kXentThreads * 8) lm_xent_kernel<8><<<grid, kXentThreads, 0, s>>>(Z, y, D, row_loss, T, V, scale);
  else if (oct <= kXentThreads * 16)
    lm_xent_kernel<16><<<grid, kXentThreads, 0, s>>>(Z, y, D, row_loss, T, V, scale);
  else if (oct <= kXentThreads * 25)   // V 51200
    lm_xent_kernel<25><<<grid, kXentThreads, 0, s>>>(Z, y, D, row_loss, T, V, scale);
  else lm_xent_kernel<32><<<grid, kXentThreads, 0, s>>>(Z, y, D, row_loss, T, V, scale);
  return cudaGetLastError();
}

cudaError_t attn_softmax_bwd(const float* S, const float* dP, const float* lse, const float* D, void* P, void* dS,
                             int64_t rows, int s, float scale, cudaStream_t st) {
  if (rows <= 0 || s <= 0 || s % 8 != 0) return cudaErrorInvalidValue;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (rows * (s / 8) + 255) / 256, cap = (int64_t)sms * 8;
  attn_softmax_bwd_kernel<<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(
      S, dP, lse, D, static_cast<__nv_bfloat16*>(P), static_cast<__nv_bfloat16*>(dS), rows, s, scale);
  return cudaGetLastError();
}

}  // namespace krt
