// sm_100a kernels of the runtime's memory path.  All are HBM-bound streaming
// kernels: 128-bit vector loads/stores, grid-stride loops over a persistent
// grid sized to 148 SMs x resident CTAs.
//
//  * update_kernel  — Adam/SGD over fp32 master shards for blocks that stay
//    on the device (distsim.py:14-16); arithmetic identical to
//    host_optim.cpp (__f*_rn intrinsics forbid FMA contraction).
//  * reduce_cast_kernel — fused gradient scale + sum over n_in sources +
//    cast (fp32/bf16) into a contiguous send/landing buffer: the "grad
//    scale/cast pack" in front of the exchange (distsim.py:205-230).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"
#include "optim.hpp"

namespace krt {
namespace {

__device__ __forceinline__ float adam_elem(float g, float& p, float& m, float& v, const OptimScalars& s) {
  if (s.weight_decay != 0.0f) g = __fadd_rn(g, __fmul_rn(s.weight_decay, p));
  float d = __fsub_rn(g, m);
  if (s.lerp_w < 0.5f) m = __fadd_rn(m, __fmul_rn(s.lerp_w, d));
  else m = __fsub_rn(g, __fmul_rn(d, __fsub_rn(1.0f, s.lerp_w)));
  v = __fadd_rn(__fmul_rn(v, s.beta2), __fmul_rn(__fmul_rn(s.one_m_b2, g), g));
  float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), s.bc2_sqrt), s.eps);
  p = __fadd_rn(p, __fmul_rn(s.neg_step, __fdiv_rn(m, denom)));
  return p;
}

__device__ __forceinline__ float sgd_elem(float g, float& p, float& m, const OptimScalars& s) {
  if (s.weight_decay != 0.0f) g = __fadd_rn(g, __fmul_rn(s.weight_decay, p));
  if (s.momentum != 0.0f) {
    float b = s.first_step ? g : __fadd_rn(__fmul_rn(m, s.momentum), g);
    m = b;
    g = b;
  }
  p = __fadd_rn(p, __fmul_rn(-s.lr, g));
  return p;
}

template <int WDT>
__global__ void __launch_bounds__(256) update_kernel(float* __restrict__ master, float* __restrict__ m,
                                                     float* __restrict__ v, const float* __restrict__ grad,
                                                     void* __restrict__ weights, size_t n, OptimScalars s) {
  size_t n4 = n / 4;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 g = reinterpret_cast<const float4*>(grad)[i];
    float4 p = reinterpret_cast<float4*>(master)[i];
    float4 mm = s.optimizer == 1 || s.momentum != 0.0f ? reinterpret_cast<float4*>(m)[i] : make_float4(0, 0, 0, 0);
    float4 vv = s.optimizer == 1 ? reinterpret_cast<float4*>(v)[i] : make_float4(0, 0, 0, 0);
    float gs[4] = {__fmul_rn(g.x, s.grad_scale), __fmul_rn(g.y, s.grad_scale), __fmul_rn(g.z, s.grad_scale),
                   __fmul_rn(g.w, s.grad_scale)};
    float ps[4] = {p.x, p.y, p.z, p.w}, ms[4] = {mm.x, mm.y, mm.z, mm.w}, vs[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (s.optimizer == 1) adam_elem(gs[k], ps[k], ms[k], vs[k], s);
      else sgd_elem(gs[k], ps[k], ms[k], s);
    }
    reinterpret_cast<float4*>(master)[i] = make_float4(ps[0], ps[1], ps[2], ps[3]);
    if (s.optimizer == 1 || s.momentum != 0.0f) reinterpret_cast<float4*>(m)[i] = make_float4(ms[0], ms[1], ms[2], ms[3]);
    if (s.optimizer == 1) reinterpret_cast<float4*>(v)[i] = make_float4(vs[0], vs[1], vs[2], vs[3]);
    if (WDT == 1) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(ps[0], ps[1]);
      __nv_bfloat162 hi = __floats2bfloat162_rn(ps[2], ps[3]);
      uint2 packed;
      packed.x = *reinterpret_cast<uint32_t*>(&lo);
      packed.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(weights)[i] = packed;
    } else if (weights != master) {
      reinterpret_cast<float4*>(weights)[i] = make_float4(ps[0], ps[1], ps[2], ps[3]);
    }
  }
  // tail (n % 4) by the first threads
  size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t i = n4 * 4 + t;
  if (i < n) {
    float g = __fmul_rn(grad[i], s.grad_scale);
    float p = master[i], mm = (s.optimizer == 1 || s.momentum != 0.0f) ? m[i] : 0.f, vv = s.optimizer == 1 ? v[i] : 0.f;
    if (s.optimizer == 1) adam_elem(g, p, mm, vv, s);
    else sgd_elem(g, p, mm, s);
    master[i] = p;
    if (s.optimizer == 1 || s.momentum != 0.0f) m[i] = mm;
    if (s.optimizer == 1) v[i] = vv;
    if (WDT == 1) reinterpret_cast<__nv_bfloat16*>(weights)[i] = __float2bfloat16_rn(p);
    else if (weights != master) reinterpret_cast<float*>(weights)[i] = p;
  }
}

constexpr int kMaxIn = 16;
struct InPtrs {
  const float* p[kMaxIn];
};

template <int ODT>
__global__ void __launch_bounds__(256) reduce_cast_kernel(InPtrs in, int n_in, void* __restrict__ out, size_t n,
                                                          float scale) {
  size_t n4 = n / 4;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 acc = __ldcs(reinterpret_cast<const float4*>(in.p[0]) + i);
    for (int r = 1; r < n_in; ++r) {
      float4 x = __ldcs(reinterpret_cast<const float4*>(in.p[r]) + i);
      acc.x = __fadd_rn(acc.x, x.x); acc.y = __fadd_rn(acc.y, x.y);
      acc.z = __fadd_rn(acc.z, x.z); acc.w = __fadd_rn(acc.w, x.w);
    }
    acc.x = __fmul_rn(acc.x, scale); acc.y = __fmul_rn(acc.y, scale);
    acc.z = __fmul_rn(acc.z, scale); acc.w = __fmul_rn(acc.w, scale);
    if (ODT == 1) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x, acc.y), hi = __floats2bfloat162_rn(acc.z, acc.w);
      uint2 packed;
      packed.x = *reinterpret_cast<uint32_t*>(&lo);
      packed.y = *reinterpret_cast<uint32_t*>(&hi);
      __stcs(reinterpret_cast<uint2*>(out) + i, packed);
    } else {
      __stcs(reinterpret_cast<float4*>(out) + i, acc);
    }
  }
  size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t i = n4 * 4 + t;
  if (i < n) {
    float acc = in.p[0][i];
    for (int r = 1; r < n_in; ++r) acc = __fadd_rn(acc, in.p[r][i]);
    acc = __fmul_rn(acc, scale);
    if (ODT == 1) reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(acc);
    else reinterpret_cast<float*>(out)[i] = acc;
  }
}

// bf16 -> fp32 (x scale): the reduce-scattered bf16 shard back to the fp32
// gradient shard the host update reads
__global__ void __launch_bounds__(256) unpack_bf16_kernel(const __nv_bfloat16* __restrict__ in,
                                                          float* __restrict__ out, size_t n, float scale) {
  size_t n4 = n / 4;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    uint2 u = __ldcs(reinterpret_cast<const uint2*>(in) + i);
    float2 lo = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
    float2 hi = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
    __stcs(reinterpret_cast<float4*>(out) + i, make_float4(__fmul_rn(lo.x, scale), __fmul_rn(lo.y, scale),
                                                            __fmul_rn(hi.x, scale), __fmul_rn(hi.y, scale)));
  }
  size_t i = n4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __fmul_rn(__bfloat162float(in[i]), scale);
}

int grid_for(size_t n4) {
  // persistent grid: 148 SMs x 8 resident 256-thread CTAs, fewer for small n
  size_t want = (n4 + 255) / 256;
  size_t cap = 148 * 8;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

cudaError_t launch_update(float* master, float* m, float* v, const float* grad, void* weights, int weight_dtype,
                          size_t n, const OptimScalars& s, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  int grid = grid_for(n / 4 + 1);
  if (weight_dtype == 1) update_kernel<1><<<grid, 256, 0, stream>>>(master, m, v, grad, weights, n, s);
  else update_kernel<0><<<grid, 256, 0, stream>>>(master, m, v, grad, weights, n, s);
  return cudaGetLastError();
}

cudaError_t launch_unpack_bf16(const void* in, float* out, size_t n, float scale, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  unpack_bf16_kernel<<<grid_for(n / 4 + 1), 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(in), out, n, scale);
  return cudaGetLastError();
}

cudaError_t launch_reduce_cast(const float* const* in, int n_in, void* out, int out_dtype, size_t n, float scale,
                               cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (n_in < 1 || n_in > kMaxIn) return cudaErrorInvalidValue;
  InPtrs ptrs{};
  for (int r = 0; r < n_in; ++r) ptrs.p[r] = in[r];
  int grid = grid_for(n / 4 + 1);
  if (out_dtype == 1) reduce_cast_kernel<1><<<grid, 256, 0, stream>>>(ptrs, n_in, out, n, scale);
  else reduce_cast_kernel<0><<<grid, 256, 0, stream>>>(ptrs, n_in, out, n, scale);
  return cudaGetLastError();
}

}  // namespace krt
