// Weight gradient of an NHWC convolution as a tcgen05 GEMM (sm_100a), with
// the batch-norm + ReLU that produced the convolution's input applied on the
// fly (cost_model.py:97-105 counts these MACs as the layer's backward work):
//
//   dW[co, (tap, ci)] = sum_p dY[p, co] * f(X)[pix(p, tap), ci]
//
//   K = output pixels p (n, oh, ow), split across CTAs (fp32 partial tiles,
//       summed in a fixed order by wgrad_reduce_kernel: deterministic)
//   M = Cout (128-row tiles), N = taps * Cin (tap-major: the OHWI weight
//       layout, so the reduced tile is the gradient in place)
//   f(X) = X, or relu(X*scale + shift) per input channel (the BN of the
//       previous layer; its output is never written and never re-read)
//
// Both operands are MN-major: a k-block is 64 pixels, each one 128-byte
// shared-memory row of 64 channels (SWIZZLE_128B), exactly what a TMA box of
// the NHWC tensor gives.  dY comes by 2D tiled TMA; X by 2D tiled TMA for a
// stride-1 1x1 convolution, else by im2col TMA (one box per (tap, 64-channel
// block): the zero padding and the stride are the TMA unit's, the shifted
// window never exists in HBM).
//
// Structure (one work unit = (k-split, m-tile, n-tile) per CTA):
//   warp 0      TMA producer (A: 2 boxes of 64 co, B: BN/64 boxes)
//   warp 1      TMEM allocator + MMA issuer (one elected thread, M=128 N=BN K=16)
//   warps 2..5  epilogue: tcgen05.ld of the accumulator -> fp32 partial tile
//   warps 6..13 prologue: relu(bn(.)) of each B stage in shared memory, with
//               the padding rows of the tap forced back to zero
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "sm100_common.cuh"
#include "wgrad_sm100.hpp"

namespace krt {
namespace {
using namespace sm100;

constexpr int kWBK = 64;             // pixels per k-block
constexpr int kWBox = 64 * kWBK * 2;  // one [64 pixels][64 channels] bf16 box: 8 KB
constexpr int kWXf0 = 6;             // first prologue warp
constexpr int kWXfThreads = 256;
constexpr int kWThreads = 64 + 128 + kWXfThreads;
constexpr int kWMaxC = 1024;  // prologue channels held in shared memory

struct WgParams {
  int64_t P;            // output pixels (the GEMM's K)
  int M, N, cin;        // Cout, taps * Cin, Cin
  int n_tiles, tiles, kbps;
  int64_t kblocks;
  float* ws;            // [splits][M][N] fp32 partial tiles
  // convolution geometry (im2col and the padding mask)
  int xh, xw, ho, wo, ks, stride, pad;
  const float* pmean;
  const float* pinvstd;
  const __nv_bfloat16* pg;
  const __nv_bfloat16* pb;
};

template <int BN, int STAGES, bool PRO>
struct WgSmem {
  alignas(1024) uint8_t a[STAGES][2 * kWBox];
  alignas(1024) uint8_t b[STAGES][BN / 64 * kWBox];
  uint64_t full[STAGES], ready[STAGES], empty[STAGES];
  uint64_t tfull;
  uint32_t tmem_base;
  alignas(16) float sc[PRO ? kWMaxC : 4];
  alignas(16) float sh[PRO ? kWMaxC : 4];
};

// UMMA descriptor of an MN-major SWIZZLE_128B operand: 64-element MN chunks
// (128-byte rows, one per K index) LBO bytes apart, 8-row K groups 1024 bytes
// apart (cute/atom/mma_traits_sm100.hpp, Major::MN B128:
// ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16-byte units)
__device__ __forceinline__ uint64_t mnmajor_desc(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::f16, D f32, A/B bf16, both MN-major, M = 128, N
__host__ __device__ constexpr uint32_t instr_desc_mn(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(kBM >> 4) << 24);
}

template <int BN, int STAGES, bool PRO, bool IM2COL>
__global__ void __launch_bounds__(kWThreads, 1)
    wgrad_kernel(const __grid_constant__ CUtensorMap map_dy, const __grid_constant__ CUtensorMap map_x, WgParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  auto& S = *reinterpret_cast<WgSmem<BN, STAGES, PRO>*>(smem_raw);
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();
  constexpr int kBoxes = BN / 64;
  constexpr uint32_t kTmemCols = BN <= 64 ? 64 : (BN <= 128 ? 128 : 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // work unit: consecutive CTAs share a k-split (same pixels: L2 reuse)
  const int split = blockIdx.x / p.tiles, tile = blockIdx.x % p.tiles;
  const int m0 = (tile / p.n_tiles) * kBM, n0 = (tile % p.n_tiles) * BN;
  const int64_t kb_lo = (int64_t)split * p.kbps;
  const int64_t kb_hi = kb_lo + p.kbps < p.kblocks ? kb_lo + p.kbps : p.kblocks;
  const int plane = p.ho * p.wo;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.ready[s], kWXfThreads);
      mbar_init(&S.empty[s], 1);
    }
    mbar_init(&S.tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(&S.tmem_base, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t kb = kb_lo; kb < kb_hi; ++kb) {
        mbar_wait(&S.empty[stage], phase ^ 1);
        mbar_expect_tx(&S.full[stage], (2 + kBoxes) * kWBox);
        const int64_t p0 = kb * kWBK;
        tma_load_2d(&map_dy, &S.full[stage], S.a[stage], m0, (int)p0);
        tma_load_2d(&map_dy, &S.full[stage], S.a[stage] + kWBox, m0 + 64, (int)p0);
        int n = 0, oh = 0, ow = 0;
        if (IM2COL) {
          n = (int)(p0 / plane);
          const int rem = (int)(p0 - (int64_t)n * plane);
          oh = rem / p.wo;
          ow = rem - oh * p.wo;
        }
#pragma unroll
        for (int b = 0; b < kBoxes; ++b) {
          const int col = n0 + 64 * b, tap = col / p.cin, c0 = col - tap * p.cin;
          if (IM2COL)
            tma_load_im2col_4d(&map_x, &S.full[stage], S.b[stage] + b * kWBox, c0, ow * p.stride - p.pad,
                               oh * p.stride - p.pad, n, (uint16_t)(tap % p.ks), (uint16_t)(tap / p.ks));
          else
            tma_load_2d(&map_x, &S.full[stage], S.b[stage] + b * kWBox, c0, (int)p0);
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = instr_desc_mn(BN);
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t kb = kb_lo; kb < kb_hi; ++kb) {
      mbar_wait(PRO ? &S.ready[stage] : &S.full[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(S.a[stage]), b0 = smem_u32(S.b[stage]);
#pragma unroll
        for (int k = 0; k < kWBK / kUmmaK; ++k)  // 16 pixels = two 8-row groups = 2048 bytes
          umma_bf16(tmem, mnmajor_desc(a0 + k * 2048, kWBox), mnmajor_desc(b0 + k * 2048, kWBox), idesc,
                    (kb != kb_lo || k != 0) ? 1u : 0u);
        umma_commit(&S.empty[stage]);
        if (kb == kb_hi - 1) umma_commit(&S.tfull);
      }
      __syncwarp();
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp < kWXf0) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter
    mbar_wait(&S.tfull, 0);
    tc_fence_after();
    float* row = p.ws + ((size_t)split * p.M + m0 + q * 32 + lane) * p.N + n0;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c * 32, v);
      float4* dst = reinterpret_cast<float4*>(row + c * 32);
#pragma unroll
      for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
  } else if (PRO) {
    // ------------------------------------------------------------ prologue transform
    const int xt = threadIdx.x - kWXf0 * 32;  // 0..255
    const int r = xt & 63, jb = 2 * (xt >> 6);  // pixel row of the box; first of two 16-byte chunks
    for (int c = xt; c < p.cin; c += kWXfThreads) {
      const float sc = p.pinvstd[c] * __bfloat162float(p.pg[c]);
      S.sc[c] = sc;
      S.sh[c] = __bfloat162float(p.pb[c]) - p.pmean[c] * sc;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kWXfThreads) : "memory");
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t kb = kb_lo; kb < kb_hi; ++kb) {
      // this row's pixel and the window origin of its input
      const int64_t pix = kb * kWBK + r;
      int ih0 = 0, iw0 = 0;
      const bool pvalid = pix < p.P;
      if (IM2COL) {
        const int n = (int)(pix / plane);
        const int rem = (int)(pix - (int64_t)n * plane);
        const int oh = rem / p.wo;
        ih0 = oh * p.stride - p.pad;
        iw0 = (rem - oh * p.wo) * p.stride - p.pad;
      }
      mbar_wait(&S.full[stage], phase);
#pragma unroll
      for (int b = 0; b < kBoxes; ++b) {
        const int col = n0 + 64 * b, tap = col / p.cin, c0 = col - tap * p.cin;
        bool valid = true;
        if (IM2COL) {
          const int ih = ih0 + tap / p.ks, iw = iw0 + tap % p.ks;
          valid = pvalid && ih >= 0 && ih < p.xh && iw >= 0 && iw < p.xw;
        }
        uint4* rowp = reinterpret_cast<uint4*>(S.b[stage] + b * kWBox + r * 128);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int j = jb + i, phys = j ^ (r & 7);
          uint4 u = rowp[phys];
          if (!valid) {
            u = make_uint4(0u, 0u, 0u, 0u);  // padding stays zero (relu(bn(0)) would not)
          } else {
            const int cc = c0 + 8 * j;
            const ulonglong2 sa = *reinterpret_cast<const ulonglong2*>(&S.sc[cc]);
            const ulonglong2 sb = *reinterpret_cast<const ulonglong2*>(&S.sc[cc + 4]);
            const ulonglong2 ha = *reinterpret_cast<const ulonglong2*>(&S.sh[cc]);
            const ulonglong2 hb = *reinterpret_cast<const ulonglong2*>(&S.sh[cc + 4]);
            const unsigned long long sc2[4] = {sa.x, sa.y, sb.x, sb.y}, sh2[4] = {ha.x, ha.y, hb.x, hb.y};
            uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t lo = w[e] << 16, hi = w[e] & 0xffff0000u;
              const unsigned long long xv = ((unsigned long long)hi << 32) | lo;
              unsigned long long yv;
              asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(yv) : "l"(xv), "l"(sc2[e]), "l"(sh2[e]));
              uint32_t packed;
              asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;"
                  : "=r"(packed)
                  : "f"(__uint_as_float((uint32_t)(yv >> 32))), "f"(__uint_as_float((uint32_t)yv)));
              w[e] = packed;
            }
          }
          rowp[phys] = u;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&S.ready[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kTmemCols);
}

// out[i] = sum over splits of ws[s][i], fixed order (float4 lanes)
__global__ void wgrad_reduce_kernel(const float4* __restrict__ ws, float4* __restrict__ out, int64_t n4, int splits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 s = ws[i];
    for (int k = 1; k < splits; ++k) {
      const float4 v = ws[(size_t)k * n4 + i];
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    out[i] = s;
  }
}

// ---------------------------------------------------------------------------
// host side
template <int BN, bool PRO, bool IM2COL>
cudaError_t wgrad_launch(const CUtensorMap& mdy, const CUtensorMap& mx, const WgParams& p, int grid, cudaStream_t s) {
  constexpr int stage_bytes = (2 + BN / 64) * kWBox;
  constexpr int fixed = PRO ? 2 * kWMaxC * 4 : 0;
  constexpr int stages_fit = (200 * 1024 - fixed) / stage_bytes;
  constexpr int STAGES = stages_fit > 8 ? 8 : stages_fit;
  static_assert(STAGES >= 3, "shared memory");
  auto k = wgrad_kernel<BN, STAGES, PRO, IM2COL>;
  const size_t smem = sizeof(WgSmem<BN, STAGES, PRO>);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k<<<grid, kWThreads, smem, s>>>(mdy, mx, p);
  return cudaGetLastError();
}

template <int BN>
cudaError_t wgrad_dispatch(bool pro, bool im2col, const CUtensorMap& mdy, const CUtensorMap& mx, const WgParams& p,
                           int grid, cudaStream_t s) {
  if (pro) return im2col ? wgrad_launch<BN, true, true>(mdy, mx, p, grid, s)
                         : wgrad_launch<BN, true, false>(mdy, mx, p, grid, s);
  return im2col ? wgrad_launch<BN, false, true>(mdy, mx, p, grid, s)
                : wgrad_launch<BN, false, false>(mdy, mx, p, grid, s);
}

int pick_bn(int N) {
  if (N % 256 == 0) return 256;
  if (N % 192 == 0) return 192;
  if (N % 128 == 0) return 128;
  return 64;
}

struct WgPlan {
  int bn, tiles, splits, kbps;
  int64_t kblocks;
};

WgPlan wgrad_plan(int64_t P, int M, int N) {
  WgPlan w;
  w.bn = pick_bn(N);
  w.tiles = (M / kBM) * (N / w.bn);
  w.kblocks = (P + kWBK - 1) / kWBK;
  int want = num_sms() / w.tiles;
  if (want < 1) want = 1;
  if (want > w.kblocks) want = (int)w.kblocks;
  w.kbps = (int)((w.kblocks + want - 1) / want);
  w.splits = (int)((w.kblocks + w.kbps - 1) / w.kbps);  // every split non-empty
  return w;
}
}  // namespace

bool conv_wgrad_supported(int cout, int cin, int k, int stride) {
  return cout % kBM == 0 && cin % 64 == 0 && (k == 1 || k == 3) && stride >= 1 && stride <= 2;
}

size_t conv_wgrad_workspace_bytes(int n, int ho, int wo, int cout, int cin, int k) {
  const int64_t P = (int64_t)n * ho * wo;
  if (P <= 0 || cout % kBM != 0 || cin % 64 != 0) return 0;
  const WgPlan w = wgrad_plan(P, cout, k * k * cin);
  return (size_t)w.splits * cout * k * k * cin * sizeof(float);
}

cudaError_t conv_wgrad(const void* dy, const void* x, float* dw, int n, int h, int w, int cin, int ho, int wo,
                       int cout, int k, int stride, int pad, const float* pmean, const float* pinvstd, const void* pg,
                       const void* pb, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (!conv_wgrad_supported(cout, cin, k, stride) || n < 1 || ho < 1 || wo < 1) return cudaErrorInvalidValue;
  if (pmean != nullptr && cin > kWMaxC) return cudaErrorInvalidValue;
  // the im2col traversal visits exactly these output rows / columns
  if (ho != (h + 2 * pad - k) / stride + 1 || wo != (w + 2 * pad - k) / stride + 1) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dw) |
       reinterpret_cast<uintptr_t>(ws)) & 15)
    return cudaErrorMisalignedAddress;
  const int64_t P = (int64_t)n * ho * wo;
  if (P > 0x7fffffffLL) return cudaErrorInvalidValue;  // TMA row coordinate
  const int N = k * k * cin;
  const WgPlan pl = wgrad_plan(P, cout, N);
  if (ws_bytes < (size_t)pl.splits * cout * N * sizeof(float)) return cudaErrorInvalidValue;
  WgParams p{};
  p.P = P;
  p.M = cout;
  p.N = N;
  p.cin = cin;
  p.n_tiles = N / pl.bn;
  p.tiles = pl.tiles;
  p.kbps = pl.kbps;
  p.kblocks = pl.kblocks;
  p.ws = static_cast<float*>(ws);
  p.xh = h;
  p.xw = w;
  p.ho = ho;
  p.wo = wo;
  p.ks = k;
  p.stride = stride;
  p.pad = pad;
  p.pmean = pmean;
  p.pinvstd = pinvstd;
  p.pg = static_cast<const __nv_bfloat16*>(pg);
  p.pb = static_cast<const __nv_bfloat16*>(pb);
  const bool im2col = k != 1 || stride != 1;
  CUtensorMap mdy, mx;
  if (!make_map(&mdy, dy, P, cout, kWBK, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  if (im2col) {
    if (!make_im2col_map(&mx, x, n, h, w, cin, k, stride, pad, kWBK)) return cudaErrorInvalidValue;
  } else if (!make_map(&mx, x, P, cin, kWBK, 64, CU_TENSOR_MAP_SWIZZLE_128B)) {
    return cudaErrorInvalidValue;
  }
  const int grid = pl.tiles * pl.splits;
  const bool pro = pmean != nullptr;
  cudaError_t e;
  switch (pl.bn) {
    case 256: e = wgrad_dispatch<256>(pro, im2col, mdy, mx, p, grid, s); break;
    case 192: e = wgrad_dispatch<192>(pro, im2col, mdy, mx, p, grid, s); break;
    case 128: e = wgrad_dispatch<128>(pro, im2col, mdy, mx, p, grid, s); break;
    default: e = wgrad_dispatch<64>(pro, im2col, mdy, mx, p, grid, s); break;
  }
  if (e != cudaSuccess) return e;
  const int64_t n4 = (int64_t)cout * N / 4;
  int64_t blocks = (n4 + 255) / 256;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  wgrad_reduce_kernel<<<(int)blocks, 256, 0, s>>>(static_cast<const float4*>(ws), reinterpret_cast<float4*>(dw), n4,
                                                  pl.splits);
  return cudaGetLastError();
}

}  // namespace krt
