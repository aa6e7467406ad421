// Weight gradient of a 3x3 / stride-1 / pad-1 convolution with few channels
// (C = cin = cout in {16, 32, 64}: ResNet-1001's bottleneck widths) on
// tcgen05, from halo windows (sm_100a):
//
//   dW[co][r][s][ci] = sum over pixels of dy[pix][co] * f(x)[pix + (r-1, s-1)][ci]
//   f = identity, or relu(x * scale + shift) per channel (the BN + ReLU the
//   forward convolved; the zero padding stays zero)
//
// The pixel dimension is the MMA's K.  Tiles are runs of V virtual rows of a
// (image, column segment) exactly as in halo_sm100.cu: the x window (whole
// padded input rows) and the dy tile (the same virtual rows, junk columns
// zeroed) sit in shared memory as rows of C channels (32 / 64 / 128 bytes,
// SWIZZLE_32B / 64B / 128B).  For each filter row r and 16-row K chunk, one
// MMA with M = 128 reads A = the window as an MN-major operand whose M atoms
// (C channels each) are consecutive window rows - atom i is filter column
// s = i (LBO = one row; atoms beyond s = 2 are junk rows of D, discarded) - and
// B = the dy tile, MN-major with N = C.  D[(s, ci)][co] accumulates in TMEM
// over every tile the CTA processes; the CTAs' partial D are summed in a fixed
// order by a finalize kernel (deterministic).  cuDNN's kernels for these
// shapes run at 9-23% of their HBM floor (profiles/round2_s3).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "halo_sm100.hpp"
#include "sm100_common.cuh"

namespace krt {
namespace {
using namespace sm100;

constexpr int wThreads = 64 + 128 + 256;  // producer, MMA, 4 drain warps, 8 transform warps
constexpr int wXf0 = 6;                   // first transform warp
constexpr int wXfThreads = 256;

struct WgParams {
  int n, H, W, C;
  int Ws, nseg, Wp, R, Rdy;
  int V;  // virtual rows per tile (multiple of 16)
  int tiles_img, tiles;
  uint32_t win_bytes, dy_bytes, slot_bytes;
  float* part;  // [gridDim.x][n_acc][128][C]
  const float* pmean;
  const float* pinvstd;
  const __nv_bfloat16* pg;
  const __nv_bfloat16* pb;
};

struct WgBars {
  uint64_t full[2], ready[2], empty[2];
  uint64_t done;
  uint32_t tmem_base;
};

// MN-major UMMA descriptor: rows of C bf16 (the swizzle span), M atoms LBO
// bytes apart, 8-row K groups SBO = 8 rows apart
template <int C>
__device__ __forceinline__ uint64_t mn_desc(uint32_t addr, uint32_t lbo) {
  constexpr uint64_t layout = C == 64 ? 2 : (C == 32 ? 4 : 6);  // SW128 / SW64 / SW32
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((8 * C * 2) >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= layout << 61;
  return d;
}

// kind::f16 instruction descriptor, D f32, A/B bf16 both MN-major, M = 128, N
__host__ __device__ constexpr uint32_t idesc_mn(int n, int m = 128) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

// M of the narrow 3x3 weight gradient's MMAs: 64 at 16 channels (four window
// atoms, filter columns 0..2 + one junk, instead of eight), else 128
template <int C>
__host__ __device__ constexpr int wg_mm() { return C == 16 ? 64 : 128; }

template <int C, bool PRO>
__global__ void __launch_bounds__(wThreads, 1) wgrad3x3_halo_kernel(const __grid_constant__ CUtensorMap map_x,
                                                                    const __grid_constant__ CUtensorMap map_dy,
                                                                    WgParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  constexpr int kRB = C * 2;           // row bytes
  constexpr int kMM = wg_mm<C>();      // MMA M
  constexpr int kApm = kMM / C;        // M atoms (filter columns) per MMA
  constexpr int kNm = (3 + kApm - 1) / kApm;  // MMAs per filter row
  constexpr int kAcc = 3 * kNm;        // accumulators of C columns
  constexpr uint32_t kCols = kAcc * C <= 32 ? 32 : (kAcc * C <= 64 ? 64 : (kAcc * C <= 128 ? 128 : (kAcc * C <= 256 ? 256 : 512)));
  uint8_t* slots = smem;  // [2][slot_bytes]: window, then dy tile
  float* sc = reinterpret_cast<float*>(smem + 2 * (size_t)p.slot_bytes);
  float* sh = sc + C;
  WgBars& B = *reinterpret_cast<WgBars*>(sh + C);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.full[i], 1);
      mbar_init(&B.ready[i], wXfThreads);
      mbar_init(&B.empty[i], 1);
    }
    mbar_init(&B.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(&B.tmem_base, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int sl = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        const int img = t / p.tiles_img, v0 = (t - img * p.tiles_img) * p.V;
        const int p_lo = v0 / p.Wp, n = img / p.nseg, seg = img - n * p.nseg;
        mbar_wait(&B.empty[sl], ph ^ 1);
        mbar_expect_tx(&B.full[sl], (uint32_t)(p.R + p.Rdy) * p.Wp * kRB);
        uint8_t* wdst = slots + (size_t)sl * p.slot_bytes;
        // x window: padded rows from p_lo - 1, columns from seg*Ws - 1
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(wdst)),
            "l"(reinterpret_cast<uint64_t>(&map_x)), "r"(smem_u32(&B.full[sl])), "r"(0), "r"(seg * p.Ws - 1),
            "r"(p_lo - 1), "r"(n)
            : "memory");
        // dy tile: the same virtual rows (row p_lo, column seg*Ws on)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(wdst + p.win_bytes)),
            "l"(reinterpret_cast<uint64_t>(&map_dy)), "r"(smem_u32(&B.full[sl])), "r"(0), "r"(seg * p.Ws),
            "r"(p_lo), "r"(n)
            : "memory");
        if (++sl == 2) {
          sl = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_mn(C, kMM);
    int sl = 0;
    uint32_t ph = 0;
    bool first = true;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int img = t / p.tiles_img, v0 = (t - img * p.tiles_img) * p.V;
      const int off = v0 - (v0 / p.Wp) * p.Wp;
      mbar_wait(&B.ready[sl], ph);
      tc_fence_after();
      const uint32_t wbase = smem_u32(slots + (size_t)sl * p.slot_bytes);
      const uint32_t dbase = wbase + p.win_bytes;
      for (int kc = 0; kc < p.V / 16; ++kc) {
        const uint64_t bdesc = mn_desc<C>(dbase + (uint32_t)(off + kc * 16) * kRB, kRB);
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int mi = 0; mi < kNm; ++mi) {
            const uint32_t arow = (uint32_t)(off + kc * 16 + r * p.Wp + mi * kApm);
            umma_bf16_elect(tmem + (r * kNm + mi) * C, mn_desc<C>(wbase + arow * kRB, kRB), bdesc, idesc,
                            first ? 0u : 1u);
          }
        first = false;
      }
      umma_commit_elect(&B.empty[sl]);
      if (++sl == 2) {
        sl = 0;
        ph ^= 1;
      }
    }
    umma_commit_elect(&B.done);
  } else if (warp >= wXf0) {
    // ------------------------------------------------------------ window prologue + dy junk rows
    const int xt = threadIdx.x - wXf0 * 32;
    if (PRO) {
      for (int c = xt; c < C; c += wXfThreads) {
        const float s = p.pinvstd[c] * __bfloat162float(p.pg[c]);
        sc[c] = s;
        sh[c] = __bfloat162float(p.pb[c]) - p.pmean[c] * s;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(wXfThreads) : "memory");
    }
    constexpr int kCPR = C / 8;              // 16-byte chunks per row
    constexpr int kRS = wXfThreads / kCPR;   // rows per pass
    const int ch = xt % kCPR;
    unsigned long long sc2[4], sh2[4];
    if (PRO) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = ch * 8 + 2 * e;
        sc2[e] = ((unsigned long long)__float_as_uint(sc[c + 1]) << 32) | __float_as_uint(sc[c]);
        sh2[e] = ((unsigned long long)__float_as_uint(sh[c + 1]) << 32) | __float_as_uint(sh[c]);
      }
    }
    int sl = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      const int img = t / p.tiles_img, v0 = (t - img * p.tiles_img) * p.V;
      const int p_lo = v0 / p.Wp, off = v0 - p_lo * p.Wp;
      const int seg = img % p.nseg, q0 = seg * p.Ws;
      mbar_wait(&B.full[sl], ph);
      uint8_t* wb = slots + (size_t)sl * p.slot_bytes;
      if (PRO) {  // relu(bn(x)) on the window rows the MMAs read; padding stays zero
        const int jhi = off + p.V + 2 * p.Wp + 2;
        const int jd = kRS / p.Wp, jm = kRS - jd * p.Wp;
        const int j0 = off + xt / kCPR;
        int wr = j0 / p.Wp, wc = j0 - (j0 / p.Wp) * p.Wp;
        for (int j = j0; j < jhi; j += kRS) {
          const int ip = p_lo - 1 + wr, iq = q0 - 1 + wc;
          if (ip >= 0 && ip < p.H && iq >= 0 && iq < p.W) {
            uint4* cp = reinterpret_cast<uint4*>(wb + (size_t)j * kRB + (swz_chunk<C>(ch, j) << 4));
            uint4 u = *cp;
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
            *cp = u;
          }
          wr += jd;
          wc += jm;
          if (wc >= p.Wp) {
            wc -= p.Wp;
            ++wr;
          }
        }
      }
      // dy rows of junk columns (beyond the segment or the image) hold the
      // neighbouring segment's pixels: zero them so they add nothing
      {
        uint8_t* db = wb + p.win_bytes;
        const int rows = p.Rdy * p.Wp;
        for (int j = xt / kCPR; j < rows; j += kRS) {
          const int q = j % p.Wp;
          if (q >= p.Ws || q0 + q >= p.W)
            *reinterpret_cast<uint4*>(db + (size_t)j * kRB + ch * 16) = make_uint4(0u, 0u, 0u, 0u);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&B.ready[sl]);
      if (++sl == 2) {
        sl = 0;
        ph ^= 1;
      }
    }
  } else {
    // ------------------------------------------------------------ drain (warps 2..5)
    // after the CTA's last MMA: every accumulator's 128 lanes x C columns
    // into this CTA's partial block
    const int q = warp & 3;
    mbar_wait_sleep(&B.done, 0, 4000);
    tc_fence_after();
    float* out = p.part + (size_t)blockIdx.x * kAcc * 128 * C;
    for (int a = 0; a < kAcc; ++a)
      for (int c = 0; c < C; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + a * C + c, v);
        float* dst = out + ((size_t)a * 128 + q * 32 + lane) * C + c;
#pragma unroll
        for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kCols);
}

// dW[co][r][s][ci] = sum over CTAs (fixed order) of D_(r, s / apm)[(s % apm) * C + ci][co]
// M = 64 accumulators: row m sits in TMEM lane (m / 16) * 32 + m % 16 (lanes
// 0..15 of each 32-lane quarter) - determined by test: lane_mode 0 passes
// tests/test_wgrad_narrow_gpu.py, 1 (lanes 0..63) fails; KRT_M64_LANES
// selects it for such checks
__device__ __forceinline__ int m64_lane(int m, int mode) { return mode ? m : (m >> 4) * 32 + (m & 15); }

template <int C>
__global__ void wgrad3x3_halo_finalize(const float* __restrict__ part, int ctas, float* __restrict__ dw,
                                       int lane_mode) {
  constexpr int kMM = wg_mm<C>();
  constexpr int kApm = kMM / C, kNm = (3 + kApm - 1) / kApm, kAcc = 3 * kNm;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over co, r, s, ci
  if (i >= C * 9 * C) return;
  const int ci = i % C, s = (i / C) % 3, r = (i / (3 * C)) % 3, co = i / (9 * C);
  const int a = r * kNm + s / kApm, mrow = (s % kApm) * C + ci;
  const int lanei = kMM == 64 ? m64_lane(mrow, lane_mode) : mrow;
  double acc = 0.0;
  for (int k = 0; k < ctas; ++k) acc += (double)part[(((size_t)k * kAcc + a) * 128 + lanei) * C + co];
  dw[i] = (float)acc;
}

int wg_rows(int Wp, int rows) { return (Wp - 1 + rows - 1 + 2 * Wp + 2) / Wp + 1; }
size_t r1k(size_t b) { return (b + 1023) / 1024 * 1024; }

struct WgPlan {
  int Ws = 0, nseg = 0, Wp = 0, R = 0, Rdy = 0, V = 0;
  size_t win = 0, dy = 0;
};

bool wg_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("KRT_WGRAD_HALO");
    return e == nullptr || std::strcmp(e, "0") != 0;
  }();
  return on;
}

// largest tile (V virtual rows) and fewest column segments whose two slots fit
bool wg_plan(int h, int w, int C, WgPlan* out) {
  if (!wg_enabled() || (C != 16 && C != 32 && C != 64) || h < 1 || w < 1) return false;
  const int rb = C * 2;
  for (int V : {1024, 512, 256, 128})
    for (int nseg = 1; nseg <= 64; ++nseg) {
      WgPlan q;
      q.V = V;
      q.nseg = nseg;
      q.Ws = (w + nseg - 1) / nseg;
      q.Wp = q.Ws + 2;
      if (q.Wp > 256) continue;
      q.R = wg_rows(q.Wp, V);
      q.Rdy = (q.Wp - 1 + V - 1) / q.Wp + 1;
      if (q.R > 256) continue;
      q.win = r1k((size_t)q.R * q.Wp * rb);
      q.dy = r1k((size_t)q.Rdy * q.Wp * rb);
      if (2 * (q.win + q.dy) + 2 * C * 4 + sizeof(WgBars) + 1024 <= 220 * 1024) {
        *out = q;
        return true;
      }
    }
  return false;
}

template <int C, bool PRO>
cudaError_t launch_wg(const CUtensorMap& mx, const CUtensorMap& mdy, const WgParams& p, int grid, size_t smem,
                      cudaStream_t s) {
  auto k = wgrad3x3_halo_kernel<C, PRO>;
  static size_t configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  k<<<grid, wThreads, smem, s>>>(mx, mdy, p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// 1x1 weight gradient with few channels: dW[co][ci] = sum over pixels of
// dy[pix][co] * f(x)[pix][ci].  The wider side (>= 64 channels) is the MMA's
// M (two 64-channel atoms per M = 128; a 64-channel side adds a junk atom),
// the narrower side (16 .. 64) its N, the pixels its K; both operands
// MN-major straight from their TMA tiles ([channel block][V rows][64 or fewer
// channels]).  The BN prologue transforms the x tile in shared memory (rows
// beyond the tensor stay zero).
struct Wg1Params {
  int64_t M;       // pixels
  int ci, co, V;   // channels, pixels per tile
  int tiles;
  int xm;          // 1: x is the M side (ci >= co)
  uint32_t x_bytes, dy_bytes, slot_bytes;
  float* part;     // [gridDim.x][n_mb][128][nch]
  const float* pmean;
  const float* pinvstd;
  const __nv_bfloat16* pg;
  const __nv_bfloat16* pb;
};

// MCH: M-side channels (64, 128, 256); NCH: N-side channels (16, 32, 64)
template <int MCH, int NCH, bool PRO>
__global__ void __launch_bounds__(wThreads, 1) wgrad1x1_narrow_kernel(const __grid_constant__ CUtensorMap map_x,
                                                                      const __grid_constant__ CUtensorMap map_dy,
                                                                      Wg1Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  constexpr int kMb = MCH / 128 > 0 ? MCH / 128 : 1;   // M = 128 MMAs per K chunk
  constexpr uint32_t kCols = kMb * NCH <= 32 ? 32 : (kMb * NCH <= 64 ? 64 : 128);
  constexpr int kNRB = NCH * 2;                          // N-side row bytes
  const int cix = p.ci < 64 ? p.ci : 64;                 // x tile channels per block
  const int cbx = (p.ci + 63) / 64, cbd = (p.co + 63) / 64;
  const int xrb = cix * 2;                               // x row bytes
  uint8_t* slots = smem;
  float* sc = reinterpret_cast<float*>(smem + 2 * (size_t)p.slot_bytes);
  float* sh = sc + p.ci;
  WgBars& B = *reinterpret_cast<WgBars*>(sh + p.ci);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.full[i], 1);
      mbar_init(&B.ready[i], wXfThreads);
      mbar_init(&B.empty[i], 1);
    }
    mbar_init(&B.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(&B.tmem_base, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_base;
  const int dyc = p.co < 64 ? p.co : 64;

  if (warp == 0) {
    if (lane == 0) {
      int sl = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        const int row0 = t * p.V;
        mbar_wait(&B.empty[sl], ph ^ 1);
        mbar_expect_tx(&B.full[sl], (uint32_t)p.V * (p.ci + p.co) * 2);
        uint8_t* dst = slots + (size_t)sl * p.slot_bytes;
        for (int cb = 0; cb < cbx; ++cb)
          tma_load_2d(&map_x, &B.full[sl], dst + (size_t)cb * p.V * xrb, cb * 64, row0);
        for (int cb = 0; cb < cbd; ++cb)
          tma_load_2d(&map_dy, &B.full[sl], dst + p.x_bytes + (size_t)cb * p.V * dyc * 2, cb * 64, row0);
        if (++sl == 2) {
          sl = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_mn(NCH);
    int sl = 0;
    uint32_t ph = 0;
    bool first = true;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      mbar_wait(&B.ready[sl], ph);
      tc_fence_after();
      const uint32_t base = smem_u32(slots + (size_t)sl * p.slot_bytes);
      const uint32_t mbase = p.xm ? base : base + p.x_bytes, nbase = p.xm ? base + p.x_bytes : base;
      for (int kc = 0; kc < p.V / 16; ++kc) {
        const uint64_t bdesc = mn_desc<NCH>(nbase + (uint32_t)(kc * 16 * kNRB), kNRB);
#pragma unroll
        for (int mb = 0; mb < kMb; ++mb) {
          // two 64-channel atoms per M = 128, p.V rows apart (a 64-channel M
          // side repeats its one atom: LBO 0, D rows 64..127 junk)
          const uint32_t a = mbase + (uint32_t)(mb * 2 * p.V * 128 + kc * 16 * 128);
          umma_bf16_elect(tmem + mb * NCH, mn_desc<64>(a, MCH == 64 ? 0u : (uint32_t)p.V * 128), bdesc, idesc,
                          first ? 0u : 1u);
        }
        first = false;
      }
      umma_commit_elect(&B.empty[sl]);
      if (++sl == 2) {
        sl = 0;
        ph ^= 1;
      }
    }
    umma_commit_elect(&B.done);
  } else if (warp >= wXf0) {
    const int xt = threadIdx.x - wXf0 * 32;
    if (PRO) {
      for (int c = xt; c < p.ci; c += wXfThreads) {
        const float s = p.pinvstd[c] * __bfloat162float(p.pg[c]);
        sc[c] = s;
        sh[c] = __bfloat162float(p.pb[c]) - p.pmean[c] * s;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(wXfThreads) : "memory");
    }
    const int cpr = cix / 8;  // 16-byte chunks per x row
    int sl = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      mbar_wait(&B.full[sl], ph);
      if (PRO) {
        // each thread keeps one 16-byte chunk (8 channels) per channel block
        // and walks the tile's rows with its coefficients in registers
        uint8_t* xb = slots + (size_t)sl * p.slot_bytes;
        const int64_t row0 = (int64_t)t * p.V;
        const int ch = xt % cpr, rs = wXfThreads / cpr;
        const int vmax = (int)(p.M - row0 < p.V ? p.M - row0 : p.V);  // rows beyond the tensor: the TMA's zeros stay
        for (int cb = 0; cb < cbx; ++cb) {
          unsigned long long sc2[4], sh2[4];
          const int c0 = cb * 64 + ch * 8;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            sc2[e] = ((unsigned long long)__float_as_uint(sc[c0 + 2 * e + 1]) << 32) | __float_as_uint(sc[c0 + 2 * e]);
            sh2[e] = ((unsigned long long)__float_as_uint(sh[c0 + 2 * e + 1]) << 32) | __float_as_uint(sh[c0 + 2 * e]);
          }
          uint8_t* cbase = xb + (size_t)cb * p.V * xrb;
          for (int j = xt / cpr; j < vmax; j += rs) {
            const int sw = cix == 64 ? (ch ^ (j & 7)) : (cix == 32 ? (ch ^ ((j >> 1) & 3)) : (ch ^ ((j >> 2) & 1)));
            uint4* cp = reinterpret_cast<uint4*>(cbase + (size_t)j * xrb + (sw << 4));
            uint4 u = *cp;
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
            *cp = u;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      mbar_arrive(&B.ready[sl]);
      if (++sl == 2) {
        sl = 0;
        ph ^= 1;
      }
    }
  } else {
    const int q = warp & 3;
    mbar_wait_sleep(&B.done, 0, 4000);
    tc_fence_after();
    float* out = p.part + (size_t)blockIdx.x * kMb * 128 * NCH;
    for (int mb = 0; mb < kMb; ++mb)
      for (int c = 0; c < NCH; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + mb * NCH + c, v);
        float* dst = out + ((size_t)mb * 128 + q * 32 + lane) * NCH + c;
#pragma unroll
        for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kCols);
}

// dW[co][ci] from the CTAs' partials (fixed order): D[m][n] with m the wide side
__global__ void wgrad1x1_narrow_finalize(const float* __restrict__ part, int ctas, int ci, int co, int xm, int nmb,
                                         int nch, float* __restrict__ dw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over co, ci
  if (i >= ci * co) return;
  const int c_in = i % ci, c_out = i / ci;
  const int m = xm ? c_in : c_out, n = xm ? c_out : c_in;
  double acc = 0.0;
  for (int k = 0; k < ctas; ++k) acc += (double)part[((size_t)k * nmb * 128 + m) * nch + n];
  dw[i] = (float)acc;
}

bool wg1_shape(int ci, int co) {
  const int mch = ci > co ? ci : co, nch = ci > co ? co : ci;
  return (mch == 64 || mch == 128 || mch == 256) && (nch == 16 || nch == 32 || nch == 64);
}

template <int MCH, int NCH, bool PRO>
cudaError_t launch_wg1(const CUtensorMap& mx, const CUtensorMap& mdy, const Wg1Params& p, int grid, size_t smem,
                       cudaStream_t s) {
  auto k = wgrad1x1_narrow_kernel<MCH, NCH, PRO>;
  static size_t configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  k<<<grid, wThreads, smem, s>>>(mx, mdy, p);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The ResNet stem's weight gradient (7x7 / stride 2 / pad 3, 4-channel padded
// RGB input, 64 output channels): dW[co][kh][kw][c] = sum over output pixels
// of dc[pix][co] * x4[2*oh - 3 + kh][2*ow - 3 + kw][c].  Per tile of V output
// pixels the gather warps build each pixel's 7x7x4 window (49 taps x 8 bytes;
// taps 49..63 zero) as four 64-element SW128 atoms ([atom][V rows][64]) - the
// MN-major A operand, M = (tap, c) in two M = 128 blocks; dc arrives by TMA
// as the MN-major B operand (N = 64); pixels are K.  cuDNN runs this on a
// legacy sm80 kernel (~9 ms per b3072 step) after an NHWC padding kernel.
struct StemWgParams {
  int n, H, W, Ho, Wo;
  int64_t M;  // output pixels
  int V, tiles;
  uint32_t a_bytes, slot_bytes;
  const uint2* x4;  // [n, H, W] pixels of 4 bf16
  float* part;      // [gridDim.x][2][128][64]
};

constexpr int sGather = 384;                      // 12 gather warps
constexpr int sThreads = 64 + 128 + sGather;

__global__ void __launch_bounds__(sThreads, 1) stem_wgrad_kernel(const __grid_constant__ CUtensorMap map_dc,
                                                                 StemWgParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  uint8_t* slots = smem;
  WgBars& B = *reinterpret_cast<WgBars*>(smem + 2 * (size_t)p.slot_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&B.full[i], 1);
      mbar_init(&B.ready[i], sGather);
      mbar_init(&B.empty[i], 1);
    }
    mbar_init(&B.done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // atom 3's chunks 1..7 (taps 50..63) are never gathered: zero them once
  for (int i = threadIdx.x; i < 2 * p.V * 7; i += blockDim.x) {
    const int sl = i / (p.V * 7), r = (i / 7) % p.V, cc = 1 + i % 7;
    *reinterpret_cast<uint4*>(slots + (size_t)sl * p.slot_bytes + (size_t)3 * p.V * 128 + (size_t)r * 128 +
                              ((cc ^ (r & 7)) << 4)) = make_uint4(0u, 0u, 0u, 0u);
  }
  if (warp == 1) tmem_alloc(&B.tmem_base, 128);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      int sl = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        mbar_wait(&B.empty[sl], ph ^ 1);
        mbar_expect_tx(&B.full[sl], (uint32_t)p.V * 128);
        tma_load_2d(&map_dc, &B.full[sl], slots + (size_t)sl * p.slot_bytes + p.a_bytes, 0, t * p.V);
        if (++sl == 2) {
          sl = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_mn(64);
    int sl = 0;
    uint32_t ph = 0;
    bool first = true;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      mbar_wait(&B.full[sl], ph);
      mbar_wait(&B.ready[sl], ph);
      tc_fence_after();
      const uint32_t abase = smem_u32(slots + (size_t)sl * p.slot_bytes), dbase = abase + p.a_bytes;
      for (int kc = 0; kc < p.V / 16; ++kc) {
        const uint64_t bdesc = mn_desc<64>(dbase + (uint32_t)(kc * 16 * 128), 128);
#pragma unroll
        for (int mb = 0; mb < 2; ++mb)
          umma_bf16_elect(tmem + mb * 64,
                          mn_desc<64>(abase + (uint32_t)(mb * 2 * p.V * 128 + kc * 16 * 128), (uint32_t)p.V * 128),
                          bdesc, idesc, first ? 0u : 1u);
        first = false;
      }
      umma_commit_elect(&B.empty[sl]);
      if (++sl == 2) {
        sl = 0;
        ph ^= 1;
      }
    }
    umma_commit_elect(&B.done);
  } else if (warp >= wXf0) {
    // gather: task = (pixel, 16-byte chunk of two taps), chunks 0..24
    const int xt = threadIdx.x - wXf0 * 32;
    int sl = 0;
    uint32_t ph = 0;
    const int plane = p.Ho * p.Wo;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      mbar_wait_sleep(&B.empty[sl], ph ^ 1, 64);  // the MMAs no longer read this slot
      uint8_t* ab = slots + (size_t)sl * p.slot_bytes;
      const int64_t pix0 = (int64_t)t * p.V;
      // eight tasks per thread in flight: all sixteen 8-byte loads issued
      // before any store; pixel coordinates stepped from the tile start
      // (no 64-bit division per task)
      const int n0 = (int)(pix0 / plane), rem0 = (int)(pix0 - (int64_t)n0 * plane);
      constexpr int kB = 8;
      for (int t0 = xt; t0 < p.V * 25; t0 += kB * sGather) {
        uint2 v[kB][2];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int task = t0 + b * sGather;
          v[b][0] = v[b][1] = make_uint2(0u, 0u);
          const int r = task / 25, c = task - r * 25;
          if (task < p.V * 25 && pix0 + r < p.M) {
            int n = n0, rem = rem0 + r;
            while (rem >= plane) {  // (only when images are smaller than a tile)
              rem -= plane;
              ++n;
            }
            const int oh = rem / p.Wo, ow = rem - oh * p.Wo;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              // tap -> (kh, kw) by arithmetic: a constant-memory table read
              // with 32 different indices per warp serialised the memory pipe
              const int tap = 2 * c + h, kh = tap / 7, kw = tap - 7 * kh;
              const int ih = 2 * oh - 3 + kh, iw = 2 * ow - 3 + kw;
              if (tap < 49 && ih >= 0 && ih < p.H && iw >= 0 && iw < p.W)
                v[b][h] = __ldg(p.x4 + ((int64_t)n * p.H + ih) * p.W + iw);
            }
          }
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int task = t0 + b * sGather;
          if (task < p.V * 25) {
            const int r = task / 25, c = task - r * 25;
            const int a = c >> 3, cc = c & 7;
            *reinterpret_cast<uint4*>(ab + ((size_t)a * p.V + r) * 128 + ((cc ^ (r & 7)) << 4)) =
                make_uint4(v[b][0].x, v[b][0].y, v[b][1].x, v[b][1].y);
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&B.ready[sl]);
      if (++sl == 2) {
        sl = 0;
        ph ^= 1;
      }
    }
  } else {
    const int q = warp & 3;
    mbar_wait_sleep(&B.done, 0, 4000);
    tc_fence_after();
    float* out = p.part + (size_t)blockIdx.x * 2 * 128 * 64;
    for (int mb = 0; mb < 2; ++mb)
      for (int c = 0; c < 64; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + mb * 64 + c, v);
        float* dst = out + ((size_t)mb * 128 + q * 32 + lane) * 64 + c;
#pragma unroll
        for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 128);
}

// dW[co][kh][kw][c] (c < 3) = sum over CTAs of D[(tap, c)][co], tap = kh * 7 + kw
__global__ void stem_wgrad_finalize(const float* __restrict__ part, int ctas, float* __restrict__ dw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over co, kh, kw, c
  if (i >= 64 * 49 * 3) return;
  const int c = i % 3, tap = (i / 3) % 49, co = i / (3 * 49);
  const int m = tap * 4 + c;
  double acc = 0.0;
  for (int k = 0; k < ctas; ++k) acc += (double)part[(((size_t)k * 2 + m / 128) * 128 + m % 128) * 64 + co];
  dw[i] = (float)acc;
}
}  // namespace

bool wgrad3x3_halo_supported(int h, int w, int C) {
  WgPlan q;
  return wg_plan(h, w, C, &q);
}

size_t wgrad3x3_halo_workspace(int C) {
  const int apm = (C == 16 ? 64 : 128) / C, nm = (3 + apm - 1) / apm;
  return (size_t)num_sms() * 3 * nm * 128 * C * sizeof(float);
}

cudaError_t wgrad3x3_halo(const void* x, const void* dy, float* dw, int n, int h, int w, int C, const float* pmean,
                          const float* pinvstd, const void* pg, const void* pb, void* ws, size_t ws_bytes,
                          cudaStream_t s) {
  WgPlan q;
  if (n < 1 || !wg_plan(h, w, C, &q)) return cudaErrorInvalidValue;
  if (ws_bytes < wgrad3x3_halo_workspace(C)) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(ws)) & 15)
    return cudaErrorMisalignedAddress;
  WgParams p{};
  p.n = n;
  p.H = h;
  p.W = w;
  p.C = C;
  p.Ws = q.Ws;
  p.nseg = q.nseg;
  p.Wp = q.Wp;
  p.R = q.R;
  p.Rdy = q.Rdy;
  p.V = q.V;
  p.tiles_img = (h * q.Wp + q.V - 1) / q.V;
  p.tiles = n * q.nseg * p.tiles_img;
  p.win_bytes = (uint32_t)q.win;
  p.dy_bytes = (uint32_t)q.dy;
  p.slot_bytes = (uint32_t)(q.win + q.dy);
  p.part = static_cast<float*>(ws);
  p.pmean = pmean;
  p.pinvstd = pinvstd;
  p.pg = static_cast<const __nv_bfloat16*>(pg);
  p.pb = static_cast<const __nv_bfloat16*>(pb);
  const CUtensorMapSwizzle sw =
      C == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : (C == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  EncodeFn enc = encode_fn();
  if (!enc) return cudaErrorInvalidValue;
  CUtensorMap mx, mdy;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)w * C * 2, (cuuint64_t)h * w * C * 2};
  cuuint32_t es[4] = {1, 1, 1, 1};
  cuuint32_t bx[4] = {(cuuint32_t)C, (cuuint32_t)q.Wp, (cuuint32_t)q.R, 1};
  cuuint32_t bd[4] = {(cuuint32_t)C, (cuuint32_t)q.Wp, (cuuint32_t)q.Rdy, 1};
  if (enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, bx, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      enc(&mdy, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(dy), dims, strides, bd, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  int grid = num_sms();
  if (grid > p.tiles) grid = p.tiles;
  const size_t smem = 2 * (size_t)p.slot_bytes + 2 * C * 4 + sizeof(WgBars) + 1024;
  const bool pro = pmean != nullptr;
  cudaError_t e = cudaErrorInvalidValue;
  if (C == 16) e = pro ? launch_wg<16, true>(mx, mdy, p, grid, smem, s) : launch_wg<16, false>(mx, mdy, p, grid, smem, s);
  else if (C == 32) e = pro ? launch_wg<32, true>(mx, mdy, p, grid, smem, s) : launch_wg<32, false>(mx, mdy, p, grid, smem, s);
  else e = pro ? launch_wg<64, true>(mx, mdy, p, grid, smem, s) : launch_wg<64, false>(mx, mdy, p, grid, smem, s);
  if (e != cudaSuccess) return e;
  const int total = C * 9 * C, thr = 256;
  static const int lane_mode = std::getenv("KRT_M64_LANES") ? std::atoi(std::getenv("KRT_M64_LANES")) : 0;
  if (C == 16) wgrad3x3_halo_finalize<16><<<(total + thr - 1) / thr, thr, 0, s>>>(p.part, grid, dw, lane_mode);
  else if (C == 32) wgrad3x3_halo_finalize<32><<<(total + thr - 1) / thr, thr, 0, s>>>(p.part, grid, dw, lane_mode);
  else wgrad3x3_halo_finalize<64><<<(total + thr - 1) / thr, thr, 0, s>>>(p.part, grid, dw, lane_mode);
  return cudaGetLastError();
}

bool wgrad1x1_narrow_supported(int ci, int co) { return wg_enabled() && wg1_shape(ci, co); }

size_t wgrad1x1_narrow_workspace(int ci, int co) {
  const int mch = ci > co ? ci : co, nch = ci > co ? co : ci;
  const int nmb = mch / 128 > 0 ? mch / 128 : 1;
  return (size_t)num_sms() * nmb * 128 * nch * sizeof(float);
}

cudaError_t wgrad1x1_narrow(const void* x, const void* dy, float* dw, int64_t M, int ci, int co, const float* pmean,
                            const float* pinvstd, const void* pg, const void* pb, void* ws, size_t ws_bytes,
                            cudaStream_t s) {
  if (M < 1 || !wgrad1x1_narrow_supported(ci, co) || ws_bytes < wgrad1x1_narrow_workspace(ci, co))
    return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(ws)) & 15)
    return cudaErrorMisalignedAddress;
  const int mch = ci > co ? ci : co, nch = ci > co ? co : ci;
  const int nmb = mch / 128 > 0 ? mch / 128 : 1;
  Wg1Params p{};
  p.M = M;
  p.ci = ci;
  p.co = co;
  p.xm = ci >= co ? 1 : 0;
  // pixels per tile: two slots of (ci + co) channels in shared memory, TMA boxes <= 256 rows
  int V = (int)((96 * 1024) / ((size_t)(ci + co) * 2)) / 16 * 16;
  if (V > 256) V = 256;
  if (V < 16) return cudaErrorInvalidValue;
  p.V = V;
  p.tiles = (int)((M + V - 1) / V);
  const int cix = ci < 64 ? ci : 64, dyc = co < 64 ? co : 64;
  p.x_bytes = (uint32_t)r1k((size_t)((ci + 63) / 64) * V * cix * 2);
  p.dy_bytes = (uint32_t)r1k((size_t)((co + 63) / 64) * V * dyc * 2);
  p.slot_bytes = p.x_bytes + p.dy_bytes;
  p.part = static_cast<float*>(ws);
  p.pmean = pmean;
  p.pinvstd = pinvstd;
  p.pg = static_cast<const __nv_bfloat16*>(pg);
  p.pb = static_cast<const __nv_bfloat16*>(pb);
  auto swz = [](int c) {
    return c == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : (c == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  };
  CUtensorMap mx, mdy;
  if (!make_map(&mx, x, M, ci, V, cix, swz(cix)) || !make_map(&mdy, dy, M, co, V, dyc, swz(dyc)))
    return cudaErrorInvalidValue;
  int grid = num_sms();
  if (grid > p.tiles) grid = p.tiles;
  const size_t smem = 2 * (size_t)p.slot_bytes + 2 * (size_t)ci * 4 + sizeof(WgBars) + 1024;
  const bool pro = pmean != nullptr;
  cudaError_t e = cudaErrorInvalidValue;
#define KRT_WG1(MC, NC)                                                                                  \
  if (mch == MC && nch == NC)                                                                            \
    e = pro ? launch_wg1<MC, NC, true>(mx, mdy, p, grid, smem, s) : launch_wg1<MC, NC, false>(mx, mdy, p, grid, smem, s);
  KRT_WG1(64, 16)
  KRT_WG1(128, 32)
  KRT_WG1(256, 64)
  KRT_WG1(64, 64)
  KRT_WG1(128, 16)
  KRT_WG1(128, 64)
  KRT_WG1(256, 16)
  KRT_WG1(256, 32)
  KRT_WG1(64, 32)
#undef KRT_WG1
  if (e != cudaSuccess) return e;
  const int total = ci * co, thr = 256;
  wgrad1x1_narrow_finalize<<<(total + thr - 1) / thr, thr, 0, s>>>(p.part, grid, ci, co, p.xm, nmb, nch, dw);
  return cudaGetLastError();
}

size_t stem_wgrad_workspace() { return (size_t)num_sms() * 2 * 128 * 64 * sizeof(float); }

cudaError_t stem_wgrad(const void* x4, const void* dc, float* dw, int n, int h, int w, void* ws, size_t ws_bytes,
                       cudaStream_t s) {
  const int ho = (h + 2 * 3 - 7) / 2 + 1, wo = (w + 2 * 3 - 7) / 2 + 1;
  if (n < 1 || ho < 1 || wo < 1 || ws_bytes < stem_wgrad_workspace()) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(x4) | reinterpret_cast<uintptr_t>(dc) | reinterpret_cast<uintptr_t>(ws)) & 15)
    return cudaErrorMisalignedAddress;
  StemWgParams p{};
  p.n = n;
  p.H = h;
  p.W = w;
  p.Ho = ho;
  p.Wo = wo;
  p.M = (int64_t)n * ho * wo;
  p.V = 128;
  p.tiles = (int)((p.M + p.V - 1) / p.V);
  p.a_bytes = 4 * p.V * 128;
  p.slot_bytes = p.a_bytes + p.V * 128;
  p.x4 = static_cast<const uint2*>(x4);
  p.part = static_cast<float*>(ws);
  CUtensorMap mdc;
  if (!make_map(&mdc, dc, p.M, 64, p.V, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  int grid = num_sms();
  if (grid > p.tiles) grid = p.tiles;
  const size_t smem = 2 * (size_t)p.slot_bytes + sizeof(WgBars) + 1024;
  static size_t configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(stem_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  stem_wgrad_kernel<<<grid, sThreads, smem, s>>>(mdc, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  stem_wgrad_finalize<<<(64 * 49 * 3 + 255) / 256, 256, 0, s>>>(p.part, grid, dw);
  return cudaGetLastError();
}

}  // namespace krt
