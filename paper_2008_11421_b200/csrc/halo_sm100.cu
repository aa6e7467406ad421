// 3x3 / stride-1 / pad-1 convolution of NHWC activations on tcgen05 with
// halo windows (sm_100a): every input pixel of a tile's window is loaded (and,
// with the BN prologue, transformed) once and serves all nine filter taps.
//
//   C[pixel, N] = sum over taps (r, s) and channels c of
//                 f(x)[n, p - 1 + r, q - 1 + s, c] * w[N, r, s, c]
//   f = identity, or relu(x * scale + shift) per input channel (the BN + ReLU
//   of the previous layer; the zero padding stays zero)
//   epilogue: C rounded to bf16 and stored, optionally the per-channel
//   partial sums of C and C^2 (the next BN's statistics) as in gemm_sm100.cu.
//
// Virtual rows.  Each image is viewed with padded width Wp = W + 2: virtual
// output row v = p * Wp + q (q < W real, q = W, W + 1 junk).  The window of a
// tile is TMA-loaded as whole padded input rows (a 4-D box {64 channels, Wp
// columns from -1, R rows from p_lo - 1, 1 image}; out-of-image coordinates
// arrive as zeros), so in shared memory input pixel (p - 1 + r, q - 1 + s)
// sits at row (v - p_lo * Wp) + r * Wp + s: for every tap the A operand of a
// 128-row block is a contiguous run of 128-byte rows, described by one UMMA
// descriptor whose start moves by r * Wp + s rows.  The cost: junk columns (2 / Wp of the
// MMA work) and the windows' extra rows (R * Wp rows loaded per 256 outputs
// instead of 9 x 256 im2col rows).
//
// Structure (one CTA per SM, persistent; a tile = 256 virtual rows of one
// image in two 128-row sub-tiles sharing every B k-block):
//   warp 0        TMA producer: window per (tile, 64-channel block) into a
//                 2-slot window ring; B k-blocks (one tap x 64 channels x N)
//                 into a kStages ring
//   warp 1        TMEM allocator + MMA issuer (M = 128 per sub-tile, N = BN)
//   warps 2..17   epilogue: tcgen05.ld, bf16, staged in shared memory (stats
//                 read it column-wise), 16-byte global stores of real rows
//   warps 18..25  prologue: relu(bn(.)) on each window in place, once
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

constexpr int hEpiWarps = 16;
constexpr int hXfWarp0 = 2 + hEpiWarps;
constexpr int hXfThreads = 256;
constexpr int hThreads = 64 + hEpiWarps * 32 + hXfThreads;
constexpr int hAcc = 16;  // accumulator barriers: up to 8 sub-tiles x double buffering
constexpr int hMaxStages = 8;

struct HaloParams {
  int n, H, W, C, N;  // images, height, width, input channels, output channels
  int Ws, nseg;       // column segments of Ws output columns (the last may be partly junk)
  int Wp, R;          // padded segment width Ws + 2, window rows
  int halves;         // 128-row sub-tiles per (image, segment)
  int sub;            // sub-tiles per tile (host copy of kSub)
  int tiles_img, tiles;
  int stages;
  int wslots;           // window ring depth (2 or 3)
  uint32_t win_bytes;   // one window (1024-aligned)
  uint32_t slot_bytes;  // one window slot (pair: + 16 KB, see below)
  uint32_t bstage;      // one B ring stage (1024-aligned)
  __nv_bfloat16* out;
  float* part;
  const float* pmean;
  const float* pinvstd;
  const __nv_bfloat16* pg;
  const __nv_bfloat16* pb;
};

struct HaloBars {
  uint64_t full[hMaxStages], empty[hMaxStages];
  uint64_t wfull[3], wready[3], wempty[3];
  uint64_t tfull[hAcc], tempty[hAcc];
  uint32_t tmem_base;
};

// UMMA descriptor of a K-major SW128 operand starting at any 128-byte row of a
// 1024-aligned, TMA-swizzled window: the tensor core applies the 128B swizzle
// to absolute shared-memory address bits (the XOR of bits [7,10) into [4,7)),
// as the TMA wrote it, so the start simply moves by whole rows and the
// descriptor's base-offset field stays 0 (measured: with base offset
// (addr >> 7) & 7 every tap but the 1024-aligned one was wrong;
// scripts/debug_halo.py)
template <int BC>
__device__ __forceinline__ uint64_t halo_desc(uint32_t addr) {
  return kmajor_desc<BC>(addr);
}

// PAIR: CTA pair (cluster of 2, cta_group::2).  Both CTAs load the same window;
// the leader (rank 0) issues M = 256 MMAs whose A descriptor addresses rows
// off + shift of its window, which the peer - its copy placed 16 KB (128 rows)
// lower in the same slot - reads as rows off + 128 + shift: the second
// sub-tile.  Each CTA loads half of B's rows per tap and drains its own
// sub-tile.  Per CTA and MMA, shared-memory operand reads drop from
// A + B (8 KB at N = 128: the whole 128 B/clk) to A + B/2.
// BC: input channels per k-block (64, 32 or 16: window rows of 128, 64 or 32
// bytes, SWIZZLE_128B / 64B / 32B); BN: output channels (16 .. 128)
template <int BN, int BC, bool PRO, bool STATS, bool PAIR>
__global__ void __launch_bounds__(hThreads, 1) conv3x3_halo_kernel(const __grid_constant__ CUtensorMap map_x,
                                                                   const __grid_constant__ CUtensorMap map_b,
                                                                   HaloParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023) != 0) __trap();
  // 128-row sub-tiles per CTA per tile: eight at <= 32 output channels (the
  // window's three halo rows then serve ~4.5 output rows of a wide image
  // instead of ~1), two at 64 / 128 (tensor memory: 2 x kSub x BN columns)
  constexpr int kSub = PAIR ? 1 : (BN <= 32 ? 8 : 2);
  constexpr int kAccN = 2 * kSub;               // accumulators (x BN columns), double-buffered
  constexpr int kTileRows = PAIR ? 256 : 128 * kSub;  // virtual rows per tile (pair: both CTAs')
  constexpr int kBRows = PAIR ? BN / 2 : BN;    // B rows per CTA per tap
  constexpr uint32_t kPeerShift = PAIR ? 16384u : 0u;
  constexpr int kRB = BC * 2;                   // window / B row bytes
  constexpr int kCW = BN < 32 ? BN : 32;        // epilogue chunk: columns per warp
  static_assert(!PAIR || BC == 64, "pair: 128-byte rows (the peer shift is 128 rows)");
  uint8_t* win = smem;                                          // [wslots][slot_bytes]
  uint8_t* bring = smem + (size_t)p.wslots * p.slot_bytes;      // [stages][bstage]
  uint8_t* stg = bring + (size_t)p.stages * p.bstage;           // [16][32 rows x kCW bf16]
  float* sc = reinterpret_cast<float*>(stg + hEpiWarps * 32 * kCW * 2);
  float* sh = sc + p.C;
  HaloBars& B = *reinterpret_cast<HaloBars*>(sh + p.C);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nunits = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  // this CTA's copy of the window: the leader's 16 KB above the peer's
  const uint32_t wload = (PAIR && rank == 0) ? kPeerShift : 0u;
  const int cblocks = p.C / BC;
  constexpr int kEpiParts = BN / kCW;       // column parts (1, 2 or 4)
  constexpr int kEpiGroups = 4 / kEpiParts;  // sub-tile groups
  constexpr uint32_t kReadyCount = PAIR ? (PRO ? 2 * hXfThreads / 32 : 2) : hXfThreads;
  constexpr uint32_t kTemptyCount = PAIR ? 2 * 4 * kEpiParts : 128 * kEpiParts;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&B.full[s], 1);
      mbar_init(&B.empty[s], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&B.wfull[i], 1);
      mbar_init(&B.wready[i], kReadyCount);
      mbar_init(&B.wempty[i], 1);
    }
    for (int i = 0; i < hAcc; ++i) {
      mbar_init(&B.tfull[i], 1);
      mbar_init(&B.tempty[i], kTemptyCount);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair(&B.tmem_base, kAccN * BN);
    else tmem_alloc(&B.tmem_base, kAccN * BN);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = B.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0, ws = 0;
      uint32_t phase = 0, wphase = 0;
      for (int t = unit; t < p.tiles; t += nunits) {
        const int img = t / p.tiles_img, v0 = (t - img * p.tiles_img) * kTileRows;
        const int p_lo = v0 / p.Wp;
        const int n = img / p.nseg, seg = img - n * p.nseg;
        for (int cb = 0; cb < cblocks; ++cb) {
          mbar_wait(&B.wempty[ws], wphase ^ 1);
          mbar_expect_tx(&B.wfull[ws], (uint32_t)p.R * p.Wp * kRB);
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(win + ws * p.slot_bytes + wload)),
              "l"(reinterpret_cast<uint64_t>(&map_x)), "r"(smem_u32(&B.wfull[ws])), "r"(cb * BC),
              "r"(seg * p.Ws - 1), "r"(p_lo - 1), "r"(n)
              : "memory");
          if (++ws == p.wslots) {
            ws = 0;
            wphase ^= 1;
          }
          for (int tap = 0; tap < 9; ++tap) {
            mbar_wait(&B.empty[stage], phase ^ 1);
            uint8_t* dst = bring + (size_t)stage * p.bstage;
            if (PAIR) {  // both halves complete on the leader's barrier
              if (rank == 0) mbar_expect_tx(&B.full[stage], 2 * kBRows * kRB);
              tma_load_2d_pair(&map_b, mapa_rank(&B.full[stage], 0), dst, tap * p.C + cb * BC, (int)rank * kBRows);
            } else {
              mbar_expect_tx(&B.full[stage], BN * kRB);
              tma_load_2d(&map_b, &B.full[stage], dst, tap * p.C + cb * BC, 0);
            }
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      if (PAIR) {  // every multicast commit has arrived before this CTA may exit
        for (int i = 0; i < p.stages; ++i) {
          mbar_wait(&B.empty[stage], phase ^ 1);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        for (int i = 0; i < p.wslots; ++i) {
          mbar_wait(&B.wempty[ws], wphase ^ 1);
          if (++ws == p.wslots) {
            ws = 0;
            wphase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (!PAIR || rank == 0) {
      constexpr uint32_t idesc = PAIR ? instr_desc_pair(BN) : instr_desc(BN);
      const uint64_t bdesc0 = kmajor_desc<BC>(smem_u32(bring));
      int stage = 0, ws = 0, it = 0;
      uint32_t phase = 0, wphase = 0;
      for (int t = unit; t < p.tiles; t += nunits, ++it) {
        const int img = t / p.tiles_img, ti = t - img * p.tiles_img, v0 = ti * kTileRows;
        const int off = v0 - (v0 / p.Wp) * p.Wp;  // first virtual row's column = its window row offset
        const int nsub = PAIR ? 1 : (p.halves - kSub * ti >= kSub ? kSub : p.halves - kSub * ti);
        const int a0 = (kSub * it) % kAccN;
        const uint32_t aph = (uint32_t)((kSub * it) / kAccN) & 1u;
        for (int u = 0; u < kSub; ++u) mbar_wait(&B.tempty[a0 + u], aph ^ 1);
        tc_fence_after();
        for (int cb = 0; cb < cblocks; ++cb) {
          if (PRO || PAIR) mbar_wait(&B.wready[ws], wphase);  // (both CTAs') window landed / transformed
          else mbar_wait(&B.wfull[ws], wphase);
          tc_fence_after();
          // descriptors: window row 0 of this slot (+ the peer shift), B stage 0
          const uint64_t wdesc = halo_desc<BC>(smem_u32(win + ws * p.slot_bytes) + kPeerShift);
          for (int tap = 0; tap < 9; ++tap) {
            mbar_wait(&B.full[stage], phase);
            tc_fence_after();
            const uint64_t bdesc = bdesc0 + (uint64_t)(stage * (p.bstage >> 4));
            const int shift = (tap / 3) * p.Wp + (tap % 3);
            for (int u = 0; u < nsub; ++u) {
              const uint64_t adesc = wdesc + (uint64_t)((off + u * 128 + shift) * (kRB >> 4));  // (row bytes) >> 4
#pragma unroll
              for (int k = 0; k < BC / kUmmaK; ++k) {
                if (PAIR)
                  umma_bf16_pair_elect(tmem + (a0 + u) * BN, adesc + 2 * k, bdesc + 2 * k, idesc, (cb | tap | k) != 0);
                else
                  umma_bf16_elect(tmem + (a0 + u) * BN, adesc + 2 * k, bdesc + 2 * k, idesc, (cb | tap | k) != 0);
              }
            }
            if (PAIR) {
              umma_commit_pair_elect(&B.empty[stage]);
              if (tap == 8) umma_commit_pair_elect(&B.wempty[ws]);
            } else {
              umma_commit_elect(&B.empty[stage]);
              if (tap == 8) umma_commit_elect(&B.wempty[ws]);
            }
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (++ws == p.wslots) {
            ws = 0;
            wphase ^= 1;
          }
        }
        if (PAIR) {
          umma_commit_pair_elect(&B.tfull[a0]);
        } else {
          for (int u = 0; u < kSub; ++u) umma_commit_elect(&B.tfull[a0 + u]);
        }
      }
    }
  } else if (warp >= hXfWarp0) {
    // ------------------------------------------------------------ prologue transform
    if (PRO) {
      const int xt = threadIdx.x - hXfWarp0 * 32;  // 0..255
      for (int c = xt; c < p.C; c += hXfThreads) {
        const float s = p.pinvstd[c] * __bfloat162float(p.pg[c]);
        sc[c] = s;
        sh[c] = __bfloat162float(p.pb[c]) - p.pmean[c] * s;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(hXfThreads) : "memory");
      constexpr int kCPR = BC / 8;             // 16-byte chunks per window row
      constexpr int kRS = hXfThreads / kCPR;   // rows per pass of the 256 threads
      const int ch = xt % kCPR;  // this thread's 16-byte chunk (8 channels) of every row it visits
      const int jd = kRS / p.Wp, jm = kRS - jd * p.Wp;  // rows advance by kRS
      int ws = 0;
      uint32_t wphase = 0;
      for (int t = unit; t < p.tiles; t += nunits) {
        const int img = t / p.tiles_img, ti = t - img * p.tiles_img, v0 = ti * kTileRows;
        const int p_lo = v0 / p.Wp;
        const int seg = img % p.nseg, q0 = seg * p.Ws - 1;  // input column of window column 0
        // only the window rows this CTA's MMAs read: its sub-tiles' 128 rows
        // each, plus two padded rows and two columns of taps
        const int off = v0 - p_lo * p.Wp;
        const int nsub = PAIR ? 1 : (p.halves - kSub * ti >= kSub ? kSub : p.halves - kSub * ti);
        const int jlo = off + (PAIR ? (int)rank * 128 : 0), jhi = jlo + 128 * nsub + 2 * p.Wp + 2;
        const int j0 = jlo + xt / kCPR;
        for (int cb = 0; cb < cblocks; ++cb) {
          // the affine of this thread's 8 channels, packed for fma.rn.f32x2
          unsigned long long sc2[4], sh2[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = cb * BC + ch * 8 + 2 * e;
            sc2[e] = ((unsigned long long)__float_as_uint(sc[c + 1]) << 32) | __float_as_uint(sc[c]);
            sh2[e] = ((unsigned long long)__float_as_uint(sh[c + 1]) << 32) | __float_as_uint(sh[c]);
          }
          mbar_wait(&B.wfull[ws], wphase);
          uint8_t* wb = win + ws * p.slot_bytes + wload;
          int wr = j0 / p.Wp, wc = j0 - (j0 / p.Wp) * p.Wp;  // window row / padded column of row j
          for (int j = j0; j < jhi; j += kRS) {
            const int ip = p_lo - 1 + wr, iq = q0 + wc;  // input pixel
            if (ip >= 0 && ip < p.H && iq >= 0 && iq < p.W) {
              uint4* cp = reinterpret_cast<uint4*>(wb + (size_t)j * kRB + (swz_chunk<BC>(ch, j) << 4));
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
            // (out-of-image window rows / padding columns keep the TMA's zeros)
            wr += jd;
            wc += jm;
            if (wc >= p.Wp) {
              wc -= p.Wp;
              ++wr;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          if (PAIR) {  // one arrival per warp on the leader's barrier
            __syncwarp();
            if (lane == 0) {
              if (rank == 0) mbar_arrive(&B.wready[ws]);
              else mbar_arrive_rank(&B.wready[ws], 0);
            }
          } else {
            mbar_arrive(&B.wready[ws]);
          }
          if (++ws == p.wslots) {
            ws = 0;
            wphase ^= 1;
          }
        }
      }
    } else if (PAIR && warp == hXfWarp0 && lane == 0) {
      // no prologue: forward this CTA's window landing to the leader's barrier
      int ws = 0;
      uint32_t wphase = 0;
      for (int t = unit; t < p.tiles; t += nunits)
        for (int cb = 0; cb < cblocks; ++cb) {
          mbar_wait(&B.wfull[ws], wphase);
          if (rank == 0) mbar_arrive(&B.wready[ws]);
          else mbar_arrive_rank(&B.wready[ws], 0);
          if (++ws == p.wslots) {
            ws = 0;
            wphase ^= 1;
          }
        }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter
    const int ew = warp - 2;
    const int part = (ew >> 2) % kEpiParts;  // column part
    const int grp = (ew >> 2) / kEpiParts;   // sub-tile group
    constexpr int kChunks = BN / kCW / kEpiParts;  // 1
    static_assert(kChunks == 1, "one chunk per warp");
    constexpr int kLPR = kCW * 2 / 16;  // lanes per row in the coalesced stores (4 or 2)
    const int col = part * kCW;
    uint8_t* sbuf = stg + ew * (32 * kCW * 2);
    float acc_s = 0.f, acc_q = 0.f;
    int it = 0;
    for (int t = unit; t < p.tiles; t += nunits, ++it) {
      const int img = t / p.tiles_img, ti = t - img * p.tiles_img, v0 = ti * kTileRows;
      const int nsub = PAIR ? 1 : (p.halves - kSub * ti >= kSub ? kSub : p.halves - kSub * ti);
      const int n = img / p.nseg, c0 = (img - n * p.nseg) * p.Ws;  // image, first column of the segment
      for (int ul = 0; ul < kSub; ++ul) {
        const int s = kSub * it + ul;  // sub-tile sequence number of this CTA
        if (s % kEpiGroups != grp) continue;
        const int u = PAIR ? (int)rank : ul;
        const int acc = s % kAccN;
        mbar_wait(&B.tfull[acc], (uint32_t)(s / kAccN) & 1u);
        tc_fence_after();
        if (ul < nsub) {
          // this lane's row: virtual row -> pixel, or junk
          const int v = v0 + u * 128 + q * 32 + lane;
          const int pr = v / p.Wp, pc = v - pr * p.Wp;
          const bool valid = pr < p.H && pc < p.Ws && c0 + pc < p.W;
          const int64_t grow = ((int64_t)n * p.H + pr) * p.W + c0 + pc;
          float x[kCW];
          if constexpr (kCW == 32) tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + col, x);
          else tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + col, x);
          // staged in shared memory: coalesced stores (four lanes per row, 64
          // contiguous bytes each) and the statistics' column sums read it
          uint4* st = reinterpret_cast<uint4*>(sbuf + lane * kCW * 2);
#pragma unroll
          for (int j = 0; j < kCW / 8; ++j) {
            uint4 w;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              h[e] = valid ? __floats2bfloat162_rn(x[8 * j + 2 * e], x[8 * j + 2 * e + 1])
                           : __floats2bfloat162_rn(0.f, 0.f);
            st[swz_chunk<kCW>(j, lane)] = w;
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < kLPR; ++i) {
            const int r = i * (32 / kLPR) + lane / kLPR, c = lane % kLPR;
            const long long gr = __shfl_sync(0xffffffffu, (long long)(valid ? grow : -1), r);
            const uint4 w = *reinterpret_cast<const uint4*>(sbuf + r * kCW * 2 + (swz_chunk<kCW>(c, r) << 4));
            if (gr >= 0) *reinterpret_cast<uint4*>(p.out + gr * p.N + col + c * 8) = w;
          }
          if (STATS) {
            // column `lane` of the staged chunk, rows in order (junk rows staged as zero)
            // (16-wide chunks: lanes 16..31 take rows 16..31 of the same
            // columns, folded in with one shuffle)
            const __nv_bfloat16* sv = reinterpret_cast<const __nv_bfloat16*>(sbuf);
            const int cl = lane % kCW, cc = cl >> 3, ce = cl & 7;
            constexpr int kRows = kCW == 32 ? 32 : 16;
            const int rb = lane / kCW * kRows;
            float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < kRows; ++i) {
              const int r = rb + i;
              const float xv = __bfloat162float(sv[r * kCW + 8 * swz_chunk<kCW>(cc, r) + ce]);
              s1[i & 3] += xv;
              s2[i & 3] = __fmaf_rn(xv, xv, s2[i & 3]);
            }
            float t1 = (s1[0] + s1[1]) + (s1[2] + s1[3]), t2 = (s2[0] + s2[1]) + (s2[2] + s2[3]);
            if constexpr (kCW == 16) {
              t1 += __shfl_down_sync(0xffffffffu, t1, 16);
              t2 += __shfl_down_sync(0xffffffffu, t2, 16);
            }
            acc_s += t1;
            acc_q += t2;
          }
          __syncwarp();  // the staging buffer is rewritten by the next sub-tile
        }
        tc_fence_before();
        if (PAIR) {  // one arrival per warp, on the leader's barrier
          __syncwarp();
          if (lane == 0) {
            if (rank == 0) mbar_arrive(&B.tempty[acc]);
            else mbar_arrive_rank(&B.tempty[acc], 0);
          }
        } else {
          mbar_arrive(&B.tempty[acc]);
        }
      }
    }
    if (STATS) {
      float* prow = p.part + (((size_t)blockIdx.x * 4 + q) * kEpiGroups + grp) * 2 * p.N;
      if (lane < kCW) {
        prow[col + lane] = acc_s;
        prow[p.N + col + lane] = acc_q;
      }
    }
  }
  tc_fence_before();
  if (PAIR) {
    cluster_sync();  // neither CTA leaves while the peer may still touch its barriers, smem or TMEM
    if (warp == 1) tmem_dealloc_pair(tmem, kAccN * BN);
  } else {
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, kAccN * BN);
  }
}

template <int BN, int BC, bool PRO, bool STATS, bool PAIR>
cudaError_t launch_halo(const CUtensorMap& mx, const CUtensorMap& mb, const HaloParams& p, int grid, size_t smem,
                        cudaStream_t s) {
  auto k = conv3x3_halo_kernel<BN, BC, PRO, STATS, PAIR>;
  static size_t configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  if (PAIR) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(hThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, mx, mb, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  k<<<grid, hThreads, smem, s>>>(mx, mb, p);
  return cudaGetLastError();
}

bool halo_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("KRT_CONV_HALO");
    return e == nullptr || std::strcmp(e, "0") != 0;
  }();
  return on;
}

// CTA pairs for the halo convolution (KRT_HALO_PAIR=0: single CTAs)
bool halo_pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("KRT_HALO_PAIR");
    return e == nullptr || std::strcmp(e, "0") != 0;
  }();
  return on;
}

// window rows for `rows` virtual rows starting at any column: the first
// row's offset (< Wp) + rows - 1 + two rows of taps + 2 columns
int halo_rows(int Wp, int rows) { return (Wp - 1 + rows - 1 + 2 * Wp + 2) / Wp + 1; }

// sub-tiles per tile, as the kernel's kSub (no pairs)
int halo_sub(int N) { return N <= 32 ? 8 : 2; }

size_t round1k(size_t b) { return (b + 1023) / 1024 * 1024; }

// How a shape runs: channel block, column segments, window / B-stage bytes
struct HaloPlan {
  int BC = 0, Ws = 0, nseg = 0, Wp = 0, R = 0;
  bool pair = false;
  size_t win = 0, slot = 0, bstage = 0, fixed = 0;
};

size_t halo_fixed(const HaloPlan& q, int cin, int N, int wslots) {
  const int cw = N < 32 ? N : 32;
  return wslots * q.slot + hEpiWarps * 32 * cw * 2 + 2 * (size_t)cin * 4 + sizeof(HaloBars) + 1024;
}

// input channels per k-block: 64 (cin % 64 == 0, 64 or 128 output channels) or
// the whole of a 16 / 32-channel input with as many output channels; image
// columns split into the fewest segments whose windows fit (TMA boxes are at
// most 256 pixels wide)
bool halo_plan(int h, int w, int cin, int N, bool pro, bool want_pair, HaloPlan* out) {
  if (!halo_enabled() || h < 1 || w < 1) return false;
  HaloPlan q;
  if (cin % 64 == 0 && (N == 64 || N == 128)) q.BC = 64;
  else if ((cin == 16 || cin == 32) && N == cin) q.BC = cin;
  else return false;
  if (pro && cin > 1024) return false;
  const int rb = q.BC * 2;
  for (int nseg = 1; nseg <= 64; ++nseg) {
    q.nseg = nseg;
    q.Ws = (w + nseg - 1) / nseg;
    q.Wp = q.Ws + 2;
    if (q.Wp > 256) continue;
    q.R = halo_rows(q.Wp, 128 * halo_sub(N));
    if (q.R > 256) return false;
    q.win = round1k((size_t)q.R * q.Wp * rb);
    q.pair = want_pair && q.BC == 64 && !pro;
    q.slot = q.win + (q.pair ? 16384 : 0);
    q.bstage = round1k((size_t)(q.pair ? N / 2 : N) * rb);
    if (halo_fixed(q, cin, N, 2) + 2 * q.bstage > 220 * 1024 && q.pair) {  // retry without the pair's shift
      q.pair = false;
      q.slot = q.win;
      q.bstage = round1k((size_t)N * rb);
    }
    if (halo_fixed(q, cin, N, 2) + 2 * q.bstage <= 220 * 1024) {
      *out = q;
      return true;
    }
  }
  return false;
}
}  // namespace

bool conv3x3_halo_supported(int h, int w, int cin, int N, bool pro) {
  HaloPlan q;
  return halo_plan(h, w, cin, N, pro, false, &q);
}

cudaError_t conv3x3_halo_fprop(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int N,
                               const float* pmean, const float* pinvstd, const void* pg, const void* pb, float* part,
                               int* part_rows, cudaStream_t s) {
  const bool pro = pmean != nullptr, st = part != nullptr;
  // CTA pairs without the prologue (measured, scripts/bench_gemm_pair.py b1024:
  // plain 0.354 -> 0.343 ms at 56x56x64, 0.241 -> 0.224 at 28x28x128); with it
  // both CTAs must transform their window halves before the pair's MMAs and
  // single CTAs are faster (0.42 vs 0.56, 0.32 vs 0.34 ms)
  HaloPlan q;
  if (n < 1 || !halo_plan(h, w, cin, N, pro, halo_pair_enabled(), &q)) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(wk) | reinterpret_cast<uintptr_t>(C)) & 15)
    return cudaErrorMisalignedAddress;
  HaloParams p{};
  p.n = n;
  p.H = h;
  p.W = w;
  p.C = cin;
  p.N = N;
  p.Ws = q.Ws;
  p.nseg = q.nseg;
  p.Wp = q.Wp;
  p.R = q.R;
  p.halves = (h * p.Wp + 127) / 128;
  p.sub = q.pair ? 2 : halo_sub(N);  // 128-row sub-tiles per tile (pair: one per CTA)
  p.tiles_img = (p.halves + p.sub - 1) / p.sub;
  p.tiles = n * q.nseg * p.tiles_img;
  p.win_bytes = (uint32_t)q.win;
  p.slot_bytes = (uint32_t)q.slot;
  p.bstage = (uint32_t)q.bstage;
  // a third window slot when it fits next to a 4-deep B ring: the next
  // window's load and prologue then have a whole tile of MMAs to hide behind
  p.wslots = halo_fixed(q, cin, N, 3) + 4 * q.bstage <= 220 * 1024 ? 3 : 2;
  const size_t fixed = halo_fixed(q, cin, N, p.wslots);
  int stages = (int)((220 * 1024 - fixed) / q.bstage);
  if (stages > hMaxStages) stages = hMaxStages;
  if (stages < 2) return cudaErrorInvalidValue;
  p.stages = stages;
  p.out = static_cast<__nv_bfloat16*>(C);
  p.part = part;
  p.pmean = pmean;
  p.pinvstd = pinvstd;
  p.pg = static_cast<const __nv_bfloat16*>(pg);
  p.pb = static_cast<const __nv_bfloat16*>(pb);
  const CUtensorMapSwizzle sw = q.BC == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                           : (q.BC == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  // x [n, h, w, cin] as a 4-D tensor {c, w, h, n}; boxes of whole padded segment rows
  EncodeFn enc = encode_fn();
  if (!enc) return cudaErrorInvalidValue;
  CUtensorMap mx, mb;
  {
    cuuint64_t dims[4] = {(cuuint64_t)cin, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)n};
    cuuint64_t strides[3] = {(cuuint64_t)cin * 2, (cuuint64_t)w * cin * 2, (cuuint64_t)h * w * cin * 2};
    cuuint32_t box[4] = {(cuuint32_t)q.BC, (cuuint32_t)p.Wp, (cuuint32_t)p.R, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (!make_map(&mb, wk, N, 9 * cin, q.pair ? N / 2 : N, q.BC, sw)) return cudaErrorInvalidValue;
  int units = q.pair ? num_sms() / 2 : num_sms();  // CTAs or CTA pairs, persistent
  if (units > p.tiles) units = p.tiles;
  const int grid = units * (q.pair ? 2 : 1);
  const int groups = 4 / (N < 32 ? 1 : N / 32);
  if (part_rows) *part_rows = grid * 4 * groups;
  const size_t smem = fixed + (size_t)stages * q.bstage;
#define KRT_HALO(BNV, BCV, PR)                                                             \
  if (N == BNV && q.BC == BCV && q.pair == PR) {                                           \
    if (pro && st) return launch_halo<BNV, BCV, true, true, PR>(mx, mb, p, grid, smem, s);  \
    if (pro) return launch_halo<BNV, BCV, true, false, PR>(mx, mb, p, grid, smem, s);       \
    if (st) return launch_halo<BNV, BCV, false, true, PR>(mx, mb, p, grid, smem, s);        \
    return launch_halo<BNV, BCV, false, false, PR>(mx, mb, p, grid, smem, s);               \
  }
  KRT_HALO(64, 64, false)
  KRT_HALO(128, 64, false)
  KRT_HALO(64, 64, true)
  KRT_HALO(128, 64, true)
  KRT_HALO(16, 16, false)
  KRT_HALO(32, 32, false)
#undef KRT_HALO
  return cudaErrorInvalidValue;
}

}  // namespace krt
