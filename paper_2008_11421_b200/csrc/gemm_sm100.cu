// 1x1 convolution of NHWC activations as a tcgen05 GEMM, fused with the
// batch-norm work around it (sm_100a):
//
//   C[M, N] = f(A)[M, K] . B[N, K]^T        (A = activations [rows, Cin],
//                                            B = weights [Cout, Cin], both K-major)
//   f(A)    = A, or relu(A*scale + shift) per K channel (the BN + ReLU of the
//             previous layer applied in shared memory: its output is never
//             written to HBM)
//   epilogue: C rounded to bf16 and stored, and per-channel partial sums of
//             C and C^2 (the next BN's batch statistics) reduced on chip, so
//             no separate statistics pass re-reads C.
//
// Structure (one CTA per SM, persistent, static tile schedule):
//   warp 0        TMA producer: A and B k-blocks (64 x bf16 = 128 B rows,
//                 SWIZZLE_128B) into a kStages-deep shared-memory ring
//   warp 1        TMEM allocator + MMA issuer: one elected thread issues
//                 tcgen05.mma (M=128, N=BN, K=16) into one of two TMEM
//                 accumulators, tcgen05.commit frees the smem stage / hands the
//                 accumulator to the epilogue
//   warps 2..17   epilogue, four warps per TMEM lane quarter (32 rows), each
//                 a quarter of the tile's columns: tcgen05.ld 32 columns at a time,
//                 bf16 round, staged through shared memory and written by TMA
//                 bulk stores; lane j then sums column j of the staged chunk
//   warps 18..25  prologue only: transform each A stage in place (half a tile
//                 row per thread) between the TMA landing and the MMA
// Statistics are deterministic: fixed tile schedule, fixed summation order,
// per-warp partial rows summed in double by bn_partials_finalize.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm_sm100.hpp"
#include "halo_sm100.hpp"
#include "sm100_common.cuh"

namespace krt {
namespace {
using namespace sm100;

constexpr int kBK = 64;        // k-block: 64 bf16 = one 128-byte swizzle row
constexpr int kEpiWarps = 16;  // four per TMEM lane quarter, each a quarter of the columns
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kXfWarp0 = 2 + kEpiWarps;        // prologue transform warps
constexpr int kXfThreads = 256;                 // two threads per tile row, four 16-byte chunks each
constexpr int kXWarp = kXfWarp0 + kXfThreads / 32;  // epilogue-operand (x / residual tile) producer
constexpr int kThreads = 64 + kEpiThreads + kXfThreads + 32;  // producer, MMA, epilogue, transform, x producer
constexpr int kEpiWarp0 = 2;
constexpr int kMaxProK = 1024;  // prologue channels held in shared memory

// ---------------------------------------------------------------------------
struct Params {
  int64_t M;
  int N, K, BN;
  int n_tiles, m_tiles;
  __nv_bfloat16* C;
  float* part;  // [gridDim.x / n_tiles * 4][2][N] or nullptr: one row per (m-group, lane quarter)
  // prologue (nullptr: none): a = relu(A*sc + sh), sc = invstd*g, sh = b - mean*sc
  const float* pmean;
  const float* pinvstd;
  const __nv_bfloat16* pg;
  const __nv_bfloat16* pb;
  // BN-backward epilogue (EPI 2): x of the BN whose output gradient C is, and
  // its statistics/affine; partials = sum gm, sum gm*xhat with gm = C*mask(x)
  const __nv_bfloat16* bx;
  const float* bmean;
  const float* binvstd;
  const __nv_bfloat16* bg;
  const __nv_bfloat16* bb;
  // residual (nullptr: none): C = acc + res, res [M, N] bf16 row-major,
  // added in fp32 before the single bf16 rounding (EPI 0/1)
  const __nv_bfloat16* res;
  // GATHER (implicit-GEMM convolution): A rows are gathered from the NHWC
  // input gx [gn, gh, gw, gc] by the transform warps: row = output pixel
  // (n, oh, ow), column k = (kh * gk + kw) * gc + c for k < gk*gk*gc, zero
  // beyond (K padded to a k-block multiple) and outside the image
  const __nv_bfloat16* gx;
  int gh, gw, gc, gho, gwo, gk, gs, gp;
};

// ASTAT (A-stationary, prologue only, K <= kMaxAstatK): the transformed A tile
// of an m-tile stays in shared memory while the CTA walks all n-tiles, so the
// relu(bn(.)) transform and the A loads happen once per m-tile instead of once
// per (m, n) tile; the ring then carries B k-blocks only.
constexpr int kMaxAstatK = 256;
// A-stationary k-block slots: a ring one larger than an m-tile's k-blocks, so
// the next m-tile's first k-block loads and transforms while this m-tile's
// last n-tile still runs (m-tile i, k-block kb -> slot (i * kblocks + kb) % 5)
constexpr int kAstatSlots = kMaxAstatK / kBK + 1;
constexpr int kMaxNT = 8;  // n-tiles per CTA in A-stationary mode (N <= 2048)

// EPI 3 / 4 residual tiles: [BN / kResW boxes][128 rows][kResW columns], each box
// TMA-loaded with the swizzle of its row width, kResBufs tiles in flight
template <int BN>
constexpr int kResW = BN < 64 ? BN : 64;
template <int BN>
constexpr int kResBufs = BN <= 64 ? 4 : 2;

// B-stationary (fixed n-tile per CTA, whole B tile <= 32 KB): the CTA's
// n-tile of B is loaded once and stays; the ring carries A only.  Re-fetching
// a small B tile for every 128-row tile starved narrow GEMMs (2x on K=16 N=64)
constexpr int kBStatBytes = 32 * 1024;
template <int BN, int BKT>
constexpr int kBSlots = kBStatBytes / (BN * BKT * 2) > 0 ? kBStatBytes / (BN * BKT * 2) : 1;

template <int BN, int STAGES, bool PRO, bool ASTAT, int EPI, int BKT, bool BSTAT = false, bool PAIR = false>
struct Smem {
  alignas(1024) uint8_t a[ASTAT ? kAstatSlots : STAGES][kBM * BKT * 2];
  // CTA pair: each CTA holds half of the n-tile's B rows
  alignas(1024) uint8_t b[BSTAT ? kBSlots<BN, BKT> : STAGES][(PAIR ? BN / 2 : BN) * BKT * 2];
  uint64_t full[STAGES], ready[STAGES], empty[STAGES];
  uint64_t bfull;
  uint64_t tfull[4], tempty[4];
  uint64_t a_full[kAstatSlots], a_ready[kAstatSlots], a_free[kAstatSlots];  // A-stationary, per slot
  uint32_t tmem_base;
  alignas(16) float sc[PRO ? kMaxProK : 4];
  alignas(16) float sh[PRO ? kMaxProK : 4];
  // per-warp C staging for the TMA store: 32 rows x 64 B, SWIZZLE_64B (16-byte
  // chunk c of row r at c ^ ((r >> 1) & 3)), so row-per-lane writes and
  // column-per-lane reads are both free of bank conflicts
  // (A-stationary: one buffer per warp, the 32 KB go to a deeper B ring)
  alignas(1024) uint8_t cstage[kEpiWarps][ASTAT ? 1 : 2][32 * 64];
  // EPI 2: the BN input x of the current tile pair, TMA-loaded by the producer
  // ahead of the epilogue (row-major [128][BN]); one buffer per accumulator.
  // EPI 3: the residual tiles (swizzled boxes), kResBufs deep
  alignas(1024) uint8_t xt[EPI == 2 ? 2 : (EPI >= 3 ? kResBufs<BN> : 1)][EPI >= 2 ? kBM * BN * 2 : 16];
  uint64_t x_full[4], x_empty[4];
};

// EPI: 0 store only, 1 + batch statistics of C, 2 + BN-backward reduce of C,
// 3 C = acc + residual (p.res through map_x), 4 = 3 + the batch statistics of
// that C (the next pre-activation unit's BN0 statistics)
// PAIR: CTA pair (cluster of 2, tcgen05 cta_group::2).  A pair tile is 256
// rows x BN columns: each CTA loads its own 128 A rows and half of the B rows,
// the leader (rank 0) issues M = 256 MMAs that write 128 accumulator rows into
// each CTA's TMEM, and each CTA drains its own rows.  Per CTA, B bytes per
// k-block halve, so the ring is deeper and the operand traffic per MMA flop
// drops by a quarter (BN = 128) to a third (BN = 256).
template <int BN, int STAGES, bool PRO, int EPI, bool ASTAT, int BKT, bool GATHER = false, bool BSTAT = false,
          bool IM2A = false, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1) conv1x1_kernel(const __grid_constant__ CUtensorMap map_a,
                                                              const __grid_constant__ CUtensorMap map_b,
                                                              const __grid_constant__ CUtensorMap map_c,
                                                              const __grid_constant__ CUtensorMap map_x, Params p) {
  // the dynamic shared-memory window starts 1024-aligned (no static shared
  // memory in this kernel); using it directly keeps every access in the shared
  // address space (an integer round-up made them generic LD.E/ST.E)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  static_assert(!BSTAT || !ASTAT, "B-stationary needs a fixed n-tile");
  auto& S = *reinterpret_cast<Smem<BN, STAGES, PRO || GATHER, ASTAT, EPI, BKT, BSTAT, PAIR>*>(smem_raw);
  static_assert(!PAIR || (!ASTAT && !GATHER && !BSTAT && BKT == kBK && EPI < 3), "pair: streamed 64-wide k-blocks");
  static_assert(!GATHER || (!PRO && !ASTAT), "gathered A has no prologue");
  static_assert(!IM2A || (!GATHER && !ASTAT && BKT == kBK), "im2col A: 64-channel k-blocks, streamed");
  static_assert(!ASTAT || (BKT == kBK && BN >= 64), "A-stationary uses 64-wide k-blocks and n-tiles");
  if ((smem_u32(smem_raw) & 1023) != 0) __trap();  // SWIZZLE_128B operands need 1024-byte alignment
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = p.K / BKT;
  const int cblocks = IM2A ? p.gc / BKT : 1;  // im2col: channel blocks per filter tap
  // epilogue column parts: one warp per (part, TMEM lane quarter); the 16
  // epilogue warps form kEpiGroups groups that drain alternate tiles, each
  // from its own accumulator (kAcc >= 2 accumulators in TMEM)
  constexpr int kEpiParts = BN >= 128 ? 4 : (BN >= 64 ? BN / 32 : 1);
  constexpr int kEpiGroups = 4 / kEpiParts;
  constexpr int kAcc = kEpiGroups > 2 ? kEpiGroups : 2;
  static_assert(EPI != 2 || kAcc == 2, "EPI 2 x tiles are double-buffered with the accumulators");
  // this CTA's tiles: m-tiles strided; either a fixed n-tile (grid is a
  // multiple of n_tiles) or, A-stationary, every n-tile of each m-tile
  // (pair: m-tiles are 256-row pair tiles, scheduled per cluster)
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int cta = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x, ncta = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int nts = ASTAT ? p.n_tiles : 1;
  const int n_fixed = ASTAT ? 0 : cta % p.n_tiles;
  const int m_first = ASTAT ? cta : cta / p.n_tiles;
  const int m_step = ASTAT ? ncta : ncta / p.n_tiles;
  // first A / C row of this CTA in m-tile mt
  auto rowbase = [&](int mt) -> int64_t { return PAIR ? (int64_t)mt * (2 * kBM) + rank * kBM : (int64_t)mt * kBM; };
  constexpr int kBRows = PAIR ? BN / 2 : BN;  // B rows per CTA
  // accumulator-drained barrier: per thread (single CTA) or per warp from both CTAs (pair)
  constexpr uint32_t kTemptyCount = PAIR ? 2 * 4 * kEpiParts : 128 * kEpiParts;

  if (threadIdx.x == 0) {
    mbar_init(&S.bfull, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.ready[s], PAIR ? 2 * kXfThreads / 32 : kXfThreads);  // pair: one arrival per warp
      mbar_init(&S.empty[s], 1);
    }
    for (int i = 0; i < 4; ++i) {  // accumulators; x / residual buffers (<= 4 each)
      mbar_init(&S.tfull[i], 1);
      mbar_init(&S.tempty[i], kTemptyCount);  // one tile group's epilogue threads / warps
      mbar_init(&S.x_full[i], 1);
      mbar_init(&S.x_empty[i], 128 * kEpiParts);
    }
    for (int kb = 0; kb < kAstatSlots; ++kb) {
      mbar_init(&S.a_full[kb], 1);
      mbar_init(&S.a_ready[kb], kXfThreads);
      mbar_init(&S.a_free[kb], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) tmem_alloc_pair(&S.tmem_base, kAcc * BN);
    else tmem_alloc(&S.tmem_base, kAcc * BN);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();  // the peer's barriers are initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0, ag = 0;  // ag: A-stationary k-block sequence number
      uint32_t phase = 0;
      if (BSTAT) {  // the CTA's n-tile of B, every k-block, once
        mbar_expect_tx(&S.bfull, BN * p.K * 2);
        for (int kb = 0; kb < kblocks; ++kb) tma_load_2d(&map_b, &S.bfull, S.b[kb], kb * BKT, n_fixed * BN);
      }
      for (int mt = m_first; mt < p.m_tiles; mt += m_step) {
        int a_n = 0, a_ih0 = 0, a_iw0 = 0;  // im2col: window origin of the m-tile's first pixel
        if (IM2A) {
          const int64_t pix = rowbase(mt), plane = (int64_t)p.gho * p.gwo;
          a_n = (int)(pix / plane);
          const int rem = (int)(pix - (int64_t)a_n * plane), oh = rem / p.gwo;
          a_ih0 = oh * p.gs - p.gp;
          a_iw0 = (rem - oh * p.gwo) * p.gs - p.gp;
        }
        if (ASTAT) {  // this m-tile's A k-blocks, each into a slot the MMAs released
          for (int kb = 0; kb < kblocks; ++kb, ++ag) {
            const int sl = ag % kAstatSlots;
            mbar_wait(&S.a_free[sl], ((uint32_t)(ag / kAstatSlots) & 1u) ^ 1u);
            mbar_expect_tx(&S.a_full[sl], kBM * BKT * 2);
            tma_load_2d(&map_a, &S.a_full[sl], S.a[sl], kb * BKT, mt * kBM);
          }
        }
        for (int nt = 0; nt < nts; ++nt) {
          const int n_tile = ASTAT ? nt : n_fixed;
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&S.empty[stage], phase ^ 1);
            if (ASTAT || GATHER) {  // A is resident / gathered by the transform warps
              // (gathered A with B stationary: an empty arrival = "slot free")
              mbar_expect_tx(&S.full[stage], BSTAT ? 0 : BN * BKT * 2);
            } else if (PAIR && !PRO) {
              // both CTAs' loads complete on the leader's barrier, which the
              // leader alone arms with the pair's bytes (its MMA waits there)
              if (rank == 0) mbar_expect_tx(&S.full[stage], 2 * (kBM + kBRows) * BKT * 2);
              const uint32_t fb = mapa_rank(&S.full[stage], 0);
              if (IM2A) {
                const int tap = kb / cblocks, c0 = (kb - tap * cblocks) * BKT;
                tma_load_im2col_4d_pair(&map_a, fb, S.a[stage], c0, a_iw0, a_ih0, a_n, (uint16_t)(tap % p.gk),
                                        (uint16_t)(tap / p.gk));
              } else {
                tma_load_2d_pair(&map_a, fb, S.a[stage], kb * BKT, (int)rowbase(mt));
              }
              tma_load_2d_pair(&map_b, fb, S.b[stage], kb * BKT, n_tile * BN + (int)rank * kBRows);
            } else {
              mbar_expect_tx(&S.full[stage], (kBM + (BSTAT ? 0 : kBRows)) * BKT * 2);
              if (IM2A) {
                // k-block kb = (tap, 64-channel block): one im2col box of the
                // m-tile's 128 output pixels at filter offset (kh, kw)
                const int tap = kb / cblocks, c0 = (kb - tap * cblocks) * BKT;
                tma_load_im2col_4d(&map_a, &S.full[stage], S.a[stage], c0, a_iw0, a_ih0, a_n, (uint16_t)(tap % p.gk),
                                   (uint16_t)(tap / p.gk));
              } else {
                tma_load_2d(&map_a, &S.full[stage], S.a[stage], kb * BKT, (int)rowbase(mt));
              }
              // (pair with a prologue: each CTA's transform warps wait on its own barrier)
              if (!BSTAT) tma_load_2d(&map_b, &S.full[stage], S.b[stage], kb * BKT, n_tile * BN + (int)rank * kBRows);
            }
            if (!BSTAT && (ASTAT || GATHER)) tma_load_2d(&map_b, &S.full[stage], S.b[stage], kb * BKT, n_tile * BN);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      if (PAIR) {  // every commit of the leader's MMAs has arrived here before the CTA may exit
        for (int i = 0; i < STAGES; ++i) {
          mbar_wait(&S.empty[stage], phase ^ 1);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // (pair: the leader's; the peer's MMA warp only allocated TMEM)
    constexpr uint32_t idesc = PAIR ? instr_desc_pair(BN) : instr_desc(BN);
    if (BSTAT) mbar_wait(&S.bfull, 0);
    if (!PAIR || rank == 0) {
    int stage = 0, ag0 = 0;  // ag0: sequence number of this m-tile's first A k-block
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int mt = m_first; mt < p.m_tiles; mt += m_step, ag0 += kblocks) {
      for (int nt = 0; nt < nts; ++nt) {
        if (PAIR) mbar_wait_cluster(&S.tempty[acc], acc_phase ^ 1);  // both CTAs' epilogues drained it
        else mbar_wait(&S.tempty[acc], acc_phase ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          const int ag = ag0 + kb, sl = ag % kAstatSlots;
          if (ASTAT && nt == 0) mbar_wait(&S.a_ready[sl], (uint32_t)(ag / kAstatSlots) & 1u);  // landed + transformed
          if (PAIR && PRO) mbar_wait_cluster(&S.ready[stage], phase);  // both CTAs' A transformed
          else if ((PRO || GATHER) && !ASTAT) mbar_wait(&S.ready[stage], phase);  // transformed / gathered
          else mbar_wait(&S.full[stage], phase);
          tc_fence_after();
          {
            // converged warp, one lane elected inside each tcgen05 asm;
            // descriptors advance by (bytes >> 4)
            const uint64_t adesc = kmajor_desc<BKT>(smem_u32(ASTAT ? S.a[sl] : S.a[stage]));
            const uint64_t bdesc = kmajor_desc<BKT>(smem_u32(S.b[BSTAT ? kb : stage]));
#pragma unroll
            for (int k = 0; k < BKT / kUmmaK; ++k) {
              if (PAIR)
                umma_bf16_pair_elect(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
              else
                umma_bf16_elect(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            }
            if (PAIR) {
              umma_commit_pair_elect(&S.empty[stage]);                       // both CTAs' stage free
              if (kb == kblocks - 1) umma_commit_pair_elect(&S.tfull[acc]);  // both CTAs' accumulator rows complete
            } else {
              umma_commit_elect(&S.empty[stage]);                       // smem stage free when these MMAs finish
              if (kb == kblocks - 1) umma_commit_elect(&S.tfull[acc]);  // accumulator complete
            }
            if (ASTAT && nt == nts - 1) umma_commit_elect(&S.a_free[sl]);  // A slot no longer read
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (++acc == kAcc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
    }
  } else if (warp == kXWarp) {
    // ------------------------------------------------ x / residual tile producer
    // its own thread, so waiting for a free buffer never holds back the A/B ring
    if (EPI >= 2 && lane == 0) {
      constexpr int kXB = EPI == 2 ? 2 : kResBufs<BN>;
      constexpr int kW = EPI == 2 ? BN : kResW<BN>;
      int xb = 0;
      uint32_t xphase = 0;
      for (int mt = m_first; mt < p.m_tiles; mt += m_step) {
        for (int nt = 0; nt < nts; ++nt) {
          const int n_tile = ASTAT ? nt : n_fixed;
          mbar_wait(&S.x_empty[xb], xphase ^ 1);
          mbar_expect_tx(&S.x_full[xb], kBM * BN * 2);
#pragma unroll
          for (int b = 0; b < BN / kW; ++b)
            tma_load_2d(&map_x, &S.x_full[xb], S.xt[xb] + b * kBM * kW * 2, n_tile * BN + b * kW, (int)rowbase(mt));
          if (++xb == kXB) {
            xb = 0;
            xphase ^= 1;
          }
        }
      }
    }
  } else if (warp >= kXfWarp0) {
    // ------------------------------------------------------------ prologue transform
    if (GATHER) {
      // implicit GEMM: each thread builds kPer 16-byte chunks of one A row per
      // k-block from the input (L1/L2-resident patch rows), into the swizzled slot
      const int xt = threadIdx.x - kXfWarp0 * 32;
      constexpr int kPer = BKT / 16;
      const int r = xt & 127, jh = kPer * (xt >> 7);
      const int kvalid = p.gk * p.gk * p.gc;
      int* ktab = reinterpret_cast<int*>(S.sc);  // k -> (kh * gw + kw) * gc + c and (kh, kw)
      int* khw = reinterpret_cast<int*>(S.sh);
      for (int k = xt; k < p.K; k += kXfThreads) {
        const int c = k % p.gc, t = k / p.gc, kw = t % p.gk, kh = t / p.gk;
        ktab[k] = k < kvalid ? (kh * p.gw + kw) * p.gc + c : 0;
        khw[k] = k < kvalid ? (kh << 16) | kw : -1;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kXfThreads) : "memory");
      const int64_t plane = (int64_t)p.gho * p.gwo;
      const unsigned short* gx = reinterpret_cast<const unsigned short*>(p.gx);
      struct Row {
        bool valid;
        int ih0, iw0;
        const unsigned short* base;
      };
      auto row_of = [&](int mt) {
        Row t;
        const int64_t row = (int64_t)mt * kBM + r;
        t.valid = row < p.M;
        const int n = t.valid ? (int)(row / plane) : 0;
        const int rem = t.valid ? (int)(row - (int64_t)n * plane) : 0;
        t.ih0 = (rem / p.gwo) * p.gs - p.gp;
        t.iw0 = (rem % p.gwo) * p.gs - p.gp;
        t.base = gx + (((int64_t)n * p.gh + t.ih0) * p.gw + t.iw0) * p.gc;
        return t;
      };
      // this thread's kPer chunks of k-block kb of a row (loads only)
      auto gather = [&](const Row& t, int kb, uint4 (&u)[kPer]) {
        if (p.gc == 4) {
          // a 16-byte chunk = two (kh, kw) pixels of 4 channels: one 8-byte load each
          const uint2* base4 = reinterpret_cast<const uint2*>(t.base);
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            uint2 v[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int q = (kb * BKT + 8 * (jh + i)) / 4 + h;
              const int hw = khw[4 * q];
              const int kh = hw >> 16, kw = hw & 0xffff;
              const int ih = t.ih0 + kh, iw = t.iw0 + kw;
              const bool in = t.valid && hw >= 0 && ih >= 0 && ih < p.gh && iw >= 0 && iw < p.gw;
              v[h] = in ? __ldg(base4 + kh * p.gw + kw) : make_uint2(0u, 0u);
            }
            u[i] = make_uint4(v[0].x, v[0].y, v[1].x, v[1].y);
          }
        } else {
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            uint32_t w2[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              uint32_t lohi[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int k = kb * BKT + 8 * (jh + i) + 2 * e + h;
                const int hw = khw[k];
                const int ih = t.ih0 + (hw >> 16), iw = t.iw0 + (hw & 0xffff);
                const bool in = t.valid && hw >= 0 && ih >= 0 && ih < p.gh && iw >= 0 && iw < p.gw;
                lohi[h] = in ? (uint32_t)__ldg(t.base + ktab[k]) : 0u;
              }
              w2[e] = lohi[0] | (lohi[1] << 16);
            }
            u[i] = make_uint4(w2[0], w2[1], w2[2], w2[3]);
          }
        }
      };
      int stage = 0;
      uint32_t phase = 0;
      auto put = [&](const uint4 (&u)[kPer]) {  // one gathered k-block into the ring
        mbar_wait(&S.full[stage], phase);  // slot free (its B landed after the MMA released it)
        uint4* rowp = reinterpret_cast<uint4*>(S.a[stage] + r * BKT * 2);
#pragma unroll
        for (int i = 0; i < kPer; ++i) rowp[swz_chunk<BKT>(jh + i, r)] = u[i];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&S.ready[stage]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      };
      bool stem_done = false;
      if constexpr (BKT == 32) {
        if (p.gk == 7 && p.gc == 4 && p.K == 224) {
          // the ResNet stem (7x7, 4-channel pixels, K = 56 pixels): k-blocks
          // unrolled so every (kh, kw) is a constant; per tile one row / column
          // validity mask replaces the per-pixel bounds arithmetic
          struct Stem {
            uint32_t rmask, cmask;
            const uint2* base;
          };
          auto stem_row = [&](int mt) {
            const Row t = row_of(mt);
            Stem st;
            st.rmask = st.cmask = 0;
#pragma unroll
            for (int d = 0; d < 7; ++d) {
              st.rmask |= (t.valid && t.ih0 + d >= 0 && t.ih0 + d < p.gh) ? 1u << d : 0u;
              st.cmask |= (t.valid && t.iw0 + d >= 0 && t.iw0 + d < p.gw) ? 1u << d : 0u;
            }
            st.base = reinterpret_cast<const uint2*>(t.base);
            return st;
          };
          auto load = [&](const Stem& st, int kb, uint4 (&u)[kPer], int half) {
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
              uint2 v[2];
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int q = kb * 8 + half * 4 + 2 * i + h;  // pixel (kh, kw) = (q / 7, q % 7)
                const int kh = q / 7, kw = q % 7;
                const bool in = q < 49 && ((st.rmask >> kh) & (st.cmask >> kw) & 1u);
                v[h] = in ? __ldg(st.base + kh * p.gw + kw) : make_uint2(0u, 0u);
              }
              u[i] = make_uint4(v[0].x, v[0].y, v[1].x, v[1].y);
            }
          };
          auto run = [&](int half) {
            int mt = m_first;
            Stem cur = stem_row(mt);
            uint4 u[kPer], un[kPer];
            if (mt < p.m_tiles) load(cur, 0, un, half);
            while (mt < p.m_tiles) {
              const int nmt = mt + m_step;
              Stem nxt = stem_row(nmt);
#pragma unroll
              for (int kb = 0; kb < 7; ++kb) {
#pragma unroll
                for (int i = 0; i < kPer; ++i) u[i] = un[i];
                if (kb < 6) load(cur, kb + 1, un, half);
                else if (nmt < p.m_tiles) load(nxt, 0, un, half);
                put(u);
              }
              cur = nxt;
              mt = nmt;
            }
          };
          if (jh == 0) run(0);  // literal halves: (kh, kw) fold to constants after inlining
          else run(1);
          stem_done = true;
        }
      }
      if (!stem_done) {
      // software pipeline over the flattened (tile, k-block) sequence: the
      // loads of the next k-block are in flight while this one is stored
      int mt = m_first, kb = 0;
      Row cur = row_of(mt);
      uint4 u[kPer], un[kPer];
      if (mt < p.m_tiles) gather(cur, 0, un);
      while (mt < p.m_tiles) {
#pragma unroll
        for (int i = 0; i < kPer; ++i) u[i] = un[i];
        int nmt = mt, nkb = kb + 1;
        if (nkb == kblocks) {
          nkb = 0;
          nmt += m_step;
          cur = row_of(nmt);
        }
        if (nmt < p.m_tiles) gather(cur, nkb, un);
        put(u);
        mt = nmt;
        kb = nkb;
      }
      }
    } else if (PRO) {
      const int xt = threadIdx.x - kXfWarp0 * 32;  // 0..255
      constexpr int kPer = BKT / 16;                // 16-byte chunks per thread (two threads per row)
      const int r = xt & 127, jh = kPer * (xt >> 7);  // tile row, first logical chunk
      // the previous BN's affine, exactly as bn_apply computes it (per input
      // channel: K columns, or the im2col input's channels)
      for (int c = xt; c < (IM2A ? p.gc : p.K); c += kXfThreads) {
        float sc = p.pinvstd[c] * __bfloat162float(p.pg[c]);
        S.sc[c] = sc;
        S.sh[c] = __bfloat162float(p.pb[c]) - p.pmean[c] * sc;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kXfThreads) : "memory");  // transform warps only
      int stage = 0, ag = 0;
      uint32_t phase = 0;
      for (int mt = m_first; mt < p.m_tiles; mt += m_step) {
        // im2col: this row's output pixel and its window origin; rows whose
        // tap falls in the zero padding (or beyond M) stay zero
        bool rvalid = true;
        int ih0 = 0, iw0 = 0;
        if (IM2A) {
          const int64_t pix = rowbase(mt) + r, plane = (int64_t)p.gho * p.gwo;
          rvalid = pix < p.M;
          const int n = (int)(pix / plane), rem = (int)(pix - (int64_t)n * plane), oh = rem / p.gwo;
          ih0 = oh * p.gs - p.gp;
          iw0 = (rem - oh * p.gwo) * p.gs - p.gp;
        }
        // a = bf16(relu(a*sc + sh)) in place.  Logical 16-byte chunk jj of row r
        // (channels kb*BKT + 8*jj .. +8) is physical chunk swz_chunk(jj, r)
        for (int kb = 0; kb < kblocks; ++kb) {
          const int sl = ag % kAstatSlots;
          if (ASTAT) mbar_wait(&S.a_full[sl], (uint32_t)(ag / kAstatSlots) & 1u);
          else mbar_wait(&S.full[stage], phase);
          uint4* rowp = reinterpret_cast<uint4*>((ASTAT ? S.a[sl] : S.a[stage]) + r * BKT * 2);
          int cbase = kb * BKT;  // prologue channel of this k-block's first column
          bool valid = true;
          if (IM2A) {
            const int tap = kb / cblocks, ih = ih0 + tap / p.gk, iw = iw0 + tap % p.gk;
            cbase = (kb - tap * cblocks) * BKT;
            valid = rvalid && ih >= 0 && ih < p.gh && iw >= 0 && iw < p.gw;
          }
          uint4 u[kPer];
#pragma unroll
          for (int i = 0; i < kPer; ++i) u[i] = rowp[swz_chunk<BKT>(jh + i, r)];  // consecutive rows: distinct columns
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            if (IM2A && !valid) {
              u[i] = make_uint4(0u, 0u, 0u, 0u);
              rowp[swz_chunk<BKT>(jh + i, r)] = u[i];
              continue;
            }
            const int c0 = cbase + 8 * (jh + i);
            // channel pairs: bf16x2 -> two fp32 (shift / mask), one packed
            // fp32x2 FMA (FFMA2, same rounding as two FFMAs), then ReLU and the
            // bf16x2 pack in one cvt.rn.relu
            const ulonglong2 sa = *reinterpret_cast<const ulonglong2*>(&S.sc[c0]);
            const ulonglong2 sb = *reinterpret_cast<const ulonglong2*>(&S.sc[c0 + 4]);
            const ulonglong2 ha = *reinterpret_cast<const ulonglong2*>(&S.sh[c0]);
            const ulonglong2 hb = *reinterpret_cast<const ulonglong2*>(&S.sh[c0 + 4]);
            const unsigned long long sc2[4] = {sa.x, sa.y, sb.x, sb.y}, sh2[4] = {ha.x, ha.y, hb.x, hb.y};
            uint32_t* w = reinterpret_cast<uint32_t*>(&u[i]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const uint32_t lo = w[e] << 16, hi = w[e] & 0xffff0000u;  // channels 2e, 2e+1 as fp32
              const unsigned long long xv = ((unsigned long long)hi << 32) | lo;
              unsigned long long yv;
              asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(yv) : "l"(xv), "l"(sc2[e]), "l"(sh2[e]));
              uint32_t packed;
              asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;"
                  : "=r"(packed)
                  : "f"(__uint_as_float((uint32_t)(yv >> 32))), "f"(__uint_as_float((uint32_t)yv)));
              w[e] = packed;
            }
            rowp[swz_chunk<BKT>(jh + i, r)] = u[i];
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the tensor core
          if (ASTAT) {
            mbar_arrive(&S.a_ready[sl]);
            ++ag;
          } else {
            if (PAIR) {  // one release per warp on the leader's barrier (its MMAs read this tile)
              __syncwarp();
              if (lane == 0) mbar_arrive_rank(&S.ready[stage], 0);
            } else {
              mbar_arrive(&S.ready[stage]);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue warps
    const int q = warp & 3;                       // TMEM lane quarter this warp may access
    const int ew = warp - kEpiWarp0;              // 0..15
    constexpr int kCW = BN < 32 ? BN : 32;        // chunk width: 32 columns (16 for BN = 16)
    constexpr int kParts = kEpiParts;
    const int half = (ew >> 2) % kParts;          // this warp's column part
    const int grp = (ew >> 2) / kParts;           // this warp's tile group
    constexpr int kChunks = BN / kCW / kParts;    // chunks per part
    {
    // statistics: one partial row per (m-group, lane quarter, tile group); lane
    // = column.  Fixed n-tile: accumulated in registers, written once at the end.
    // A-stationary (the n-tile varies per tile): accumulated in the thread's
    // own slots of the partial rows, zeroed first and then added to with
    // fire-and-forget reductions (no load latency in the epilogue; no
    // dynamically indexed local arrays)
    constexpr bool kStats = EPI == 1 || EPI == 2 || EPI == 4;
    const int mgroup = PAIR ? 2 * m_first + (int)rank : m_first;  // partial-row group of this CTA
    float* part_row = kStats ? p.part + (((size_t)mgroup * 4 + q) * kEpiGroups + grp) * 2 * p.N : nullptr;
    if (ASTAT && kStats) {
      for (int nt = 0; nt < nts; ++nt)
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          float* slot = part_row + (size_t)nt * BN + half * (BN / kParts) + c * kCW + lane;
          slot[0] = 0.f;
          slot[p.N] = 0.f;
        }
    }
    float acc_s[kChunks], acc_q[kChunks];
#pragma unroll
    for (int c = 0; c < kChunks; ++c) acc_s[c] = acc_q[c] = 0.f;
    int sbuf = 0;
    int t = -1;  // tile sequence number, as the MMA warp counts it
    for (int mt = m_first; mt < p.m_tiles; mt += m_step) {
     for (int nt = 0; nt < nts; ++nt) {
      if (++t % kEpiGroups != grp) continue;      // another group's tile
      const int acc = t % kAcc;
      const uint32_t acc_phase = (uint32_t)(t / kAcc) & 1u;
      const int n_tile = ASTAT ? nt : n_fixed;
      const int64_t row0 = rowbase(mt) + q * 32;
      const bool valid = row0 + lane < p.M;
      const int rb = EPI >= 3 ? t % kResBufs<BN> : 0;  // residual buffer of this tile
      mbar_wait(&S.tfull[acc], acc_phase);
      if (EPI >= 3) mbar_wait(&S.x_full[rb], (uint32_t)(t / kResBufs<BN>) & 1u);
      if (EPI == 2) mbar_wait(&S.x_full[acc], acc_phase);  // x tiles alternate with the accumulators
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        const int col = half * (BN / kParts) + c * kCW;  // within the tile
        float v[kCW];
        if constexpr (kCW == 32) tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + col, v);
        else tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + col, v);
        // this warp's staging buffer must be free: the TMA store issued two chunks ago has read it
        if (lane == 0) {
          if (ASTAT) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
        __syncwarp();
        uint4* st = reinterpret_cast<uint4*>(S.cstage[ew][sbuf] + lane * kCW * 2);
#pragma unroll
        for (int j = 0; j < kCW / 8; ++j) {
          if (EPI >= 3) {
            // chunk j of this row in its residual box (row-per-lane reads of
            // the swizzled box: 8 lanes of a phase hit 8 distinct bank groups)
            constexpr int RW = kResW<BN>;
            const int row = q * 32 + lane, cb = col / RW, cj = (col % RW) / 8 + j;
            const uint4 rw = *reinterpret_cast<const uint4*>(S.xt[rb] + cb * kBM * RW * 2 + row * RW * 2 +
                                                             swz_chunk<RW>(cj, row) * 16);
            const __nv_bfloat162* rh = reinterpret_cast<const __nv_bfloat162*>(&rw);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(rh[e]);
              v[8 * j + 2 * e] += f.x;
              v[8 * j + 2 * e + 1] += f.y;
            }
          }
          uint4 u;
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            h[e] = valid ? __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1])
                         : __floats2bfloat162_rn(0.f, 0.f);
          }
          st[swz_chunk<kCW>(j, lane)] = u;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          // rows beyond M are clipped by the TMA unit
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&map_c)),
              "r"(n_tile * BN + col), "r"((int)row0), "r"(smem_u32(S.cstage[ew][sbuf]))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (EPI == 2) {
          // BN backward reduce on the stored (rounded) gradient: lane = column,
          // rows in order; x read straight from global (a warp reads 64
          // contiguous bytes per row), the mask recomputed as bn_backward does
          const __nv_bfloat16* stg = reinterpret_cast<const __nv_bfloat16*>(S.cstage[ew][sbuf]);
          const int cc = lane >> 3, ce = lane & 7;
          const int gc = n_tile * BN + col + lane;  // global column
          const float is = __ldg(p.binvstd + gc), mu = __ldg(p.bmean + gc);
          const float sc = is * __bfloat162float(p.bg[gc]);
          const float sh = __bfloat162float(p.bb[gc]) - mu * sc;
          // x of this (row, column) from the TMA-loaded tile (OOB rows are zeros)
          const __nv_bfloat16* xs = reinterpret_cast<const __nv_bfloat16*>(S.xt[acc]) + (q * 32) * BN + col + lane;
          float xv[32];
#pragma unroll
          for (int r = 0; r < 32; ++r) xv[r] = __bfloat162float(xs[r * BN]);
          float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int r = 0; r < 32; ++r) {
            float gm = __bfloat162float(stg[r * 32 + 8 * (cc ^ ((r >> 1) & 3)) + ce]);
            // bf16(fma) > 0 <=> fma > 2^-134 (bn_kernels.cu relu_mask); rows beyond M: staged gm = 0
            gm = __fmaf_rn(xv[r], sc, sh) > 0x1p-134f ? gm : 0.0f;
            s1[r & 3] += gm;
            s2[r & 3] += gm * ((xv[r] - mu) * is);
          }
          const float t1 = (s1[0] + s1[1]) + (s1[2] + s1[3]), t2 = (s2[0] + s2[1]) + (s2[2] + s2[3]);
          if (ASTAT) {
            float* slot = part_row + (size_t)n_tile * BN + col + lane;
            atomicAdd(slot, t1);  // fire-and-forget RED: only this thread touches the slot,
            atomicAdd(slot + p.N, t2);  // so the sum order (and result) is fixed
          } else {
            acc_s[c] += t1;
            acc_q[c] += t2;
          }
        }
        if (EPI == 1 || EPI == 4) {
          // column `lane` of the staged (stored) bf16 chunk, rows in order;
          // rows beyond M were staged as zeros.  16-wide chunks: lanes 16..31
          // take rows 16..31 of the same columns, folded in with one shuffle
          const __nv_bfloat16* stg = reinterpret_cast<const __nv_bfloat16*>(S.cstage[ew][sbuf]);
          const int cl = lane % kCW, cc = cl >> 3, ce = cl & 7;  // column, logical chunk, element
          constexpr int kRows = kCW == 32 ? 32 : 16;
          const int rb = lane / kCW * kRows;
          float s1[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent chains
#pragma unroll
          for (int i = 0; i < kRows; ++i) {
            const int r = rb + i;
            float x = __bfloat162float(stg[r * kCW + 8 * swz_chunk<kCW>(cc, r) + ce]);
            s1[i & 3] += x;
            s2[i & 3] = __fmaf_rn(x, x, s2[i & 3]);
          }
          float t1 = (s1[0] + s1[1]) + (s1[2] + s1[3]), t2 = (s2[0] + s2[1]) + (s2[2] + s2[3]);
          if constexpr (kCW == 16) {
            t1 += __shfl_down_sync(0xffffffffu, t1, 16);
            t2 += __shfl_down_sync(0xffffffffu, t2, 16);
          }
          if (ASTAT) {
            float* slot = part_row + (size_t)n_tile * BN + col + lane;
            atomicAdd(slot, t1);  // fire-and-forget RED: only this thread touches the slot,
            atomicAdd(slot + p.N, t2);  // so the sum order (and result) is fixed
          } else {
            acc_s[c] += t1;
            acc_q[c] += t2;
          }
        }
        if (!ASTAT) sbuf ^= 1;
      }
      tc_fence_before();
      if (PAIR) {  // one arrival per warp, on the leader's barrier
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&S.tempty[acc]);
          else mbar_arrive_rank(&S.tempty[acc], 0);
        }
      } else {
        mbar_arrive(&S.tempty[acc]);
      }
      if (EPI == 2) mbar_arrive(&S.x_empty[acc]);
      if (EPI >= 3) mbar_arrive(&S.x_empty[rb]);
     }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
    if (kStats && !ASTAT) {
      float* out = part_row + (size_t)n_fixed * BN + half * (BN / kParts);
#pragma unroll
      for (int c = 0; c < kChunks; ++c) {
        if (lane < kCW) {
          out[c * kCW + lane] = acc_s[c];
          out[p.N + c * kCW + lane] = acc_q[c];
        }
      }
    }
    }
  }
  tc_fence_before();
  if (PAIR) {
    cluster_sync();  // neither CTA leaves while the peer may still touch its barriers or TMEM
    if (warp == 1) tmem_dealloc_pair(tmem, kAcc * BN);
  } else {
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, kAcc * BN);
  }
}

// per-channel mean / invstd from the partial rows: CTA = 32 channels, 32 warps
// stride the rows (4 loads in flight each), then a fixed-order pass over the
// warps in double (deterministic)
__global__ void __launch_bounds__(1024) partials_finalize_kernel(const float* __restrict__ part, int rows_part, int N,
                                                                 int64_t M, float eps, float* __restrict__ mean,
                                                                 float* __restrict__ invstd) {
  __shared__ double sh[2][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double s = 0, q = 0;
  if (c < N) {
    int r = w;
    for (; r + 96 < rows_part; r += 128) {
      float a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = part[(size_t)(r + 32 * u) * 2 * N + c];
        b[u] = part[(size_t)(r + 32 * u) * 2 * N + N + c];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        s += (double)a[u];
        q += (double)b[u];
      }
    }
    for (; r < rows_part; r += 32) {
      s += (double)part[(size_t)r * 2 * N + c];
      q += (double)part[(size_t)r * 2 * N + N + c];
    }
  }
  sh[0][w][lane] = s;
  sh[1][w][lane] = q;
  __syncthreads();
  if (w != 0 || c >= N) return;
  s = 0;
  q = 0;
  for (int k = 0; k < 32; ++k) {
    s += sh[0][k][lane];
    q += sh[1][k][lane];
  }
  const double mu = s / (double)M;
  double var = q / (double)M - mu * mu;
  if (var < 0) var = 0;
  mean[c] = (float)mu;
  invstd[c] = (float)(1.0 / sqrt(var + (double)eps));
}

// BN backward from the partial rows (EPI 2): dbeta = sum gm, dgamma = sum
// gm*xhat, and the dx coefficients A, B, D of bn_kernels.cu (dx = A*gm + B*x + D)
__global__ void __launch_bounds__(1024) partials_bwd_finalize_kernel(
    const float* __restrict__ part, int rows_part, int N, int64_t M, const float* __restrict__ mean,
    const float* __restrict__ invstd, const __nv_bfloat16* __restrict__ g, float* __restrict__ dgamma,
    float* __restrict__ dbeta, float* __restrict__ coef) {
  __shared__ double sh[2][32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double s = 0, q = 0;
  if (c < N)
    for (int r = w; r < rows_part; r += 32) {
      s += (double)part[(size_t)r * 2 * N + c];
      q += (double)part[(size_t)r * 2 * N + N + c];
    }
  sh[0][w][lane] = s;
  sh[1][w][lane] = q;
  __syncthreads();
  if (w != 0 || c >= N) return;
  s = 0;
  q = 0;
  for (int k = 0; k < 32; ++k) {
    s += sh[0][k][lane];
    q += sh[1][k][lane];
  }
  if (dbeta) dbeta[c] = (float)s;
  if (dgamma) dgamma[c] = (float)q;
  const double is = invstd[c], mu = mean[c];
  const double gs = (double)__bfloat162float(g[c]) * is;
  const double k1 = s / (double)M, k2 = q / (double)M;
  coef[c] = (float)gs;
  coef[N + c] = (float)(-gs * is * k2);
  coef[2 * N + c] = (float)(gs * (mu * is * k2 - k1));
}

// ---------------------------------------------------------------------------
// host side

template <int BN, int STAGES, bool PRO, int EPI, bool ASTAT, int BKT, bool GATHER, bool BSTAT, bool IM2A, bool PAIR>
cudaError_t launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const CUtensorMap& mx,
                   const Params& p, int grid, cudaStream_t s) {
  auto k = conv1x1_kernel<BN, STAGES, PRO, EPI, ASTAT, BKT, GATHER, BSTAT, IM2A, PAIR>;
  const size_t smem = sizeof(Smem<BN, STAGES, PRO || GATHER, ASTAT, EPI, BKT, BSTAT, PAIR>);
  static bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (PAIR) {  // clusters of two CTAs on one TPC
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, ma, mb, mc, mx, p);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  k<<<grid, kThreads, smem, s>>>(ma, mb, mc, mx, p);
  return cudaGetLastError();
}

template <int BN, bool PRO, int EPI, bool ASTAT, int BKT, bool GATHER, bool bstat, bool IM2A = false, bool PAIR = false>
cudaError_t dispatch_ring(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                          const CUtensorMap& mx, const Params& p, int grid, cudaStream_t s) {
  // deepest ring that fits next to everything else (227 KB per CTA)
  constexpr int fixed = (PRO || GATHER ? 2 * kMaxProK * 4 : 0) + kEpiWarps * (ASTAT ? 1 : 2) * 32 * 64 +
                        (ASTAT ? kAstatSlots * kBM * kBK * 2 : 0) + (EPI == 2 ? 2 * kBM * BN * 2 : 0) +
                        (EPI >= 3 ? kResBufs<BN> * kBM * BN * 2 : 0) + (bstat ? kBSlots<BN, BKT> * BN * BKT * 2 : 0);
  constexpr int stage_bytes = (ASTAT ? BN : kBM + (bstat ? 0 : (PAIR ? BN / 2 : BN))) * BKT * 2;
  constexpr int avail = 220 * 1024 - fixed;
  constexpr int max_stages = 8 * kBK / BKT;  // same bytes in flight for narrow k-blocks
  constexpr int stages = avail / stage_bytes > max_stages ? max_stages : avail / stage_bytes;
  static_assert(stages >= 2, "shared memory");
  return launch<BN, stages, PRO, EPI, ASTAT, BKT, GATHER, bstat, IM2A, PAIR>(ma, mb, mc, mx, p, grid, s);
}

// CTA-pair instantiations: streamed A and B, 64-wide k-blocks
template <int BN, bool PRO, int EPI, bool IM2A>
cudaError_t dispatch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const CUtensorMap& mx,
                          const Params& p, int grid, cudaStream_t s) {
  return dispatch_ring<BN, PRO, EPI, false, kBK, false, false, IM2A, true>(ma, mb, mc, mx, p, grid, s);
}

// im2col A (3x3 / strided convolutions): streamed 64-channel k-blocks, B too
// wide to stay resident
template <int BN, bool PRO, int EPI>
cudaError_t dispatch_im2col(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, const CUtensorMap& mx,
                            const Params& p, int grid, bool pair, cudaStream_t s) {
  if (pair) return dispatch_pair<BN, PRO, EPI, true>(ma, mb, mc, mx, p, grid, s);
  return dispatch_ring<BN, PRO, EPI, false, kBK, false, false, true>(ma, mb, mc, mx, p, grid, s);
}

// CTA pairs for streamed GEMMs (KRT_GEMM_PAIR=0 turns them off)
bool pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("KRT_GEMM_PAIR");
    return e == nullptr || std::strcmp(e, "0") != 0;
  }();
  return on;
}

template <int BN, bool PRO, int EPI, bool ASTAT, int BKT = kBK, bool GATHER = false>
cudaError_t dispatch_stages(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                            const CUtensorMap& mx, const Params& p, int grid, cudaStream_t s) {
  if constexpr (!ASTAT) {
    if (p.K / BKT <= kBSlots<BN, BKT> && BN * p.K * 2 <= kBStatBytes)
      return dispatch_ring<BN, PRO, EPI, ASTAT, BKT, GATHER, true>(ma, mb, mc, mx, p, grid, s);
  }
  return dispatch_ring<BN, PRO, EPI, ASTAT, BKT, GATHER, false>(ma, mb, mc, mx, p, grid, s);
}

// EPI 3 (residual) instantiations: n-tiles up to 128 columns, never
// A-stationary (its A region and the residual ring do not both fit)
template <int BKT>
cudaError_t dispatch_res(int BN, bool pro, bool st, const CUtensorMap& ma, const CUtensorMap& mb,
                         const CUtensorMap& mc, const CUtensorMap& mx, const Params& p, int grid, cudaStream_t s) {
#define KRT_GEMM_RES(BNV)                                                                                   \
  if (BN == BNV) {                                                                                          \
    if (st) return pro ? dispatch_stages<BNV, true, 4, false, BKT>(ma, mb, mc, mx, p, grid, s)               \
                       : dispatch_stages<BNV, false, 4, false, BKT>(ma, mb, mc, mx, p, grid, s);             \
    return pro ? dispatch_stages<BNV, true, 3, false, BKT>(ma, mb, mc, mx, p, grid, s)                       \
               : dispatch_stages<BNV, false, 3, false, BKT>(ma, mb, mc, mx, p, grid, s);                     \
  }
  KRT_GEMM_RES(16)
  KRT_GEMM_RES(32)
  KRT_GEMM_RES(64)
  KRT_GEMM_RES(128)
#undef KRT_GEMM_RES
  return cudaErrorInvalidValue;
}

}  // namespace

// partial rows: (m-group <= SMs) x (lane quarter) x (epilogue tile group <= 4)
size_t conv1x1_partials_bytes(int N) { return (size_t)num_sms() * 16 * 2 * N * sizeof(float); }

bool conv1x1_supported(int64_t M, int N, int K) {
  return M > 0 && (K == 16 || K == 32 || K % kBK == 0) && K <= 65536 &&
         (N == 16 || N == 32 || N == 64 || N == 128 || N % 256 == 0);
}

namespace {
cudaError_t conv1x1_impl(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                         const float* pinvstd, const void* pg, const void* pb, float* part, int* part_rows,
                         const void* bx, const float* bmean, const float* binvstd, const void* bg, const void* bb,
                         const void* res, cudaStream_t s) {
  if (!conv1x1_supported(M, N, K) || (pmean != nullptr && K > kMaxProK)) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) & 15)
    return cudaErrorMisalignedAddress;
  const bool bwd_mode = bx != nullptr;
  // the BN-backward epilogue keeps two x tiles in shared memory, the residual
  // epilogue a ring of residual tiles: 128-column tiles
  const bool res_mode = res != nullptr;
  const int BN = (bwd_mode || res_mode) ? (N < 128 ? N : 128) : (N <= 256 ? N : 256);
  Params p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.BN = BN;
  p.n_tiles = N / BN;
  p.m_tiles = (int)((M + kBM - 1) / kBM);
  p.C = static_cast<__nv_bfloat16*>(C);
  p.part = part;
  p.pmean = pmean;
  p.pinvstd = pinvstd;
  p.pg = static_cast<const __nv_bfloat16*>(pg);
  p.pb = static_cast<const __nv_bfloat16*>(pb);
  p.bx = static_cast<const __nv_bfloat16*>(bx);
  p.bmean = bmean;
  p.binvstd = binvstd;
  p.bg = static_cast<const __nv_bfloat16*>(bg);
  p.bb = static_cast<const __nv_bfloat16*>(bb);
  p.res = static_cast<const __nv_bfloat16*>(res);
  if (res != nullptr && (reinterpret_cast<uintptr_t>(res) & 15)) return cudaErrorMisalignedAddress;
  const bool bwd = bx != nullptr;
  if (bwd && (pmean != nullptr || part == nullptr || N < 64 || res != nullptr)) return cudaErrorInvalidValue;
  // narrow reductions (K = 16, 32: the first stages of ResNet-1001) use one
  // K-wide k-block whose row is the 32/64-byte swizzle span
  const int bkt = K < kBK ? K : kBK;
  const CUtensorMapSwizzle ksw = bkt == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                           : (bkt == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  CUtensorMap ma, mb, mc, mx;
  if (!make_map(&ma, A, M, K, kBM, bkt, ksw) || !make_map(&mb, B, N, K, BN, bkt, ksw) ||
      !make_map(&mc, C, M, N, 32, N < 32 ? N : 32, N < 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  if (bwd_mode) {
    if (!make_map(&mx, bx, M, N, kBM, BN, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
  } else if (res_mode) {
    const int rw = BN < 64 ? BN : 64;
    if (!make_map(&mx, res, M, N, kBM, rw,
                  rw == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                           : (rw == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B)))
      return cudaErrorInvalidValue;
  } else {
    mx = mc;  // unused
  }
  const bool pro = pmean != nullptr, st = part != nullptr;
  // A-stationary when the prologue would otherwise transform the same A tile once per n-tile
  const bool astat = pro && !res_mode && bkt == kBK && p.n_tiles > 1 && K <= kMaxAstatK && p.n_tiles <= kMaxNT;
  // CTA pairs for the streamed 64-wide k-block path at 256-column n-tiles with
  // K >= 256 (measured, scripts/bench_gemm_pair.py: 2-8% faster there, up to
  // 16% slower at K = 128 where the epilogue, not the operand ring, bounds it)
  const bool pair = pair_enabled() && !astat && !res_mode && bkt == kBK && BN == 256 && K >= 256;
  if (pair) p.m_tiles = (int)((M + 2 * kBM - 1) / (2 * kBM));
  // whole n-tile groups (or, A-stationary, whole m-tiles), at most one CTA per SM
  const int units = pair ? num_sms() / 2 : num_sms();  // CTAs or CTA pairs
  int per = astat ? units : units / p.n_tiles;
  if (per < 1) per = 1;
  if (per > p.m_tiles) per = p.m_tiles;
  const int grid = (astat ? per : per * p.n_tiles) * (pair ? 2 : 1);
  const int epi_groups = 4 / (BN >= 128 ? 4 : (BN >= 64 ? BN / 32 : 1));
  if (part_rows) *part_rows = per * (pair ? 2 : 1) * 4 * epi_groups;  // every row and column written exactly once
  if (pair && !make_map(&mb, B, N, K, BN / 2, bkt, ksw)) return cudaErrorInvalidValue;  // half the n-tile per CTA
  if (res_mode) {
    if (bkt == 16) return dispatch_res<16>(BN, pro, st, ma, mb, mc, mx, p, grid, s);
    if (bkt == 32) return dispatch_res<32>(BN, pro, st, ma, mb, mc, mx, p, grid, s);
    return dispatch_res<kBK>(BN, pro, st, ma, mb, mc, mx, p, grid, s);
  }
  if (bkt != kBK) {  // no A-stationary instantiations for narrow k-blocks
    if (bwd) {
      if (BN == 64) return bkt == 16 ? dispatch_stages<64, false, 2, false, 16>(ma, mb, mc, mx, p, grid, s)
                                     : dispatch_stages<64, false, 2, false, 32>(ma, mb, mc, mx, p, grid, s);
      if (BN == 128) return bkt == 16 ? dispatch_stages<128, false, 2, false, 16>(ma, mb, mc, mx, p, grid, s)
                                      : dispatch_stages<128, false, 2, false, 32>(ma, mb, mc, mx, p, grid, s);
      return cudaErrorInvalidValue;
    }
#define KRT_GEMM_NARROW(BNV, BKV)                                                                  \
  if (BN == BNV && bkt == BKV) {                                                                  \
    if (pro && st) return dispatch_stages<BNV, true, 1, false, BKV>(ma, mb, mc, mx, p, grid, s); \
    if (pro) return dispatch_stages<BNV, true, 0, false, BKV>(ma, mb, mc, mx, p, grid, s);       \
    if (st) return dispatch_stages<BNV, false, 1, false, BKV>(ma, mb, mc, mx, p, grid, s);       \
    return dispatch_stages<BNV, false, 0, false, BKV>(ma, mb, mc, mx, p, grid, s);               \
  }
    KRT_GEMM_NARROW(16, 16)
    KRT_GEMM_NARROW(32, 16)
    KRT_GEMM_NARROW(64, 16)
    KRT_GEMM_NARROW(128, 16)
    KRT_GEMM_NARROW(256, 16)
    KRT_GEMM_NARROW(16, 32)
    KRT_GEMM_NARROW(32, 32)
    KRT_GEMM_NARROW(64, 32)
    KRT_GEMM_NARROW(128, 32)
    KRT_GEMM_NARROW(256, 32)
#undef KRT_GEMM_NARROW
    return cudaErrorInvalidValue;
  }
  if (bwd) {
    if (BN == 64) return pair ? dispatch_pair<64, false, 2, false>(ma, mb, mc, mx, p, grid, s)
                              : dispatch_stages<64, false, 2, false>(ma, mb, mc, mx, p, grid, s);
    if (BN == 128) return pair ? dispatch_pair<128, false, 2, false>(ma, mb, mc, mx, p, grid, s)
                               : dispatch_stages<128, false, 2, false>(ma, mb, mc, mx, p, grid, s);
    return cudaErrorInvalidValue;
  }
#define KRT_GEMM_BN(BNV)                                                                          \
  if (BN == BNV) {                                                                                \
    if (pair && pro && st) return dispatch_pair<BNV, true, 1, false>(ma, mb, mc, mx, p, grid, s); \
    if (pair && pro) return dispatch_pair<BNV, true, 0, false>(ma, mb, mc, mx, p, grid, s);       \
    if (pair && st) return dispatch_pair<BNV, false, 1, false>(ma, mb, mc, mx, p, grid, s);       \
    if (pair) return dispatch_pair<BNV, false, 0, false>(ma, mb, mc, mx, p, grid, s);             \
    if (astat && st) return dispatch_stages<BNV, true, 1, true>(ma, mb, mc, mx, p, grid, s);     \
    if (astat) return dispatch_stages<BNV, true, 0, true>(ma, mb, mc, mx, p, grid, s);           \
    if (pro && st) return dispatch_stages<BNV, true, 1, false>(ma, mb, mc, mx, p, grid, s);      \
    if (pro) return dispatch_stages<BNV, true, 0, false>(ma, mb, mc, mx, p, grid, s);            \
    if (st) return dispatch_stages<BNV, false, 1, false>(ma, mb, mc, mx, p, grid, s);            \
    return dispatch_stages<BNV, false, 0, false>(ma, mb, mc, mx, p, grid, s);                   \
  }
  if (BN < 64) {  // one n-tile: never A-stationary
    if (BN == 16) return pro ? (st ? dispatch_stages<16, true, 1, false>(ma, mb, mc, mx, p, grid, s)
                                   : dispatch_stages<16, true, 0, false>(ma, mb, mc, mx, p, grid, s))
                             : (st ? dispatch_stages<16, false, 1, false>(ma, mb, mc, mx, p, grid, s)
                                   : dispatch_stages<16, false, 0, false>(ma, mb, mc, mx, p, grid, s));
    if (BN == 32) return pro ? (st ? dispatch_stages<32, true, 1, false>(ma, mb, mc, mx, p, grid, s)
                                   : dispatch_stages<32, true, 0, false>(ma, mb, mc, mx, p, grid, s))
                             : (st ? dispatch_stages<32, false, 1, false>(ma, mb, mc, mx, p, grid, s)
                                   : dispatch_stages<32, false, 0, false>(ma, mb, mc, mx, p, grid, s));
    return cudaErrorInvalidValue;
  }
  KRT_GEMM_BN(64)
  KRT_GEMM_BN(128)
  KRT_GEMM_BN(256)
#undef KRT_GEMM_BN
  return cudaErrorInvalidValue;
}
}  // namespace

cudaError_t conv1x1_bn_fprop(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                             const float* pinvstd, const void* pg, const void* pb, float* part, int* part_rows,
                             cudaStream_t s) {
  return conv1x1_impl(A, B, C, M, N, K, pmean, pinvstd, pg, pb, part, part_rows, nullptr, nullptr, nullptr, nullptr,
                      nullptr, nullptr, s);
}

namespace {
// RGB NHWC bf16 -> 4-channel pixels (4th = 0): two pixels per thread, 12-byte
// (3 x 4-byte) loads, one 16-byte store
__global__ void pad_rgb4_kernel(const uint32_t* __restrict__ x, uint4* __restrict__ y, int64_t pixels) {
  const int64_t pairs = pixels / 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < pairs; t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = __ldg(x + 3 * t), b = __ldg(x + 3 * t + 1), c = __ldg(x + 3 * t + 2);
    // pixel 0 = (a.lo, a.hi, b.lo), pixel 1 = (b.hi, c.lo, c.hi)
    y[t] = make_uint4(a, b & 0xffffu, (b >> 16) | (c << 16), c >> 16);
  }
  if ((pixels & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd count: the last pixel alone
    const unsigned short* xs = reinterpret_cast<const unsigned short*>(x) + 3 * (pixels - 1);
    reinterpret_cast<uint2*>(y)[pixels - 1] = make_uint2(xs[0] | ((uint32_t)xs[1] << 16), xs[2]);
  }
}
}  // namespace

cudaError_t pad_rgb4(const void* x, void* y, int64_t pixels, cudaStream_t s) {
  if (pixels < 1 || (reinterpret_cast<uintptr_t>(x) & 3) || (reinterpret_cast<uintptr_t>(y) & 15))
    return cudaErrorInvalidValue;
  const int64_t pairs = pixels / 2;
  int64_t blocks = (pairs + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  pad_rgb4_kernel<<<(int)blocks, 256, 0, s>>>(static_cast<const uint32_t*>(x), static_cast<uint4*>(y), pixels);
  return cudaGetLastError();
}

cudaError_t conv_gather_fprop(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int ho, int wo,
                              int k, int stride, int pad, int N, int K, float* part, int* part_rows, cudaStream_t s) {
  const int64_t M = (int64_t)n * ho * wo;
  if (M <= 0 || N != 64 || K % 32 != 0 || K < k * k * cin || K > kMaxProK || cin < 1 || k < 1 || stride < 1)
    return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(wk) | reinterpret_cast<uintptr_t>(C)) & 15) return cudaErrorMisalignedAddress;
  Params p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.BN = N;
  p.n_tiles = 1;
  p.m_tiles = (int)((M + kBM - 1) / kBM);
  p.C = static_cast<__nv_bfloat16*>(C);
  p.part = part;
  p.gx = static_cast<const __nv_bfloat16*>(x);
  p.gh = h;
  p.gw = w;
  p.gc = cin;
  p.gho = ho;
  p.gwo = wo;
  p.gk = k;
  p.gs = stride;
  p.gp = pad;
  CUtensorMap mb, mc;
  if (!make_map(&mb, wk, N, K, N, 32, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_map(&mc, C, M, N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  int per = num_sms();
  if (per > p.m_tiles) per = p.m_tiles;
  if (part_rows) *part_rows = per * 4 * 2;  // BN 64: two epilogue tile groups
  if (part != nullptr) return dispatch_stages<64, false, 1, false, 32, true>(mb, mb, mc, mc, p, per, s);
  return dispatch_stages<64, false, 0, false, 32, true>(mb, mb, mc, mc, p, per, s);
}

cudaError_t conv1x1_bn_res_fprop(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                                 const float* pinvstd, const void* pg, const void* pb, const void* res, float* part,
                                 int* part_rows, cudaStream_t s) {
  if (res == nullptr) return cudaErrorInvalidValue;
  return conv1x1_impl(A, B, C, M, N, K, pmean, pinvstd, pg, pb, part, part_rows, nullptr, nullptr, nullptr, nullptr,
                      nullptr, res, s);
}

cudaError_t conv1x1_bn_dgrad(const void* dY, const void* Wt, void* dX, int64_t M, int N, int K, const void* x,
                             const float* mean, const float* invstd, const void* g, const void* b, float* part,
                             int* part_rows, cudaStream_t s) {
  if (x == nullptr || mean == nullptr || invstd == nullptr || g == nullptr || b == nullptr)
    return cudaErrorInvalidValue;
  return conv1x1_impl(dY, Wt, dX, M, N, K, nullptr, nullptr, nullptr, nullptr, part, part_rows, x, mean, invstd, g,
                      b, nullptr, s);
}

cudaError_t bn_partials_bwd_finalize(const float* part, int part_rows, int N, int64_t M, const float* mean,
                                     const float* invstd, const void* g, float* dgamma, float* dbeta, float* coef,
                                     cudaStream_t s) {
  partials_bwd_finalize_kernel<<<(N + 31) / 32, 1024, 0, s>>>(part, part_rows, N, M, mean, invstd,
                                                              static_cast<const __nv_bfloat16*>(g), dgamma, dbeta,
                                                              coef);
  return cudaGetLastError();
}

cudaError_t bn_partials_finalize(const float* part, int part_rows, int N, int64_t M, float eps, float* mean,
                                 float* invstd, cudaStream_t s) {
  partials_finalize_kernel<<<(N + 31) / 32, 1024, 0, s>>>(part, part_rows, N, M, eps, mean, invstd);
  return cudaGetLastError();
}

cudaError_t conv_im2col_fprop(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int ho, int wo,
                              int k, int stride, int pad, int N, const float* pmean, const float* pinvstd,
                              const void* pg, const void* pb, float* part, int* part_rows, const void* bx,
                              const float* bmean, const float* binvstd, const void* bg, const void* bb,
                              cudaStream_t s) {
  const int64_t M = (int64_t)n * ho * wo;
  const int K = k * k * cin;
  const bool bwd = bx != nullptr, pro = pmean != nullptr, st = part != nullptr;
  // 3x3 / stride 1 / pad 1 forward at 64/128 output channels (cin % 64 == 0)
  // or 16/32 -> 16/32 channels: halo windows (each input pixel loaded and
  // transformed once for all nine taps; halo_sm100.cu)
  if (!bwd && k == 3 && stride == 1 && pad == 1 && ho == h && wo == w && conv3x3_halo_supported(h, w, cin, N, pro))
    return conv3x3_halo_fprop(x, wk, C, n, h, w, cin, N, pmean, pinvstd, pg, pb, part, part_rows, s);
  if (M <= 0 || cin % kBK != 0 || k < 1 || k > 7 || stride < 1 || stride > 2 || (pro && cin > kMaxProK))
    return cudaErrorInvalidValue;
  // the im2col traversal visits exactly these output rows / columns
  if (ho != (h + 2 * pad - k) / stride + 1 || wo != (w + 2 * pad - k) / stride + 1) return cudaErrorInvalidValue;
  if (bwd ? (N != 64 && N != 128 && N % 128 != 0) || pro || part == nullptr
          : (N != 64 && N != 128 && N % 256 != 0))
    return cudaErrorInvalidValue;
  if (M > 0x7fffffffLL) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(wk) | reinterpret_cast<uintptr_t>(C)) & 15)
    return cudaErrorMisalignedAddress;
  const int BN = bwd ? (N < 128 ? N : 128) : (N <= 256 ? N : 256);
  Params p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.BN = BN;
  p.n_tiles = N / BN;
  p.m_tiles = (int)((M + kBM - 1) / kBM);
  p.C = static_cast<__nv_bfloat16*>(C);
  p.part = part;
  p.pmean = pmean;
  p.pinvstd = pinvstd;
  p.pg = static_cast<const __nv_bfloat16*>(pg);
  p.pb = static_cast<const __nv_bfloat16*>(pb);
  p.bx = static_cast<const __nv_bfloat16*>(bx);
  p.bmean = bmean;
  p.binvstd = binvstd;
  p.bg = static_cast<const __nv_bfloat16*>(bg);
  p.bb = static_cast<const __nv_bfloat16*>(bb);
  p.gh = h;
  p.gw = w;
  p.gc = cin;
  p.gho = ho;
  p.gwo = wo;
  p.gk = k;
  p.gs = stride;
  p.gp = pad;
  const bool pair = pair_enabled();
  if (pair) p.m_tiles = (int)((M + 2 * kBM - 1) / (2 * kBM));
  CUtensorMap ma, mb, mc, mx;
  if (!make_im2col_map(&ma, x, n, h, w, cin, k, stride, pad, kBM) ||
      !make_map(&mb, wk, N, K, pair ? BN / 2 : BN, kBK, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map(&mc, C, M, N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
    return cudaErrorInvalidValue;
  if (bwd) {
    if (!make_map(&mx, bx, M, N, kBM, BN, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
  } else {
    mx = mc;
  }
  int per = (pair ? num_sms() / 2 : num_sms()) / p.n_tiles;
  if (per < 1) per = 1;
  if (per > p.m_tiles) per = p.m_tiles;
  const int grid = per * p.n_tiles * (pair ? 2 : 1);
  const int epi_groups = 4 / (BN >= 128 ? 4 : BN / 32);
  if (part_rows) *part_rows = per * (pair ? 2 : 1) * 4 * epi_groups;
  if (bwd) {
    if (BN == 64) return dispatch_im2col<64, false, 2>(ma, mb, mc, mx, p, grid, pair, s);
    return dispatch_im2col<128, false, 2>(ma, mb, mc, mx, p, grid, pair, s);
  }
#define KRT_IM2COL_BN(BNV)                                                            \
  if (BN == BNV) {                                                                    \
    if (pro && st) return dispatch_im2col<BNV, true, 1>(ma, mb, mc, mx, p, grid, pair, s); \
    if (pro) return dispatch_im2col<BNV, true, 0>(ma, mb, mc, mx, p, grid, pair, s);       \
    if (st) return dispatch_im2col<BNV, false, 1>(ma, mb, mc, mx, p, grid, pair, s);       \
    return dispatch_im2col<BNV, false, 0>(ma, mb, mc, mx, p, grid, pair, s);              \
  }
  KRT_IM2COL_BN(64)
  KRT_IM2COL_BN(128)
  KRT_IM2COL_BN(256)
#undef KRT_IM2COL_BN
  return cudaErrorInvalidValue;
}

}  // namespace krt
