// Microbenchmark: back-to-back tcgen05.mma (kind::f16, M = 128, both operands
// in shared memory, SW128 K-major) at N = 64 / 128 / 256, one CTA per SM, no
// global traffic: cycles per MMA instruction, with a commit every 4 MMAs (one
// 64-wide k-block, as the conv kernels do) or only at the end.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2008_11421_b200/csrc mma_rate.cu -o mma_rate
#include <cstdio>

#include "sm100_common.cuh"

using namespace krt::sm100;

template <int N, bool COMMIT, int NACC, int AOFF = 0, int SUB = 1>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* a = smem;                 // 128 x 64 bf16
  uint8_t* b = smem + 512 * 128;     // N x 64 bf16 (A region: 512 rows)
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (512 + N) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(&tbase, N * NACC >= 32 ? N * NACC : 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && lane == 0) {
    constexpr uint32_t idesc = instr_desc(N);
    const uint32_t a0 = smem_u32(a), b0 = smem_u32(b);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      // AOFF: A starts AOFF rows into the buffer, moving by (it % 9) rows (the halo taps)
      const uint32_t ar = AOFF ? (uint32_t)(AOFF + (it % 9) * 7) * 128 : 0u;
#pragma unroll
      for (int u = 0; u < SUB; ++u)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tbase + ((it * SUB + u) % NACC) * N, kmajor_desc<64>(a0 + ar + u * 128 * 128 + k * 32),
                    kmajor_desc<64>(b0 + k * 32), idesc, (it | k) != 0);
      if (COMMIT) umma_commit(&bar);
    }
    umma_commit(&bar);
    mbar_wait(&bar, COMMIT ? (uint32_t)(iters & 1) : 0u);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, N * NACC >= 32 ? N * NACC : 32);
}

template <int N, bool COMMIT, int NACC, int AOFF = 0, int SUB = 1>
void run(int sms) {
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = (512 + N) * 128 + 1024;
  auto k = mma_kernel<N, COMMIT, NACC, AOFF, SUB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  k<<<sms, 128, smem>>>(16, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double mmas = 4.0 * iters * SUB;
  const double tflops = 2.0 * 128 * N * 16 * mmas * sms / (ms * 1e-3) / 1e12;
  printf("N=%3d aoff=%d sub=%d commit_per_kblock=%d acc=%d: %.1f cycles/MMA (floor %d), %.0f TFLOP/s over %d SMs  %s\n", N, AOFF, SUB, COMMIT,
         NACC, cyc / mmas, 128 * N / 256, tflops, sms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, true, 1>(sms);
  run<64, true, 1, 3>(sms);
  run<64, true, 4, 3, 2>(sms);
  run<64, true, 4, 0, 2>(sms);
  run<128, true, 1>(sms);
  run<128, true, 1, 3>(sms);
  run<128, true, 4, 3, 2>(sms);
  run<128, true, 4, 0, 2>(sms);
  run<256, true, 1>(sms);
  run<256, true, 1, 3>(sms);
  return 0;
}
