// Measured denominator of the FP4 roofline: tcgen05.mma.cta_group::2.kind::mxf4 (N = 192, the
// library's tile) issued back to back on every SM pair with RANDOM +-1 e2m1 operands (the
// bitwise GEMMs' data; operand toggling sets the power draw and with it the clock), first as a
// single burst launch, then launched back to back for ~4 s so the power limiter settles.
// Prints JSON: TMAC/s and TFLOP/s (2 ops per MAC), burst and sustained, plus the SM clock the
// MMA loop saw (clock64 cycles / elapsed time).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2306_08960_b200/csrc mxf4_sustained.cu -o mxf4_sustained
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace bitmm_dev;

constexpr int N = 192, STAGES = 7, STAGE = 16384 + N / 2 * 128;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_loop(int iters, unsigned long long seed, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  // random +-1 e2m1 nibbles (0x2 / 0xA), as the sign expansion writes them
  unsigned long long x = seed ^ (blockIdx.x * 0x9E3779B97F4A7C15ull) ^ threadIdx.x;
  for (int i = threadIdx.x; i < STAGES * STAGE / 4; i += blockDim.x) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    reinterpret_cast<uint32_t*>(smem)[i] = (static_cast<uint32_t>(x) & 0x88888888u) | 0x22222222u;
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 1) tmem_alloc_pair(&tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  tmem_st_32x32b_x32_fill(tmem + lane_off + 448, 0x7F7F7F7Fu);
  tmem_st_32x32b_x32_fill(tmem + lane_off + 480, 0x7F7F7F7Fu);
  tmem_st_wait();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  fence_proxy_async_smem();
  unsigned long long t0 = clock64();
  if (warp == 0 && rank == 0) {
    constexpr uint32_t idesc = make_idesc_mxf4(256, N);
    const uint64_t d0 = sw128_kmajor_desc(smem_u32(smem));
    int st = 0;
    for (int it = 0; it < iters; ++it) {
      const uint64_t ad = d0 + static_cast<uint64_t>((st * STAGE) >> 4);
      const uint64_t bd = ad + (16384 >> 4);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_pair_elect<2>(tmem + (it & 1) * N, ad + 2 * k, bd + 2 * k, idesc, 1, tmem + 448, tmem + 480);
      if (++st == STAGES) st = 0;
    }
    mma_commit_pair_elect(&bar, 0x3);
  }
  if (rank == 0 && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    atomicAdd(cycles, clock64() - t0);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) { tc_fence_after(); tmem_dealloc_pair(tmem, 512); }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int clusters = sms / 2;
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, STAGES * STAGE);
  const int iters = 8192;  // 4 MMAs each: ~3 ms per launch at full rate
  const double macs = double(clusters) * iters * 4 * 256.0 * N * 64;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mma_loop<<<2 * clusters, 128, STAGES * STAGE>>>(64, 1, d);  // warm
  cudaDeviceSynchronize();
  // burst: one launch after an idle second
  cudaMemset(d, 0, 8);
  cudaEventRecord(e0);
  mma_loop<<<2 * clusters, 128, STAGES * STAGE>>>(iters, 2, d);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double burst = macs / (ms * 1e-3) / 1e12;
  const double burst_mhz = double(cyc) / clusters / (ms * 1e-3) / 1e6;
  // sustained: back-to-back launches for ~4 s, timed over the last ~2 s
  int launches = 0;
  float tot = 0;
  while (tot < 2000.f) {
    mma_loop<<<2 * clusters, 128, STAGES * STAGE>>>(iters, 3 + launches, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&tot, e0, e1);
    ++launches;
  }
  cudaMemset(d, 0, 8);
  cudaEventRecord(e0);
  const int timed = launches;
  for (int i = 0; i < timed; ++i) mma_loop<<<2 * clusters, 128, STAGES * STAGE>>>(iters, 100 + i, d);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  cudaEventElapsedTime(&ms, e0, e1);
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double sus = macs * timed / (ms * 1e-3) / 1e12;
  const double sus_mhz = double(cyc) / clusters / (ms * 1e-3) / 1e6;
  printf("{\"kind\": \"tcgen05.mma.cta_group::2.kind::mxf4 M256 N%d K64, random +-1 e2m1, unit E8M0 scales\", "
         "\"sms\": %d, \"burst_tmacs\": %.1f, \"burst_tflops\": %.1f, \"burst_clock_mhz\": %.0f, "
         "\"sustained_tmacs\": %.1f, \"sustained_tflops\": %.1f, \"sustained_clock_mhz\": %.0f, "
         "\"sustained_window_ms\": %.0f, \"error\": \"%s\"}\n",
         N, sms, burst, 2 * burst, burst_mhz, sus, 2 * sus, sus_mhz, ms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
