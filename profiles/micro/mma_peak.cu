// Microbenchmark: back-to-back tcgen05.mma (cta_group::2) on resident shared memory, no TMA
// and no barriers in the loop, to measure the instruction's own throughput per shape.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2306_08960_b200/csrc mma_peak.cu -o mma_peak
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace bitmm_dev;

// STAGES > 1: cycle A/B through that many distinct stage buffers (like the GEMM's ring).
template <int KIND_ID, int N, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 1) tmem_alloc_pair(&tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (KIND_ID == 2) {  // unit scale factors
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    tmem_st_32x32b_x32_fill(tmem + lane_off + 448, 0x7F7F7F7Fu);
    tmem_st_32x32b_x32_fill(tmem + lane_off + 480, 0x7F7F7F7Fu);
    tmem_st_wait();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  fence_proxy_async_smem();
  unsigned long long t0 = clock64();
  if (warp == 0 && rank == 0) {
    constexpr uint32_t idesc = KIND_ID == 2 ? make_idesc_mxf4(256, N) : make_idesc(2u, 1u, 1u, 256, N);
    constexpr int STAGE = 16384 + N / 2 * 128;  // A 128 rows + B N/2 rows of 128 B
    const uint64_t d0 = sw128_kmajor_desc(smem_u32(smem));
    int st = 0;
    for (int it = 0; it < iters; ++it) {
      const uint64_t ad = d0 + static_cast<uint64_t>((st * STAGE) >> 4);
      const uint64_t bd = ad + (16384 >> 4);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_pair_elect<KIND_ID>(tmem, ad + 2 * k, bd + 2 * k, idesc, 1, tmem + 448, tmem + 480);
      if (++st == STAGES) st = 0;
    }
    mma_commit_pair_elect(&bar, 0x3);
  }
  if (rank == 0 && threadIdx.x == 0) {
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    atomicAdd(cycles, t1 - t0);
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) { tc_fence_after(); tmem_dealloc_pair(tmem, 512); }
}

template <int KIND_ID, int N, int STAGES = 1>
void run(const char* name, int clusters) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaMemset(d, 0, 8);
  auto k = mma_loop<KIND_ID, N, STAGES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 4096;
  k<<<2 * clusters, 128, 200 * 1024>>>(16, d);
  cudaDeviceSynchronize();
  cudaMemset(d, 0, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<2 * clusters, 128, 200 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double kel = KIND_ID == 2 ? 64 : 32;  // elements per MMA along K
  const double macs = double(clusters) * iters * 4 * 256.0 * N * kel;
  printf("%-6s stages=%d N=%3d clusters=%2d: %.3f ms  %.0f TMAC/s  (%.1f cyc/MMA per pair) %s\n", name,
         STAGES, N, clusters, ms, macs / (ms * 1e-3) / 1e12, double(cyc) / clusters / (iters * 4.0),
         cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  run<2, 192, 1>("mxf4", 74);
  run<2, 192, 7>("mxf4", 74);
  run<2, 256, 6>("mxf4", 74);
  run<0, 256, 1>("i8", 74);
  run<0, 256, 6>("i8", 74);
  return 0;
}
