// Microbenchmark: tcgen05 mxf4 MMAs (cta_group::2, N=192) issued back to back over a 7-stage
// smem ring while (optionally) a TMA producer streams 28 KB per stage into the same ring with
// no dependency on the MMAs. Shows how much TMA smem writes slow the MMA's operand reads.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace bitmm_dev;

constexpr int STAGES = 7, N = 192;
constexpr int A_BYTES = 16384, B_BYTES = 12288, STAGE = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE + 2048;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_mma_tma(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int iters,
              int with_tma, unsigned long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(slot, 512);
  tc_fence_before(); cluster_sync(); tc_fence_after();
  const uint32_t tmem = *slot;
  {
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    tmem_st_32x32b_x32_fill(tmem + lane_off + 448, 0x7F7F7F7Fu);
    tmem_st_32x32b_x32_fill(tmem + lane_off + 480, 0x7F7F7F7Fu);
    tmem_st_wait();
  }
  tc_fence_before(); cluster_sync(); tc_fence_after();
  const long long t0 = clock64();
  const int loads = with_tma ? iters : 0;
  if (warp == 0 && lane == 0) {  // TMA producer (own CTA only)
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < loads; ++it) {
      mbar_wait(&empty[st], ph ^ 1u);
      mbar_arrive_expect_tx(&full[st], STAGE);
      tma_load_2d(smem + st * STAGE, &ma, &full[st], (it % 16) * 128, (blockIdx.x * 128) % 8192);
      tma_load_2d(smem + st * STAGE + A_BYTES, &mb, &full[st], (it % 16) * 128, (blockIdx.x * 96) % 8192);
      if (++st == STAGES) { st = 0; ph ^= 1u; }
    }
  } else if (warp == 3 && lane == 0) {  // time until the last load has landed
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < loads; ++it) {
      if (it == loads - 1) mbar_wait(&full[st], ph);
      if (++st == STAGES) { st = 0; ph ^= 1u; }
    }
    (void)0;
  } else if (warp == 2 && lane == 0) {  // consumer of the loads (releases stages at once)
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < loads; ++it) {
      mbar_wait(&full[st], ph);
      mbar_arrive(&empty[st]);
      if (++st == STAGES) { st = 0; ph ^= 1u; }
    }
    if (loads) atomicAdd(cycles + 1, static_cast<unsigned long long>(clock64() - t0));
  } else if (warp == 1 && rank == 0) {  // MMAs over the ring, no dependency on the loads
    const uint64_t d0 = sw128_kmajor_desc(smem_u32(smem));
    constexpr uint32_t idesc = make_idesc_mxf4(256, N);
    int st = 0;
    for (int it = 0; it < iters; ++it) {
      const uint64_t ad = d0 + static_cast<uint64_t>((st * STAGE) >> 4);
      const uint64_t bd = ad + (A_BYTES >> 4);
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_pair_elect<2>(tmem, ad + 2 * k, bd + 2 * k, idesc, 1, tmem + 448, tmem + 480);
      if (++st == STAGES) st = 0;
    }
    mma_commit_pair_elect(done, 0x1);
    if (lane == 0) {
      mbar_wait(done, 0);
      atomicAdd(cycles, static_cast<unsigned long long>(clock64() - t0));
    }
  }
  tc_fence_before(); cluster_sync();
  if (warp == 1) { tc_fence_after(); tmem_dealloc_pair(tmem, 512); }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int rows = 8192, cols = 2048;  // 16 MiB source (L2-resident)
  uint8_t* buf = nullptr;
  if (cudaMalloc(&buf, size_t(rows) * cols) != cudaSuccess) return 1;
  cudaMemset(buf, 0x22, size_t(rows) * cols);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return 2;
  Enc enc = reinterpret_cast<Enc>(fn);
  CUtensorMap ma, mb;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols)};
  cuuint32_t boxa[2] = {128, 128}, boxb[2] = {128, 96}, es[2] = {1, 1};
  if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) return 3;
  if (enc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) return 4;
  if (cudaFuncSetAttribute(k_mma_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess) return 5;
  unsigned long long* d = nullptr;
  cudaMalloc(&d, 16);
  for (int clusters : {74, 9}) {
    for (int with_tma : {0, 1}) {
      const int iters = 4096;
      cudaMemset(d, 0, 16);
      k_mma_tma<<<2 * clusters, 128, SMEM>>>(ma, mb, 64, with_tma, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("warmup error %s\n", cudaGetErrorString(e)); return 6; }
      cudaMemset(d, 0, 16);
      k_mma_tma<<<2 * clusters, 128, SMEM>>>(ma, mb, iters, with_tma, d);
      e = cudaDeviceSynchronize();
      unsigned long long cyc[2] = {0, 0};
      cudaMemcpy(cyc, d, 16, cudaMemcpyDeviceToHost);
      printf("clusters=%2d tma=%d: %.1f cycles per MMA (ideal 96); loads: %.1f B/cycle per SM %s\n", clusters,
             with_tma, double(cyc[0]) / clusters / (iters * 4.0),
             cyc[1] ? double(STAGE) * iters / (double(cyc[1]) / (2 * clusters)) : 0.0, cudaGetErrorString(e));
    }
  }
  return 0;
}
