// The library's tc_gemm_kernel (F4, 1 problem) launched directly on a synthetic e2m1 buffer:
// separates kernel-code effects from the API / unpack environment, and checks 4096 sampled
// outputs against a host dot product. Build options:
//   -DTC_GEMM_STATS   per-CTA wait counters (MMA on tempty / full, epilogue on tfull / busy)
//   -DRK_BN=224       output tile width (TMEM: 2 * BN + 64 scale-factor columns <= 512)
//   -DRK_MC=2         four-CTA clusters, A rows multicast between the two pairs
//   -DRK_NOTMA        epilogue stores through the LSU fallback instead of TMA stores
//   -DRK_ZERO_ONE     {0, +1} operand data (timing only; the sampled check assumes +-1)
#include <cstdio>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include "tc_gemm.cuh"
using namespace bitmm_dev;

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

#ifndef RK_MC
#define RK_MC 1
#endif
#ifndef RK_BN
#define RK_BN 192
#endif
int main() {
  const int M = 8192, N = 8192, K = 4096, RB = K / 2;  // e2m1 row bytes
  uint8_t* a = nullptr; uint8_t* b = nullptr; int32_t* c = nullptr;
  cudaMalloc(&a, size_t(M) * RB); cudaMalloc(&b, size_t(N) * RB); cudaMalloc(&c, size_t(M) * N * 4);
  unsigned char* h = nullptr;
  {
#ifdef RK_ZERO_ONE
    const unsigned char codes[2] = {0x0, 0x2};  // {0, +1}: timing only (the check assumes +-1)
#else
    const unsigned char codes[2] = {0x2, 0xA};
#endif
    h = static_cast<unsigned char*>(malloc(size_t(M) * RB));
    unsigned long long x = 88172645463325252ull;
    for (size_t i = 0; i < size_t(M) * RB; ++i) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      h[i] = static_cast<unsigned char>(codes[x & 1] | (codes[(x >> 1) & 1] << 4));
    }
    cudaMemcpy(a, h, size_t(M) * RB, cudaMemcpyHostToDevice);
    cudaMemcpy(b, h, size_t(N) * RB, cudaMemcpyHostToDevice);
  }
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return 2;
  Enc enc = reinterpret_cast<Enc>(fn);
  using S = TcShape<true, RK_BN>;
  TcGroup<1> g;
  memset(&g, 0, sizeof(g));
  cuuint64_t dims[2] = {cuuint64_t(RB), cuuint64_t(M)};
  cuuint64_t strides[1] = {cuuint64_t(RB)};
  cuuint32_t boxa[2] = {128, S::A_ROWS / RK_MC}, boxb[2] = {128, S::B_ROWS}, es[2] = {1, 1};
  enc(&g.a[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a, dims, strides, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&g.b[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, b, dims, strides, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t cd[2] = {cuuint64_t(N), cuuint64_t(M)};
  cuuint64_t cs[1] = {cuuint64_t(N) * 4};
  cuuint32_t cb[2] = {32, 32};
  enc(&g.c[0], CU_TENSOR_MAP_DATA_TYPE_INT32, 2, c, cd, cs, cb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TcParams& p = g.prob[0];
  p.M = M; p.N = N; p.num_kb = RB / 128; p.shift = 0; p.scale = 1.0f; p.out_i32 = c; p.ldc = N;
  p.small_acc = 1; p.shift_mul = 1.0f; p.tma_store = 1;
#ifdef RK_NOTMA
  p.tma_store = 0;
#endif
 p.epi = 0;
  p.num_m_blocks = M / 256; p.num_n_blocks = (N + RK_BN - 1) / RK_BN; p.num_tiles = p.num_m_blocks * ((p.num_n_blocks + RK_MC - 1) / RK_MC);
  p.group_m = TC_GROUP_M;
  g.count = 1; g.tile_begin[0] = 0; g.tile_begin[1] = p.num_tiles;
  auto k = tc_gemm_kernel<Kind::F4, Epi::I32, RK_BN, 1, RK_MC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(RK_MC == 2 ? 132 : 148); cfg.blockDim = dim3(TC_THREADS); cfg.dynamicSmemBytes = S::SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2 * RK_MC; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  {
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    cfg.gridDim = dim3(ncl * 2 * RK_MC);
    printf("clusters of %d: %d active -> grid %d\n", 2 * RK_MC, ncl, ncl * 2 * RK_MC);
  }
  for (int rep = 0; rep < 6; ++rep) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaError_t err = cudaLaunchKernelEx(&cfg, k, g);
    cudaEventRecord(e1);
    cudaError_t e2 = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("real tc_gemm_kernel 8192x8192x4096 (synthetic +-1 operands): %.1f us  %.0f TMAC/s  %s %s\n", ms * 1e3,
           double(M) * N * K / (ms * 1e-3) / 1e12, cudaGetErrorString(err), cudaGetErrorString(e2));
  }
  {
    int* hc = static_cast<int*>(malloc(size_t(M) * N * 4));
    cudaMemcpy(hc, c, size_t(M) * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    unsigned long long x = 1234567;
    auto val = [](unsigned char nib) { return nib == 0x2 ? 1 : -1; };
    for (int t = 0; t < 4096; ++t) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      const int i = int(x % M), j = int((x >> 20) % N);
      int ref = 0;
      for (int q = 0; q < RB; ++q) {
        const unsigned char u = h[size_t(i) * RB + q], v = h[size_t(j) * RB + q];
        ref += val(u & 15) * val(v & 15) + val(u >> 4) * val(v >> 4);
      }
      if (hc[size_t(i) * N + j] != ref && bad++ < 5) printf("mismatch (%d,%d): %d vs %d\n", i, j, hc[size_t(i) * N + j], ref);
    }
    printf("check: %d / 4096 sampled outputs wrong\n", bad);
  }
#ifdef TC_GEMM_STATS
  static unsigned long long hs[6][160];
  cudaMemcpyFromSymbol(hs, tcg_stats, sizeof(hs));
  double te = 0, fu = 0, tot = 0, tf = 0, busy = 0;
  for (int i = 0; i < (RK_MC == 2 ? 132 : 148); i += 2) { te += hs[0][i]; fu += hs[1][i]; tot += hs[2][i]; }
  for (int i = 0; i < (RK_MC == 2 ? 132 : 148); ++i) { tf += hs[3][i]; busy += hs[4][i]; }
  printf("stats (cycles/CTA): mma total %.0f  tempty-wait %.0f  full-wait %.0f | epi tfull-wait %.0f  busy %.0f\n",
         tot / (RK_MC == 2 ? 66 : 74), te / (RK_MC == 2 ? 66 : 74), fu / (RK_MC == 2 ? 66 : 74), tf / (RK_MC == 2 ? 132 : 148), busy / (RK_MC == 2 ? 132 : 148));
#endif
  return 0;
}
