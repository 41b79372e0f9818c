// Two concurrent launches of the library's tc_gemm_kernel over one 8192x8192x4096 problem:
// four-CTA clusters with A multicast (MC = 2) on the N-blocks [0, nA) -- these clusters only fit
// on 132 of the 148 SMs -- and CTA pairs (MC = 1) on the remaining N-blocks, meant for the 16
// SMs the four-CTA clusters leave free. Measures whether the two overlap and beat one launch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../../paper_2306_08960_b200/csrc hybrid.cu -o hybrid -lcuda
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include "tc_gemm.cuh"
using namespace bitmm_dev;

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
constexpr int M = 8192, N = 8192, K = 4096, RB = K / 2, BN = 192;
using S = TcShape<true, BN>;

// Group over output columns [nb0 * BN, nb0 * BN + ncols) through offset B / C base pointers.
static void make_group(Enc enc, TcGroup<1>& g, int mc, uint8_t* a, uint8_t* b, int32_t* c, int nb0, int ncols) {
  memset(&g, 0, sizeof(g));
  cuuint64_t da[2] = {cuuint64_t(RB), cuuint64_t(M)}, db[2] = {cuuint64_t(RB), cuuint64_t(ncols)};
  cuuint64_t st[1] = {cuuint64_t(RB)};
  cuuint32_t boxa[2] = {128, cuuint32_t(S::A_ROWS / mc)}, boxb[2] = {128, S::B_ROWS}, es[2] = {1, 1};
  enc(&g.a[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, a, da, st, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&g.b[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, b + size_t(nb0) * BN * RB, db, st, boxb, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t cd[2] = {cuuint64_t(ncols), cuuint64_t(M)};
  cuuint64_t cs[1] = {cuuint64_t(N) * 4};
  cuuint32_t cb[2] = {32, 32};
  enc(&g.c[0], CU_TENSOR_MAP_DATA_TYPE_INT32, 2, c + size_t(nb0) * BN, cd, cs, cb, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TcParams& p = g.prob[0];
  p.M = M; p.N = ncols; p.num_kb = RB / 128; p.shift = 0; p.scale = 1.0f; p.out_i32 = c + size_t(nb0) * BN;
  p.ldc = N; p.small_acc = 1; p.shift_mul = 1.0f; p.tma_store = 1; p.epi = 0;
  p.num_m_blocks = M / 256; p.num_n_blocks = (ncols + BN - 1) / BN;
  p.num_tiles = p.num_m_blocks * ((p.num_n_blocks + mc - 1) / mc);
  p.group_m = TC_GROUP_M;
  g.count = 1; g.tile_begin[0] = 0; g.tile_begin[1] = p.num_tiles;
}

template <int MC>
static cudaError_t launch(const TcGroup<1>& g, int grid, cudaStream_t s) {
  auto k = tc_gemm_kernel<Kind::F4, Epi::I32, BN, 1, MC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(TC_THREADS); cfg.dynamicSmemBytes = S::SMEM; cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2 * MC; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, g);
}

int main(int argc, char** argv) {
  const int nA = argc > 1 ? atoi(argv[1]) : 38;  // N-blocks for the four-CTA clusters (even)
  uint8_t *a, *b; int32_t* c;
  cudaMalloc(&a, size_t(M) * RB); cudaMalloc(&b, size_t(N) * RB); cudaMalloc(&c, size_t(M) * N * 4);
  {
    unsigned char* h = static_cast<unsigned char*>(malloc(size_t(M) * RB));
    unsigned long long x = 88172645463325252ull;
    const unsigned char codes[2] = {0x2, 0xA};
    for (size_t i = 0; i < size_t(M) * RB; ++i) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      h[i] = static_cast<unsigned char>(codes[x & 1] | (codes[(x >> 1) & 1] << 4));
    }
    cudaMemcpy(a, h, size_t(M) * RB, cudaMemcpyHostToDevice);
    cudaMemcpy(b, h, size_t(N) * RB, cudaMemcpyHostToDevice);
    free(h);
  }
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return 2;
  Enc enc = reinterpret_cast<Enc>(fn);
  const int nnb = (N + BN - 1) / BN;
  TcGroup<1> gA, gB, gAll;
  make_group(enc, gA, 2, a, b, c, 0, nA * BN);
  make_group(enc, gB, 1, a, b, c, nA, N - nA * BN);
  make_group(enc, gAll, 1, a, b, c, 0, N);
  int clA = 0;
  {
    auto k = tc_gemm_kernel<Kind::F4, Epi::I32, BN, 1, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(TC_THREADS); cfg.dynamicSmemBytes = S::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaOccupancyMaxActiveClusters(&clA, k, &cfg);
  }
  const int gridA = 4 * clA, gridB = 148 - gridA;
  printf("N-blocks %d: %d to four-CTA clusters (grid %d), %d to pairs (grid %d)\n", nnb, nA, gridA, nnb - nA, gridB);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1, eB, eS;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&eB); cudaEventCreate(&eS);
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0, s1);
    launch<1>(gAll, 148, s1);
    cudaEventRecord(e1, s1);
    cudaStreamSynchronize(s1);
    float ms1; cudaEventElapsedTime(&ms1, e0, e1);
    cudaEventRecord(e0, s1);
    cudaStreamWaitEvent(s2, e0, 0);
    cudaError_t ea = launch<2>(gA, gridA, s1);
    cudaError_t eb = launch<1>(gB, gridB, s2);
    cudaEventRecord(eB, s2);
    cudaStreamWaitEvent(s1, eB, 0);
    cudaEventRecord(e1, s1);
    cudaError_t es = cudaDeviceSynchronize();
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    printf("one launch %.1f us | hybrid %.1f us (%s %s %s)\n", ms1 * 1e3, ms2 * 1e3, cudaGetErrorString(ea),
           cudaGetErrorString(eb), cudaGetErrorString(es));
  }
  return 0;
}
