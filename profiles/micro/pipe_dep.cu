// Microbenchmark: the GEMM main loop without epilogue — pair TMA loads (leader barrier counts
// both CTAs' bytes) -> tcgen05 mxf4 MMAs (N=192) -> commit releases the stage to both CTAs.
// Cycles per MMA vs the number of ring stages show how much latency the ring must cover.
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace bitmm_dev;

constexpr int N = 192, A_BYTES = 16384, B_BYTES = 12288, STAGE = A_BYTES + B_BYTES;
constexpr int MAXST = 7, SMEM = MAXST * STAGE + 2048;

// TILES: every 16 stages the MMA switches between two accumulators (waiting for the epilogue
// warps 2..5 of both CTAs to release it) and commits the finished one, like the GEMM.
// WALK: like the GEMM's persistent schedule, the rows change every 16 stages (tile t of this
// pair = unit + t * num_units over a 32 x 42 tile grid of 8192-row operands).
// SPLIT: all A stages, then all B stages (the GEMM's smem layout) instead of A|B per stage.
template <int STAGES, bool TILES = false, int SFCOL = 448, bool WALK = false, bool SPLIT = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    k_pipe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int iters,
           unsigned long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + MAXST * STAGE);
  uint64_t* empty = full + MAXST;
  uint64_t* done = empty + MAXST;
  uint64_t* tfull = done + 1;
  uint64_t* tempty = tfull + 2;
  uint32_t* slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 256); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(slot, 512);
  tc_fence_before(); cluster_sync(); tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp >= 2) {
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    tmem_st_32x32b_x32_fill(tmem + lane_off + SFCOL, 0x7F7F7F7Fu);
    tmem_st_32x32b_x32_fill(tmem + lane_off + SFCOL + 32, 0x7F7F7F7Fu);
    tmem_st_wait();
  }
  tc_fence_before(); cluster_sync(); tc_fence_after();
  const long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    int st = 0; uint32_t ph = 0;
    int arow = (blockIdx.x * 128) % 8192, brow = (blockIdx.x * 96) % 8064;
    for (int it = 0; it < iters; ++it) {
      if (WALK && (it % 16) == 0) {
        const int tile = static_cast<int>(blockIdx.x >> 1) + (it / 16) * static_cast<int>(gridDim.x >> 1);
        const int mb = tile % 32, nb = (tile / 32) % 42;
        arow = mb * 256 + static_cast<int>(rank) * 128;
        brow = 8192 + nb * 192 + static_cast<int>(rank) * 96;
      }
      mbar_wait(&empty[st], ph ^ 1u);
      if (rank == 0) mbar_arrive_expect_tx(&full[st], 2 * STAGE);
      uint8_t* da = SPLIT ? smem + st * A_BYTES : smem + st * STAGE;
      uint8_t* db = SPLIT ? smem + STAGES * A_BYTES + st * B_BYTES : smem + st * STAGE + A_BYTES;
      tma_load_2d_pair(da, &ma, &full[st], (it % 16) * 128, arow);
      tma_load_2d_pair(db, &mb, &full[st], (it % 16) * 128, brow);
      if (++st == STAGES) { st = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && rank == 0) {
    const uint64_t d0 = sw128_kmajor_desc(smem_u32(smem));
    constexpr uint32_t idesc = make_idesc_mxf4(256, N);
    int st = 0; uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      const int tile = it / 16, acc = TILES ? (tile & 1) : 0;
      if (TILES && (it % 16) == 0) {
        mbar_wait(&tempty[acc], ((tile >> 1) & 1) ^ 1u);
        tc_fence_after();
      }
      mbar_wait(&full[st], ph);
      tc_fence_after();
      const uint64_t ad = SPLIT ? d0 + static_cast<uint64_t>((st * A_BYTES) >> 4)
                                : d0 + static_cast<uint64_t>((st * STAGE) >> 4);
      const uint64_t bd = SPLIT ? d0 + static_cast<uint64_t>((STAGES * A_BYTES + st * B_BYTES) >> 4)
                                : ad + (A_BYTES >> 4);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_pair_elect<2>(tmem + acc * 192, ad + 2 * k, bd + 2 * k, idesc, (it % 16) | k, tmem + SFCOL, tmem + SFCOL + 32);
      mma_commit_pair_elect(&empty[st], 0x3);
      if (TILES && (it % 16) == 15) mma_commit_pair_elect(&tfull[acc], 0x3);
      if (++st == STAGES) { st = 0; ph ^= 1u; }
    }
    mma_commit_pair_elect(done, 0x1);
    if (lane == 0) {
      mbar_wait(done, 0);
      atomicAdd(cycles, static_cast<unsigned long long>(clock64() - t0));
    }
  }
  if (TILES && warp >= 2) {  // epilogue warps: wait for each accumulator, release it
    for (int tile = 0; tile < iters / 16; ++tile) {
      const int acc = tile & 1;
      mbar_wait(&tfull[acc], (tile >> 1) & 1);
      tc_fence_after();
      tc_fence_before();
      mbar_arrive_cluster(smem_u32(&tempty[acc]) & kPeerBitMask);
    }
  }
  tc_fence_before(); cluster_sync();
  if (warp == 1) { tc_fence_after(); tmem_dealloc_pair(tmem, 512); }
}

// Rewrites the operand buffer on the device right before the timed kernel (like the unpack).
__global__ void rewrite(uint4* buf, size_t n16) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    uint4 v = buf[i];
    buf[i] = make_uint4(v.y, v.x, v.w, v.z);  // still +-1 nibbles
  }
}
static uint8_t* g_buf = nullptr;
static size_t g_bytes = 0;
static bool g_rewrite = false;
static int g_iters = 65536;

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int STAGES, bool TILES = false, int SFCOL = 448, bool WALK = false, bool SPLIT = false>
int run(const CUtensorMap& ma, const CUtensorMap& mb, unsigned long long* d, int clusters) {
  if (cudaFuncSetAttribute(k_pipe<STAGES, TILES, SFCOL, WALK, SPLIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess) return 5;
  const int iters = g_iters;
  cudaMemset(d, 0, 8);
  k_pipe<STAGES, TILES, SFCOL, WALK, SPLIT><<<2 * clusters, 192, SMEM>>>(ma, mb, 64, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("warmup error %s\n", cudaGetErrorString(e)); return 6; }
  cudaMemset(d, 0, 8);
  if (g_rewrite) rewrite<<<1184, 256>>>(reinterpret_cast<uint4*>(g_buf), g_bytes / 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_pipe<STAGES, TILES, SFCOL, WALK, SPLIT><<<2 * clusters, 192, SMEM>>>(ma, mb, iters, d);
  cudaEventRecord(e1);
  e = cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double cyc_per_cluster = double(cyc) / clusters;
  printf("iters=%d rewrite=%d split=%d walk=%d sf=%d tiles=%d stages=%d clusters=%2d: %.1f cycles per MMA (ideal 96), %.0f TMAC/s wall, clock %.0f MHz %s\n", g_iters, int(g_rewrite), int(SPLIT), int(WALK), SFCOL, int(TILES), STAGES,
         clusters, cyc_per_cluster / (iters * 4.0), double(clusters) * iters * 4 * 256.0 * N * 64 / (ms * 1e-3) / 1e12,
         cyc_per_cluster / (ms * 1e3), cudaGetErrorString(e));
  return 0;
}

static void fill(uint8_t* buf, size_t n, const unsigned char* codes) {
  unsigned char* h = static_cast<unsigned char*>(malloc(n));
  unsigned long long x = 88172645463325252ull;
  for (size_t i = 0; i < n; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = static_cast<unsigned char>(codes[x & 7] | (codes[(x >> 3) & 7] << 4));
  }
  cudaMemcpy(buf, h, n, cudaMemcpyHostToDevice);
  free(h);
}

int main() {
  const int rows = 16384, cols = 2048;  // A rows [0,8192), B rows [8192,16384) in the walk
  uint8_t* buf = nullptr;
  if (cudaMalloc(&buf, size_t(rows) * cols) != cudaSuccess) return 1;

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
  unsigned long long* d = nullptr;
  cudaMalloc(&d, 8);
  const unsigned char pm1[8] = {0x2, 0xA, 0x2, 0xA, 0x2, 0xA, 0x2, 0xA};   // random +-1
  const unsigned char b01[8] = {0x0, 0x2, 0x0, 0x2, 0x0, 0x2, 0x0, 0x2};   // random {0,1}
  const unsigned char lv[8] = {0x0, 0x2, 0x4, 0x5, 0x0, 0x2, 0x4, 0x5};    // random levels 0..3
  const unsigned char cst[8] = {0x2, 0x2, 0x2, 0x2, 0x2, 0x2, 0x2, 0x2};   // constant 1.0
  const unsigned char* pats[4] = {pm1, b01, lv, cst};
  const char* names[4] = {"+-1", "{0,1}", "levels", "const"};
  fill(buf, size_t(rows) * cols, pm1);
  g_buf = buf;
  g_bytes = size_t(rows) * cols;
  for (int it : {65536, 304}) {
    g_iters = it;
    for (int rep = 0; rep < 2; ++rep) {
      g_rewrite = false;
      run<7, true, 448, true, true>(ma, mb, d, 74);
      g_rewrite = true;
      run<7, true, 448, true, true>(ma, mb, d, 74);
    }
  }
  return 0;
}
