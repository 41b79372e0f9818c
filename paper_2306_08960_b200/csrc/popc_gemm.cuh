// CUDA-core LOP3 + POPC 1/1 GEMM on the packed bits, kept as the measured
// alternative to the tensor-core path (BASELINE.json north star: the tensor
// path is used only if it beats the popc path). It is the direct GPU analogue
// of the reference's xor_popcount_many (kernels_avx512.cpp:31-44 /
// kernels_scalar.cpp:19-27): C[r][c] = K - 2 * sum_w popc(a_r[w] ^ b_c[w]).
//
// Tile 128 x 128 outputs per CTA of 256 threads, 8 x 8 register micro-tile per
// thread, K staged through shared memory 16 words (512 bits) at a time, double
// buffered. Zero padding makes the xor of padding words vanish, so only
// ceil(K/32) words are walked.
#pragma once

#include <cstdint>

namespace bitmm_dev {

constexpr int PC_BM = 128, PC_BN = 128, PC_BKW = 16, PC_THREADS = 256;

template <bool F32OUT>
__global__ void __launch_bounds__(PC_THREADS)
    popc_gemm_1x1(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B, int M, int N,
                  int K, int wpr32, float scale, int32_t* __restrict__ out_i32,
                  float* __restrict__ out_f32, long long ldc) {
  __shared__ uint32_t sa[2][PC_BKW][PC_BM];
  __shared__ uint32_t sb[2][PC_BKW][PC_BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * PC_BM, n0 = blockIdx.x * PC_BN;
  const int nwords = (K + 31) / 32;
  const int nsteps = (nwords + PC_BKW - 1) / PC_BKW;

  uint32_t acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0;

  // each thread stages 8 words of A and 8 of B per step: idx = tid + 256*q
  uint32_t ra[8], rb[8];
  auto gload = [&](int step) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + PC_THREADS * q;
      const int row = idx / PC_BKW, w = idx % PC_BKW;
      const int kw = step * PC_BKW + w;
      const int ar = m0 + row, br = n0 + row;
      ra[q] = (ar < M && kw < nwords) ? A[static_cast<long long>(ar) * wpr32 + kw] : 0u;
      rb[q] = (br < N && kw < nwords) ? B[static_cast<long long>(br) * wpr32 + kw] : 0u;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int idx = tid + PC_THREADS * q;
      const int row = idx / PC_BKW, w = idx % PC_BKW;
      sa[buf][w][row] = ra[q];
      sb[buf][w][row] = rb[q];
    }
  };

  gload(0);
  sstore(0);
  __syncthreads();
  for (int step = 0; step < nsteps; ++step) {
    const int buf = step & 1;
    if (step + 1 < nsteps) gload(step + 1);
#pragma unroll
    for (int w = 0; w < PC_BKW; ++w) {
      uint32_t a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = sa[buf][w][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = sb[buf][w][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] += __popc(a[i] ^ b[j]);
    }
    if (step + 1 < nsteps) {
      sstore(buf ^ 1);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = m0 + ty + 16 * i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = n0 + tx + 16 * j;
      if (c >= N) continue;
      const int units = K - 2 * static_cast<int>(acc[i][j]);
      if (F32OUT)
        out_f32[static_cast<long long>(r) * ldc + c] = __fmul_rn(scale, static_cast<float>(units));
      else
        out_i32[static_cast<long long>(r) * ldc + c] = units;
    }
  }
}

// Plain CSR x dense product, standalone spmm_csr (kernels.cpp:334-352): one warp
// per output row segment of 128 columns, nonzeros walked in col_idx order,
// separate fp32 multiply and add exactly as the reference row loop. accumulate: C += R.B
// (one more fp32 add per cell, the layer's bin_part + res_part).
__global__ void spmm_csr_kernel(long long rows, const unsigned long long* __restrict__ row_ptr,
                                const unsigned long long* __restrict__ col_idx,
                                const float* __restrict__ vals, const float* __restrict__ b,
                                long long ldb, int N, float* __restrict__ c, long long ldc,
                                int accumulate) {
  const long long warp_global = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int segs = (N + 127) / 128;
  const long long r = warp_global / segs;
  if (r >= rows) return;
  const int col0 = static_cast<int>(warp_global % segs) * 128;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const unsigned long long i0 = row_ptr[r], i1 = row_ptr[r + 1];
  for (unsigned long long i = i0; i < i1; ++i) {
    const float v = vals[i];
    const float* br = b + static_cast<long long>(col_idx[i]) * ldb;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int cc = col0 + lane + 32 * e;
      if (cc < N) acc[e] = __fadd_rn(acc[e], __fmul_rn(v, br[cc]));
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int cc = col0 + lane + 32 * e;
    if (cc < N) c[r * ldc + cc] = accumulate ? __fadd_rn(c[r * ldc + cc], acc[e]) : acc[e];
  }
}

}  // namespace bitmm_dev
