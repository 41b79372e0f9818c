// APB layer forward (apb.cpp:158-164): C = alpha_r * (sign(bin) . X) + residual . X.
//
// Two kernels, chained with programmatic dependent launch (the GEMM runs first):
//
// 1. spmm_xchunk_kernel — the sparse full-precision residual (spmm_csr,
//    kernels.cpp:334-352). A block stages an X column chunk [K][32] fp32 in shared
//    memory (coalesced, read once from L2), then walks CSR rows: an 8-lane octet owns one
//    output row, lane l owns 4 consecutive columns, nonzeros are broadcast with
//    octet shuffles and accumulated in col_idx order. ACCUM adds R.X onto C (the layer);
//    otherwise it writes R.X (spmm_csr). EXACT = true reproduces the reference's rounding
//    (separate fp32 multiply and add, in order); the layer uses fma for R.X.
//
// 2. apb_gemm_kernel — the binary part on the tensor cores, cta_group::2 (a CTA pair
//    owns 256 output rows x 128 columns). A = sign(bin) as fp16 +-1 (exact); B = X^T
//    scaled per token by 2^e_n and split into two fp16 parts x * 2^e_n = hi + lo
//    (split_x_f16, unpack.cuh; 22 significant bits). One smem stage holds one 64-wide K
//    slice of A and of both B parts, so A is fetched once per slice. The hi products
//    accumulate in one TMEM accumulator and the lo products in a second one: the tensor
//    core's fp32 accumulation truncates small addends against a large running sum, and
//    keeping the magnitudes apart removes that bias (measured: 3e-6 -> ~1e-7 relative at
//    K=768). TMEM holds 2 tiles x 2 accumulators x 128 columns = 512 columns, so the
//    epilogue of tile i overlaps the MMAs of i+1. Two fp16 parts at the f16 rate replace
//    three bf16 parts (the earlier bf16x3 split): 2 MMAs per update instead of 3.
//    Epilogue: C = (alpha_r * (hi + lo)) * 2^-e_n, stored.
//    layer_forward folds the residual into A instead (apb_fold_kernel below): A holds
//    W' = hi + lo, and a fold phase of kpad/64 extra K blocks adds W'_lo . X_hi into the low
//    accumulator, so C = m_r * W' . X comes out of one GEMM with no sparse pass over C.
//    Kernel 1 remains the standalone spmm_csr and the 2-bit layer's residual.
#pragma once

#include "ptx.cuh"
#include "tc_gemm.cuh"
#include "unpack.cuh"

namespace bitmm_dev {

constexpr int SPMM_TOK = 32;       // columns per block (X chunk [K][32] fp32 in smem)
constexpr int SPMM_THREADS = 512;  // 64 octets: an 8-lane octet owns one output row, 4 columns/lane
constexpr int SPMM_QUADS = SPMM_THREADS / 8;  // rows in flight per block

// Dynamic smem: X chunk [K][SPMM_TOK] fp32 plus one zero row (the target of padded
// nonzeros, so they contribute 0 * 0 without a branch), then the row offsets (u32).
inline int spmm_smem_bytes(long long K, int rows_per_split) {
  return static_cast<int>((K + 1) * SPMM_TOK * 4 + (rows_per_split + 1) * 4);
}



// ACCUM (both layers): the GEMM has already stored the binary part in C, and each output
// row becomes C = bin + R.X (apb.cpp:161-162; fp32 add commutes).
template <bool EXACT, bool PDL_CHAIN, bool LEVELS, bool ACCUM = LEVELS>
__global__ void __launch_bounds__(SPMM_THREADS, 2)
    spmm_xchunk_kernel(int rows, int K, int N, const unsigned long long* __restrict__ row_ptr,
                       const unsigned long long* __restrict__ col_idx,
                       const float* __restrict__ vals, const float* __restrict__ X, long long ldx,
                       float* __restrict__ C, long long ldc, int rows_per_split,
                       const SpmmLevels lv) {
  extern __shared__ float xs[];  // [K][SPMM_TOK], then u32 row offsets
  // PDL: wait for the predecessor first (a wait deferred to the end of the kernel can park
  // blocks on SM slots the predecessor still needs), then let the GEMM launch early.
  if (PDL_CHAIN) {
    pdl_wait();
    pdl_launch_dependents();
  }
  unsigned* rps = reinterpret_cast<unsigned*>(xs + static_cast<long long>(K + 1) * SPMM_TOK);
  if (threadIdx.x < SPMM_TOK) xs[K * SPMM_TOK + threadIdx.x] = 0.f;
  const int c0 = blockIdx.x * SPMM_TOK;
  const int r0 = blockIdx.y * rows_per_split;
  const int r1 = min(rows, r0 + rows_per_split);
  const bool vec = ((N & 3) == 0) && ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0) &&
                   (LEVELS || (((ldx & 3) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0)));
  if constexpr (LEVELS) {
    // lane = token, warp step = one 64-bit plane word: each smem store instruction writes
    // 32 tokens of one k (conflict-free). Level p = 2*(t|h) + (t | ~(h|m)) per bit
    // (decompose_thm states, transform.cpp:56-71); tokens past N stage zeros.
    const int words = (K + 63) >> 6;
    for (int i = threadIdx.x; i < words * SPMM_TOK; i += SPMM_THREADS) {
      const int tok = i & (SPMM_TOK - 1), word = i / SPMM_TOK;
      const int c = c0 + tok;
      unsigned long long hi = 0, lo = 0;
      if (c < N) {
        const long long o = static_cast<long long>(c) * lv.wpr + word;
        const unsigned long long t = lv.t[o], h = lv.h[o], m = lv.m[o];
        hi = t | h;
        lo = t | ~(h | m);
      }
      const int k0 = word * 64;
      const int nb = min(64, K - k0);
      float* dst = &xs[k0 * SPMM_TOK + tok];
      if (nb == 64) {
        // constant bit positions: each element is two predicate tests, two selects, one store
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const unsigned hw = static_cast<unsigned>(hi >> (32 * half));
          const unsigned lw = static_cast<unsigned>(lo >> (32 * half));
#pragma unroll
          for (int b = 0; b < 32; ++b) {
            const float lo_v = (lw & (1u << b)) ? lv.d1 : 0.f;
            const float hi_v = (lw & (1u << b)) ? lv.d3 : lv.d2;
            dst[(32 * half + b) * SPMM_TOK] = (hw & (1u << b)) ? hi_v : lo_v;
          }
        }
      } else {
        for (int b = 0; b < nb; ++b) {
          const int lvl = static_cast<int>(((hi >> b) & 1ull) * 2ull + ((lo >> b) & 1ull));
          dst[b * SPMM_TOK] = lvl == 0 ? 0.f : lvl == 1 ? lv.d1 : lvl == 2 ? lv.d2 : lv.d3;
        }
      }
    }
  } else {
    // X chunk: every 16-byte piece in flight at once (cp.async), zero-filled past N
    for (int i = threadIdx.x; i < K * (SPMM_TOK / 4); i += SPMM_THREADS) {
      const int k = i / (SPMM_TOK / 4), q = (i % (SPMM_TOK / 4)) * 4;
      const float* src = X + static_cast<long long>(k) * ldx + c0 + q;
      float* dst = &xs[k * SPMM_TOK + q];
      if (vec && c0 + q + 3 < N) {
        cp_async16(dst, src);
      } else {
        for (int e = 0; e < 4; ++e) dst[e] = (c0 + q + e < N) ? src[e] : 0.f;
      }
    }
  }
  const unsigned long long nz0 = row_ptr[r0];
  for (int i = threadIdx.x; i <= r1 - r0; i += SPMM_THREADS)
    rps[i] = static_cast<unsigned>(row_ptr[r0 + i] - nz0);
  cp_async_wait_all();
  __syncthreads();

  // All loops below are warp-uniform (trip counts are warp maxima; short rows are padded
  // with zero weights) so the full-warp shuffles never need divergence handling.
  // An octet (8 lanes) owns one output row and its 32 columns: each shared-memory phase
  // then reads one whole 128-byte X row (conflict-free). Loops are warp-uniform (trip
  // counts are warp maxima, short rows padded with zero weights) so the full-warp
  // shuffles never need divergence handling.
  const int oct = threadIdx.x >> 3;
  const int ol = threadIdx.x & 7;
  const int lane = threadIdx.x & 31;
  const int obase = lane & ~7;
  const int col = c0 + ol * 4;
  const unsigned long long* cbase = col_idx + nz0;
  const float* vbase = vals + nz0;
  const int iters = (r1 - r0 + SPMM_QUADS - 1) / SPMM_QUADS;
  const unsigned zero_row = static_cast<unsigned>(K);  // X row index of the zero row
  // Nonzero slot `idx` of a row as (X row index, weight); padded slots point at the zero row
  // with weight 0 (0 * 0 leaves an accumulator that started at +0 bit-identical: it can never
  // be -0, so no branch is needed, and EXACT keeps the order). Loaded raw: the index becomes
  // a byte offset only where it is used (step8, an iteration later for prefetched slots), so
  // the warp does not stall on the load right after issuing it.
  auto fetch = [&](unsigned i0, unsigned n, unsigned idx, unsigned& kk, float& vv) {
    kk = zero_row;
    vv = 0.f;
    if (idx < n) {
      kk = static_cast<unsigned>(cbase[i0 + idx]);
      vv = vbase[i0 + idx];
    }
  };
  const char* xrow = reinterpret_cast<const char*>(xs) + ol * 16;
  auto step8 = [&](unsigned kk, float vv, float (&acc)[4]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const unsigned koff = __shfl_sync(0xFFFFFFFFu, kk, obase + j) * (SPMM_TOK * 4);
      const float v = __shfl_sync(0xFFFFFFFFu, vv, obase + j);
      const float4 x = *reinterpret_cast<const float4*>(xrow + koff);
      if (EXACT) {
        acc[0] = __fadd_rn(acc[0], __fmul_rn(v, x.x));
        acc[1] = __fadd_rn(acc[1], __fmul_rn(v, x.y));
        acc[2] = __fadd_rn(acc[2], __fmul_rn(v, x.z));
        acc[3] = __fadd_rn(acc[3], __fmul_rn(v, x.w));
      } else {
        acc[0] = __fmaf_rn(v, x.x, acc[0]);
        acc[1] = __fmaf_rn(v, x.y, acc[1]);
        acc[2] = __fmaf_rn(v, x.z, acc[2]);
        acc[3] = __fmaf_rn(v, x.w, acc[3]);
      }
    }
  };
  // Software pipeline: the first 16 nonzero slots of the next row are loaded from global
  // memory while the current row computes (rows of a 2% residual rarely have more).
  unsigned i0 = 0, n = 0, kk0 = zero_row, kk1 = zero_row;
  float vv0 = 0.f, vv1 = 0.f;
  {
    const int r = r0 + oct;
    if (r < r1) {
      i0 = rps[r - r0];
      n = rps[r - r0 + 1] - i0;
    }
    fetch(i0, n, ol, kk0, vv0);
    fetch(i0, n, ol + 8, kk1, vv1);
  }
  // ACCUM: C of the row one iteration ahead is loaded with the next row's slots, so an HBM
  // round trip overlaps a whole row's nonzero loop instead of a part of it.
  auto load_c = [&](int r, float (&p)[4]) {
    p[0] = p[1] = p[2] = p[3] = 0.f;
    if (ACCUM && r < r1) {
      const float* src = C + static_cast<long long>(r) * ldc + col;
      if (vec && col + 3 < N) {
        const float4 p4 = *reinterpret_cast<const float4*>(src);
        p[0] = p4.x; p[1] = p4.y; p[2] = p4.z; p[3] = p4.w;
      } else {
        for (int e = 0; e < 4; ++e)
          if (col + e < N) p[e] = src[e];
      }
    }
  };
  float prev[4];
  load_c(r0 + oct, prev);
  for (int it = 0; it < iters; ++it) {
    const int r = r0 + it * SPMM_QUADS + oct;
    const bool live = r < r1;
    const unsigned nmax = __reduce_max_sync(0xFFFFFFFFu, n);
    float* dst = C + static_cast<long long>(r) * ldc + col;
    float nprev[4];
    load_c(r + SPMM_QUADS, nprev);
    // prefetch the next row's first 16 slots
    unsigned ni0 = 0, nn = 0, nkk0 = zero_row, nkk1 = zero_row;
    float nvv0 = 0.f, nvv1 = 0.f;
    {
      const int rn = r + SPMM_QUADS;
      if (rn < r1) {
        ni0 = rps[rn - r0];
        nn = rps[rn - r0 + 1] - ni0;
      }
      fetch(ni0, nn, ol, nkk0, nvv0);
      fetch(ni0, nn, ol + 8, nkk1, nvv1);
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (nmax > 0) step8(kk0, vv0, acc);
    if (nmax > 8) step8(kk1, vv1, acc);
    for (unsigned base = 16; base < nmax; base += 8) {
      unsigned kk;
      float vv;
      fetch(i0, n, base + ol, kk, vv);
      step8(kk, vv, acc);
    }
    if (ACCUM) {
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] = __fadd_rn(prev[e], acc[e]);
    }
    if (live) {
      if (vec && col + 3 < N) {
        *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      } else {
        for (int e = 0; e < 4; ++e)
          if (col + e < N) dst[e] = acc[e];
      }
    }
    i0 = ni0;
    n = nn;
    kk0 = nkk0;
    kk1 = nkk1;
    vv0 = nvv0;
    vv1 = nvv1;
#pragma unroll
    for (int e = 0; e < 4; ++e) prev[e] = nprev[e];
  }
}

// Large-K fallback of the LEVELS source: dequantize the planes into a dense [K][N] fp32
// matrix (the layout spmm_csr's b operand has, kernels.hpp:76) for the global-gather SpMM.
// Adjacent threads own adjacent tokens, so every store instruction is coalesced.
__global__ void dequant_levels_kernel(const SpmmLevels lv, int K, int N, float* __restrict__ out) {
  const int words = (K + 63) >> 6;
  const long long total = static_cast<long long>(words) * N;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % N), word = static_cast<int>(i / N);
    const long long o = static_cast<long long>(c) * lv.wpr + word;
    const unsigned long long t = lv.t[o], h = lv.h[o], m = lv.m[o];
    const unsigned long long hi = t | h, lo = t | ~(h | m);
    const int k0 = word * 64, nb = min(64, K - k0);
    for (int b = 0; b < nb; ++b) {
      const int lvl = static_cast<int>(((hi >> b) & 1ull) * 2ull + ((lo >> b) & 1ull));
      out[static_cast<long long>(k0 + b) * N + c] =
          lvl == 0 ? 0.f : lvl == 1 ? lv.d1 : lvl == 2 ? lv.d2 : lv.d3;
    }
  }
}

// ----------------------------------------------------------------------------------
// Residual folded into the tensor-core operand (layer_forward, apb.cpp:158-164).
//   C_r = alpha_r * sum_k s_rk x_k + sum_{residual (r,k)} v_rk x_k = m_r * sum_k W'_rk x_k
// with W'_rk = (alpha_r * s_rk + v_rk) / m_r. For a normal row m_r = alpha_r, so W' = s + v/alpha_r:
// +-1 everywhere (exact in fp16) except at the ~2% residual positions. W' is stored as two
// fp16 parts, W' = hi + lo (22 significant bits), hi in the row's first kpad elements and lo
// in the second kpad elements (zero except at residual positions). The GEMM adds lo . X_hi
// into its low accumulator (apb_gemm_kernel's fold phase), which replaces the sparse pass over
// C. A row whose alpha is 0 or not finite, or whose residuals exceed 2^14 alpha (fp16 range),
// takes m_r = max(|alpha_r|, max|v_rk|) and the rounded parts of (alpha_r/m_r) s + v/m_r.
// A repeated column adds to the running value (spmm_csr sums repeated entries).
__device__ __forceinline__ void f16_split(float w, uint16_t& hi, uint16_t& lo) {
  const __half h = __float2half_rn(w);
  hi = __half_as_ushort(h);
  lo = __half_as_ushort(__float2half_rn(w - __half2float(h)));  // w - hi is exact in fp32
}

// One warp per row. Lane i loads nonzero i up front (rows of a 2% residual have at most a few
// dozen; a row with more than 32 takes the serial path below). The row's largest |v| (warp
// reduction) decides normal vs not. Lane j then expands 32-bit sign words j, j+32, ... into
// both parts (hi = +-1 and lo = 0 for a normal row; zero past K up to kpad) and checks the
// padding bits (ERR_PADDING, as unpack_sign_f16). Finally each lane folds its nonzero into
// its column: the value there is the sign entry, known from the bit, so nothing is read
// back. A row with a repeated column, or with more than 32 nonzeros, is folded serially by
// lane 0 in col_idx order, reading the running value back (spmm_csr sums repeated entries).
__global__ void __launch_bounds__(256) apb_fold_kernel(
    const uint32_t* __restrict__ words, int wpr32, int rows, int K, int kpad, long long ld,
    const unsigned long long* __restrict__ row_ptr, const unsigned long long* __restrict__ col_idx,
    const float* __restrict__ vals, float alpha, const float* __restrict__ row_alpha,
    uint16_t* __restrict__ A, float* __restrict__ row_mul, int* __restrict__ err) {
  pdl_wait();  // the previous kernel may still read the workspace we overwrite
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float a = row_alpha ? row_alpha[r] : alpha;
  const unsigned long long i0 = row_ptr[r], i1 = row_ptr[r + 1];
  const unsigned long long n = i1 - i0;
  const bool mine = static_cast<unsigned long long>(lane) < n;
  const unsigned long long kc = mine ? col_idx[i0 + lane] : ~0ull;
  const float v = mine ? vals[i0 + lane] : 0.f;
  const bool kc_ok = kc < static_cast<unsigned long long>(K);
  const uint32_t kw = kc_ok ? words[static_cast<long long>(r) * wpr32 + static_cast<int>(kc >> 5)] : 0u;
  float vmax = fabsf(v);
  for (unsigned long long i = i0 + 32 + lane; i < i1; i += 32) vmax = fmaxf(vmax, fabsf(vals[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xFFFFFFFFu, vmax, o));
  const bool normal = isfinite(a) && a != 0.f && isfinite(vmax) && vmax <= 16384.f * fabsf(a);
  float m = a;
  if (!normal) {
    m = fmaxf(isfinite(a) ? fabsf(a) : 0.f, vmax);
    if (!(m > 0.f) || !isfinite(m)) m = 1.f;
  }
  uint16_t h1 = 0x3C00u, l1 = 0u;  // the parts of +1 (normal) or +alpha_r/m_r
  if (!normal) f16_split(a / m, h1, l1);
  const uint32_t hpos = h1, lpos = l1, hneg = h1 ^ 0x8000u, lneg = l1 ? (l1 ^ 0x8000u) : 0u;
  uint16_t* hi_row = A + static_cast<long long>(r) * ld;
  uint16_t* lo_row = hi_row + kpad;
  const int groups = max(kpad / 32, wpr32);
  for (int g = lane; g < groups; g += 32) {
    const uint32_t w = (g < wpr32) ? words[static_cast<long long>(r) * wpr32 + g] : 0u;
    const uint32_t valid = valid_mask32(g * 32, K);
    if (w & ~valid) atomicOr(err, ERR_PADDING);
    if (g * 32 >= kpad) continue;
    uint32_t oh[16], ol[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      uint32_t eh[2], el[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int bit = 2 * q + e;
        const bool vb = (valid >> bit) & 1u, b = (w >> bit) & 1u;
        eh[e] = vb ? (b ? hpos : hneg) : 0u;
        el[e] = vb ? (b ? lpos : lneg) : 0u;
      }
      oh[q] = eh[0] | (eh[1] << 16);
      ol[q] = el[0] | (el[1] << 16);
    }
    uint4* dh = reinterpret_cast<uint4*>(hi_row + g * 32);
    uint4* dl = reinterpret_cast<uint4*>(lo_row + g * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      dh[q] = make_uint4(oh[4 * q], oh[4 * q + 1], oh[4 * q + 2], oh[4 * q + 3]);
      dl[q] = make_uint4(ol[4 * q], ol[4 * q + 1], ol[4 * q + 2], ol[4 * q + 3]);
    }
  }
  // repeated columns among the (up to 32) lanes' entries
  const unsigned peers = __match_any_sync(0xFFFFFFFFu, kc);
  const bool serial = n > 32 || __any_sync(0xFFFFFFFFu, mine && __popc(peers) > 1);
  __syncwarp();  // the sign expansion's stores before the folds that overwrite some of them
  const float sv = __half2float(__ushort_as_half(h1)) + __half2float(__ushort_as_half(l1));
  if (!serial) {
    if (mine && kc_ok) {
      const float cur = ((kw >> (kc & 31)) & 1u) ? sv : -sv;
      f16_split(cur + v / m, hi_row[kc], lo_row[kc]);
    }
  } else if (lane == 0) {
    for (unsigned long long i = i0; i < i1; ++i) {
      const unsigned long long k = col_idx[i];
      if (k >= static_cast<unsigned long long>(K)) continue;
      const float cur = __half2float(__ushort_as_half(hi_row[k])) + __half2float(__ushort_as_half(lo_row[k]));
      f16_split(cur + vals[i] / m, hi_row[k], lo_row[k]);
    }
  }
  if (lane == 0) row_mul[r] = m;
}

constexpr int APB_BN = 128;        // output columns per pair tile
constexpr int APB_PARTS = 2;       // fp16 split parts of X (hi, lo)
constexpr int APB_STAGES = 6;
constexpr int APB_A_STAGE = 128 * TC_BK_BYTES;                       // 128 rows x 64 fp16
constexpr int APB_B_PART = (APB_BN / 2) * TC_BK_BYTES;               // 64 rows x 64 fp16
constexpr int APB_STAGE = APB_A_STAGE + APB_PARTS * APB_B_PART;      // 32 KB
constexpr int APB_EPI_BYTES = 4 * 32 * TC_EPI_STRIDE * 4;
constexpr int APB_SMEM = 1024 + APB_STAGES * APB_STAGE + APB_EPI_BYTES + (2 * APB_STAGES + 4) * 8 + 16;

// AP = A parts per smem stage. AP = 1: A = sign(bin) (or W'_hi, with the fold phase after the
// main K loop); AP = 2: a stage holds W'_hi and W'_lo of one K slice with both X parts, so X_hi
// is loaded once for both products (48 KB stages, 4 of them).
// BN = output columns per pair tile: 128 keeps the hi and lo products in separate TMEM
// accumulators (2 x 2 x 128 columns); 256 (AP = 2 only) sums all three products in one
// accumulator per tile (2 x 256 columns) and halves the operand bytes per MAC (64 KB stages,
// 3 of them).
template <int AP, int BN = APB_BN>
struct ApbCfg {
  static constexpr int B_PART = (BN / 2) * TC_BK_BYTES;
  static constexpr int STAGES = AP == 1 ? APB_STAGES : (BN == 256 ? 3 : 4);
  static constexpr int STAGE = AP * APB_A_STAGE + APB_PARTS * B_PART;
  static constexpr int SMEM = 1024 + STAGES * STAGE + APB_EPI_BYTES + (2 * STAGES + 4) * 8 + 16;
  static constexpr bool ONE_ACC = BN == 256;
};
static_assert(ApbCfg<2>::SMEM <= 227 * 1024, "APB stages exceed shared memory");
static_assert(ApbCfg<2, 256>::SMEM <= 227 * 1024, "APB stages exceed shared memory");

struct ApbParams {
  int M, N, kb_per_part;     // kb_per_part = kpad / 64
  int kpad;                  // elements per part row segment
  int fold_kb;               // 0, or kb_per_part: the lo . X_hi phase of the folded residual
  float alpha;               // scalar alpha (row_alpha == nullptr)
  const float* row_alpha;
  const float* tok_scale;    // per output column 2^-e_n (split_x_f16)
  float* C;                  // C = alpha_r * S.X (the residual SpMM then adds R.X onto C)
  long long ldc;
  int num_m_blocks, num_n_blocks, num_tiles;
};

__device__ __forceinline__ void apb_tile_coords(int t, const ApbParams& p, int& mb, int& nb) {
  const int group_tiles = TC_GROUP_M * p.num_n_blocks;
  const int g = t / group_tiles;
  const int first_m = g * TC_GROUP_M;
  const int gm = min(TC_GROUP_M, p.num_m_blocks - first_m);
  const int within = t - g * group_tiles;
  mb = first_m + within % gm;
  nb = within / gm;
}

template <int AP, int BN = APB_BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    apb_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const ApbParams p) {
  using CFG = ApbCfg<AP, BN>;
  constexpr int B_PART = CFG::B_PART;
  constexpr int B_OFF = AP * APB_A_STAGE;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (base_u32 & 1023u)) & 1023u);
  uint8_t* stages = smem;
  float* sEpi = reinterpret_cast<float*>(stages + CFG::STAGES * CFG::STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sEpi) + APB_EPI_BYTES);
  uint64_t* empty = full + CFG::STAGES;
  uint64_t* tfull = empty + CFG::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int unit = static_cast<int>(cluster_id_x());
  const int num_units = static_cast<int>(num_clusters_x());

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < CFG::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 256);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // operands (split X, bf16 signs) and C = R.X come from the preceding kernels
  const int num_kb = p.kb_per_part;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = unit; tile < p.num_tiles; tile += num_units) {
        int mb, nb;
        apb_tile_coords(tile, p, mb, nb);
        const int a_row = mb * 256 + static_cast<int>(rank) * 128;
        const int b_row = nb * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = 0; kb < num_kb + p.fold_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* st = stages + stage * CFG::STAGE;
          if (kb < num_kb) {
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * CFG::STAGE);
            tma_load_2d_pair(st, &tmA, &full[stage], kb * 64, a_row);
            if constexpr (AP == 2) tma_load_2d_pair(st + APB_A_STAGE, &tmA, &full[stage], p.kpad + kb * 64, a_row);
#pragma unroll
            for (int q = 0; q < APB_PARTS; ++q)
              tma_load_2d_pair(st + B_OFF + q * B_PART, &tmB, &full[stage],
                               q * p.kpad + kb * 64, b_row);
          } else {  // fold phase: the lo part of W' against X_hi
            const int kf = kb - num_kb;
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (APB_A_STAGE + B_PART));
            tma_load_2d_pair(st, &tmA, &full[stage], p.kpad + kf * 64, a_row);
            tma_load_2d_pair(st + APB_A_STAGE, &tmB, &full[stage], kf * 64, b_row);
          }
          if (++stage == CFG::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = make_idesc(1u, 0u, 0u, 256, BN);  // f32 <- f16 x f16
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = unit; tile < p.num_tiles; tile += num_units, ++it) {
        const int buf = it & 1;
        const uint32_t bphase = (it >> 1) & 1;
        mbar_wait(&tempty[buf], bphase ^ 1u);
        tc_fence_after();
        // ONE_ACC: every product of the tile into one accumulator (d_lo == d_hi)
        const uint32_t d_hi = tmem_base + buf * (CFG::ONE_ACC ? BN : 2 * BN);
        const uint32_t d_lo = CFG::ONE_ACC ? d_hi : d_hi + BN;
        for (int kb = 0; kb < num_kb + p.fold_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(stages + stage * CFG::STAGE);
          if (kb < num_kb) {
#pragma unroll
            for (int q = 0; q < APB_PARTS; ++q) {
              const uint32_t b_addr = a_addr + B_OFF + q * B_PART;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = sw128_kmajor_desc(a_addr + k * 32);
                const uint64_t bd = sw128_kmajor_desc(b_addr + k * 32);
                const uint32_t acc = (q == 0) ? ((kb | k) != 0)
                                              : (CFG::ONE_ACC ? 1u : !(q == 1 && kb == 0 && k == 0));
                mma_f16_pair(q == 0 ? d_hi : d_lo, ad, bd, idesc, acc);
              }
            }
            if constexpr (AP == 2) {  // W'_lo . X_hi into the low accumulator
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_f16_pair(d_lo, sw128_kmajor_desc(a_addr + APB_A_STAGE + k * 32),
                             sw128_kmajor_desc(a_addr + B_OFF + k * 32), idesc, 1u);
            }
          } else {  // fold phase: W'_lo . X_hi joins the low accumulator (same magnitude)
            const uint32_t b_addr = a_addr + APB_A_STAGE;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_f16_pair(d_lo, sw128_kmajor_desc(a_addr + k * 32), sw128_kmajor_desc(b_addr + k * 32),
                           idesc, 1u);
          }
          mma_commit_pair(&empty[stage], 0x3);
          if (++stage == CFG::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit_pair(&tfull[buf], 0x3);
      }
    }
  } else {
    const int quad = warp & 3;
    float* stg = sEpi + (warp - 2) * 32 * TC_EPI_STRIDE;
    const bool vec_ok = ((p.N & 3) == 0) && ((p.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.C) & 15) == 0);
    int it = 0;
    for (int tile = unit; tile < p.num_tiles; tile += num_units, ++it) {
      int mb, nb;
      apb_tile_coords(tile, p, mb, nb);
      const int buf = it & 1;
      const uint32_t bphase = (it >> 1) & 1;
      const int row_base = mb * 256 + static_cast<int>(rank) * 128 + quad * 32;
      const int my_row = row_base + lane;
      // loaded before the accumulator wait so the latency hides behind it
      const float alpha = (p.row_alpha != nullptr) ? (my_row < p.M ? p.row_alpha[my_row] : 0.f)
                                                   : p.alpha;
      mbar_wait(&tfull[buf], bphase);
      tc_fence_after();
      const uint32_t t_hi = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                            buf * (CFG::ONE_ACC ? BN : 2 * BN);
      const int cl = (lane & 7) * 4;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        const int col0 = nb * BN + c * 32;
        if (col0 >= p.N) break;
        uint32_t vh[32], vl[32];
        tmem_ld_32x32b_x32(t_hi + c * 32, vh);
        if constexpr (!CFG::ONE_ACC) tmem_ld_32x32b_x32(t_hi + BN + c * 32, vl);
        // the chunk's 32 token scales: same address in every lane (broadcast); past N: 0
        float ts[32];
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          if (col0 + j + 3 < p.N) {
            const float4 t4 = __ldg(reinterpret_cast<const float4*>(p.tok_scale + col0 + j));
            ts[j] = t4.x; ts[j + 1] = t4.y; ts[j + 2] = t4.z; ts[j + 3] = t4.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) ts[j + e] = (col0 + j + e < p.N) ? p.tok_scale[col0 + j + e] : 0.f;
          }
        }
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float of[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)  // x 2^-e_n is exact
            of[e] = __fmul_rn(__fmul_rn(alpha, CFG::ONE_ACC ? __uint_as_float(vh[j + e])
                                                            : __fadd_rn(__uint_as_float(vh[j + e]),
                                                                        __uint_as_float(vl[j + e]))),
                              ts[j + e]);
          *reinterpret_cast<float4*>(&stg[lane * TC_EPI_STRIDE + j]) = make_float4(of[0], of[1], of[2], of[3]);
        }
        __syncwarp();
#pragma unroll
        for (int r8 = 0; r8 < 8; ++r8) {
          const int rl = r8 * 4 + (lane >> 3);
          const int grow = row_base + rl;
          const int gcol = col0 + cl;
          if (grow < p.M && gcol < p.N) {
            const float4 r = *reinterpret_cast<const float4*>(&stg[rl * TC_EPI_STRIDE + cl]);
            float* dst = p.C + static_cast<long long>(grow) * p.ldc + gcol;
            if (vec_ok && gcol + 3 < p.N) {
              *reinterpret_cast<float4*>(dst) = r;
            } else {
              const float* rf = reinterpret_cast<const float*>(&r);
              for (int e = 0; e < 4; ++e)
                if (gcol + e < p.N) dst[e] = rf[e];
            }
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive_cluster(smem_u32(&tempty[buf]) & kPeerBitMask);
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace bitmm_dev
