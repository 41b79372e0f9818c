// 2-bit activation levels for the APB residual (sm_100a): the planes' level codes as bf16
// patterns of p in {0, 1, 2, 3}, staged per 64-token chunk as [K + 1][SL_ROW_WORDS] 32-bit words
// (two tokens each; row K is zeros). Used by spmm_levels_kernel (staged in the kernel) and by
// the fused layer (staged for every chunk by unpack_operands, then bulk-copied).
#pragma once

#include <cstdint>

namespace bitmm_dev {

constexpr int SL_TOK = 64;                   // tokens per block
constexpr int SL_ROW_WORDS = SL_TOK / 2;     // u32 words per staged column (two bf16 levels each)

// LEVELS source: activation planes {t,h,m} [tokens][wpr] (K-packed per token, the a_packed
// orientation of gemm_1x2), dequantized to d[p] = float(p) * (s * gamma_a).
struct SpmmLevels {
  const unsigned long long* t;
  const unsigned long long* h;
  const unsigned long long* m;
  int wpr;
  float d1, d2, d3;  // d0 = 0
  float neg_zero;    // -0.0f, passed at run time (spmm_levels_kernel's exact products)
};

// bf16 bit pattern of the level p = 2 hi + lo (0, 1.0, 2.0, 3.0)
__device__ __forceinline__ unsigned level_bf16(bool lo, bool hi) {
  return hi ? (lo ? 0x4040u : 0x4000u) : (lo ? 0x3F80u : 0u);
}

// One staging item of the level chunk of tokens [c0, c0 + SL_TOK): (64-bit plane word, half of
// it, token pair) -> 32 words of xw [K + 1][SL_ROW_WORDS] (two bf16 levels each). p = 2 (t|h) +
// (t | ~(h|m)) (decompose_thm states, transform.cpp:56-71); bits past K are never staged,
// tokens past N stage level 0.
__device__ __forceinline__ void sl_stage_item(unsigned* xw, int K, int N, int c0, const SpmmLevels& lv, int i) {
  const int pair = i & (SL_ROW_WORDS - 1), hw = i / SL_ROW_WORDS;
  const int word = hw >> 1, half = hw & 1;
  const int ta = c0 + 2 * pair;
  unsigned loA = 0, hiA = 0, loB = 0, hiB = 0;
  if (ta < N) {
    const long long o = static_cast<long long>(ta) * lv.wpr + word;
    const unsigned long long t = lv.t[o], h = lv.h[o], m = lv.m[o];
    hiA = static_cast<unsigned>((t | h) >> (32 * half));
    loA = static_cast<unsigned>((t | ~(h | m)) >> (32 * half));
  }
  if (ta + 1 < N) {
    const long long o = static_cast<long long>(ta + 1) * lv.wpr + word;
    const unsigned long long t = lv.t[o], h = lv.h[o], m = lv.m[o];
    hiB = static_cast<unsigned>((t | h) >> (32 * half));
    loB = static_cast<unsigned>((t | ~(h | m)) >> (32 * half));
  }
  const int k0 = word * 64 + half * 32;
  unsigned* dst = &xw[static_cast<long long>(k0) * SL_ROW_WORDS + pair];
  if (k0 + 32 <= K) {
#pragma unroll
    for (int b = 0; b < 32; ++b)
      dst[b * SL_ROW_WORDS] = level_bf16((loA >> b) & 1u, (hiA >> b) & 1u) |
                              (level_bf16((loB >> b) & 1u, (hiB >> b) & 1u) << 16);
  } else {
    for (int b = 0; b < K - k0; ++b)
      dst[b * SL_ROW_WORDS] = level_bf16((loA >> b) & 1u, (hiA >> b) & 1u) |
                              (level_bf16((loB >> b) & 1u, (hiB >> b) & 1u) << 16);
  }
}

// Every level chunk of the activations, for the fused layer: out [chunks][K + 1][SL_ROW_WORDS]
// (L2-resident: tokens x (K + 1) x 2 bytes). chunks = 0: none.
struct LevelChunkJob {
  SpmmLevels lv;
  int K, N, chunks;
  unsigned* out;
};

__device__ __forceinline__ long long level_chunk_items(const LevelChunkJob& j) {
  return static_cast<long long>(((j.K + 63) >> 6) * 2 * SL_ROW_WORDS + SL_ROW_WORDS) * j.chunks;
}

// Item i of the job (one (chunk, plane word, half, token pair), or a word of a zero row).
__device__ __forceinline__ void level_chunk_item(const LevelChunkJob& j, long long i) {
  const int items = ((j.K + 63) >> 6) * 2 * SL_ROW_WORDS;
  const long long per_chunk = items + SL_ROW_WORDS;
  const int chunk = static_cast<int>(i / per_chunk), q = static_cast<int>(i - chunk * per_chunk);
  unsigned* xw = j.out + static_cast<long long>(chunk) * (j.K + 1) * SL_ROW_WORDS;
  if (q < items)
    sl_stage_item(xw, j.K, j.N, chunk * SL_TOK, j.lv, q);
  else
    xw[static_cast<long long>(j.K) * SL_ROW_WORDS + (q - items)] = 0u;
}

}  // namespace bitmm_dev
