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

// The byte format of the fused layer's chunks ("L8", [K + 1][SL_TOK] bytes, row K = level 0):
// level p is stored as 0x80 + 0x20 p, the second-highest byte of the fp32 value p + 4
// (0x40800000, 0x40A00000, 0x40C00000, 0x40E00000), so one PRMT with the constant 0x40 rebuilds
// p + 4 in fp32, and fma(p + 4, sg, -4 sg) = fl(p * sg) exactly (the product and the exact
// -4 sg are summed before the one rounding). Half the bytes of the bf16 patterns.
constexpr int L8_ROW_WORDS = SL_TOK / 4;  // u32 words per staged column (four levels each)
__device__ __forceinline__ unsigned level_l8(bool lo, bool hi) { return 0x80u + 0x20u * (2u * hi + lo); }

// sl_stage_item's item (plane word, half, token pair) in the L8 format: 32 u16 (two tokens each)
// of xb [K + 1][SL_TOK] bytes.
__device__ __forceinline__ void l8_stage_item(unsigned char* xb, int K, int N, int c0, const SpmmLevels& lv, int i) {
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
  unsigned short* dst = reinterpret_cast<unsigned short*>(xb + static_cast<long long>(k0) * SL_TOK) + pair;
  const int nb = min(32, K - k0);
  for (int b = 0; b < nb; ++b)
    dst[b * (SL_TOK / 2)] = static_cast<unsigned short>(level_l8((loA >> b) & 1u, (hiA >> b) & 1u) |
                                                        (level_l8((loB >> b) & 1u, (hiB >> b) & 1u) << 8));
}

// Every level chunk of the activations, for the fused layer: out [chunks][K + 1][SL_ROW_WORDS]
// words (bf16 patterns; L2-resident: tokens x (K + 1) x 2 bytes), or with l8 [chunks][K + 1]
// [L8_ROW_WORDS] (the L8 bytes, half that). chunks = 0: none.
struct LevelChunkJob {
  SpmmLevels lv;
  int K, N, chunks;
  unsigned* out;
  int l8;
};

__device__ __forceinline__ int level_chunk_row_words(const LevelChunkJob& j) { return j.l8 ? L8_ROW_WORDS : SL_ROW_WORDS; }

__device__ __forceinline__ long long level_chunk_items(const LevelChunkJob& j) {
  return static_cast<long long>(((j.K + 63) >> 6) * 2 * SL_ROW_WORDS + level_chunk_row_words(j)) * j.chunks;
}

// Item i of the job (one (chunk, plane word, half, token pair), or a word of a zero row).
__device__ __forceinline__ void level_chunk_item(const LevelChunkJob& j, long long i) {
  const int items = ((j.K + 63) >> 6) * 2 * SL_ROW_WORDS;
  const int rw = level_chunk_row_words(j);
  const long long per_chunk = items + rw;
  const int chunk = static_cast<int>(i / per_chunk), q = static_cast<int>(i - chunk * per_chunk);
  unsigned* xw = j.out + static_cast<long long>(chunk) * (j.K + 1) * rw;
  if (q < items) {
    if (j.l8)
      l8_stage_item(reinterpret_cast<unsigned char*>(xw), j.K, j.N, chunk * SL_TOK, j.lv, q);
    else
      sl_stage_item(xw, j.K, j.N, chunk * SL_TOK, j.lv, q);
  } else {
    xw[static_cast<long long>(j.K) * rw + (q - items)] = j.l8 ? 0x80808080u : 0u;
  }
}

}  // namespace bitmm_dev
