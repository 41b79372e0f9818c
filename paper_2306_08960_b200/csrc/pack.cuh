// GPU packers: dense fp32 -> the reference's packed layouts.
//
//   pack_signs_kernel      : tensor.cpp:155-164 — bit i of row r = (a[r][i] >= 0), sign(0)=+1
//   quantize_thm_kernel    : transform.cpp:21-36 (lround(v/s), clamp to [0,3]) followed by
//                            decompose_thm, transform.cpp:47-75 (p0=(0,0,1) p1=(0,0,0)
//                            p2=(0,1,0) p3=(1,0,1))
//   decompose_thm_kernel   : decompose_thm alone, from 2-bit levels (TwoBitMatrix, one byte per
//                            element); a level above 3 sets ERR_LEVEL (transform.cpp:70-71)
//   decompose_apb_*        : decompose_apb, apb.cpp:119-142 — the residual CSR of every entry
//                            with |a| != alpha, value rounded with ties away from zero
//
// Output rows are `wpr` uint64 words (wpr >= ceil(cols/64), e.g. 512-bit lanes), element i
// at word i/64 bit i%64, and every padding bit is zero (tensor.hpp:14-16). A warp covers 32
// consecutive elements per __ballot_sync; two ballots form one uint64 word, written by lane 0.
// Reads are coalesced (32 consecutive floats per warp step); each warp walks a row segment of
// 64 * WORDS_PER_WARP elements so every warp writes whole words.
#pragma once

#include <cmath>
#include <cstdint>

namespace bitmm_dev {

constexpr int PACK_WORDS_PER_WARP = 4;  // 256 elements per warp work unit

// lround(v / s) clamped to [0, 3]: halves away from zero (std::lround) on the fp32 quotient,
// as quantize_uniform_2bit computes `v / s` in float (transform.cpp:224). `/` is IEEE
// round-to-nearest division here (no fast-math), matching the host.
__device__ __forceinline__ int quantize_level(float v, float s) {
  long p = lroundf(v / s);
  p = p < 0 ? 0 : p;
  return static_cast<int>(p > 3 ? 3 : p);
}

// One warp per (row, 256-element segment); grid-stride over units.
__global__ void pack_signs_kernel(const float* __restrict__ a, long long rows, int cols,
                                  long long lda, int wpr, unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const int segs = (wpr + PACK_WORDS_PER_WARP - 1) / PACK_WORDS_PER_WARP;
  for (long long u = warp; u < rows * segs; u += nwarps) {
    const long long r = u / segs;
    const int w0 = static_cast<int>(u - r * segs) * PACK_WORDS_PER_WARP;
    const float* row = a + r * lda;
#pragma unroll
    for (int w = 0; w < PACK_WORDS_PER_WARP; ++w) {
      const int word = w0 + w;
      if (word >= wpr) break;
      const int e0 = word * 64 + lane, e1 = e0 + 32;
      const unsigned lo = __ballot_sync(0xFFFFFFFFu, e0 < cols && row[e0] >= 0.0f);
      const unsigned hi = __ballot_sync(0xFFFFFFFFu, e1 < cols && row[e1] >= 0.0f);
      if (lane == 0)
        out[r * wpr + word] = (static_cast<unsigned long long>(hi) << 32) | lo;
    }
  }
}

__global__ void quantize_thm_kernel(const float* __restrict__ a, long long rows, int cols,
                                    long long lda, float s, int wpr,
                                    unsigned long long* __restrict__ t,
                                    unsigned long long* __restrict__ h,
                                    unsigned long long* __restrict__ m) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const int segs = (wpr + PACK_WORDS_PER_WARP - 1) / PACK_WORDS_PER_WARP;
  for (long long u = warp; u < rows * segs; u += nwarps) {
    const long long r = u / segs;
    const int w0 = static_cast<int>(u - r * segs) * PACK_WORDS_PER_WARP;
    const float* row = a + r * lda;
#pragma unroll
    for (int w = 0; w < PACK_WORDS_PER_WARP; ++w) {
      const int word = w0 + w;
      if (word >= wpr) break;
      unsigned tb[2], hb[2], mb[2];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int e = word * 64 + half * 32 + lane;
        const int p = e < cols ? quantize_level(row[e], s) : 1;  // padding: (0,0,0)
        tb[half] = __ballot_sync(0xFFFFFFFFu, p == 3);
        hb[half] = __ballot_sync(0xFFFFFFFFu, p == 2);
        mb[half] = __ballot_sync(0xFFFFFFFFu, p == 0 || p == 3);
      }
      if (lane == 0) {
        const long long o = r * wpr + word;
        t[o] = (static_cast<unsigned long long>(tb[1]) << 32) | tb[0];
        h[o] = (static_cast<unsigned long long>(hb[1]) << 32) | hb[0];
        m[o] = (static_cast<unsigned long long>(mb[1]) << 32) | mb[0];
      }
    }
  }
}

constexpr int ERR_LEVEL = 4;  // a 2-bit level above 3 (decompose_thm's invalid_argument)
constexpr int ERR_ALPHA = 8;  // a non-positive alpha (decompose_apb's invalid_argument)

__global__ void decompose_thm_kernel(const uint8_t* __restrict__ levels, long long rows, int cols,
                                     int wpr, unsigned long long* __restrict__ t,
                                     unsigned long long* __restrict__ h,
                                     unsigned long long* __restrict__ m, int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const int segs = (wpr + PACK_WORDS_PER_WARP - 1) / PACK_WORDS_PER_WARP;
  bool bad = false;
  for (long long u = warp; u < rows * segs; u += nwarps) {
    const long long r = u / segs;
    const int w0 = static_cast<int>(u - r * segs) * PACK_WORDS_PER_WARP;
    const uint8_t* row = levels + r * cols;
#pragma unroll
    for (int w = 0; w < PACK_WORDS_PER_WARP; ++w) {
      const int word = w0 + w;
      if (word >= wpr) break;
      unsigned tb[2], hb[2], mb[2];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int e = word * 64 + half * 32 + lane;
        const int p = e < cols ? row[e] : 1;  // padding: (0,0,0)
        bad |= p > 3;
        tb[half] = __ballot_sync(0xFFFFFFFFu, p == 3);
        hb[half] = __ballot_sync(0xFFFFFFFFu, p == 2);
        mb[half] = __ballot_sync(0xFFFFFFFFu, p == 0 || p == 3);
      }
      if (lane == 0) {
        const long long o = r * wpr + word;
        t[o] = (static_cast<unsigned long long>(tb[1]) << 32) | tb[0];
        h[o] = (static_cast<unsigned long long>(hb[1]) << 32) | hb[0];
        m[o] = (static_cast<unsigned long long>(mb[1]) << 32) | mb[0];
      }
    }
  }
  if (bad) atomicOr(err, ERR_LEVEL);
}

// apb.cpp:35-46 with away_from_zero = true: double -> float, round to nearest, a tie goes to
// the neighbour of larger magnitude.
__device__ __forceinline__ float round_tie_away(double x) {
  const float nearf = __double2float_rn(x);
  const double dn = static_cast<double>(nearf);
  if (dn == x) return nearf;
  const float other = nextafterf(nearf, dn < x ? INFINITY : -INFINITY);
  const double en = fabs(x - dn), eo = fabs(static_cast<double>(other) - x);
  if (en != eo) return en < eo ? nearf : other;
  return fabs(dn) > fabs(static_cast<double>(other)) ? nearf : other;
}

__device__ __forceinline__ float apb_alpha(float alpha, const float* row_alpha, long long r) {
  return row_alpha != nullptr ? row_alpha[r] : alpha;
}

// decompose_apb, pass 1: residual entries per row (one warp per row) into counts[r + 1].
__global__ void decompose_apb_count_kernel(const float* __restrict__ a, long long rows, int cols,
                                           long long lda, float alpha,
                                           const float* __restrict__ row_alpha,
                                           unsigned long long* __restrict__ counts,
                                           int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  for (long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const float al = apb_alpha(alpha, row_alpha, r);
    if (!(al > 0.0f) && lane == 0) atomicOr(err, ERR_ALPHA);
    const float* row = a + r * lda;
    unsigned long long n = 0;
    for (int c0 = 0; c0 < cols; c0 += 32) {
      const int c = c0 + lane;
      n += __popc(__ballot_sync(0xFFFFFFFFu, c < cols && fabsf(row[c]) != al));
    }
    if (lane == 0) counts[r + 1] = n;
  }
}

// decompose_apb, pass 2: column indices (ascending) and values of every residual entry, at
// row_ptr[r] onward (one warp per row; a ballot and a prefix popcount place each entry).
__global__ void decompose_apb_fill_kernel(const float* __restrict__ a, long long rows, int cols,
                                          long long lda, float alpha,
                                          const float* __restrict__ row_alpha,
                                          const unsigned long long* __restrict__ row_ptr,
                                          unsigned long long* __restrict__ col_idx,
                                          float* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const unsigned below = (1u << lane) - 1u;
  for (long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const float al = apb_alpha(alpha, row_alpha, r);
    const float* row = a + r * lda;
    unsigned long long pos = row_ptr[r];
    for (int c0 = 0; c0 < cols; c0 += 32) {
      const int c = c0 + lane;
      const float v = c < cols ? row[c] : 0.0f;
      const bool keep = c < cols && fabsf(v) != al;
      const unsigned mask = __ballot_sync(0xFFFFFFFFu, keep);
      if (keep) {
        const unsigned long long i = pos + __popc(mask & below);
        col_idx[i] = static_cast<unsigned long long>(c);
        const float base = al * (v >= 0.0f ? 1.0f : -1.0f);  // sign(0) = +1
        vals[i] = round_tie_away(static_cast<double>(v) - static_cast<double>(base));
      }
      pos += __popc(mask);
    }
  }
}

// Row ops (kernels.cpp:120-140), batched: one warp per row pair.
//   dot_binary: n - 2 * popc(u ^ v)           (xor_popcount_many's int32 count, kernels.cpp:124-127)
//   mbm:        popc(z) - 2 * popc((x ^ y) & z)
__global__ void row_ops_kernel(const unsigned long long* __restrict__ a,
                               const unsigned long long* __restrict__ b,
                               const unsigned long long* __restrict__ z, long long count,
                               long long words, long long n, long long* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5; r < count;
       r += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    long long flip = 0, act = 0;
    for (long long i = lane; i < words; i += 32) {
      const unsigned long long d = a[r * words + i] ^ b[r * words + i];
      if (z != nullptr) {
        const unsigned long long zw = z[r * words + i];
        flip += __popcll(d & zw);
        act += __popcll(zw);
      } else {
        flip += __popcll(d);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      flip += __shfl_xor_sync(0xFFFFFFFFu, flip, o);
      act += __shfl_xor_sync(0xFFFFFFFFu, act, o);
    }
    if (lane == 0)
      out[r] = z != nullptr ? act - 2 * flip : n - 2 * static_cast<long long>(static_cast<int>(flip));
  }
}

// ThmPlanes::validate on device (tensor.cpp:133-153), exact precedence: nonzero padding in any
// plane wins; otherwise the first violating word in row-major order decides, and within it
// the first failing check (1: t&h, 2: t&~m, 3: h&m). Results: *pad_bad |= 1, and
// *first_bad = min over violating words of (word index << 2 | check).
__global__ void validate_planes_kernel(const unsigned long long* __restrict__ t,
                                       const unsigned long long* __restrict__ h,
                                       const unsigned long long* __restrict__ m, long long rows,
                                       long long cols, long long wpr, int* pad_bad,
                                       unsigned long long* first_bad) {
  const long long total = rows * wpr;
  const long long full = cols / 64;
  const int tail = static_cast<int>(cols % 64);
  const unsigned long long keep = tail ? ((1ull << tail) - 1) : ~0ull;
  unsigned long long best = ~0ull;
  int pad = 0;
  for (long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long tw = t[g], hw = h[g], mw = m[g];
    const long long cw = g % wpr;
    if (cw >= full) {
      const unsigned long long all = tw | hw | mw;
      if ((cw == full && tail) ? (all & ~keep) : all) pad = 1;
    }
    const int code = (tw & hw) ? 1 : (tw & ~mw) ? 2 : (hw & mw) ? 3 : 0;
    if (code && best == ~0ull) best = (static_cast<unsigned long long>(g) << 2) | code;
  }
  if (pad) atomicOr(pad_bad, 1);
  if (best != ~0ull) atomicMin(first_bad, best);
}

}  // namespace bitmm_dev
