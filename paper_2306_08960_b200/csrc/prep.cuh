// Operand preparation for fx_gemm (in-GEMM expansion): one launch over every operand of a
// call that needs a pass before the GEMM.
//   planes -> codes : ThmPlanes {t,h,m} (tensor.hpp:134-145) -> 2-bit codes p = 2 hi + lo,
//                     hi = t | h, lo = t | ~(h | m) (legal states per transform.cpp:56-71:
//                     p0 = (0,0,1), p1 = (0,0,0), p2 = (0,1,0), p3 = (1,0,1)), validated like
//                     ThmPlanes::validate (tensor.cpp:133-153: illegal triples and nonzero
//                     padding set ERR_ENCODING). 32 elements -> one 64-bit code word laid out
//                     for fx_expand_code: element 4n+q sits in 32-bit half q >> 1 at bit pair
//                     4n + 2 (q & 1). Rows are padded with zero codes to kcode (a multiple of
//                     512 elements, one packed slot).
//   sign tail check : a BitMatrix needs no pass (fx_gemm reads its words), only the padding
//                     check of tensor.cpp:78-89 for the words that hold bits past K: nonzero
//                     padding sets ERR_PADDING.
#pragma once

#include <cstdint>

#include "ptx.cuh"
#include "unpack.cuh"

namespace bitmm_dev {

struct PrepOperand {
  const uint64_t* t;  // planes (codes) or sign words (tail check)
  const uint64_t* h;
  const uint64_t* m;
  uint2* codes;       // [rows][kcode / 32] (codes only)
  long long rows;
  int wpr;            // 64-bit words per input row
  int K;
  int first_word;     // tail check: first 64-bit word holding bits past K
  int out_words;      // codes: kcode / 64 (two code words per input word)
  int code;           // 1: planes -> codes, 0: sign tail check
  long long items;    // rows * words per row handled
};

constexpr int PREP_MAX_OPS = 8;
struct PrepSet {
  PrepOperand op[PREP_MAX_OPS];
  int count;
  int* err;
};

__device__ __forceinline__ uint64_t valid_mask64(int kbase, int K) {
  if (kbase + 64 <= K) return ~0ull;
  if (kbase >= K) return 0ull;
  return (1ull << (K - kbase)) - 1ull;
}

// One 32-element group: hi / lo bit words -> the 64-bit code word (see the header).
__device__ __forceinline__ uint2 codes_of(uint32_t H, uint32_t L) {
  const uint32_t lo = (L & 0x11111111u) | ((H & 0x11111111u) << 1) | ((L & 0x22222222u) << 1) |
                      ((H & 0x22222222u) << 2);
  const uint32_t hi = ((L & 0x44444444u) >> 2) | ((H & 0x44444444u) >> 1) | ((L & 0x88888888u) >> 1) |
                      (H & 0x88888888u);
  return make_uint2(lo, hi);
}

// Thread per 64-bit input word (codes: per output word pair as well).
__global__ void __launch_bounds__(256) prep_operands_kernel(const __grid_constant__ PrepSet P) {
  pdl_wait();  // the previous GEMM may still read the code workspace we overwrite
  pdl_launch_dependents();
  const PrepOperand& o = P.op[blockIdx.y];
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= o.items) return;
  int bad = 0;
  if (o.code) {
    const int per_row = max(o.wpr, o.out_words);
    const long long r = i / per_row;
    const int w = static_cast<int>(i - r * per_row);
    uint64_t t = 0, h = 0, m = 0;
    if (w < o.wpr) {
      const long long idx = r * o.wpr + w;
      t = __ldg(reinterpret_cast<const unsigned long long*>(o.t) + idx);
      h = __ldg(reinterpret_cast<const unsigned long long*>(o.h) + idx);
      m = __ldg(reinterpret_cast<const unsigned long long*>(o.m) + idx);
    }
    const uint64_t valid = valid_mask64(w * 64, o.K);
    if (((t | h | m) & ~valid) | (t & h) | (t & ~m) | (h & m)) bad = ERR_ENCODING;
    if (w < o.out_words) {
      const uint64_t H = (t | h) & valid, L = (t | ~(h | m)) & valid;
      const uint2 c0 = codes_of(static_cast<uint32_t>(H), static_cast<uint32_t>(L));
      const uint2 c1 = codes_of(static_cast<uint32_t>(H >> 32), static_cast<uint32_t>(L >> 32));
      reinterpret_cast<uint4*>(o.codes)[r * o.out_words + w] = make_uint4(c0.x, c0.y, c1.x, c1.y);
    }
  } else {
    const int per_row = o.wpr - o.first_word;
    const long long r = i / per_row;
    const int w = o.first_word + static_cast<int>(i - r * per_row);
    const uint64_t v = __ldg(reinterpret_cast<const unsigned long long*>(o.t) + r * o.wpr + w);
    if (v & ~valid_mask64(w * 64, o.K)) bad = ERR_PADDING;
  }
  if (bad) atomicOr(P.err, bad);  // invalid input only: no contention on valid calls
}

}  // namespace bitmm_dev
