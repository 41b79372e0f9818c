// Operand expansion: reference packed layouts -> tensor-core operand rows.
//
// Input layouts are exactly the reference's (proj/include/bitmm/tensor.hpp:59-112):
// row-major uint64 words, bit i of a row in word i/64 at position i%64, padded to
// words_per_row (512-bit lanes by default) with zero padding. Read as uint32 the
// order is unchanged on little-endian (element i -> u32 i/32, bit i%32).
//
// Outputs are K-major operand rows padded to kpad elements with zeros, so the
// padding never contributes to a product:
//   unpack_operands   : both GEMM operands in one launch:
//                      bit b -> int8 (2b-1)                (BitMatrix, tensor.hpp:59)
//                      planes {t,h,m} -> int8 level p      (ThmPlanes, tensor.hpp:134;
//                      legal states per transform.cpp:47-75: p0=(0,0,1) p1=(0,0,0)
//                      p2=(0,1,0) p3=(1,0,1), so p = 2(t|h) + (t | ~(h|m)))
//   unpack_sign_f16  : bit b -> fp16 (+1/-1)               (APB binary plane)
//   split_x_f16      : fp32 X[K][N] -> fp16 parts XT[N][part*kpad + k], transposed to
//                      K-major: per token n a power of two 2^e_n brings max_k |X[k][n]|
//                      into [2^14, 2^15), and x * 2^e_n = hi + lo (+ <= 2^-22 relative);
//                      2^-e_n goes to the GEMM epilogue as the column scale.
// Validation folded into the same pass (the reference checks these on the host,
// tensor.cpp:78-89 and tensor.cpp:133-153): nonzero padding of a BitMatrix sets
// ERR_PADDING, an illegal plane triple or nonzero plane padding sets ERR_ENCODING.
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

#include "levels.cuh"
#include "ptx.cuh"

namespace bitmm_dev {

constexpr int ERR_PADDING = 1;
constexpr int ERR_ENCODING = 2;

// 4 bits -> 4 bytes holding 0/1 (no carries: the shifted copies never overlap).
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

__device__ __forceinline__ uint32_t valid_mask32(int kbase, int K) {
  if (kbase + 32 <= K) return 0xFFFFFFFFu;
  if (kbase >= K) return 0u;
  return (1u << (K - kbase)) - 1u;
}

// Operand descriptors for the pair expansion (blockIdx.y / op index selects the operand).
struct UnpackOperand {
  const uint32_t* w0;  // sign words, or the t plane
  const uint32_t* w1;  // h plane (levels only)
  const uint32_t* w2;  // m plane (levels only)
  uint8_t* out;        // [rows][kpad]
  long long rows;
  long long groups_per_row;  // slices of 128 words (4096 elements) per row
  int wpr32;
  int levels;  // 0: +-1 signs, 1: 2-bit levels
  int K;       // logical columns (bits past K must be zero)
  int kpad;    // expanded elements per row (zero past K)
};

// Every operand of one launch: the two of a GEMM, or all operands of a GEMM group.
constexpr int UNPACK_MAX_OPS = 8;
struct UnpackSet {
  UnpackOperand op[UNPACK_MAX_OPS];
  int count;
  int* err;
  int fp4;          // 1: packed e2m1 nibbles, rows of kpad/2 bytes (Kind::F4 operands)
  LevelChunkJob lc;  // the fused 2-bit APB layer's level chunks (grid row 0), if any
};

// One warp expands one 4096-element slice of one operand row (128 input words, 4 KB of
// int8 output), split into a load step (all 128 words in flight: lane t holds words
// j*32 + t) and an expand/store step, so a warp looping over slices can prefetch the next
// slice while expanding the current one. Store v of lane t writes output bytes
// [16*(32v+t), +16): every warp store instruction covers 512 contiguous bytes, and its 16
// source bits (half of word 16v + t/2) come from the loading lane via a shuffle.
struct SliceWords {
  uint32_t w0[4], w1[4], w2[4];
};

__device__ __forceinline__ void load_slice_warp(const UnpackOperand& o, long long r, int sl,
                                                int lane, SliceWords& s) {
  const long long rbase = r * o.wpr32;
  const int word0 = sl * 128;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int g = word0 + j * 32 + lane;
    s.w0[j] = s.w1[j] = s.w2[j] = 0u;
    if (g < o.wpr32) {
      s.w0[j] = __ldg(o.w0 + rbase + g);
      if (o.levels) {
        s.w1[j] = __ldg(o.w1 + rbase + g);
        s.w2[j] = __ldg(o.w2 + rbase + g);
      }
    }
  }
}

// Returns the warp-wide OR of the slice's error flags.
__device__ __forceinline__ int expand_slice_warp(const UnpackOperand& o, long long r, int sl,
                                                 int K, int kpad, int lane, SliceWords& s,
                                                 bool fp4 = false) {
  const int word0 = sl * 128;
  int bad = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t valid = valid_mask32((word0 + j * 32 + lane) * 32, K);
    if (o.levels == 0) {
      bad |= (s.w0[j] & ~valid) ? ERR_PADDING : 0;
    } else {
      const uint32_t tw = s.w0[j], hw = s.w1[j], mw = s.w2[j];
      if (((tw | hw | mw) & ~valid) | (tw & hw) | (tw & ~mw) | (hw & mw)) bad |= ERR_ENCODING;
      // fold the planes into (hi, lo) level bits in place: p = 2*hi + lo
      s.w0[j] = (tw | hw) & valid;
      s.w1[j] = (tw | ~(hw | mw)) & valid;
    }
  }
  if (fp4) {
    // e2m1 operands with a K-permutation inside each 32-element group: source bit j of a
    // 32-bit word goes to output word j % 4, nibble j / 4, so output word q collects bits
    // q, q+4, ... shifted into one bit position of every nibble. Both GEMM operands use the
    // same permutation, so every dot product is unchanged. Codes (e2m1 values):
    //   signs : +1 -> 0x2 (1.0), -1 -> 0xA (-1.0), padding -> 0x0
    //   levels: p -> p as a nibble = p / 2 (0, 0.5, 1, 1.5), exact; the GEMM's epilogue
    //           shift adds a factor 2 per level operand (fp4_shift, bitmm_capi.cu)
    // Full words take two instructions per output word (a funnel shift and one LOP3).
    // Lane t writes the 16 output bytes of its own word: each warp store covers 512
    // contiguous bytes.
    uint8_t* out_row = o.out + r * (kpad / 2);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int g = word0 + j * 32 + lane;
      if (g * 32 >= kpad) continue;
      uint32_t ow[4];
      const uint32_t valid = valid_mask32(g * 32, K);
      if (o.levels == 0) {
        if (valid == 0xFFFFFFFFu) {
          const uint32_t w = s.w0[j];
          // bit 4n+q -> nibble n bit 3 (the sign), then 0x2 in every nibble
          ow[0] = (~(w << 3) & 0x88888888u) | 0x22222222u;
          ow[1] = (~(w << 2) & 0x88888888u) | 0x22222222u;
          ow[2] = (~(w << 1) & 0x88888888u) | 0x22222222u;
          ow[3] = (~w & 0x88888888u) | 0x22222222u;
        } else {
          const uint32_t neg = valid & ~s.w0[j];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            ow[q] = (((valid >> q) & 0x11111111u) << 1) | (((neg >> q) & 0x11111111u) << 3);
        }
      } else {
        const uint32_t hi = s.w0[j], lo = s.w1[j];  // already masked to K
        ow[0] = ((hi << 1) & 0x22222222u) | (lo & 0x11111111u);
        ow[1] = (hi & 0x22222222u) | ((lo >> 1) & 0x11111111u);
        ow[2] = ((hi >> 1) & 0x22222222u) | ((lo >> 2) & 0x11111111u);
        ow[3] = ((hi >> 2) & 0x22222222u) | ((lo >> 3) & 0x11111111u);
      }
      *reinterpret_cast<uint4*>(out_row + static_cast<long long>(g) * 16) =
          make_uint4(ow[0], ow[1], ow[2], ow[3]);
    }
    return __reduce_or_sync(0xFFFFFFFFu, bad);
  }
  uint8_t* out_row = o.out + r * kpad;
  const bool full_slice = (word0 + 128) * 32 <= K;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int chunk = v * 32 + lane;
    const int elem = word0 * 32 + chunk * 16;
    const int src_lane = (v & 1) * 16 + (lane >> 1);
    const int shift = (lane & 1) * 16;
    const uint32_t a = __shfl_sync(0xFFFFFFFFu, s.w0[v >> 1], src_lane);
    const uint32_t b = __shfl_sync(0xFFFFFFFFu, s.w1[v >> 1], src_lane);
    if (elem >= kpad) continue;
    uint32_t ow[4];
    if (o.levels == 0) {
      const uint32_t bits = (a >> shift) & 0xFFFFu;
      if (full_slice) {  // warp-uniform: every element of the slice is inside K
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ow[q] = ~(spread4((bits >> (4 * q)) & 0xFu) * 0xFEu);  // 1 -> +1, 0 -> -1
      } else {
        const int g = word0 + (chunk >> 1);
        const uint32_t valid = (valid_mask32(g * 32, K) >> shift) & 0xFFFFu;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t bb = spread4((bits >> (4 * q)) & 0xFu);
          const uint32_t vm = spread4((valid >> (4 * q)) & 0xFu);
          ow[q] = ((bb * 0xFEu) ^ 0xFFFFFFFFu) & (vm * 0xFFu);  // 1 -> +1, 0 -> -1, pad -> 0
        }
      }
    } else {
      const uint32_t hi = (a >> shift) & 0xFFFFu;
      const uint32_t lo = (b >> shift) & 0xFFFFu;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        ow[q] = (spread4((hi >> (4 * q)) & 0xFu) << 1) + spread4((lo >> (4 * q)) & 0xFu);
    }
    *reinterpret_cast<uint4*>(out_row + elem) = make_uint4(ow[0], ow[1], ow[2], ow[3]);
  }
  return __reduce_or_sync(0xFFFFFFFFu, bad);
}

// Fast path of the e2m1 expansion for a slice lying wholly inside K and inside the words
// of the row (every slice when K is a multiple of 4096): no per-word bounds checks, one base
// address per plane and immediate offsets, so the warp spends its instructions on loads,
// validation, expansion and stores. Same output and flags as expand_slice_warp.
__device__ __forceinline__ int unpack_slice_fp4_full(const UnpackOperand& o, long long r, int sl,
                                                     int lane) {
  const long long src = r * o.wpr32 + sl * 128 + lane;
  uint4* dst = reinterpret_cast<uint4*>(o.out + r * (o.kpad / 2)) + sl * 128 + lane;
  if (o.levels == 0) {
    const uint32_t* w0 = o.w0 + src;
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) w[j] = __ldg(w0 + 32 * j);
#pragma unroll
    for (int j = 0; j < 4; ++j)  // +1 -> 0x2, -1 -> 0xA (see expand_slice_warp)
      dst[32 * j] = make_uint4((~(w[j] << 3) & 0x88888888u) | 0x22222222u,
                               (~(w[j] << 2) & 0x88888888u) | 0x22222222u,
                               (~(w[j] << 1) & 0x88888888u) | 0x22222222u,
                               (~w[j] & 0x88888888u) | 0x22222222u);
    return 0;
  }
  const uint32_t *pt = o.w0 + src, *ph = o.w1 + src, *pm = o.w2 + src;
  uint32_t t[4], h[4], m[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    t[j] = __ldg(pt + 32 * j);
    h[j] = __ldg(ph + 32 * j);
    m[j] = __ldg(pm + 32 * j);
  }
  uint32_t illegal = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    // legal (t,h,m): (0,0,1) (0,0,0) (0,1,0) (1,0,1) (transform.cpp:56-71)
    illegal |= (t[j] & h[j]) | (t[j] & ~m[j]) | (h[j] & m[j]);
    const uint32_t hi = t[j] | h[j], lo = t[j] | ~(h[j] | m[j]);  // p = 2 hi + lo
    dst[32 * j] = make_uint4(((hi << 1) & 0x22222222u) | (lo & 0x11111111u),
                             (hi & 0x22222222u) | ((lo >> 1) & 0x11111111u),
                             ((hi >> 1) & 0x22222222u) | ((lo >> 2) & 0x11111111u),
                             ((hi >> 2) & 0x22222222u) | ((lo >> 3) & 0x11111111u));
  }
  return __any_sync(0xFFFFFFFFu, illegal != 0) ? ERR_ENCODING : 0;
}

__device__ __forceinline__ int unpack_slice_warp(const UnpackOperand& o, long long r, int sl, int K,
                                                 int kpad, int lane, bool fp4) {
  SliceWords s;
  load_slice_warp(o, r, sl, lane, s);
  return expand_slice_warp(o, r, sl, K, kpad, lane, s, fp4);
}

// Standalone expansion of both GEMM operands (blockIdx.y selects the operand).
// PDL: waits for its predecessor before touching the workspace, then lets the GEMM that
// consumes its output launch early (the GEMM's prologue overlaps this kernel's tail).
// A variant that deferred this wait to the end, to overlap with the previous GEMM, deadlocked
// nondeterministically on B200 (dependent blocks parked in griddepcontrol.wait while holding
// SM slots); see DESIGN.md.
__global__ void __launch_bounds__(256) unpack_operands(const __grid_constant__ UnpackSet P) {
  pdl_wait();
  pdl_launch_dependents();
  // Grid row 0 holds the level chunks when there are any (scheduled first, so they overlap the
  // operand rows instead of trailing them); the operands follow.
  const int y = static_cast<int>(blockIdx.y) - (P.lc.chunks > 0 ? 1 : 0);
  if (y < 0) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < level_chunk_items(P.lc)) level_chunk_item(P.lc, i);
    return;
  }
  const UnpackOperand& o = P.op[y];
  const long long unit = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long slices = o.groups_per_row;  // slices of 128 words per row
  if (unit >= o.rows * slices) return;
  long long r;
  int sl;
  if (slices == 1) {  // K <= 4096: one slice per row
    r = unit;
    sl = 0;
  } else if (o.rows * slices < (1ll << 31)) {  // 32-bit division (the 64-bit one is ~4x longer)
    const unsigned q = static_cast<unsigned>(unit) / static_cast<unsigned>(slices);
    r = q;
    sl = static_cast<int>(static_cast<unsigned>(unit) - q * static_cast<unsigned>(slices));
  } else {
    r = unit / slices;
    sl = static_cast<int>(unit - r * slices);
  }
  // warp-uniform: the slice's 4096 elements are all inside K and inside the row's words
  const bool full = (sl + 1) * 128 <= o.wpr32 && (sl + 1) * 4096 <= o.K;
  const int bad = !P.fp4 ? unpack_slice_warp(o, r, sl, o.K, o.kpad, lane, false)
                  : full ? unpack_slice_fp4_full(o, r, sl, lane)
                         : unpack_slice_warp(o, r, sl, o.K, o.kpad, lane, true);
  if (bad && lane == 0) atomicOr(P.err, bad);
}

// ---- Flat expansion through the bulk-copy engine (e2m1 operands without padding) ----
// An operand whose rows hold no padding (K = 32 * wpr32, a multiple of 256, so kpad = K) is a
// flat array of words whose e2m1 image is position-preserving: word i (row-major) expands to
// output bytes [16 i, 16 i + 16), nibble order as unpack_slice_fp4_full. A block streams chunks
// of UF_CHUNK words into shared memory with one bulk copy per plane, expands them with shared
// loads and stores, and writes the chunk's e2m1 bytes back with one bulk store, double-buffered:
// no per-thread global loads or stores, so neither the warps' load latency nor the load/store
// unit's queue (the per-slice kernel above: long-scoreboard and lg_throttle stalls) paces it.
constexpr int UF_CHUNK = 2048;   // words per chunk
constexpr int UF_THREADS = 256;
constexpr int UF_IN = 3 * UF_CHUNK * 4;  // 24 KB: up to three planes
constexpr int UF_OUT = UF_CHUNK * 16;    // 32 KB of e2m1
constexpr int UF_SMEM = 2 * (UF_IN + UF_OUT) + 128;

struct UnpackFlat {
  UnpackOperand op[UNPACK_MAX_OPS];
  long long chunk_begin[UNPACK_MAX_OPS + 1];  // operand i owns chunks [chunk_begin[i], chunk_begin[i + 1])
  int count;
  int* err;
};

__global__ void __launch_bounds__(UF_THREADS) unpack_flat_kernel(const __grid_constant__ UnpackFlat P) {
  extern __shared__ __align__(128) uint8_t uf_smem[];
  uint8_t* in_s = uf_smem;                 // [stage][plane][UF_CHUNK words]
  uint8_t* out_s = uf_smem + 2 * UF_IN;    // [stage][UF_OUT]
  uint64_t* full = reinterpret_cast<uint64_t*>(out_s + 2 * UF_OUT);
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();  // the previous kernel may still read the workspace we overwrite
  pdl_launch_dependents();
  const long long total = P.chunk_begin[P.count];
  // chunk c -> operand, first word, word count
  auto locate = [&](long long c, int& oi, long long& w0, int& nw) {
    oi = 0;
    for (int i = 1; i < P.count; ++i)
      if (c >= P.chunk_begin[i]) oi = i;
    const UnpackOperand& o = P.op[oi];
    w0 = (c - P.chunk_begin[oi]) * UF_CHUNK;
    nw = static_cast<int>(min(static_cast<long long>(UF_CHUNK), o.rows * o.wpr32 - w0));
  };
  auto issue = [&](long long c, int stage) {  // thread 0: the chunk's planes into `stage`
    int oi, nw;
    long long w0;
    locate(c, oi, w0, nw);
    const UnpackOperand& o = P.op[oi];
    const uint32_t bytes = static_cast<uint32_t>(nw) * 4;
    fence_proxy_async_smem();  // earlier generic reads of the stage before the async writes
    mbar_arrive_expect_tx(&full[stage], bytes * (o.levels ? 3 : 1));
    uint8_t* dst = in_s + stage * UF_IN;
    bulk_load_1d(dst, o.w0 + w0, bytes, &full[stage]);
    if (o.levels) {
      bulk_load_1d(dst + UF_CHUNK * 4, o.w1 + w0, bytes, &full[stage]);
      bulk_load_1d(dst + 2 * UF_CHUNK * 4, o.w2 + w0, bytes, &full[stage]);
    }
  };
  uint32_t illegal = 0;
  uint32_t phase = 0;  // bit s: parity of stage s
  if (tid == 0 && static_cast<long long>(blockIdx.x) < total) issue(blockIdx.x, 0);
  int it = 0;
  for (long long c = blockIdx.x; c < total; c += gridDim.x, ++it) {
    const int st = it & 1;
    // the other stage's input was read by every thread before the last __syncthreads
    if (tid == 0 && c + gridDim.x < total) issue(c + gridDim.x, st ^ 1);
    mbar_wait(&full[st], (phase >> st) & 1u);
    phase ^= 1u << st;
    if (tid == 0) bulk_wait_group_read<1>();  // out_s[st]'s store (two chunks ago) has read it
    __syncthreads();
    int oi, nw;
    long long w0;
    locate(c, oi, w0, nw);
    const UnpackOperand& o = P.op[oi];
    const uint32_t* pin = reinterpret_cast<const uint32_t*>(in_s + st * UF_IN);
    uint4* pout = reinterpret_cast<uint4*>(out_s + st * UF_OUT);
    if (!o.levels) {
      for (int i = tid; i < nw; i += UF_THREADS) {  // +1 -> 0x2, -1 -> 0xA
        const uint32_t w = pin[i];
        pout[i] = make_uint4((~(w << 3) & 0x88888888u) | 0x22222222u, (~(w << 2) & 0x88888888u) | 0x22222222u,
                             (~(w << 1) & 0x88888888u) | 0x22222222u, (~w & 0x88888888u) | 0x22222222u);
      }
    } else {
      for (int i = tid; i < nw; i += UF_THREADS) {
        const uint32_t t = pin[i], h = pin[UF_CHUNK + i], m = pin[2 * UF_CHUNK + i];
        // legal (t,h,m): (0,0,1) (0,0,0) (0,1,0) (1,0,1) (transform.cpp:56-71)
        illegal |= (t & h) | (t & ~m) | (h & m);
        const uint32_t hi = t | h, lo = t | ~(h | m);  // p = 2 hi + lo
        pout[i] = make_uint4(((hi << 1) & 0x22222222u) | (lo & 0x11111111u),
                             (hi & 0x22222222u) | ((lo >> 1) & 0x11111111u),
                             ((hi >> 1) & 0x22222222u) | ((lo >> 2) & 0x11111111u),
                             ((hi >> 2) & 0x22222222u) | ((lo >> 3) & 0x11111111u));
      }
    }
    fence_proxy_async_smem();  // the expanded bytes before the bulk store reads them
    __syncthreads();
    if (tid == 0) {
      bulk_store_1d(o.out + w0 * 16, pout, static_cast<uint32_t>(nw) * 16);
      bulk_commit_group();
    }
  }
  if (tid == 0) bulk_wait_group_all();
  if (__syncthreads_or(illegal != 0) && tid == 0) atomicOr(P.err, ERR_ENCODING);
}

__global__ void unpack_level_i8(const uint32_t* __restrict__ t, const uint32_t* __restrict__ h,
                                const uint32_t* __restrict__ m, long long rows, int wpr32, int K,
                                int kpad, uint8_t* __restrict__ out, int* __restrict__ err) {
  const int groups_out = kpad / 32;
  const int groups = max(groups_out, wpr32);
  const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= rows * groups) return;
  const long long r = gid / groups;
  const int g = static_cast<int>(gid - r * groups);
  uint32_t tw = 0, hw = 0, mw = 0;
  if (g < wpr32) {
    tw = t[r * wpr32 + g];
    hw = h[r * wpr32 + g];
    mw = m[r * wpr32 + g];
  }
  const uint32_t valid = valid_mask32(g * 32, K);
  if (((tw | hw | mw) & ~valid) | (tw & hw) | (tw & ~mw) | (hw & mw)) atomicOr(err, ERR_ENCODING);
  if (g >= groups_out) return;
  const uint32_t hi = (tw | hw) & valid;
  const uint32_t lo = (tw | ~(hw | mw)) & valid;
  uint32_t o[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    o[q] = (spread4((hi >> (4 * q)) & 0xFu) << 1) + spread4((lo >> (4 * q)) & 0xFu);
  }
  uint4* dst = reinterpret_cast<uint4*>(out + r * kpad + g * 32);
  dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
  dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
}

__global__ void unpack_sign_f16(const uint32_t* __restrict__ words, long long rows, int wpr32,
                                int K, int kpad, uint16_t* __restrict__ out,
                                int* __restrict__ err) {
  pdl_wait();  // the previous kernel may still read the workspace we overwrite
  pdl_launch_dependents();
  const int groups_out = kpad / 32;
  const int groups = max(groups_out, wpr32);
  const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= rows * groups) return;
  const long long r = gid / groups;
  const int g = static_cast<int>(gid - r * groups);
  const uint32_t w = (g < wpr32) ? words[r * wpr32 + g] : 0u;
  const uint32_t valid = valid_mask32(g * 32, K);
  if (w & ~valid) atomicOr(err, ERR_PADDING);
  if (g >= groups_out) return;
  uint32_t o[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const uint32_t b0 = (w >> (2 * q)) & 1u, b1 = (w >> (2 * q + 1)) & 1u;
    const uint32_t v0 = (valid >> (2 * q)) & 1u, v1 = (valid >> (2 * q + 1)) & 1u;
    const uint32_t e0 = v0 ? (b0 ? 0x3C00u : 0xBC00u) : 0u;  // +1.0 / -1.0 fp16
    const uint32_t e1 = v1 ? (b1 ? 0x3C00u : 0xBC00u) : 0u;
    o[q] = e0 | (e1 << 16);
  }
  uint4* dst = reinterpret_cast<uint4*>(out + r * kpad + g * 32);
#pragma unroll
  for (int q = 0; q < 4; ++q) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
}

// Per-token scale of the fp16 split: tok_scale[n] = 2^-e_n with max_k |X[k][n]| * 2^e_n in
// [2^14, 2^15) (e_n = 0 when the maximum is 0 or not finite; |e_n| <= 126). One block per
// 32-token strip, 32 warps each reading every 32nd K row (coalesced 128-byte rows).
__global__ void __launch_bounds__(1024) x_token_scale(const float* __restrict__ X, long long ldx,
                                                      int K, int N, float* __restrict__ tok_scale) {
  __shared__ float red[32][33];
  pdl_wait();
  pdl_launch_dependents();
  const int n0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  float mx = 0.f;
  if (n0 + tx < N) {
#pragma unroll 4
    for (int k = ty; k < K; k += 32) mx = fmaxf(mx, fabsf(X[static_cast<long long>(k) * ldx + n0 + tx]));
  }
  red[ty][tx] = mx;
  __syncthreads();
  if (ty == 0) {
#pragma unroll
    for (int i = 1; i < 32; ++i) mx = fmaxf(mx, red[i][tx]);
    int e = 0;
    if (mx > 0.f && mx <= 3.402823466e38f) {
      int q;
      frexpf(mx, &q);  // mx = f * 2^q, f in [0.5, 1)
      e = min(126, max(-126, 15 - q));
    }
    if (n0 + tx < N) tok_scale[n0 + tx] = ldexpf(1.0f, -e);
  }
}

// X [K][ldx] fp32 -> XT [N][2*kpad] fp16, hi at column 0 and lo at column kpad, with x
// scaled by 1 / tok_scale[n] = 2^e_n (exact). hi = rn_f16(x * 2^e_n), lo = rn_f16(x * 2^e_n
// - hi) (the difference is exact in fp32), so only lo's rounding is lost: <= 2^-22 of |x|
// while lo stays a normal fp16 number. Block = 256 threads, tile 64 k x 32 n; reads
// coalesced along n, writes 128 B segments along k per part.
__global__ void split_x_f16(const float* __restrict__ X, long long ldx, int K, int N, int kpad,
                            const float* __restrict__ tok_scale, uint16_t* __restrict__ XT) {
  __shared__ float tile[64][33];
  pdl_wait();
  pdl_launch_dependents();
  const int k0 = blockIdx.x * 64;
  const int n0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = k0 + ty + 8 * i;
    const int n = n0 + tx;
    tile[ty + 8 * i][tx] = (k < K && n < N) ? X[static_cast<long long>(k) * ldx + n] : 0.0f;
  }
  __syncthreads();
  const int nl = threadIdx.x >> 3;        // 0..31
  const int kl = (threadIdx.x & 7) * 8;   // 0..56
  const int n = n0 + nl;
  if (n >= N) return;
  const float sc = __frcp_rn(tok_scale[n]);  // 2^e_n, exact
  uint32_t hi2[4], lo2[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t h[2], l[2];
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      const float xs = tile[kl + 2 * q + d][nl] * sc;  // exact: a power of two
      const __half hv = __float2half_rn(xs);
      const __half lv = __float2half_rn(xs - __half2float(hv));
      h[d] = __half_as_ushort(hv);
      l[d] = __half_as_ushort(lv);
    }
    hi2[q] = h[0] | (h[1] << 16);
    lo2[q] = l[0] | (l[1] << 16);
  }
  uint16_t* row = XT + static_cast<long long>(n) * 2 * kpad + k0 + kl;
  *reinterpret_cast<uint4*>(row) = make_uint4(hi2[0], hi2[1], hi2[2], hi2[3]);
  *reinterpret_cast<uint4*>(row + kpad) = make_uint4(lo2[0], lo2[1], lo2[2], lo2[3]);
}

// x_token_scale + split_x_f16 in one pass for K small enough that a 32-token strip of X
// fits in shared memory (kpad * 128 B; config 4: 96 KB, two blocks per SM): the block stages
// its strip [kpad][32] fp32 (16-byte chunk c of row k at c ^ ((k >> 3) & 7), so both the
// cp.async writes and the transposed reads below are conflict-free), takes each token's
// maximum, and splits from shared memory. X is read once instead of twice, and the whole
// matrix is in flight in one wave. Same outputs as the two-kernel path.
__device__ __forceinline__ int strip_idx(int k, int n) {
  return k * 32 + ((((n >> 2) ^ (k >> 3)) & 7) << 2) + (n & 3);
}

__global__ void __launch_bounds__(256) split_x_f16_strip(const float* __restrict__ X, long long ldx,
                                                         int K, int N, int kpad,
                                                         float* __restrict__ tok_scale,
                                                         uint16_t* __restrict__ XT) {
  extern __shared__ float xs[];  // [kpad][32], swizzled
  __shared__ float red[8][33];
  __shared__ float sscale[32];
  pdl_wait();
  pdl_launch_dependents();
  const int n0 = blockIdx.x * 32;
  const int tid = threadIdx.x;
  const bool vec = n0 + 32 <= N && (ldx & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  // stage the strip: 8 chunks of 16 B per row; rows past K and tokens past N are zero
  for (int i = tid; i < kpad * 8; i += 256) {
    const int k = i >> 3, c = i & 7;
    float* dst = &xs[k * 32 + (((c ^ (k >> 3)) & 7) << 2)];
    const float* src = X + static_cast<long long>(k) * ldx + n0 + 4 * c;
    if (k < K && vec) {
      cp_async16(dst, src);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) dst[e] = (k < K && n0 + 4 * c + e < N) ? src[e] : 0.0f;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  {
    const int n = tid & 31;
    float mx = 0.f;
    for (int k = tid >> 5; k < K; k += 8) mx = fmaxf(mx, fabsf(xs[strip_idx(k, n)]));
    red[tid >> 5][n] = mx;
  }
  __syncthreads();
  if (tid < 32) {
    float mx = red[0][tid];
#pragma unroll
    for (int i = 1; i < 8; ++i) mx = fmaxf(mx, red[i][tid]);
    int e = 0;
    if (mx > 0.f && mx <= 3.402823466e38f) {
      int q;
      frexpf(mx, &q);  // mx = f * 2^q, f in [0.5, 1)
      e = min(126, max(-126, 15 - q));
    }
    sscale[tid] = ldexpf(1.0f, e);
    if (n0 + tid < N) tok_scale[n0 + tid] = ldexpf(1.0f, -e);
  }
  __syncthreads();
  const int nl = tid >> 3;        // token 0..31
  const int kl = (tid & 7) * 8;   // 8 consecutive k per thread
  const int n = n0 + nl;
  if (n >= N) return;
  const float sc = sscale[nl];
  uint16_t* row = XT + static_cast<long long>(n) * 2 * kpad;
  for (int k0 = 0; k0 < kpad; k0 += 64) {
    uint32_t hi2[4], lo2[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t h[2], l[2];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        const float xv = xs[strip_idx(k0 + kl + 2 * q + d, nl)] * sc;  // exact: a power of two
        const __half hv = __float2half_rn(xv);
        const __half lv = __float2half_rn(xv - __half2float(hv));
        h[d] = __half_as_ushort(hv);
        l[d] = __half_as_ushort(lv);
      }
      hi2[q] = h[0] | (h[1] << 16);
      lo2[q] = l[0] | (l[1] << 16);
    }
    *reinterpret_cast<uint4*>(row + k0 + kl) = make_uint4(hi2[0], hi2[1], hi2[2], hi2[3]);
    *reinterpret_cast<uint4*>(row + kpad + k0 + kl) = make_uint4(lo2[0], lo2[1], lo2[2], lo2[3]);
  }
}

}  // namespace bitmm_dev
