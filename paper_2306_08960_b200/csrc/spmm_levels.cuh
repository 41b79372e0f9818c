// Residual pass of the APB layer with 2-bit activations (sm_100a): C[r][t] += S[r][t],
//   S[r][t] = (...((+0 + v_1 * D[c_1][t]) + v_2 * D[c_2][t]) + ...)   in col_idx order,
//   D[c][t] = float(p_t(c)) * (s * gamma_a)                            (kernels.cpp:334-352,
// each product and sum rounded to fp32, the reference's spmm_csr over the dequantized levels of
// apb.cpp:158-164 / PAPER.md:1119-1122), then C = fl(G + S) over the binary part G the 1/2 GEMM
// stored. Bit for bit.
//
// The earlier form (spmm_xchunk_kernel<..., LEVELS>) staged D as fp32 and read 4 bytes of
// shared memory per product: it was bound by the shared-memory/shuffle (MIO) pipe. Here a
// block stages the level of each (column, token) as the bf16 pattern of p in {0, 1, 2, 3}
// (exact; 2 bytes), and the arithmetic runs on fp32 pairs (FMUL2 / FADD2, sm_100a):
//   d  = fl(p * sg)        one FMUL2 per two tokens (= the reference's D[c][t] exactly)
//   q  = fl(v * d)         one FMUL2
//   S  = fl(S + q)         one FADD2
// so a product costs 2 bytes of shared memory and 1.5 pair instructions instead of 4 bytes and
// 2 scalar instructions. bf16 -> fp32 is a shift / mask of the 32-bit word holding two
// tokens. Layout: an 8-lane octet owns one output row and a 64-token chunk, lane l owns 8
// consecutive tokens (one 16-byte load per nonzero; an octet reads one whole 128-byte X row,
// conflict-free), nonzeros are broadcast with octet shuffles.
#pragma once

#include "apb_gemm.cuh"
#include "levels.cuh"

namespace bitmm_dev {

#ifndef SL_THREADS_CFG  // profiling builds sweep these (profiles/dev/ab_spmm_levels.py)
#define SL_THREADS_CFG 768
#endif
#ifndef SL_MINB_CFG
#define SL_MINB_CFG 1
#endif
#ifndef SL_CPREF
#define SL_CPREF 1
#endif
constexpr int SL_THREADS = SL_THREADS_CFG;   // 96 octets, one block per SM (measured best of 256..1024 x 1..3)
constexpr int SL_BLOCKS_PER_SM = SL_MINB_CFG;
constexpr int SL_OCTETS = SL_THREADS / 8;    // rows in flight per block

// Dynamic smem: the level chunk [K + 1][SL_TOK] bf16 (row K is zero: the target of padded
// nonzeros), then the block's row offsets (u32).
inline int spmm_levels_smem_bytes(long long K, int rows_per_split, bool f32 = false) {
  return static_cast<int>((K + 1) * (f32 ? SL_TOK * 4 : SL_ROW_WORDS * 4) + (rows_per_split + 1) * 4);
}

__device__ __forceinline__ unsigned long long f32x2_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
// fl(a * b) per element, written as fma(a, b, z) with z = (-0, -0) (exact: adding -0 changes no
// product, and +0 + -0 = +0 keeps a zero product's sign). ptxas contracts a mul.rn.f32x2 that
// feeds an add.rn.f32x2 into FFMA2 even with the explicit rounding modifier, and folds an fma
// with a constant -0 addend back into a multiply; z comes from a kernel parameter, so neither
// happens and each product is rounded as in the reference.
__device__ __forceinline__ unsigned long long f32x2_mul(unsigned long long a, unsigned long long b,
                                                         unsigned long long z) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(z));
  return r;
}
__device__ __forceinline__ unsigned long long f32x2_add(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}


// The whole chunk (rows [0, K) plus the zero row K), by threads tid of nthreads. Each store
// instruction of a warp writes one whole 128-byte column row.
__device__ __forceinline__ void sl_stage(unsigned* xw, int K, int N, int c0, const SpmmLevels& lv, int tid,
                                         int nthreads) {
  if (tid < SL_ROW_WORDS) xw[K * SL_ROW_WORDS + tid] = 0u;
  const int items = ((K + 63) >> 6) * 2 * SL_ROW_WORDS;
  for (int i = tid; i < items; i += nthreads) sl_stage_item(xw, K, N, c0, lv, i);
}

// One octet's view of a staged chunk: lane `ol` of the octet owns tokens [8 ol, 8 ol + 8).
struct SlOctet {
  const char* xrow;         // chunk base + 16 ol bytes
  int obase;                // first lane of the octet in the warp
  unsigned long long dd;    // (d1, d1), d1 = fl(1 * sg) = sg
  unsigned long long z;     // (-0, -0) from a kernel parameter (see f32x2_mul)
};

// Eight nonzeros of the octet's row, (kk, vv) held by octet lane j for slot j (padded slots:
// the zero row, weight 0 — they add fl(0 * 0) = +0, which leaves a sum that started at +0
// bit-identical: it never becomes -0). acc[q] = token pair (8 ol + 2 q, 8 ol + 2 q + 1).
__device__ __forceinline__ void sl_step8(const SlOctet& o, unsigned kk, float vv, unsigned long long (&acc)[4]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const unsigned koff = __shfl_sync(0xFFFFFFFFu, kk, o.obase + j) * (SL_ROW_WORDS * 4);
    const float v = __shfl_sync(0xFFFFFFFFu, vv, o.obase + j);
    const uint4 x = *reinterpret_cast<const uint4*>(o.xrow + koff);
    const unsigned long long v2 = f32x2_pack(v, v);
    const unsigned xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // low token: PRMT (ALU pipe; a plain shift becomes IMAD.U32 on the FMA pipe, which the
      // pair arithmetic already saturates); high token: mask
      unsigned lo16;
      asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(lo16) : "r"(xs[q]));
      const unsigned long long p2 = f32x2_pack(__uint_as_float(lo16), __uint_as_float(xs[q] & 0xFFFF0000u));
      acc[q] = f32x2_add(acc[q], f32x2_mul(v2, f32x2_mul(p2, o.dd, o.z), o.z));
    }
  }
}

// sl_step8 for two rows of the octet at once (independent chains: twice the work in flight per
// warp, for kernels with few residual warps per SM).
__device__ __forceinline__ void sl_step8x2(const SlOctet& o, unsigned kka, float vva, unsigned long long (&acca)[4],
                                           unsigned kkb, float vvb, unsigned long long (&accb)[4]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const unsigned koffa = __shfl_sync(0xFFFFFFFFu, kka, o.obase + j) * (SL_ROW_WORDS * 4);
    const float va = __shfl_sync(0xFFFFFFFFu, vva, o.obase + j);
    const unsigned koffb = __shfl_sync(0xFFFFFFFFu, kkb, o.obase + j) * (SL_ROW_WORDS * 4);
    const float vb = __shfl_sync(0xFFFFFFFFu, vvb, o.obase + j);
    const uint4 xa = *reinterpret_cast<const uint4*>(o.xrow + koffa);
    const uint4 xb = *reinterpret_cast<const uint4*>(o.xrow + koffb);
    const unsigned long long va2 = f32x2_pack(va, va), vb2 = f32x2_pack(vb, vb);
    const unsigned xsa[4] = {xa.x, xa.y, xa.z, xa.w}, xsb[4] = {xb.x, xb.y, xb.z, xb.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      unsigned la, lb;
      asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(la) : "r"(xsa[q]));
      asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(lb) : "r"(xsb[q]));
      const unsigned long long pa = f32x2_pack(__uint_as_float(la), __uint_as_float(xsa[q] & 0xFFFF0000u));
      const unsigned long long pb = f32x2_pack(__uint_as_float(lb), __uint_as_float(xsb[q] & 0xFFFF0000u));
      acca[q] = f32x2_add(acca[q], f32x2_mul(va2, f32x2_mul(pa, o.dd, o.z), o.z));
      accb[q] = f32x2_add(accb[q], f32x2_mul(vb2, f32x2_mul(pb, o.dd, o.z), o.z));
    }
  }
}

// sl_step8 over an fp32 chunk [K + 1][SL_TOK] (the standalone spmm_csr): lane l of the octet owns
// tokens [4 l, 4 l + 4) and [32 + 4 l, 32 + 4 l + 4), so each of its two 16-byte loads is part of
// one contiguous 128-byte octet read. acc[0..1] = the first four tokens, acc[2..3] the second.
__device__ __forceinline__ void sl_step8_f32(const SlOctet& o, unsigned kk, float vv, unsigned long long (&acc)[4]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const unsigned koff = __shfl_sync(0xFFFFFFFFu, kk, o.obase + j) * (SL_TOK * 4);
    const float v = __shfl_sync(0xFFFFFFFFu, vv, o.obase + j);
    const uint4 x0 = *reinterpret_cast<const uint4*>(o.xrow + koff);
    const uint4 x1 = *reinterpret_cast<const uint4*>(o.xrow + koff + 128);
    const unsigned long long v2 = f32x2_pack(v, v);
    const unsigned long long xs[4] = {f32x2_pack(__uint_as_float(x0.x), __uint_as_float(x0.y)),
                                      f32x2_pack(__uint_as_float(x0.z), __uint_as_float(x0.w)),
                                      f32x2_pack(__uint_as_float(x1.x), __uint_as_float(x1.y)),
                                      f32x2_pack(__uint_as_float(x1.z), __uint_as_float(x1.w))};
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = f32x2_add(acc[q], f32x2_mul(v2, xs[q], o.z));  // fl(S + fl(v x))
  }
}

// Persistent: gridDim.x = blocks resident at once (SL_BLOCKS_PER_SM per SM), block b owns the contiguous
// range [b W, (b + 1) W) of the (token chunk, row) work space in chunk-major order, so every block
// gets the same number of rows (no partial last wave) and restages only when its range crosses
// into the next chunk (at most twice).
// F32: the standalone exact spmm_csr (kernels.cpp:334-352) over an fp32 X [K][ldx]: the chunk is
// [K + 1][SL_TOK] fp32 (cp.async), products fl(v * x), and C = S is stored (no binary part).
template <bool PDL_CHAIN, bool F32 = false>
__global__ void __launch_bounds__(SL_THREADS, SL_BLOCKS_PER_SM)
    spmm_levels_kernel(int rows, int K, int N, const unsigned long long* __restrict__ row_ptr,
                       const unsigned long long* __restrict__ col_idx, const float* __restrict__ vals,
                       const SpmmLevels lv, float* __restrict__ C, long long ldc, long long work_per_block,
                       const float* __restrict__ X = nullptr, long long ldx = 0) {
  extern __shared__ unsigned xw[];  // [K + 1][SL_ROW_WORDS] (F32: [K + 1][SL_TOK]), then u32 row offsets
  constexpr int ROW_WORDS = F32 ? SL_TOK : SL_ROW_WORDS;
  if (PDL_CHAIN) {
    pdl_wait();  // C holds the GEMM's binary part
    pdl_launch_dependents();
  }
  unsigned* rps = xw + static_cast<long long>(K + 1) * ROW_WORDS;
  const long long chunks = (N + SL_TOK - 1) / SL_TOK;
  const long long total = chunks * rows;
  long long lo = blockIdx.x * work_per_block;
  const long long hi = min(total, lo + work_per_block);
  while (lo < hi) {
    const int chunk = static_cast<int>(lo / rows);
    const long long seg_end = min(hi, (chunk + 1LL) * rows);
    const int c0 = chunk * SL_TOK;
    const int r0 = static_cast<int>(lo - static_cast<long long>(chunk) * rows);
    const int r1 = static_cast<int>(seg_end - static_cast<long long>(chunk) * rows);
    lo = seg_end;
    __syncthreads();  // the previous segment's rows are done with the chunk and the offsets

    if constexpr (F32) {
      // X rows [0, K) of the chunk: every 16-byte piece in flight at once, zero past N
      const bool xvec = ((ldx & 3) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
      float* xf = reinterpret_cast<float*>(xw);
      if (threadIdx.x < SL_TOK) xf[static_cast<long long>(K) * SL_TOK + threadIdx.x] = 0.f;
      for (int i = threadIdx.x; i < K * (SL_TOK / 4); i += SL_THREADS) {
        const int k = i / (SL_TOK / 4), q = (i % (SL_TOK / 4)) * 4;
        const float* src = X + static_cast<long long>(k) * ldx + c0 + q;
        float* dst = &xf[static_cast<long long>(k) * SL_TOK + q];
        if (xvec && c0 + q + 3 < N) {
          cp_async16(dst, src);
        } else {
          for (int e = 0; e < 4; ++e) dst[e] = (c0 + q + e < N) ? src[e] : 0.f;
        }
      }
      cp_async_wait_all();
    } else {
      sl_stage(xw, K, N, c0, lv, threadIdx.x, SL_THREADS);
    }
    const unsigned long long nz0 = row_ptr[r0];
    for (int i = threadIdx.x; i <= r1 - r0; i += SL_THREADS) rps[i] = static_cast<unsigned>(row_ptr[r0 + i] - nz0);
    __syncthreads();

    const int oct = threadIdx.x >> 3;
    const int ol = threadIdx.x & 7;
    const int lane = threadIdx.x & 31;
    const int obase = lane & ~7;
    const int col = c0 + ol * 8;
    const bool vec = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && col + 7 < N;
    const unsigned long long* cbase = col_idx + nz0;
    const float* vbase = vals + nz0;
    const int iters = (r1 - r0 + SL_OCTETS - 1) / SL_OCTETS;
    const unsigned zero_row = static_cast<unsigned>(K);
    const SlOctet so{reinterpret_cast<const char*>(xw) + ol * 16, obase, f32x2_pack(lv.d1, lv.d1),
                     f32x2_pack(lv.neg_zero, lv.neg_zero)};
    auto step = [&](unsigned kk, float vv, unsigned long long (&acc)[4]) {
      if constexpr (F32)
        sl_step8_f32(so, kk, vv, acc);
      else
        sl_step8(so, kk, vv, acc);
    };
    auto fetch = [&](unsigned i0, unsigned n, unsigned idx, unsigned& kk, float& vv) {
      kk = zero_row;
      vv = 0.f;
      if (idx < n) {
        kk = static_cast<unsigned>(cbase[i0 + idx]);
        vv = vbase[i0 + idx];
      }
    };
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
    for (int it = 0; it < iters; ++it) {
      const int r = r0 + it * SL_OCTETS + oct;
      const bool live = r < r1;
      const unsigned nmax = __reduce_max_sync(0xFFFFFFFFu, n);
      // the next row's first 16 slots load while this row computes
      unsigned ni0 = 0, nn = 0, nkk0 = zero_row, nkk1 = zero_row;
      float nvv0 = 0.f, nvv1 = 0.f;
      {
        const int rn = r + SL_OCTETS;
        if (rn < r1) {
          ni0 = rps[rn - r0];
          nn = rps[rn - r0 + 1] - ni0;
        }
        fetch(ni0, nn, ol, nkk0, nvv0);
        fetch(ni0, nn, ol + 8, nkk1, nvv1);
      }
      // this row's binary part, loaded before the nonzero loop so the HBM round trip overlaps it
      float* dst = C + static_cast<long long>(r) * ldc + col;
      float g[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      auto load_g = [&]() {
        if (vec) {
          *reinterpret_cast<float4*>(&g[0]) = *reinterpret_cast<const float4*>(dst);
          *reinterpret_cast<float4*>(&g[4]) = *reinterpret_cast<const float4*>(dst + 4);
        } else {
          for (int e = 0; e < 8; ++e)
            if (col + e < N) g[e] = dst[e];
        }
      };
      if (!F32 && SL_CPREF && live) load_g();
      unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};  // +0 pairs
      if (nmax > 0) step(kk0, vv0, acc);
      if (nmax > 8) step(kk1, vv1, acc);
      for (unsigned base = 16; base < nmax; base += 8) {
        unsigned kk;
        float vv;
        fetch(i0, n, base + ol, kk, vv);
        step(kk, vv, acc);
      }
      if (F32 && live) {
        // C = S: tokens [4 ol, +4) and [32 + 4 ol, +4) of the chunk
        const float* af = reinterpret_cast<const float*>(acc);
        float* d0 = C + static_cast<long long>(r) * ldc + c0 + ol * 4;
        float* d1 = d0 + 32;
        const bool v0 = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
        if (v0 && c0 + ol * 4 + 3 < N) {
          *reinterpret_cast<float4*>(d0) = make_float4(af[0], af[1], af[2], af[3]);
        } else {
          for (int e = 0; e < 4; ++e)
            if (c0 + ol * 4 + e < N) d0[e] = af[e];
        }
        if (v0 && c0 + 32 + ol * 4 + 3 < N) {
          *reinterpret_cast<float4*>(d1) = make_float4(af[4], af[5], af[6], af[7]);
        } else {
          for (int e = 0; e < 4; ++e)
            if (c0 + 32 + ol * 4 + e < N) d1[e] = af[4 + e];
        }
      } else if (live) {
        if (!SL_CPREF) load_g();
        // C = fl(G + S) (apb.cpp:161-162)
        unsigned long long o[4];
  #pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = f32x2_add(f32x2_pack(g[2 * q], g[2 * q + 1]), acc[q]);
        const float* of = reinterpret_cast<const float*>(o);
        if (vec) {
          *reinterpret_cast<float4*>(dst) = make_float4(of[0], of[1], of[2], of[3]);
          *reinterpret_cast<float4*>(dst + 4) = make_float4(of[4], of[5], of[6], of[7]);
        } else {
          for (int e = 0; e < 8; ++e)
            if (col + e < N) dst[e] = of[e];
        }
      }
      i0 = ni0;
      n = nn;
      kk0 = nkk0;
      kk1 = nkk1;
      vv0 = nvv0;
      vv1 = nvv1;
    }
  }  // segments
}

}  // namespace bitmm_dev
