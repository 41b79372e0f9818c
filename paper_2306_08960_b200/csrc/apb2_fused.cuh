// APB layer with 2-bit activations, the residual fused into the 1/2 GEMM (sm_100a).
//
// C = gemm_1x2(bin, alpha_r, planes) + spmm_csr(R, D) added elementwise (apb.cpp:158-164 with
// the 2-bit activations of PAPER.md:1119-1122), D[c][t] = float(p_t(c)) * (s * gamma_a):
//   G[r][t] = ((0.5 * alpha_r) * s) * gamma_a * units[r][t]       (kernels.cpp:193, 216)
//   S[r][t] = (...((+0 + v_1 * D[c_1][t]) + v_2 * D[c_2][t]) + ...)  in col_idx order, each
//             product and sum rounded to fp32 (kernels.cpp:347)
//   C[r][t] = G[r][t] + S[r][t]                                      (apb.cpp:161-162)
// bit for bit, with C written once. The two-pass form (GEMM stores G, spmm_levels_kernel reads it
// back, adds S, stores C) moves 300 MB of C at config 4; this kernel moves 100 MB and runs the
// tensor-core GEMM under the CUDA-core residual.
//
// Tiles are 256 rows x 64 tokens (cta_group::2, a CTA pair; each CTA owns 128 rows). A cluster
// owns a contiguous range of tiles in token-block-major order, so its two CTAs load the levels
// of a 64-token block once (bf16 patterns of p, [K + 1][64], staged for every block by
// unpack_operands beside the operand expansion, bulk-copied from L2) and reuse them for every
// row block of the range (a range crosses at most two or three token blocks).
//
// Warp roles per CTA (22 warps):
//   warp 0       TMA producer: the tile's operand k-blocks (as tc_gemm)
//   warp 1       MMA issuer (leader CTA): tcgen05.mma kind::mxf4 into one of two TMEM
//                accumulators, commit to tfull
//   warps 2..5   epilogue, thread = row (TMEM lane quadrant warp % 4): G from TMEM, S from the
//                staging buffer, C = fl(G + S) written back in place, TMA store
//   warps 6..21  residual: 64 octets (spmm_levels.cuh's layout: octet = row, lane = 8 tokens),
//                two rows each per tile, computed together; S goes to one of two staging
//                buffers in the epilogue's 128B-swizzled 32x32 block layout.
// Handshakes: sfull (16 residual warps -> epilogue), sfree (epilogue, after its TMA store read the
// buffer -> residual), tfull / tempty (MMA <-> epilogue, both CTAs), full / empty (TMA <-> MMA).
#pragma once

#include "spmm_levels.cuh"

namespace bitmm_dev {

constexpr int A3_BN = SL_TOK;                 // 64 tokens per tile = one staged level chunk
constexpr int A3_STAGES = 2;                  // operand stages (a tile has K/256 k-blocks)
constexpr int A3_EPI_WARPS = 4;
constexpr int A3_RES_WARPS = 16;              // 64 octets
constexpr int A3_THREADS = (2 + A3_EPI_WARPS + A3_RES_WARPS) * 32;  // 704
constexpr int A3_RES_THREADS = A3_RES_WARPS * 32;
constexpr int A3_RES_BAR = 1;                 // named barrier of the residual warps
constexpr int A3_A_STAGE = 128 * TC_BK_BYTES;             // 16 KB
constexpr int A3_B_STAGE = (A3_BN / 2) * TC_BK_BYTES;     // 4 KB
constexpr int A3_SBUF = 128 * A3_BN * 4;                  // 32 KB: 4 quadrants x 2 blocks of 32x32 fp32
constexpr int A3_BARS = 256;
constexpr int A3_FIXED = 1024 + A3_STAGES * (A3_A_STAGE + A3_B_STAGE) + 2 * A3_SBUF + A3_BARS;

inline int apb2_fused_smem_bytes(long long K) {
  return static_cast<int>(A3_FIXED + ((K + 1) * SL_ROW_WORDS * 4 + 15) / 16 * 16);
}

#ifdef A3_STATS
// Profiling builds only (-DA3_STATS): cycles per CTA of residual warp 6 ([0] staging, [1] S
// compute, [2] waiting for a free staging buffer, [3] total) and epilogue warp 2 ([4] waiting
// for the accumulator, [5] waiting for S, [6] add + store issue, [7] waiting for the store).
__device__ unsigned long long a3_stats[8][160];
#define A3_T(v) const long long v = clock64()
#else
#define A3_T(v)
#endif

struct Apb2Params {
  TcParams p;              // tc_gemm's problem record (F32R scale terms, tiles)
  const unsigned long long* row_ptr;
  const unsigned long long* col_idx;
  const float* vals;
  SpmmLevels lv;
  // [chunks][K + 1][SL_ROW_WORDS] bf16 patterns, or (L8) [chunks][K + 1][L8_ROW_WORDS] bytes
  // (LevelChunkJob, unpack_operands)
  const unsigned* level_chunks;
  int K;
  float neg4sg;            // L8: -4 * sg (exact), the fma addend that turns p + 4 into p
};

// sl_step8x2 over an L8 chunk (levels.cuh): lane ol of the octet owns tokens [8 ol, 8 ol + 8),
// one 8-byte load per nonzero. Per token pair: two PRMTs rebuild (p + 4) in fp32 from the stored
// bytes and the constant 0x40, then d = fma(p + 4, sg, -4 sg) = fl(p * sg) exactly,
// q = fl(v * d) and S = fl(S + q) as in sl_step8x2.
struct L8Octet {
  const char* xrow;         // chunk buffer + 8 ol bytes
  int obase;                // first lane of the octet in the warp
  unsigned long long dd;    // (sg, sg)
  unsigned long long z4;    // (-4 sg, -4 sg) from a kernel parameter
  unsigned long long z;     // (-0, -0) from a kernel parameter
};

template <int SEL>
__device__ __forceinline__ unsigned l8_level(unsigned w) {
  unsigned r;
  asm("prmt.b32 %0, %1, 0x40, %2;" : "=r"(r) : "r"(w), "n"(SEL));
  return r;
}

__device__ __forceinline__ void l8_step8x2(const L8Octet& o, unsigned kka, float vva, unsigned long long (&acca)[4],
                                           unsigned kkb, float vvb, unsigned long long (&accb)[4]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const unsigned koffa = __shfl_sync(0xFFFFFFFFu, kka, o.obase + j) * SL_TOK;
    const float va = __shfl_sync(0xFFFFFFFFu, vva, o.obase + j);
    const unsigned koffb = __shfl_sync(0xFFFFFFFFu, kkb, o.obase + j) * SL_TOK;
    const float vb = __shfl_sync(0xFFFFFFFFu, vvb, o.obase + j);
    const uint2 xa = *reinterpret_cast<const uint2*>(o.xrow + koffa);
    const uint2 xb = *reinterpret_cast<const uint2*>(o.xrow + koffb);
    const unsigned long long va2 = f32x2_pack(va, va), vb2 = f32x2_pack(vb, vb);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned wa = q < 2 ? xa.x : xa.y, wb = q < 2 ? xb.x : xb.y;
      // result bytes (low to high): 0, 0, the token's byte, 0x40 (PRMT bytes 5, 5, i, 4 of {0x40, w});
      // token pair q of the lane = bytes 2 (q & 1), 2 (q & 1) + 1 of word q / 2
      unsigned la, ha, lb, hb;
      if ((q & 1) == 0) {
        la = l8_level<0x4055>(wa);
        ha = l8_level<0x4155>(wa);
        lb = l8_level<0x4055>(wb);
        hb = l8_level<0x4155>(wb);
      } else {
        la = l8_level<0x4255>(wa);
        ha = l8_level<0x4355>(wa);
        lb = l8_level<0x4255>(wb);
        hb = l8_level<0x4355>(wb);
      }
      const unsigned long long pa = f32x2_pack(__uint_as_float(la), __uint_as_float(ha));
      const unsigned long long pb = f32x2_pack(__uint_as_float(lb), __uint_as_float(hb));
      acca[q] = f32x2_add(acca[q], f32x2_mul(va2, f32x2_mul(pa, o.dd, o.z4), o.z));
      accb[q] = f32x2_add(accb[q], f32x2_mul(vb2, f32x2_mul(pb, o.dd, o.z4), o.z));
    }
  }
}

// L8: the level chunks in the byte format (levels.cuh), double-buffered: the next token block's
// chunk loads while the current one is in use (two buffers of (K + 1) x 64 bytes in the space of
// one bf16 chunk). Otherwise one bf16 chunk, reloaded after every residual warp is done with it.
template <bool L8>
__global__ void __launch_bounds__(A3_THREADS, 1)
    apb2_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC, const Apb2Params ap) {
  const TcParams& p = ap.p;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (base_u32 & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + A3_STAGES * A3_A_STAGE;
  float* sbuf = reinterpret_cast<float*>(sB + A3_STAGES * A3_B_STAGE);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sbuf) + 2 * A3_SBUF);
  uint64_t* empty = full + A3_STAGES;
  uint64_t* tfull = empty + A3_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sfree = sfull + 2;
  uint64_t* lfull = sfree + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lfull + 2);
  unsigned* levels = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(full) + A3_BARS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank() & 1u;
  const int unit = static_cast<int>(cluster_id_x());
  const int num_units = static_cast<int>(num_clusters_x());
  // this cluster's tiles: [t0, t1) of the token-block-major order, balanced to +-1 tile
  const int t0 = static_cast<int>(static_cast<long long>(p.num_tiles) * unit / num_units);
  const int t1 = static_cast<int>(static_cast<long long>(p.num_tiles) * (unit + 1) / num_units);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < A3_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * A3_EPI_WARPS);  // both CTAs' epilogue warps
      mbar_init(&sfull[b], A3_RES_WARPS);
      mbar_init(&sfree[b], A3_EPI_WARPS);
    }
    mbar_init(lfull, 1);
    mbar_init(lfull + 1, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 256);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  constexpr uint32_t kSfCol = 2 * A3_BN;
  if (warp >= 2 && warp < 6) {  // E8M0 scale factors = 1.0 (0x7F) for both operands
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    tmem_st_32x32b_x32_fill(tmem_base + lane_off + kSfCol, 0x7F7F7F7Fu);
    tmem_st_32x32b_x32_fill(tmem_base + lane_off + kSfCol + 32, 0x7F7F7F7Fu);
    tmem_st_wait();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  pdl_wait();  // the expanded operands come from the preceding kernel

  const int nmb = p.num_m_blocks;
  if (warp == 0) {
    // ======================= TMA producer: operand k-blocks =======================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = t0; tile < t1; ++tile) {
        const int nb = tile / nmb, mb = tile - nb * nmb;
        const int a_row = mb * 256 + static_cast<int>(rank) * 128;
        const int b_row = nb * A3_BN + static_cast<int>(rank) * (A3_BN / 2);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (A3_A_STAGE + A3_B_STAGE));
          tma_load_2d_pair(sA + stage * A3_A_STAGE, &tmA, &full[stage], kb * TC_BK_BYTES, a_row);
          tma_load_2d_pair(sB + stage * A3_B_STAGE, &tmB, &full[stage], kb * TC_BK_BYTES, b_row);
          if (++stage == A3_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ========================= MMA issuer (leader CTA) =========================
    constexpr uint32_t idesc = make_idesc_mxf4(256, A3_BN);
    if (rank == 0) {
      const uint64_t a_desc0 = sw128_kmajor_desc(smem_u32(sA));
      const uint64_t b_desc0 = sw128_kmajor_desc(smem_u32(sB));
      const uint32_t sfa = tmem_base + kSfCol, sfb = tmem_base + kSfCol + 32;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = t0; tile < t1; ++tile, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * A3_BN;
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint64_t>((stage * A3_A_STAGE) >> 4);
          const uint64_t bd = b_desc0 + static_cast<uint64_t>((stage * A3_B_STAGE) >> 4);
#pragma unroll
          for (int k = 0; k < TC_BK_BYTES / 32; ++k)
            mma_pair_elect<2>(d_tmem, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0, sfa, sfb);
          mma_commit_pair_elect(&empty[stage], 0x3);
          if (++stage == A3_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit_pair_elect(&tfull[acc], 0x3);
      }
    }
  } else if (warp < 6) {
    // ====== epilogue, thread = row: C = fl(fl(row_mul * units) + S), one TMA store ======
    const int quad = warp & 3;
    int it = 0;
#ifdef A3_STATS
    long long st_acc = 0, st_s = 0, st_work = 0, st_store = 0;
#endif
    for (int tile = t0; tile < t1; ++tile, ++it) {
      const int nb = tile / nmb, mb = tile - nb * nmb;
      const int b = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      const int row_base = mb * 256 + static_cast<int>(rank) * 128 + quad * 32;
      const float row_mul = tc_row_mul<Epi::F32R>(p, row_base + lane);
      A3_T(q0);
      mbar_wait(&tfull[b], ph);
      tc_fence_after();
      A3_T(q1);
      mbar_wait(&sfull[b], ph);
      A3_T(q2);
      float* blk0 = sbuf + b * (A3_SBUF / 4) + quad * 2 * 1024;
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) {
        uint32_t g[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + b * A3_BN + cb * 32, g);
        tmem_ld_wait();
        float* blk = blk0 + cb * 1024;
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          float4* at = reinterpret_cast<float4*>(&blk[lane * 32 + (((j >> 2) ^ (lane & 7)) << 2)]);
          float4 v = *at;
          float* vf = reinterpret_cast<float*>(&v);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float units = __fmul_rn(__uint_as_float(g[j + e]), p.shift_mul);  // exact
            vf[e] = __fadd_rn(__fmul_rn(row_mul, units), vf[e]);                    // G + S
          }
          *at = v;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(smem_u32(&tempty[b]) & kPeerBitMask);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&tmC, blk0, nb * A3_BN, row_base);
        tma_store_2d(&tmC, blk0 + 1024, nb * A3_BN + 32, row_base);
        bulk_commit_group();
      }
      A3_T(q3);
      if (lane == 0) {
        bulk_wait_group_read<0>();  // the stores have read the staging block
        mbar_arrive(&sfree[b]);
      }
      __syncwarp();
#ifdef A3_STATS
      A3_T(q4);
      st_acc += q1 - q0;
      st_s += q2 - q1;
      st_work += q3 - q2;
      st_store += q4 - q3;
#endif
    }
    if (lane == 0) bulk_wait_group_all();
#ifdef A3_STATS
    if (warp == 2 && lane == 0) {
      a3_stats[4][blockIdx.x] = st_acc;
      a3_stats[5][blockIdx.x] = st_s;
      a3_stats[6][blockIdx.x] = st_work;
      a3_stats[7][blockIdx.x] = st_store;
    }
#endif
  } else {
    // ============ residual S: 64 octets, two rows each per tile (spmm_levels.cuh) ============
    const int rt = threadIdx.x - 6 * 32;  // 0 .. A3_RES_THREADS - 1
    const int oct = rt >> 3, ol = rt & 7;
    const SlOctet so{reinterpret_cast<const char*>(levels) + ol * 16, lane & ~7, f32x2_pack(ap.lv.d1, ap.lv.d1),
                     f32x2_pack(ap.lv.neg_zero, ap.lv.neg_zero)};
    // L8: two chunk buffers; block nb_first + k lives in buffer k & 1
    const uint32_t l8_bytes = static_cast<uint32_t>(ap.K + 1) * SL_TOK;
    const char* l8base = reinterpret_cast<const char*>(levels);  // buffer j at l8base + j * l8_bytes
    L8Octet lo8{l8base + ol * 8, lane & ~7, so.dd, f32x2_pack(ap.neg4sg, ap.neg4sg), so.z};
    const int nb_first = t0 / nmb, nb_last = t1 > t0 ? (t1 - 1) / nmb : -1;
    uint32_t l8ph = 0;  // bit j: phase of buffer j
    auto l8_issue = [&](int k) {  // token block nb_first + k into buffer k & 1
      if (L8 && rt == 0 && nb_first + k <= nb_last) {
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&lfull[k & 1], l8_bytes);
        bulk_load_1d(const_cast<char*>(l8base) + (k & 1) * l8_bytes,
                     ap.level_chunks + static_cast<long long>(nb_first + k) * (ap.K + 1) * L8_ROW_WORDS, l8_bytes,
                     &lfull[k & 1]);
      }
    };
    if (L8) {
      l8_issue(0);
      l8_issue(1);
    }
    const unsigned zero_row = static_cast<unsigned>(ap.K);
    // Per tile the octet computes its two rows (oct, oct + 64 of the CTA's 128) together
    // (sl_step8x2: two independent chains). Software pipeline over tiles: the row offsets two
    // tiles ahead and the first 16 slots of each row one tile ahead load while this tile computes;
    // offsets stay raw until the tile after the one that loaded them (consuming a load right away
    // would stall the warp on it).
    struct Row {
      unsigned long long lo, hi;
    };
    // tile coordinates advance incrementally (no integer division in the loop)
    auto advance = [&](int& nb, int& mb) {
      if (++mb == nmb) {
        mb = 0;
        ++nb;
      }
    };
    auto load_rp = [&](bool valid, int mb, int pass) {
      Row x{0, 0};
      const int r = mb * 256 + static_cast<int>(rank) * 128 + oct + 64 * pass;
      if (valid && r < p.M) {
        x.lo = ap.row_ptr[r];
        x.hi = ap.row_ptr[r + 1];
      }
      return x;
    };
    auto fetch = [&](unsigned long long e0, unsigned n, unsigned idx, unsigned& kk, float& vv) {
      kk = zero_row;
      vv = 0.f;
      if (idx < n) {
        kk = static_cast<unsigned>(ap.col_idx[e0 + idx]);
        vv = ap.vals[e0 + idx];
      }
    };
    int nbc = t0 / nmb, mbc = t0 - (t0 / nmb) * nmb;  // tile t0 + it
    int nb2 = nbc, mb2 = mbc;                          // tile t0 + it + 2
    int nb1 = nbc, mb1 = mbc;
    advance(nb1, mb1);
    advance(nb2, mb2);
    advance(nb2, mb2);
    Row ra = load_rp(t0 < t1, mbc, 0), rb = load_rp(t0 < t1, mbc, 1);
    Row ra1 = load_rp(t0 + 1 < t1, mb1, 0), rb1 = load_rp(t0 + 1 < t1, mb1, 1);
    unsigned na = static_cast<unsigned>(ra.hi - ra.lo), nb_ = static_cast<unsigned>(rb.hi - rb.lo);
    unsigned ka0, ka1, kb0, kb1;
    float va0, va1, vb0, vb1;
    fetch(ra.lo, na, ol, ka0, va0);
    fetch(ra.lo, na, ol + 8, ka1, va1);
    fetch(rb.lo, nb_, ol, kb0, vb0);
    fetch(rb.lo, nb_, ol + 8, kb1, vb1);
    int cur_nb = -1;
    uint32_t lphase = 0;
    int it = 0;
#ifdef A3_STATS
    long long st_stage = 0, st_comp = 0, st_free = 0;
    A3_T(s_begin);
#endif
    for (int tile = t0; tile < t1; ++tile, ++it) {
      const int nb = nbc;
      A3_T(p0);
      const int b = it & 1;
      const uint32_t ph = (it >> 1) & 1;
      if (L8 && nb != cur_nb) {  // new token block: its chunk was issued one block ahead
        const int k = nb - nb_first;
        if (k >= 1) {  // every octet is done with block k - 1: its buffer takes block k + 1
          named_bar_sync(A3_RES_BAR, A3_RES_THREADS);
          l8_issue(k + 1);
        }
        mbar_wait(&lfull[k & 1], (l8ph >> (k & 1)) & 1u);
        l8ph ^= 1u << (k & 1);
        lo8.xrow = l8base + (k & 1) * l8_bytes + ol * 8;
        cur_nb = nb;
      } else if (nb != cur_nb) {  // new token block: bulk-copy its levels once every octet is done with the old
        named_bar_sync(A3_RES_BAR, A3_RES_THREADS);
        if (rt == 0) {
          const uint32_t bytes = static_cast<uint32_t>(ap.K + 1) * SL_ROW_WORDS * 4;
          fence_proxy_async_smem();  // the octets' reads of the old chunk before the async writes
          mbar_arrive_expect_tx(lfull, bytes);
          bulk_load_1d(levels, ap.level_chunks + static_cast<long long>(nb) * (ap.K + 1) * SL_ROW_WORDS, bytes,
                       lfull);
        }
        mbar_wait(lfull, lphase);
        lphase ^= 1u;
        cur_nb = nb;
      }
      A3_T(p1);
      const Row ra2 = load_rp(tile + 2 < t1, mb2, 0), rb2 = load_rp(tile + 2 < t1, mb2, 1);
      advance(nbc, mbc);
      advance(nb2, mb2);
      const unsigned na1 = static_cast<unsigned>(ra1.hi - ra1.lo), nb1 = static_cast<unsigned>(rb1.hi - rb1.lo);
      unsigned nka0, nka1, nkb0, nkb1;
      float nva0, nva1, nvb0, nvb1;
      fetch(ra1.lo, na1, ol, nka0, nva0);
      fetch(ra1.lo, na1, ol + 8, nka1, nva1);
      fetch(rb1.lo, nb1, ol, nkb0, nvb0);
      fetch(rb1.lo, nb1, ol + 8, nkb1, nvb1);

      const unsigned nmax = __reduce_max_sync(0xFFFFFFFFu, max(na, nb_));
      unsigned long long acca[4] = {0ull, 0ull, 0ull, 0ull}, accb[4] = {0ull, 0ull, 0ull, 0ull};  // +0 pairs
      auto step = [&](unsigned kka, float vva, unsigned kkb, float vvb) {
        if constexpr (L8)
          l8_step8x2(lo8, kka, vva, acca, kkb, vvb, accb);
        else
          sl_step8x2(so, kka, vva, acca, kkb, vvb, accb);
      };
      if (nmax > 0) step(ka0, va0, kb0, vb0);
      if (nmax > 8) step(ka1, va1, kb1, vb1);
      for (unsigned base = 16; base < nmax; base += 8) {
        unsigned kka, kkb;
        float vva, vvb;
        fetch(ra.lo, na, base + ol, kka, vva);
        fetch(rb.lo, nb_, base + ol, kkb, vvb);
        step(kka, vva, kkb, vvb);
      }
      A3_T(p2);
      mbar_wait(&sfree[b], ph ^ 1u);
#ifdef A3_STATS
      A3_T(p3);
      st_stage += p1 - p0;
      st_comp += p2 - p1;
      st_free += p3 - p2;
#endif
      // S of tokens [8 ol, 8 ol + 8) of row R -> 32x32 block (R / 32, ol / 4), row R % 32,
      // 16-byte chunks 2 (ol % 4) and 2 (ol % 4) + 1, 128B-swizzled by (R % 8)
      const int c0 = 2 * (ol & 3);
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const int R = oct + 64 * pass;
        float* blk = sbuf + b * (A3_SBUF / 4) + ((R >> 5) * 2 + (ol >> 2)) * 1024 + (R & 31) * 32;
        const float* af = reinterpret_cast<const float*>(pass ? accb : acca);
        *reinterpret_cast<float4*>(&blk[((c0 ^ (R & 7)) << 2)]) = make_float4(af[0], af[1], af[2], af[3]);
        *reinterpret_cast<float4*>(&blk[(((c0 + 1) ^ (R & 7)) << 2)]) = make_float4(af[4], af[5], af[6], af[7]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sfull[b]);
      ra = ra1;
      rb = rb1;
      na = na1;
      nb_ = nb1;
      ra1 = ra2;
      rb1 = rb2;
      ka0 = nka0;
      ka1 = nka1;
      kb0 = nkb0;
      kb1 = nkb1;
      va0 = nva0;
      va1 = nva1;
      vb0 = nvb0;
      vb1 = nvb1;
    }
#ifdef A3_STATS
    if (warp == 6 && lane == 0) {
      a3_stats[0][blockIdx.x] = st_stage;
      a3_stats[1][blockIdx.x] = st_comp;
      a3_stats[2][blockIdx.x] = st_free;
      a3_stats[3][blockIdx.x] = clock64() - s_begin;
    }
#endif
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 256);
  }
}

}  // namespace bitmm_dev
