// Bitwise GEMM with the operand expansion inside the tensor-core kernel (sm_100a).
// A measured alternative to unpack.cuh + tc_gemm.cuh, selected with BITMM_FX=1 (not the
// default): the expanders' st.shared writes of 28 KB per stage and CTA bound it (DESIGN.md
// "In-GEMM expansion"; profiles/fx_r02.md).
//
// tc_gemm.cuh multiplies operands that a separate pass (unpack.cuh) expanded to e2m1 nibbles:
// 4 bits per element in HBM/L2, re-read by every tile that uses them. Here the kernel reads
// the PACKED operands and expands them in shared memory:
//   sign operand  : the reference BitMatrix words themselves (tensor.hpp:59-112), 1 bit per
//                   element, loaded by TMA straight from the caller's buffer;
//   level operand : 2-bit codes (p = 2 hi + lo) that prep_codes_kernel (prep.cuh) derives from
//                   the {t,h,m} planes once per call, validating them (transform.cpp:47-75).
// so a tile's operand bytes through L2 are 1/4 (signs) or 1/2 (levels) of the expanded ones.
//
// Structure (persistent; one CTA pair per cluster, cta_group::2, 256 x 192 output tiles):
//   warp 0        : TMA producer of the packed ring: P slots, each 512 K elements of the
//                   CTA's 128 A rows and 96 B rows (64 B per row for signs, 128 B for codes)
//   warp 1        : TMEM allocator + MMA issuer (leader CTA), as in tc_gemm
//   warps 2..5    : epilogue (tc_epilogue_tile), as in tc_gemm
//   warps 6..     : NEXP expander warps: packed slot -> e2m1 stage of 256 K elements in the
//                   128B-swizzled K-major layout the UMMA descriptors read (16-byte chunk j of
//                   row r at chunk j ^ (r & 7)), then fence.proxy.async and one arrival per
//                   warp on the leader CTA's `full` barrier (both CTAs' warps: 2 * NEXP).
// The e2m1 nibble order is the one unpack.cuh writes: inside every 32-element group, element
// 4n + q goes to output word q, nibble n (the same permutation on both operands, so every dot
// product is unchanged). Signs: +1 -> 0x2, -1 -> 0xA; levels p -> p (value p / 2; the
// epilogue shift restores the factor 2 per level operand); elements past K -> 0.
#pragma once

#include "tc_gemm.cuh"
#include "unpack.cuh"

namespace bitmm_dev {

constexpr int FX_KSTAGE = 256;  // K elements per expanded stage (128 bytes of e2m1 per row)
constexpr int FX_KSLOT = 512;   // K elements per packed slot (two stages)
// Expander groups: with 2, the warps split in two halves that take alternate stages, so one
// half's shared-memory store burst overlaps the other half's loads and bit arithmetic.
#ifndef FX_GROUPS
#define FX_GROUPS 2
#endif

// SLOT_ROW: packed slot bytes per row, 64 (sign operands only) or 128 (2-bit codes possible).
// AX (hybrid, BITMM_FX=2): A arrives already expanded (unpack.cuh's e2m1 rows, TMA-loaded into
// the stage as tc_gemm does) and only B is expanded here: the expanders write 12 KB per stage
// instead of 28 KB, and the packed ring holds B alone, so six stages fit instead of four.
template <int NEXP, int SLOT_ROW, bool AX = false>
struct FxShape {
  static constexpr int BN = 192;
  static constexpr int A_ROWS = 128;
  static constexpr int B_ROWS = BN / 2;
  static constexpr int TILE_M = 256;
  static constexpr int STAGE_A = A_ROWS * 128;
  static constexpr int STAGE_B = B_ROWS * 128;
  static constexpr int STAGE = STAGE_A + STAGE_B;  // 28 KB
  static constexpr int SLOT_A = AX ? 0 : A_ROWS * SLOT_ROW;
  static constexpr int SLOT = SLOT_A + B_ROWS * SLOT_ROW;
  static constexpr int EPI_BUFS = 1;
  static constexpr int EPI_WARP_BYTES = 5120;
  static constexpr int EPI_BYTES = 4 * EPI_WARP_BYTES;
  static constexpr int COLS_BYTES = BN * 4;
  static constexpr int E = AX ? 6 : 4;  // expanded stages
  static constexpr int P = (232448 - 1024 - E * STAGE - EPI_BYTES - COLS_BYTES - 512) / SLOT;
  static constexpr int BAR_BYTES = (2 * E + 2 * P + 4) * 8 + 16;
  static constexpr int SMEM = 1024 + E * STAGE + P * SLOT + EPI_BYTES + COLS_BYTES + BAR_BYTES;
  static constexpr int THREADS = (6 + NEXP) * 32;
  static_assert(P >= 2, "packed ring needs two slots");
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(E % 2 == 0, "expander groups alternate over an even ring");
};

template <int NP>
struct FxGroup {
  CUtensorMap a[NP], b[NP], c[NP];  // packed A / B (sign words or 2-bit codes), output
  TcParams prob[NP];                // num_kb = expanded stages = ceil(K / 256)
  int a_code[NP], b_code[NP];       // 0: sign bits (64 B per slot row), 1: 2-bit codes (128 B)
  int K[NP];                        // logical shared dimension (elements past K expand to 0)
  int count;
  int tile_begin[NP + 1];
};

#ifdef FX_STATS
// Profiling build only: cycles per CTA spent waiting. [0] MMA on full, [1] MMA total,
// [2] expander warp 6 on pfull, [3] on empty, [4] its total, [5] producer on pempty.
__device__ unsigned long long fx_stats[8][160];
#define FX_T0() long long _t0 = clock64()
#define FX_ACC(v) v += clock64() - _t0
#else
#define FX_T0()
#define FX_ACC(v)
#endif

template <int NP>
__device__ __forceinline__ int fx_problem_of(const FxGroup<NP>& g, int t) {
  if constexpr (NP == 1) return 0;
  int pi = 0;
#pragma unroll
  for (int i = 1; i < NP; ++i)
    if (i < g.count && t >= g.tile_begin[i]) pi = i;
  return pi;
}

// One 32-element group of a sign row -> 16 bytes of e2m1 (unpack.cuh's K permutation).
__device__ __forceinline__ uint4 fx_expand_sign(uint32_t w, int kel, int K) {
  if (kel + 32 <= K)
    return make_uint4((~(w << 3) & 0x88888888u) | 0x22222222u, (~(w << 2) & 0x88888888u) | 0x22222222u,
                      (~(w << 1) & 0x88888888u) | 0x22222222u, (~w & 0x88888888u) | 0x22222222u);
  const uint32_t valid = valid_mask32(kel, K);
  const uint32_t neg = valid & ~w;
  uint32_t o[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) o[q] = (((valid >> q) & 0x11111111u) << 1) | (((neg >> q) & 0x11111111u) << 3);
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// One 32-element group of 2-bit codes (prep.cuh layout: the low word holds elements 4n and
// 4n+1 at bit pairs 4n and 4n+2, the high word elements 4n+2 and 4n+3) -> 16 bytes of e2m1.
__device__ __forceinline__ uint4 fx_expand_code(uint2 x) {
  return make_uint4(x.x & 0x33333333u, (x.x >> 2) & 0x33333333u, x.y & 0x33333333u,
                    (x.y >> 2) & 0x33333333u);
}

// ITS rows of one operand (rows r0, r0 + STEP, ...) for one 32-element chunk j of a stage:
// packed slot (row pitch 64 B for signs, 128 B for codes; `sub` selects the stage's half)
// -> 16-byte e2m1 chunks in registers (fx_store_rows writes them).
template <int ITS, int STEP>
__device__ __forceinline__ void fx_load_rows(const uint8_t* slot, uint4 (&v)[ITS], int r0, int j, int sub,
                                             int kel, int K, bool code) {
  if (code) {
    uint2 x[ITS];
#pragma unroll
    for (int i = 0; i < ITS; ++i)
      x[i] = *reinterpret_cast<const uint2*>(slot + (r0 + i * STEP) * 128 + sub * 64 + j * 8);
#pragma unroll
    for (int i = 0; i < ITS; ++i) v[i] = fx_expand_code(x[i]);
  } else {
    uint32_t w[ITS];
#pragma unroll
    for (int i = 0; i < ITS; ++i)
      w[i] = *reinterpret_cast<const uint32_t*>(slot + (r0 + i * STEP) * 64 + sub * 32 + j * 4);
    if (kel + 32 <= K) {
#pragma unroll
      for (int i = 0; i < ITS; ++i)
        v[i] = make_uint4((~(w[i] << 3) & 0x88888888u) | 0x22222222u, (~(w[i] << 2) & 0x88888888u) | 0x22222222u,
                          (~(w[i] << 1) & 0x88888888u) | 0x22222222u, (~w[i] & 0x88888888u) | 0x22222222u);
    } else {
#pragma unroll
      for (int i = 0; i < ITS; ++i) v[i] = fx_expand_sign(w[i], kel, K);
    }
  }
}

// The chunks into the 128B-swizzled stage: chunk j of row r at j ^ (r & 7) (conflict-free:
// the 8 lanes of a store phase cover the 8 chunks of one row).
template <int ITS, int STEP>
__device__ __forceinline__ void fx_store_rows(uint8_t* st, const uint4 (&v)[ITS], int r0, int j) {
#pragma unroll
  for (int i = 0; i < ITS; ++i) {
    const int r = r0 + i * STEP;
    *reinterpret_cast<uint4*>(st + r * 128 + ((j ^ (r & 7)) << 4)) = v[i];
  }
}

template <Epi EPI, int NP, int NEXP, int SLOT_ROW, bool AX = false>
__global__ void __launch_bounds__(FxShape<NEXP, SLOT_ROW, AX>::THREADS, 1)
    fx_gemm_kernel(const __grid_constant__ FxGroup<NP> g) {
  using S = FxShape<NEXP, SLOT_ROW, AX>;
  constexpr int BN = S::BN;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (base_u32 & 1023u)) & 1023u);
  uint8_t* sStage = smem;                          // E expanded stages (A then B per stage)
  uint8_t* sSlot = sStage + S::E * S::STAGE;       // P packed slots (A then B per slot)
  float* sEpi = reinterpret_cast<float*>(sSlot + S::P * S::SLOT);
  float* sCols = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sEpi) + S::EPI_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sCols) + S::COLS_BYTES);
  uint64_t* empty = full + S::E;
  uint64_t* pfull = empty + S::E;
  uint64_t* pempty = pfull + S::P;
  uint64_t* tfull = pempty + S::P;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank() & 1u;
  const int unit = static_cast<int>(cluster_id_x());
  const int num_units = static_cast<int>(num_clusters_x());
  const int num_tiles = g.tile_begin[g.count];

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < g.count; ++i) {
      tma_prefetch_desc(&g.a[i]);
      tma_prefetch_desc(&g.b[i]);
      if (g.prob[i].tma_store) tma_prefetch_desc(&g.c[i]);
    }
    for (int s = 0; s < S::E; ++s) {
      // every expander warp of the stage's group, both CTAs (+ the leader's A loads under AX)
      mbar_init(&full[s], 2 * NEXP / FX_GROUPS + (AX ? 1 : 0));
      mbar_init(&empty[s], 1);        // the pair's MMA commit
    }
    for (int s = 0; s < S::P; ++s) {
      mbar_init(&pfull[s], 1);
      mbar_init(&pempty[s], NEXP);
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
  constexpr uint32_t kSfCol = 2 * BN;  // E8M0 scale factors after the two accumulators
  if (warp >= 2 && warp < 6) {         // every scale-factor cell = 1.0 (0x7F)
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    tmem_st_32x32b_x32_fill(tmem_base + lane_off + kSfCol, 0x7F7F7F7Fu);
    tmem_st_32x32b_x32_fill(tmem_base + lane_off + kSfCol + 32, 0x7F7F7F7Fu);
    tmem_st_wait();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  // Everything above overlapped the previous kernel (PDL); from here on we read its output.
  pdl_wait();

  if (AX && warp == 0) {
    // ============ TMA producer (AX): B's packed ring, and A's e2m1 rows into the stages ============
    if (lane == 0) {
      int ps = 0, stage = 0;
      uint32_t pph = 0, phase = 0;
      for (int tile = unit; tile < num_tiles; tile += num_units) {
        const int pi = fx_problem_of(g, tile);
        const TcParams& p = g.prob[pi];
        int mb, nb;
        tc_tile_coords(tile - g.tile_begin[pi], p, p.num_n_blocks, mb, nb);
        const int a_row = mb * S::TILE_M + static_cast<int>(rank) * S::A_ROWS;
        const int b_row = nb * BN + static_cast<int>(rank) * S::B_ROWS;
        const int b_box = g.b_code[pi] ? 128 : 64;
        const CUtensorMap* ma = &g.a[pi];
        const CUtensorMap* mbm = &g.b[pi];
        for (int kb = 0; kb < p.num_kb; ++kb) {
          if ((kb & 1) == 0) {  // a packed slot holds two stages of B
            mbar_wait(&pempty[ps], pph ^ 1u);
            mbar_arrive_expect_tx(&pfull[ps], static_cast<uint32_t>(S::B_ROWS * b_box));
            tma_load_2d(sSlot + ps * S::SLOT, mbm, &pfull[ps], (kb >> 1) * b_box, b_row);
            if (++ps == S::P) {
              ps = 0;
              pph ^= 1u;
            }
          }
          mbar_wait(&empty[stage], phase ^ 1u);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * S::STAGE_A);
          tma_load_2d_pair(sStage + stage * S::STAGE, ma, &full[stage], kb * 128, a_row);
          if (++stage == S::E) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 0) {
    // ===================== TMA producer of the packed ring (each CTA its own rows) ==========
    if (lane == 0) {
      int ps = 0;
      uint32_t pph = 0;
#ifdef FX_STATS
      long long st_pe = 0;
#endif
      for (int tile = unit; tile < num_tiles; tile += num_units) {
        const int pi = fx_problem_of(g, tile);
        const TcParams& p = g.prob[pi];
        int mb, nb;
        tc_tile_coords(tile - g.tile_begin[pi], p, p.num_n_blocks, mb, nb);
        const int a_row = mb * S::TILE_M + static_cast<int>(rank) * S::A_ROWS;
        const int b_row = nb * BN + static_cast<int>(rank) * S::B_ROWS;
        const int a_box = g.a_code[pi] ? 128 : 64, b_box = g.b_code[pi] ? 128 : 64;
        const uint32_t tx = static_cast<uint32_t>(S::A_ROWS * a_box + S::B_ROWS * b_box);
        const CUtensorMap* ma = &g.a[pi];
        const CUtensorMap* mbm = &g.b[pi];
        const int npk = (p.num_kb + 1) >> 1;
        for (int pk = 0; pk < npk; ++pk) {
          {
            FX_T0();
            mbar_wait(&pempty[ps], pph ^ 1u);
            FX_ACC(st_pe);
          }
          mbar_arrive_expect_tx(&pfull[ps], tx);
          uint8_t* slot = sSlot + ps * S::SLOT;
          tma_load_2d(slot, ma, &pfull[ps], pk * a_box, a_row);
          tma_load_2d(slot + S::SLOT_A, mbm, &pfull[ps], pk * b_box, b_row);
          if (++ps == S::P) {
            ps = 0;
            pph ^= 1u;
          }
        }
      }
#ifdef FX_STATS
      fx_stats[5][blockIdx.x] = st_pe;
#endif
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA, whole warp) =====================
    constexpr uint32_t idesc = make_idesc_mxf4(S::TILE_M, BN);
    if (rank == 0) {
      const uint64_t a_desc0 = sw128_kmajor_desc(smem_u32(sStage));
      const uint64_t b_desc0 = sw128_kmajor_desc(smem_u32(sStage + S::STAGE_A));
      const uint32_t sfa = tmem_base + kSfCol, sfb = tmem_base + kSfCol + 32;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
#ifdef FX_STATS
      long long st_fu = 0, st_start = clock64();
#endif
      for (int tile = unit; tile < num_tiles; tile += num_units, ++it) {
        const int num_kb = g.prob[fx_problem_of(g, tile)].num_kb;
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aphase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          {
            FX_T0();
            mbar_wait(&full[stage], phase);
            FX_ACC(st_fu);
          }
          tc_fence_after();
          const uint64_t off = static_cast<uint64_t>((stage * S::STAGE) >> 4);
#ifndef FX_NO_MMA  // timing experiment only (wrong results): no MMAs
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_pair_elect<2>(d_tmem, a_desc0 + off + 2 * k, b_desc0 + off + 2 * k, idesc, (kb | k) != 0,
                              sfa, sfb);
#endif
          mma_commit_pair_elect(&empty[stage], 0x3);
          if (++stage == S::E) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit_pair_elect(&tfull[acc], 0x3);
      }
#ifdef FX_STATS
      if (lane == 0) {
        fx_stats[0][blockIdx.x] = st_fu;
        fx_stats[1][blockIdx.x] = clock64() - st_start;
      }
#endif
    }
  } else if (warp < 6) {
    // ===================== epilogue (warps 2..5 of every CTA) =====================
    const int quad = warp & 3;
    float* stg = sEpi + (warp - 2) * (S::EPI_WARP_BYTES / 4);
    uint32_t buf = 0;
    int it = 0;
    for (int tile = unit; tile < num_tiles; tile += num_units, ++it) {
      const int pi = fx_problem_of(g, tile);
      const TcParams p = g.prob[pi];
      int mb, nb;
      tc_tile_coords(tile - g.tile_begin[pi], p, p.num_n_blocks, mb, nb);
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int row_base = mb * S::TILE_M + static_cast<int>(rank) * 128 + quad * 32;
      float row_mul = p.scale;
      if constexpr (EPI == Epi::ANY) {
        if (p.epi != static_cast<int>(Epi::I32)) row_mul = tc_row_mul<Epi::F32>(p, row_base + lane);
      } else {
        row_mul = tc_row_mul<EPI>(p, row_base + lane);
      }
      const bool has_cs = p.col_scale != nullptr && p.epi != static_cast<int>(Epi::I32);
      constexpr int CS_PER_THREAD = (BN + 127) / 128;
      float csv[CS_PER_THREAD];
      if (has_cs) {
#pragma unroll
        for (int j = 0; j < CS_PER_THREAD; ++j) {
          const int i = (warp - 2) * 32 + lane + j * 128;
          const int cc = nb * BN + i;
          csv[j] = (i < BN && cc < p.N) ? p.col_scale[cc] : 0.0f;
        }
      }
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const uint32_t tacc = tmem_base + acc * BN;
      const float* cs = nullptr;
      if (has_cs) {
        named_bar_sync(1, 128);
#pragma unroll
        for (int j = 0; j < CS_PER_THREAD; ++j) {
          const int i = (warp - 2) * 32 + lane + j * 128;
          if (i < BN) sCols[i] = csv[j];
        }
        named_bar_sync(1, 128);
        cs = sCols;
      }
      if constexpr (EPI == Epi::ANY) {
        if (p.epi == static_cast<int>(Epi::I32))
          tc_epilogue_tile<Epi::I32, BN, true, S::EPI_BUFS>(p, &g.c[pi], tacc, quad, lane, row_base, nb * BN,
                                                            stg, buf, cs, row_mul);
        else
          tc_epilogue_tile<Epi::F32, BN, true, S::EPI_BUFS>(p, &g.c[pi], tacc, quad, lane, row_base, nb * BN,
                                                            stg, buf, cs, row_mul);
      } else {
        tc_epilogue_tile<EPI, BN, true, S::EPI_BUFS>(p, &g.c[pi], tacc, quad, lane, row_base, nb * BN, stg,
                                                     buf, cs, row_mul);
      }
      tc_fence_before();
      mbar_arrive_cluster(smem_u32(&tempty[acc]) & kPeerBitMask);
    }
    if (lane == 0) bulk_wait_group_all();  // stores land before the grid ends
  } else {
    // ===================== expanders (warps 6.. of every CTA) =====================
    constexpr int T = NEXP / FX_GROUPS * 32;  // threads per group
    constexpr int ROWS_PER_IT = T / 8;  // 8 lanes per row: one 16-byte output chunk each
    constexpr int A_ITS = AX ? 1 : S::A_ROWS / ROWS_PER_IT, B_ITS = S::B_ROWS / ROWS_PER_IT;
    static_assert(AX || (A_ITS * ROWS_PER_IT == S::A_ROWS && B_ITS * ROWS_PER_IT == S::B_ROWS), "task split");
    static_assert(B_ITS * ROWS_PER_IT == S::B_ROWS, "task split");
    const int group = (threadIdx.x - 6 * 32) / T;
    const int tid = threadIdx.x - 6 * 32 - group * T;
    const int r0 = tid >> 3, j = tid & 7;
    int gs = 0;            // stages walked so far (all groups walk every stage)
    bool waited = false;   // this warp has observed the current packed slot's pfull
    const uint32_t full_base = smem_u32(full) & kPeerBitMask;  // the leader CTA's barriers
    int stage = 0, ps = 0;
    uint32_t phase = 0, pph = 0;
#ifdef FX_STATS
    long long st_pf = 0, st_em = 0, st_start = clock64();
#endif
    for (int tile = unit; tile < num_tiles; tile += num_units) {
      const int pi = fx_problem_of(g, tile);
      const int num_kb = g.prob[pi].num_kb;
      const int K = g.K[pi];
      const bool a_code = g.a_code[pi] != 0, b_code = g.b_code[pi] != 0;
      for (int kb = 0; kb < num_kb; ++kb) {
        const int sub = kb & 1;
        if ((gs++ % FX_GROUPS) == group) {
        if (!waited) {
          FX_T0();
          mbar_wait(&pfull[ps], pph);
          FX_ACC(st_pf);
          waited = true;
        }
        {
          FX_T0();
          mbar_wait(&empty[stage], phase ^ 1u);
          FX_ACC(st_em);
        }
        const uint8_t* slot = sSlot + ps * S::SLOT;
        uint8_t* st = sStage + stage * S::STAGE;
        // Every task of this thread covers the same 32 K elements (chunk j of the stage), so
        // the K bound is one thread-uniform test; all packed loads are issued before the
        // first store (the stores could alias them as far as the compiler knows).
        const int kel = kb * FX_KSTAGE + j * 32;
        uint4 va[A_ITS], vb[B_ITS];
        if constexpr (!AX) fx_load_rows<A_ITS, ROWS_PER_IT>(slot, va, r0, j, sub, kel, K, a_code);
        fx_load_rows<B_ITS, ROWS_PER_IT>(slot + S::SLOT_A, vb, r0, j, sub, kel, K, b_code);
#ifdef FX_NO_STS  // timing experiment only (wrong results): no stage writes
        if (vb[0].x == 0x12345678u && vb[0].y == 0x9abcdef0u) {
#endif
        if constexpr (!AX) fx_store_rows<A_ITS, ROWS_PER_IT>(st, va, r0, j);
        fx_store_rows<B_ITS, ROWS_PER_IT>(st + S::STAGE_A, vb, r0, j);
#ifdef FX_NO_STS
        }
#endif
#ifdef FX_FENCE_ALL
        fence_proxy_async_all();
#elif defined(FX_NO_FENCE)  // timing experiment only
#else
        fence_proxy_async_smem();
#endif
        __syncwarp();
        // Plain (default .release.cta) remote arrival: release at cluster scope compiles to
        // MEMBAR.ALL.GPU per warp and stage (measured 4x slower overall); the fence above
        // already publishes the stage's st.shared writes to the async proxy.
        if (lane == 0) mbar_arrive_cluster(full_base + stage * 8);
        }
        if (sub == 1 || kb + 1 == num_kb) {
          if (lane == 0) mbar_arrive(&pempty[ps]);  // every warp, whether or not it read the slot
          waited = false;
          if (++ps == S::P) {
            ps = 0;
            pph ^= 1u;
          }
        }
        if (++stage == S::E) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
#ifdef FX_STATS
    if (threadIdx.x == 6 * 32) {
      fx_stats[2][blockIdx.x] = st_pf;
      fx_stats[3][blockIdx.x] = st_em;
      fx_stats[4][blockIdx.x] = clock64() - st_start;
    }
#endif
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace bitmm_dev
