// Tensor-core bitwise GEMM for sm_100a.
//
// The reference (proj/src/kernels.cpp:163-275) evaluates every output cell as an exact
// integer ("units") built from xor/and + popcount over K-packed bit rows, then multiplies by
// one float scale. sm_100a has no b1 tensor-core MMA, so the operands are
// expanded first (unpack.cuh) and multiplied on tcgen05:
//   1/1 : A = sign(a) in {-1,+1},  B = sign(b) in {-1,+1}   units = acc
//   1/2 : A = sign(w) in {-1,+1},  B = level p in {0..3}   units = 2*acc
//   2/2 : A = level p_w in {0..3}, B = level p_a in {0..3} units = 4*acc
// with acc = sum_k A[r][k]*B[c][k]. Kind::F4 (default) feeds these as packed e2m1 through
// kind::mxf4 with unit E8M0 scale factors and fp32 accumulators, which hold every partial sum
// exactly (|acc| <= 9*2^20 < 2^24); Kind::I8 uses kind::i8 with s32 accumulators.
//
// Structure (persistent; one CTA pair per cluster, cta_group::2):
//   warp 0     : TMA producer, multi-stage smem ring of 128-byte K slices (each CTA stages
//                128 rows of A and BN/2 rows of B; the pair's MMA reads both CTAs' halves)
//   warp 1     : TMEM allocator + MMA issuer (leader CTA; whole warp, one elected lane issues)
//   warps 2..5 : epilogue: TMEM -> registers (next chunk's load in flight) -> transform ->
//                128B-swizzled smem block -> TMA bulk tensor store. Two TMEM accumulators of
//                BN columns, so the epilogue of tile i overlaps the MMAs of tile i+1; F4 keeps
//                its scale factors in the 64 columns after them (hence BN = 192, not 256).
// A launch covers a group of problems (TcGroup): their tiles are concatenated, so several
// GEMMs pay one ramp-up and one tail. The 2-bit-activation APB layer runs it with the F32R
// epilogue (reference-order per-row scales); the fp32-activation APB layer has its own bf16
// kernel (apb_gemm.cuh).
#pragma once

#include "ptx.cuh"

namespace bitmm_dev {

// I8: int8 operands, s32 accumulators. F4: packed e2m1 operands (+-1 and levels 0..3 are
// exact e2m1 values) through kind::mxf4 with unit scale factors, fp32 accumulators that hold
// exact integers (|sum| <= 9 * 2^20 < 2^24).
enum class Kind : int { I8 = 0, BF16 = 1, F4 = 2 };
// I32: integer units. F32: scale * units. F32R: half_r * units with the reference's per-row
// scale order ((row_pre * alpha_r) * act_scale) * act_gamma (kernels.cpp:193), used by the
// 2-bit-activation APB layer (whose residual SpMM then adds onto C).
enum class Epi : int { I32 = 0, F32 = 1, F32R = 2, ANY = 3 };

constexpr int TC_BN = 256;         // widest output tile (TMEM columns per accumulator)
constexpr int TC_BK_BYTES = 128;   // one 128-byte swizzle row per operand row per stage
constexpr int TC_THREADS = 192;
constexpr int TC_EPI_STRIDE = 36;  // fallback staging row stride in words (conflict-free)
constexpr int TC_GROUP_M = 16;     // tile raster: groups of 16 M-tiles for L2 reuse
constexpr int TC_EPI_BUF = 32 * 32 * 4;        // one 32x32 fp32/int32 block, 128B-swizzled
constexpr int TC_EPI_BYTES = 4 * 2 * TC_EPI_BUF;  // 4 epilogue warps x 2 buffers (widest case)

// BN = output columns per tile (256, or 128 when 256-wide tiles leave a ragged last wave).
template <bool PAIR, int BN = TC_BN>
struct TcShape {
  static constexpr int A_ROWS = 128;                 // A rows staged per CTA
  static constexpr int B_ROWS = PAIR ? BN / 2 : BN;  // B rows staged per CTA
  static constexpr int TILE_M = PAIR ? 256 : 128;    // output rows per tile
  // Epilogue staging per warp: two swizzled 4 KB blocks, or (BN = 192, whose operand stages
  // are smaller) one block in a 5 KB slot so a seventh operand stage fits; the slot also
  // holds the stride-36 fallback staging (4.5 KB).
  static constexpr int EPI_BUFS = (PAIR && BN == 192) ? 1 : 2;
  static constexpr int EPI_WARP_BYTES = EPI_BUFS == 2 ? 2 * TC_EPI_BUF : 5120;
  static constexpr int EPI_BYTES = 4 * EPI_WARP_BYTES;
  static constexpr int COLS_BYTES = BN * 4;  // the tile's column scales (F32 epilogue)
  static constexpr int STAGES =
      PAIR ? (232448 - 1024 - EPI_BYTES - COLS_BYTES - 256) / ((128 + BN / 2) * TC_BK_BYTES) : 4;
  static constexpr int A_STAGE = A_ROWS * TC_BK_BYTES;
  static constexpr int B_STAGE = B_ROWS * TC_BK_BYTES;
  static constexpr int BAR_BYTES = (2 * STAGES + 4) * 8 + 16;
  static constexpr int SMEM =
      1024 + STAGES * (A_STAGE + B_STAGE) + EPI_BYTES + COLS_BYTES + BAR_BYTES;
  static_assert(SMEM <= 232448, "shared memory budget");
};

struct TcParams {
  int M, N;          // output rows / columns
  int num_kb;        // K blocks (of 128 bytes) walked along B
  int shift;         // integer units = acc << shift
  float scale;       // scalar multiplier (reference scale, built on the host)
  const float* row_scale;  // optional per-output-row multiplier [M]
  const float* col_scale;  // optional per-output-column multiplier [N]
  int32_t* out_i32;
  float* out_f32;
  long long ldc;
  // F32R: per-row scale factors in the reference's multiplication order
  float row_pre, act_scale, act_gamma;
  int tma_store;     // 1: output through the tensor map (ldc*4 % 16 == 0, 16B-aligned base)
  int small_acc;     // F4: every |units| < 2^22 (36 * kpad < 2^22), float -> int by magic add
  float shift_mul;   // F4: 2^shift
  int epi;           // this problem's epilogue (Epi::I32 / Epi::F32) under Epi::ANY
  int num_m_blocks, num_n_blocks, num_tiles;
  int group_m;       // tile raster: groups of group_m M-blocks walked column by column
};

// Tile t of a grid with num_n column groups -> (mb, n-group), raster in groups of group_m
// M-blocks so the CTAs working at the same time share operand blocks in L2.
__device__ __forceinline__ void tc_tile_coords(int t, const TcParams& p, int num_n, int& mb, int& nb) {
  const int group_tiles = p.group_m * num_n;
  const int g = t / group_tiles;
  const int first_m = g * p.group_m;
  const int gm = min(p.group_m, p.num_m_blocks - first_m);
  const int within = t - g * group_tiles;
  mb = first_m + within % gm;
  nb = within / gm;
}

// Drains one 128-row x 256-column TMEM accumulator owned by this CTA into global
// memory. Warp w (2..5) reads TMEM lanes 32*(w%4).. (one output row per thread) in
// 32-column blocks. TMA path: the block is written into one of the warp's two 4 KB
// buffers in the 128B-swizzled layout (16-byte chunk j of row r at chunk j ^ (r & 7):
// conflict-free), then lane 0 issues one bulk tensor store and moves on; a buffer is
// rewritten only after the store issued from it two blocks earlier has finished reading.
// Fallback (unaligned ldc): stride-36 staging and coalesced 4-row x 128 B stores.
// cs: the tile's column scales staged in shared memory (nullptr: no column scale).
// This thread's row multiplier (F32: scale * row_scale[r]; F32R: the reference-order
// product). Loaded by the caller before it waits for the accumulator.
template <Epi EPI>
__device__ __forceinline__ float tc_row_mul(const TcParams& p, int my_row) {
  float row_mul = p.scale;
  if constexpr (EPI == Epi::F32) {
    if (p.row_scale != nullptr && my_row < p.M) row_mul = p.scale * p.row_scale[my_row];
  } else if constexpr (EPI == Epi::F32R) {
    if (p.row_scale != nullptr && my_row < p.M)
      row_mul = __fmul_rn(__fmul_rn(__fmul_rn(p.row_pre, p.row_scale[my_row]), p.act_scale),
                          p.act_gamma);
  }
  return row_mul;
}

template <Epi EPI, int BN, bool F32ACC = false, int EPI_BUFS = 2>
__device__ __forceinline__ void tc_epilogue_tile(const TcParams& p, const CUtensorMap* tmC,
                                                 uint32_t tmem_acc, int quad, int lane,
                                                 int row_base, int col_base, float* stg,
                                                 uint32_t& buf, const float* cs, float row_mul,
                                                 int width = BN) {
  // 16-byte stores in the fallback only when every row start is 16-byte aligned
  const void* out_base = (EPI == Epi::I32) ? static_cast<const void*>(p.out_i32) : static_cast<const void*>(p.out_f32);
  const bool vec_ok = ((p.N | static_cast<int>(p.ldc & 3)) & 3) == 0 && (reinterpret_cast<uintptr_t>(out_base) & 15) == 0;
  const uint32_t lane_base = tmem_acc + (static_cast<uint32_t>(quad * 32) << 16);
  const int nch = min(width / 32, (p.N - col_base + 31) / 32);
  // One 32-column chunk: per-thread (row) transform, staged into smem, then stored.
  auto drain = [&](uint32_t (&v)[32], int c) {
    const int col0 = col_base + c * 32;
    float* sb = stg + buf * (TC_EPI_BUF / 4);
    if (p.tma_store) {
      if (lane == 0) bulk_wait_group_read<EPI_BUFS - 1>();
      __syncwarp();
    }
    // Transform f(i) of the 32 columns, staged as four-word groups.
    auto stage = [&](auto f) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o;
        float* of = reinterpret_cast<float*>(&o);
#pragma unroll
        for (int e = 0; e < 4; ++e) of[e] = f(j + e);
        const int off = p.tma_store ? lane * 32 + (((j >> 2) ^ (lane & 7)) << 2) : lane * TC_EPI_STRIDE + j;
        *reinterpret_cast<float4*>(&sb[off]) = o;
      }
    };
    if constexpr (F32ACC && EPI == Epi::I32) {
      // fp32 accumulator holding an exact integer acc; units = acc * 2^shift, exact in fp32.
      // Small accumulators (|units| < 2^22) convert with one FFMA magic add (1.5 * 2^23) and
      // one integer subtract; the branch is uniform, outside the element loop.
      if (p.small_acc) {
        stage([&](int i) {
          return __int_as_float(__float_as_int(__fmaf_rn(__uint_as_float(v[i]), p.shift_mul, 12582912.0f)) -
                                0x4B400000);
        });
      } else {
        stage([&](int i) { return __int_as_float(__float2int_rn(__fmul_rn(__uint_as_float(v[i]), p.shift_mul))); });
      }
    } else if constexpr (F32ACC) {
      stage([&](int i) {
        const float units = __fmul_rn(__uint_as_float(v[i]), p.shift_mul);  // exact: x 1, 2 or 4
        float s = row_mul;
        if constexpr (EPI == Epi::F32) {
          if (cs != nullptr) s = __fmul_rn(s, cs[c * 32 + i]);
        }
        return __fmul_rn(s, units);
      });
    } else if constexpr (EPI == Epi::I32) {
      stage([&](int i) { return __int_as_float(static_cast<int>(v[i]) << p.shift); });
    } else if constexpr (EPI == Epi::F32) {
      stage([&](int i) {
        const float units = static_cast<float>(static_cast<int>(v[i]) << p.shift);
        float s = row_mul;
        if (cs != nullptr) s = __fmul_rn(s, cs[c * 32 + i]);
        return __fmul_rn(s, units);
      });
    } else {
      stage([&](int i) { return __fmul_rn(row_mul, static_cast<float>(static_cast<int>(v[i]) << p.shift)); });
    }
    if (p.tma_store) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmC, sb, col0, row_base);
        bulk_commit_group();
      }
      if constexpr (EPI_BUFS == 2) buf ^= 1u;
      return;
    }
    __syncwarp();
    // ---- fallback write-out: 4 rows x 128 B per warp instruction ----
#pragma unroll
    for (int r8 = 0; r8 < 8; ++r8) {
      const int rl = r8 * 4 + (lane >> 3);
      const int cl = (lane & 7) * 4;
      const int grow = row_base + rl;
      const int gcol = col0 + cl;
      if (grow < p.M) {
        const float4 val = *reinterpret_cast<const float4*>(&sb[rl * TC_EPI_STRIDE + cl]);
        void* dst_base = (EPI == Epi::I32) ? static_cast<void*>(p.out_i32)
                                           : static_cast<void*>(p.out_f32);
        uint32_t* dst = static_cast<uint32_t*>(dst_base) + static_cast<long long>(grow) * p.ldc;
        if (vec_ok && gcol + 3 < p.N) {
          *reinterpret_cast<float4*>(dst + gcol) = val;
        } else {
          const float* vf = reinterpret_cast<const float*>(&val);
          for (int e = 0; e < 4; ++e)
            if (gcol + e < p.N) dst[gcol + e] = __float_as_uint(vf[e]);
        }
      }
    }
    __syncwarp();
  };
  // Software pipeline over chunks: the TMEM load of chunk c+1 is in flight while chunk c is
  // transformed and stored (tcgen05.wait::ld waits for every earlier load of the thread).
  uint32_t va[32], vb[32];
  if (nch > 0) tmem_ld_32x32b_x32(lane_base, va);
#pragma unroll 1
  for (int c = 0; c < nch; c += 2) {
    tmem_ld_wait();
    if (c + 1 < nch) tmem_ld_32x32b_x32(lane_base + (c + 1) * 32, vb);
    drain(va, c);
    if (c + 1 >= nch) break;
    tmem_ld_wait();
    if (c + 2 < nch) tmem_ld_32x32b_x32(lane_base + (c + 2) * 32, va);
    drain(vb, c + 1);
  }
}

// A launch covers a group of up to NP independent GEMM problems (a single call is a group of
// one): every problem has its own operand / output tensor maps and parameters, and the
// persistent grid walks the concatenation of their tiles, so a step of several GEMMs pays one
// ramp-up and one tail instead of one per GEMM.
constexpr int TC_GROUP_MAX = 4;
#ifdef TC_GEMM_STATS
// Profiling build only (profiles/micro/real_kernel.cu): cycles per CTA the MMA issuer waits on
// tempty [0] / full [1] and its total [2]; epilogue warp 2 waiting on tfull [3] / draining [4].
__device__ unsigned long long tcg_stats[6][160];
#endif

template <int NP>
struct TcGroup {
  CUtensorMap a[NP], b[NP], c[NP];
  TcParams prob[NP];
  int count;
  int tile_begin[NP + 1];  // problem i owns tiles [tile_begin[i], tile_begin[i+1])
  // Balanced schedule (optional): CTA pair u walks pieces [unit_begin[u], unit_begin[u + 1]) of
  // `sched`, each {problem | width << 16, m block, first column, 0}: a contiguous stretch of the
  // output column-work, cut into pieces of at most BN columns (multiples of 32), so every pair
  // gets the same number of columns instead of a whole number of BN-wide tiles. Null: tiles
  // round-robin.
  const int4* sched;
  const int* unit_begin;
};

template <int NP>
__device__ __forceinline__ int tc_problem_of(const TcGroup<NP>& g, int t) {
  if constexpr (NP == 1) return 0;
  int pi = 0;
#pragma unroll
  for (int i = 1; i < NP; ++i)
    if (i < g.count && t >= g.tile_begin[i]) pi = i;
  return pi;
}

// The tiles (or balanced pieces) one CTA pair walks, in order: problem, m block, first output
// column and width of each.
template <int NP, int BN, int MC>
struct TcTileIter {
  const TcGroup<NP>& g;
  int i, end, step, pair;
  __device__ __forceinline__ TcTileIter(const TcGroup<NP>& g_, int unit, int num_units, int pair_)
      : g(g_), pair(pair_) {
    if (g.sched) {
      i = g.unit_begin[unit];
      end = g.unit_begin[unit + 1];
      step = 1;
    } else {
      i = unit;
      end = g.tile_begin[g.count];
      step = num_units;
    }
  }
  __device__ __forceinline__ bool next(int& pi, int& mb, int& n0, int& width) {
    if (i >= end) return false;
    if (g.sched) {
      const int4 r = g.sched[i];
      pi = r.x & 0xFFFF;
      width = r.x >> 16;
      mb = r.y;
      n0 = r.z;
    } else {
      pi = tc_problem_of(g, i);
      const TcParams& p = g.prob[pi];
      int nb;
      tc_tile_coords(i - g.tile_begin[pi], p, (p.num_n_blocks + MC - 1) / MC, mb, nb);
      n0 = (nb * MC + pair) * BN;
      width = BN;
    }
    i += step;
    return true;
  }
};


// Persistent cta_group::2 GEMM (one CTA pair per cluster). EPI == Epi::ANY dispatches each
// problem's epilogue (I32 or F32) at run time.
// MC = CTA pairs per cluster. MC = 2 (measured, not used by the library: DESIGN.md) runs two
// pairs of a four-CTA cluster on horizontally adjacent tiles; each pair loads half of the
// shared A rows and multicasts it to the same-rank CTA of the other pair, and every stage
// release is committed to all four CTAs. The host then builds the A map with A_ROWS / 2-row
// boxes, counts tiles in pairs of N blocks and launches clusters of four.
template <Kind KIND, Epi EPI, int BN, int NP, int MC = 1>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ TcGroup<NP> g) {
  using S = TcShape<true, BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (base_u32 & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + S::STAGES * S::A_STAGE;
  float* sEpi = reinterpret_cast<float*>(sB + S::STAGES * S::B_STAGE);
  float* sCols = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sEpi) + S::EPI_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sCols) + S::COLS_BYTES);
  uint64_t* empty = full + S::STAGES;
  uint64_t* tfull = empty + S::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1u;               // rank within the CTA pair
  const int pair = static_cast<int>(crank >> 1);  // pair within the cluster (MC = 2)
  const int unit = static_cast<int>(cluster_id_x());
  const int num_units = static_cast<int>(num_clusters_x());

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < g.count; ++i) {
      tma_prefetch_desc(&g.a[i]);
      tma_prefetch_desc(&g.b[i]);
      if (g.prob[i].tma_store) tma_prefetch_desc(&g.c[i]);
    }
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);  // one release per pair of the cluster
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
  constexpr uint32_t kSfCol = 2 * BN;  // F4: scale factors after the two accumulators
  if constexpr (KIND == Kind::F4) {
    // every scale-factor cell = E8M0 1.0 (0x7F), for both the A and B scale regions
    if (warp >= 2) {
      const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
      tmem_st_32x32b_x32_fill(tmem_base + lane_off + kSfCol, 0x7F7F7F7Fu);
      tmem_st_32x32b_x32_fill(tmem_base + lane_off + kSfCol + 32, 0x7F7F7F7Fu);
      tmem_st_wait();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
  }
  // Everything above overlapped the producer of our operands (PDL); from here on
  // we read its output.
  pdl_wait();

  // TMA inner coordinate per 128-byte K block (operand maps are in bytes for I8 and F4)
  constexpr int BK_ELEMS = (KIND == Kind::BF16) ? TC_BK_BYTES / 2 : TC_BK_BYTES;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs of a pair) =====================
    // At FP4 rates a stage lasts ~384 cycles, and this single thread issues every load, so
    // the k-block loop is kept to a handful of instructions (no division / modulo: a
    // dependent MUFU.RCP chain per stage starved the MMA).
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      constexpr uint32_t kTx = 2 * (S::A_STAGE + S::B_STAGE);
      TcTileIter<NP, BN, MC> tiles(g, unit, num_units, pair);
      int pi, mb, n0, width;
      while (tiles.next(pi, mb, n0, width)) {
        const TcParams& p = g.prob[pi];
        const int a_row = mb * S::TILE_M + static_cast<int>(rank) * S::A_ROWS;
        // each CTA stages its half of the piece's B rows (a narrower piece leaves the box's
        // last rows unused by the MMA)
        const int b_row = n0 + static_cast<int>(rank) * (width / 2);
        const CUtensorMap* ma = &g.a[pi];
        const CUtensorMap* mbm = &g.b[pi];
        const int nkb = p.num_kb;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], kTx);
          if constexpr (MC == 2) {
            // this pair's half of the A rows, to this CTA and its twin in the other pair
            constexpr int HALF = S::A_ROWS / 2;
            tma_load_2d_pair_mc(sA + stage * S::A_STAGE + pair * HALF * TC_BK_BYTES, ma, &full[stage],
                                kb * BK_ELEMS, a_row + pair * HALF, static_cast<uint16_t>(0x5u << rank));
          } else {
            tma_load_2d_pair(sA + stage * S::A_STAGE, ma, &full[stage], kb * BK_ELEMS, a_row);
          }
          tma_load_2d_pair(sB + stage * S::B_STAGE, mbm, &full[stage], kb * BK_ELEMS, b_row);
          if (++stage == S::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA, whole warp) =====================
    // Warp-uniform state; one elected lane issues each tcgen05 instruction. Descriptors:
    // the stage-0 descriptor plus (byte offset >> 4) in the address field.
    constexpr uint32_t idesc = (KIND == Kind::I8)   ? make_idesc(2u, 1u, 1u, S::TILE_M, BN)
                               : (KIND == Kind::F4) ? make_idesc_mxf4(S::TILE_M, BN)
                                                    : make_idesc(1u, 1u, 1u, S::TILE_M, BN);
    if (rank == 0) {
      constexpr int KID = (KIND == Kind::I8) ? 0 : (KIND == Kind::F4) ? 2 : 1;
      const uint64_t a_desc0 = sw128_kmajor_desc(smem_u32(sA));
      const uint64_t b_desc0 = sw128_kmajor_desc(smem_u32(sB));
      const uint32_t sfa = tmem_base + kSfCol, sfb = tmem_base + kSfCol + 32;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
#ifdef TC_GEMM_STATS
      long long st_te = 0, st_fu = 0, st_start = clock64();
#endif
      TcTileIter<NP, BN, MC> tiles(g, unit, num_units, pair);
      int pi, mb, n0, width;
      for (; tiles.next(pi, mb, n0, width); ++it) {
        const int num_kb = g.prob[pi].num_kb;
        // the piece's width as the MMA's N (a multiple of 32, so of 16 as M = 256 requires)
        const uint32_t idesc_t = (idesc & ~(0x3Fu << 17)) | ((static_cast<uint32_t>(width) >> 3) << 17);
        const int acc = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
#ifdef TC_GEMM_STATS
        long long t0 = clock64();
#endif
        mbar_wait(&tempty[acc], aphase ^ 1u);
#ifdef TC_GEMM_STATS
        st_te += clock64() - t0;
#endif
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
#ifdef TC_GEMM_STATS
          long long t1 = clock64();
#endif
          mbar_wait(&full[stage], phase);
#ifdef TC_GEMM_STATS
          st_fu += clock64() - t1;
#endif
          tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint64_t>((stage * S::A_STAGE) >> 4);
          const uint64_t bd = b_desc0 + static_cast<uint64_t>((stage * S::B_STAGE) >> 4);
#pragma unroll
          for (int k = 0; k < TC_BK_BYTES / 32; ++k)
            mma_pair_elect<KID>(d_tmem, ad + 2 * k, bd + 2 * k, idesc_t, (kb | k) != 0, sfa, sfb);
          mma_commit_pair_elect(&empty[stage], MC == 2 ? 0xF : 0x3);
          if (++stage == S::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit_pair_elect(&tfull[acc], static_cast<uint16_t>(0x3u << (2 * pair)));
      }
#ifdef TC_GEMM_STATS
      if (lane == 0) {
        tcg_stats[0][blockIdx.x] = st_te;
        tcg_stats[1][blockIdx.x] = st_fu;
        tcg_stats[2][blockIdx.x] = clock64() - st_start;
      }
#endif
    }
  } else {
    // ===================== epilogue (warps 2..5 of every CTA) =====================
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    float* stg = sEpi + (warp - 2) * (S::EPI_WARP_BYTES / 4);
    uint32_t buf = 0;
    int it = 0;
#ifdef TC_GEMM_STATS
    long long st_tf = 0, st_busy = 0;
#endif
    TcTileIter<NP, BN, MC> tiles(g, unit, num_units, pair);
    int pi, mb, n0, width;
    for (; tiles.next(pi, mb, n0, width); ++it) {
      const TcParams p = g.prob[pi];  // by value: its fields stay in registers in the epilogue
      const int acc = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int row_base = mb * S::TILE_M + static_cast<int>(rank) * 128 + quad * 32;
      // Row multiplier and column scales of this tile are loaded before the accumulator wait
      // so their latency hides behind it; the column scales are staged into smem below
      // (broadcast reads in the transform).
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
          const int cc = n0 + i;
          csv[j] = (i < width && cc < p.N) ? p.col_scale[cc] : 0.0f;
        }
      }
#ifdef TC_GEMM_STATS
      long long t2 = clock64();
#endif
      mbar_wait(&tfull[acc], aphase);
#ifdef TC_GEMM_STATS
      long long t3 = clock64();
      st_tf += t3 - t2;
#endif
      tc_fence_after();
      constexpr bool kF32Acc = KIND == Kind::F4;
      const uint32_t tacc = tmem_base + acc * BN;
      // Column scales -> smem. The first barrier keeps the previous tile's readers ahead of
      // the overwrite.
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
          tc_epilogue_tile<Epi::I32, BN, kF32Acc, S::EPI_BUFS>(p, &g.c[pi], tacc, quad, lane,
                                                               row_base, n0, stg, buf, cs, row_mul, width);
        else
          tc_epilogue_tile<Epi::F32, BN, kF32Acc, S::EPI_BUFS>(p, &g.c[pi], tacc, quad, lane,
                                                               row_base, n0, stg, buf, cs, row_mul, width);
      } else {
        tc_epilogue_tile<EPI, BN, kF32Acc, S::EPI_BUFS>(p, &g.c[pi], tacc, quad, lane, row_base,
                                                        n0, stg, buf, cs, row_mul, width);
      }
#ifdef TC_GEMM_STATS
      st_busy += clock64() - t3;
#endif
      tc_fence_before();
      mbar_arrive_cluster(smem_u32(&tempty[acc]) & kPeerBitMask);
    }
#ifdef TC_GEMM_STATS
    if (lane == 0 && warp == 2) {
      tcg_stats[3][blockIdx.x] = st_tf;
      tcg_stats[4][blockIdx.x] = st_busy;
    }
#endif
    if (lane == 0) bulk_wait_group_all();  // stores land before the grid ends
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace bitmm_dev
