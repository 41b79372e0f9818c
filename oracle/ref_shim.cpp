// ref_shim.cpp — extern "C" bridge onto the UNMODIFIED reference library, compiled
// from its own sources under /root/reference/proj by oracle/Makefile into
// oracle/_ref/libbitmm_ref.so. TEST INFRASTRUCTURE ONLY: used to pin the oracle
// (tests/golden/make_golden.py) and as bench.py's CPU baseline / reference arm.
//
// Each wrapper adopts caller words with BitMatrix::from_words (tensor.cpp:62-76),
// calls the reference entry point, and copies the DenseMatrix result out. The
// `seconds` out-parameter (nullable) times only the reference call itself, which
// — like the reference's own bench_routine (bench.cpp:129-153) — includes its
// output allocation.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "bitmm/apb.hpp"
#include "bitmm/errors.hpp"
#include "bitmm/kernels.hpp"
#include "bitmm/simd.hpp"
#include "bitmm/tensor.hpp"
#include "bitmm/tensor_io.hpp"
#include "bitmm/transform.hpp"

using namespace bitmm;

namespace {

thread_local std::string g_msg;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const InvalidEncoding& e) {
    g_msg = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_msg = e.what();
    return 1;
  } catch (const IoError& e) {
    g_msg = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 9;
  }
}

BitMatrix bits(const uint64_t* w, int64_t rows, int64_t cols, int64_t wpr) {
  std::vector<uint64_t> v(w, w + rows * wpr);
  return BitMatrix::from_words(rows, cols, static_cast<std::size_t>(wpr), std::move(v));
}

ThmPlanes planes(const uint64_t* t, const uint64_t* h, const uint64_t* m, int64_t rows,
                 int64_t cols, int64_t wpr, float scale, int has_gamma, float gamma) {
  ThmPlanes p;
  p.t = bits(t, rows, cols, wpr);
  p.h = bits(h, rows, cols, wpr);
  p.m = bits(m, rows, cols, wpr);
  p.scale = scale;
  if (has_gamma) p.gamma = gamma;
  return p;
}

DenseMatrix dense(const float* d, int64_t rows, int64_t cols) {
  return DenseMatrix(rows, cols, std::vector<float>(d, d + rows * cols));
}

CsrMatrix csr(int64_t rows, int64_t cols, const uint64_t* row_ptr, const uint64_t* col_idx,
              const float* vals, int64_t nnz) {
  return CsrMatrix::create(rows, cols, std::vector<uint64_t>(row_ptr, row_ptr + rows + 1),
                           std::vector<uint64_t>(col_idx, col_idx + nnz),
                           std::vector<float>(vals, vals + nnz));
}

void copy_out(const DenseMatrix& c, float* out) {
  std::memcpy(out, c.data().data(), c.data().size() * sizeof(float));
}

template <typename Fn>
DenseMatrix timed(double* seconds, Fn&& fn) {
  auto t0 = std::chrono::steady_clock::now();
  DenseMatrix c = fn();
  if (seconds)
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return c;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }

int ref_set_simd(const char* level) {
  return guarded([&] { set_simd_level(parse_simd_level(level)); });
}

const char* ref_active_simd(void) { return simd_level_name(active_simd_level()); }

int ref_gemm_1x1(const uint64_t* a, int64_t m, const uint64_t* b, int64_t n, int64_t k, int64_t wpr,
                 float gamma_a, float gamma_b, int threads, float* out, double* seconds) {
  return guarded([&] {
    BitMatrix A = bits(a, m, k, wpr), B = bits(b, n, k, wpr);
    copy_out(timed(seconds, [&] { return gemm_1x1(A, B, gamma_a, gamma_b, threads); }), out);
  });
}

int ref_gemm_1x2(const uint64_t* w, int64_t m, float gamma, const uint64_t* t, const uint64_t* h,
                 const uint64_t* mm, int64_t n, int64_t k, int64_t wpr, float scale, int has_gamma,
                 float a_gamma, int threads, float* out, double* seconds) {
  return guarded([&] {
    BitMatrix W = bits(w, m, k, wpr);
    ThmPlanes P = planes(t, h, mm, n, k, wpr, scale, has_gamma, a_gamma);
    copy_out(timed(seconds, [&] { return gemm_1x2(W, gamma, P, threads); }), out);
  });
}

int ref_gemm_2x2(const uint64_t* wt, const uint64_t* wh, const uint64_t* wm, int64_t m,
                 float w_scale, int has_w_gamma, float w_gamma, const uint64_t* at,
                 const uint64_t* ah, const uint64_t* am, int64_t n, int64_t k, int64_t wpr,
                 float a_scale, int has_a_gamma, float a_gamma, int threads, float* out,
                 double* seconds) {
  return guarded([&] {
    ThmPlanes W = planes(wt, wh, wm, m, k, wpr, w_scale, has_w_gamma, w_gamma);
    ThmPlanes A = planes(at, ah, am, n, k, wpr, a_scale, has_a_gamma, a_gamma);
    copy_out(timed(seconds, [&] { return gemm_2x2(W, A, threads); }), out);
  });
}

int ref_gemm_1x32(const uint64_t* w, int64_t m, int64_t k, int64_t wpr, float gamma,
                  const float* b, int64_t n, int threads, float* out, double* seconds) {
  return guarded([&] {
    BitMatrix W = bits(w, m, k, wpr);
    DenseMatrix B = dense(b, k, n);
    copy_out(timed(seconds, [&] { return gemm_1x32_ref(W, gamma, B, threads); }), out);
  });
}

int ref_spmm_csr(int64_t rows, int64_t cols, const uint64_t* row_ptr, const uint64_t* col_idx,
                 const float* vals, int64_t nnz, const float* b, int64_t n, int threads,
                 float* out, double* seconds) {
  return guarded([&] {
    CsrMatrix A = csr(rows, cols, row_ptr, col_idx, vals, nnz);
    DenseMatrix B = dense(b, cols, n);
    copy_out(timed(seconds, [&] { return spmm_csr(A, B, threads); }), out);
  });
}

int ref_layer_forward(int64_t rows, int64_t cols, float alpha, const uint64_t* bin, int64_t wpr,
                      const uint64_t* row_ptr, const uint64_t* col_idx, const float* vals,
                      int64_t nnz, const float* b, int64_t n, int threads, float* out,
                      double* seconds) {
  return guarded([&] {
    ApbLayer l;
    l.rows = rows;
    l.cols = cols;
    l.alpha = alpha;
    l.bin = bits(bin, rows, cols, wpr);
    l.residual = csr(rows, cols, row_ptr, col_idx, vals, nnz);
    DenseMatrix B = dense(b, cols, n);
    copy_out(timed(seconds, [&] { return layer_forward(l, B, threads); }), out);
  });
}

int ref_apb_forward(const float* w, int64_t rows, int64_t cols, float alpha, float delta,
                    float* out) {
  return guarded([&] { copy_out(apb_forward(dense(w, rows, cols), ApbParams{alpha, delta}), out); });
}

// decompose_apb: first call with col_idx == NULL to learn nnz (returned in *nnz_out).
int ref_decompose_apb(const float* a, int64_t rows, int64_t cols, float alpha, int lane_bits,
                      uint64_t* bin, int64_t* wpr_out, uint64_t* row_ptr, uint64_t* col_idx,
                      float* vals, int64_t* nnz_out) {
  return guarded([&] {
    ApbLayer l = decompose_apb(dense(a, rows, cols), alpha, lane_bits);
    *wpr_out = static_cast<int64_t>(l.bin.words_per_row());
    *nnz_out = static_cast<int64_t>(l.residual.nnz());
    if (bin) std::memcpy(bin, l.bin.words().data(), l.bin.words().size() * 8);
    if (row_ptr) std::memcpy(row_ptr, l.residual.row_ptr.data(), l.residual.row_ptr.size() * 8);
    if (col_idx) std::memcpy(col_idx, l.residual.col_idx.data(), l.residual.col_idx.size() * 8);
    if (vals) std::memcpy(vals, l.residual.vals.data(), l.residual.vals.size() * 4);
  });
}

int ref_pack_signs(const float* a, int64_t rows, int64_t cols, int lane_bits, uint64_t* words,
                   int64_t* wpr_out) {
  return guarded([&] {
    BitMatrix b = pack_signs(dense(a, rows, cols), lane_bits);
    *wpr_out = static_cast<int64_t>(b.words_per_row());
    if (words) std::memcpy(words, b.words().data(), b.words().size() * 8);
  });
}

int ref_decompose_thm(const uint8_t* levels, int64_t rows, int64_t cols, float scale, int lane_bits,
                      uint64_t* t, uint64_t* h, uint64_t* m, int64_t* wpr_out) {
  return guarded([&] {
    TwoBitMatrix q;
    q.rows = rows;
    q.cols = cols;
    q.scale = scale;
    q.levels.assign(levels, levels + rows * cols);
    ThmPlanes p = decompose_thm(q, std::nullopt, lane_bits);
    *wpr_out = static_cast<int64_t>(p.t.words_per_row());
    if (t) std::memcpy(t, p.t.words().data(), p.t.words().size() * 8);
    if (h) std::memcpy(h, p.h.words().data(), p.h.words().size() * 8);
    if (m) std::memcpy(m, p.m.words().data(), p.m.words().size() * 8);
  });
}

int ref_quantize_2bit(const float* a, int64_t rows, int64_t cols, float s, uint8_t* levels) {
  return guarded([&] {
    TwoBitMatrix q = quantize_uniform_2bit(dense(a, rows, cols), s);
    std::memcpy(levels, q.levels.data(), q.levels.size());
  });
}

int ref_dot_binary(const uint64_t* u, const uint64_t* v, int64_t words, int64_t n, int64_t* out) {
  return guarded([&] {
    *out = dot_binary({u, static_cast<std::size_t>(words)}, {v, static_cast<std::size_t>(words)}, n);
  });
}

int ref_mbm(const uint64_t* x, const uint64_t* y, const uint64_t* z, int64_t words, int64_t* out) {
  return guarded([&] {
    const auto w = static_cast<std::size_t>(words);
    *out = mbm({x, w}, {y, w}, {z, w});
  });
}

// ---- BTSR containers through the reference's own writer / reader (tensor_io.cpp) ----
int ref_store_dense(const char* path, const float* a, int64_t rows, int64_t cols) {
  return guarded([&] { store_tensor(path, dense(a, rows, cols)); });
}

int ref_store_bit(const char* path, const uint64_t* w, int64_t rows, int64_t cols, int64_t wpr) {
  return guarded([&] { store_tensor(path, bits(w, rows, cols, wpr)); });
}

int ref_store_csr(const char* path, int64_t rows, int64_t cols, const uint64_t* row_ptr,
                  const uint64_t* col_idx, const float* vals, int64_t nnz) {
  return guarded([&] { store_tensor(path, csr(rows, cols, row_ptr, col_idx, vals, nnz)); });
}

// The reference CLI's `pack --mode apb` branch (tools/bitmm_main.cpp:195-207): params given
// (has_params) or init_alpha_delta(w), apb_forward, decompose_apb, store_apb_layer(prefix).
// Writes the chosen alpha / delta back.
int ref_pack_apb(const float* w, int64_t rows, int64_t cols, int has_params, float* alpha,
                 float* delta, const char* prefix) {
  return guarded([&] {
    DenseMatrix W = dense(w, rows, cols);
    ApbParams p;
    if (has_params) {
      p.alpha = *alpha;
      p.delta = *delta;
    } else {
      p = init_alpha_delta(W);
    }
    store_apb_layer(prefix, decompose_apb(apb_forward(W, p), p.alpha));
    *alpha = p.alpha;
    *delta = p.delta;
  });
}

int ref_store_thm_planes(const char* prefix, const uint64_t* t, const uint64_t* h, const uint64_t* m,
                         int64_t rows, int64_t cols, int64_t wpr, float scale, int has_gamma,
                         float gamma) {
  return guarded([&] {
    store_thm_planes(prefix, planes(t, h, m, rows, cols, wpr, scale, has_gamma, gamma));
  });
}

// Loads with the reference reader; kind -1 any, 0 dense, 1 bit, 2 csr (load_dense / load_bit /
// load_csr), 3 thm plane prefix. Returns 0 or the error class (message via ref_last_error).
int ref_load_check(const char* path, int kind) {
  return guarded([&] {
    if (kind == 0) (void)load_dense(path);
    else if (kind == 1) (void)load_bit(path);
    else if (kind == 2) (void)load_csr(path);
    else if (kind == 3) (void)load_thm_planes(path);
    else (void)load_tensor(path);
  });
}

}  // extern "C"
