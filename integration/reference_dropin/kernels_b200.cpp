// kernels_b200.cpp — reference-side binding of the B200 library (drop-in for the GEMM
// bodies of /root/reference/proj/src/kernels.cpp:163-352 and apb.cpp:158-164, and for the
// packers pack_signs (tensor.cpp:155-164), decompose_thm (transform.cpp:47-75) and
// decompose_apb (apb.cpp:119-142)).
//
// Compiled against the reference's OWN headers (include/bitmm/*.hpp) and linked in place
// of those function bodies, it keeps every public signature, argument check, exception
// type and message order of the reference, and routes the arithmetic through the C ABI
// in include/bitmm_b200.h (host-pointer flavour: the result comes back as the
// reference's DenseMatrix). The `threads` argument is validated and otherwise ignored
// (results never depended on it, kernels.cpp:47-49).
//
// Build recipe (see INTEGRATION.md and oracle/Makefile target `dropin`): compile the
// reference sources unmodified, weaken the nine replaced symbols in their objects
// (objcopy --weaken-symbol), link this file plus libbitmm_b200.so.
#include <optional>
#include <span>
#include <stdexcept>
#include <string>

#include "bitmm/apb.hpp"
#include "bitmm/errors.hpp"
#include "bitmm/kernels.hpp"
#include "bitmm/tensor.hpp"
#include "bitmm/transform.hpp"
#include "bitmm_b200.h"

namespace bitmm {

namespace {

void raise_on(int rc) {
  if (rc == BITMM_OK) return;
  const std::string msg = bitmm_last_error();
  if (rc == BITMM_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == BITMM_ERR_INVALID_ENCODING) throw InvalidEncoding(msg);
  throw std::runtime_error("bitmm_b200: " + msg);
}

void check_threads(int threads) {
  if (threads < 1) throw std::invalid_argument("thread count must be at least 1");
}

void check_packed_pair(std::int64_t cols_a, std::size_t wpr_a, std::int64_t cols_b,
                       std::size_t wpr_b) {
  if (cols_a != cols_b || wpr_a != wpr_b)
    throw std::invalid_argument("gemm dimension mismatch (packed rows must share K and padding)");
}

float plane_gamma(const ThmPlanes& p) { return p.gamma.value_or(1.0f); }

}  // namespace

// ---- packers: the GPU packers behind the host ABI (same layouts, checks and messages) ----
BitMatrix pack_signs(const DenseMatrix& m, int lane_bits) {
  BitMatrix b(m.rows(), m.cols(), lane_bits);  // the reference's lane / dimension checks
  if (m.rows() == 0 || b.words_per_row() == 0) return b;
  raise_on(bitmm_pack_signs_host(m.cols() > 0 ? m.row_data(0) : nullptr, m.rows(), m.cols(),
                                 m.cols(), b.row_data(0),
                                 static_cast<std::int64_t>(b.words_per_row())));
  return b;
}

ThmPlanes decompose_thm(const TwoBitMatrix& q, std::optional<float> gamma, int lane_bits) {
  ThmPlanes p;
  p.t = BitMatrix(q.rows, q.cols, lane_bits);
  p.h = BitMatrix(q.rows, q.cols, lane_bits);
  p.m = BitMatrix(q.rows, q.cols, lane_bits);
  p.scale = q.scale;
  p.gamma = gamma;
  if (q.rows == 0 || p.t.words_per_row() == 0) return p;
  // a level above 3 -> std::invalid_argument("2-bit level out of range"), transform.cpp:70-71
  raise_on(bitmm_decompose_thm_host(q.levels.data(), q.rows, q.cols, p.t.row_data(0),
                                    p.h.row_data(0), p.m.row_data(0),
                                    static_cast<std::int64_t>(p.t.words_per_row())));
  return p;
}

ApbLayer decompose_apb(const DenseMatrix& a, float alpha, int lane_bits) {
  if (!(alpha > 0.0f)) throw std::invalid_argument("alpha must be positive");
  ApbLayer l;
  l.rows = a.rows();
  l.cols = a.cols();
  l.alpha = alpha;
  l.bin = BitMatrix(a.rows(), a.cols(), lane_bits);
  std::vector<std::uint64_t> row_ptr(static_cast<std::size_t>(a.rows()) + 1, 0);
  const float* src = a.rows() > 0 && a.cols() > 0 ? a.row_data(0) : nullptr;
  std::uint64_t* bin = l.bin.words_per_row() > 0 && a.rows() > 0 ? l.bin.row_data(0) : nullptr;
  const auto wpr = static_cast<std::int64_t>(l.bin.words_per_row());
  std::int64_t nnz = 0;
  raise_on(bitmm_decompose_apb_host(src, a.rows(), a.cols(), a.cols(), alpha, nullptr, bin, wpr,
                                    row_ptr.data(), nullptr, nullptr, 0, &nnz));
  std::vector<std::uint64_t> col_idx(static_cast<std::size_t>(nnz));
  std::vector<float> vals(static_cast<std::size_t>(nnz));
  if (nnz > 0)
    raise_on(bitmm_decompose_apb_host(src, a.rows(), a.cols(), a.cols(), alpha, nullptr, bin, wpr,
                                      row_ptr.data(), col_idx.data(), vals.data(), nnz, &nnz));
  l.residual = CsrMatrix::create(a.rows(), a.cols(), std::move(row_ptr), std::move(col_idx),
                                 std::move(vals));
  return l;
}

#ifdef BITMM_DROPIN_ROWOPS_GPU
// ---- row ops (kernels.cpp:120-140) on the GPU, one row pair per call. Not in the default
// drop-in: a call costs a launch plus two tiny copies (tens of microseconds) where the
// reference's AVX-512 loop takes nanoseconds, and verify.cpp / acceptance.cpp call them
// millions of times; the batched device calls are the GPU's form. ----
std::int64_t dot_binary(std::span<const std::uint64_t> u, std::span<const std::uint64_t> v,
                        std::int64_t n) {
  if (u.size() != v.size()) throw std::invalid_argument("bit row word counts differ");
  if (n < 0 || static_cast<std::size_t>((n + 63) / 64) > u.size())
    throw std::invalid_argument("logical length does not fit the row words");
  if (u.empty()) return 0;
  std::int64_t out = 0;
  raise_on(bitmm_dot_binary_host(u.data(), v.data(), 1, static_cast<std::int64_t>(u.size()), n, &out));
  return out;
}

std::int64_t mbm(std::span<const std::uint64_t> x, std::span<const std::uint64_t> y,
                 std::span<const std::uint64_t> z) {
  if (x.size() != y.size() || x.size() != z.size())
    throw std::invalid_argument("bit row word counts differ");
  if (x.empty()) return 0;
  std::int64_t out = 0;
  raise_on(bitmm_mbm_host(x.data(), y.data(), z.data(), 1, static_cast<std::int64_t>(x.size()), &out));
  return out;
}
#endif

// The three GEMMs return a fresh DenseMatrix (kernels.cpp:163-275). The binding hands the
// library a callback that constructs it (the reference's zero-filling constructor) once the
// call's copies and kernels are enqueued, so that allocation overlaps the device work
// (bitmm_gemm_host_late); the result is then copied straight into it.
namespace {

struct LateDense {
  std::int64_t rows, cols;
  std::optional<DenseMatrix> c;
};

int make_late_dense(void* user, bitmm_host_out* out) {
  auto* l = static_cast<LateDense*>(user);
  l->c.emplace(l->rows, l->cols);
  out->c = l->c->row_data(0);
  out->ldc = l->cols;
  return 0;
}

DenseMatrix run_late(const bitmm_gemm_item& it) {
  LateDense l{it.m, it.n, std::nullopt};
  raise_on(bitmm_gemm_host_late(&it, BITMM_WANT_C, &make_late_dense, &l));
  return std::move(*l.c);
}

}  // namespace

DenseMatrix gemm_1x1(const BitMatrix& a, const BitMatrix& b_packed, float gamma_a, float gamma_b,
                     int threads) {
  check_packed_pair(a.cols(), a.words_per_row(), b_packed.cols(), b_packed.words_per_row());
  GemmProblem{a.rows(), a.cols(), b_packed.rows()}.validate();
  check_threads(threads);
  bitmm_gemm_item it{};
  it.routine = BITMM_ROUTINE_1X1;
  it.a0 = a.row_data(0);
  it.b0 = b_packed.row_data(0);
  it.m = a.rows();
  it.n = b_packed.rows();
  it.k = a.cols();
  it.wpr = static_cast<std::int64_t>(a.words_per_row());
  it.a_scale = gamma_a;
  it.b_scale = gamma_b;
  return run_late(it);
}

DenseMatrix gemm_1x2(const BitMatrix& w, float gamma, const ThmPlanes& a_packed, int threads) {
  a_packed.validate();  // InvalidEncoding first, as kernels.cpp:186
  check_packed_pair(w.cols(), w.words_per_row(), a_packed.cols(), a_packed.t.words_per_row());
  GemmProblem{w.rows(), w.cols(), a_packed.rows()}.validate();
  check_threads(threads);
  bitmm_gemm_item it{};
  it.routine = BITMM_ROUTINE_1X2;
  it.a0 = w.row_data(0);
  it.b0 = a_packed.t.row_data(0);
  it.b1 = a_packed.h.row_data(0);
  it.b2 = a_packed.m.row_data(0);
  it.m = w.rows();
  it.n = a_packed.rows();
  it.k = w.cols();
  it.wpr = static_cast<std::int64_t>(w.words_per_row());
  it.a_scale = gamma;
  it.b_scale = a_packed.scale;
  it.has_b_gamma = a_packed.gamma.has_value() ? 1 : 0;
  it.b_gamma = plane_gamma(a_packed);
  return run_late(it);
}

DenseMatrix gemm_2x2(const ThmPlanes& w, const ThmPlanes& a_packed, int threads) {
  w.validate();  // kernels.cpp:224-225
  a_packed.validate();
  check_packed_pair(w.cols(), w.t.words_per_row(), a_packed.cols(), a_packed.t.words_per_row());
  GemmProblem{w.rows(), w.cols(), a_packed.rows()}.validate();
  check_threads(threads);
  bitmm_gemm_item it{};
  it.routine = BITMM_ROUTINE_2X2;
  it.a0 = w.t.row_data(0);
  it.a1 = w.h.row_data(0);
  it.a2 = w.m.row_data(0);
  it.b0 = a_packed.t.row_data(0);
  it.b1 = a_packed.h.row_data(0);
  it.b2 = a_packed.m.row_data(0);
  it.m = w.rows();
  it.n = a_packed.rows();
  it.k = w.cols();
  it.wpr = static_cast<std::int64_t>(w.t.words_per_row());
  it.a_scale = w.scale;
  it.has_a_gamma = w.gamma.has_value() ? 1 : 0;
  it.a_gamma = plane_gamma(w);
  it.b_scale = a_packed.scale;
  it.has_b_gamma = a_packed.gamma.has_value() ? 1 : 0;
  it.b_gamma = plane_gamma(a_packed);
  return run_late(it);
}

DenseMatrix gemm_1x32_ref(const BitMatrix& w, float gamma, const DenseMatrix& b, int threads) {
  if (w.cols() != b.rows()) throw std::invalid_argument("gemm dimension mismatch");
  GemmProblem{w.rows(), w.cols(), b.cols()}.validate();
  check_threads(threads);
  DenseMatrix c(w.rows(), b.cols());
  raise_on(bitmm_gemm_1x32_host(w.row_data(0), w.rows(), w.cols(),
                                static_cast<std::int64_t>(w.words_per_row()), gamma, nullptr,
                                b.row_data(0), b.cols(), b.cols(), c.row_data(0), c.cols()));
  return c;
}

DenseMatrix spmm_csr(const CsrMatrix& a, const DenseMatrix& b, int threads) {
  if (a.cols != b.rows()) throw std::invalid_argument("gemm dimension mismatch");
  if (a.rows <= 0 || b.cols() <= 0 || a.cols <= 0)
    throw std::invalid_argument("gemm dimensions must be positive");
  if (a.cols > kMaxSharedDim)
    throw std::invalid_argument("shared dimension exceeds the 2^20 accumulator bound");
  check_threads(threads);
  DenseMatrix c(a.rows, b.cols());
  raise_on(bitmm_spmm_csr_host(a.rows, a.cols, a.row_ptr.data(), a.col_idx.data(), a.vals.data(),
                               static_cast<std::int64_t>(a.nnz()), b.row_data(0), b.cols(),
                               b.cols(), c.row_data(0), c.cols()));
  return c;
}

DenseMatrix layer_forward(const ApbLayer& l, const DenseMatrix& b, int threads) {
  // the reference's two calls (apb.cpp:159-160) perform these checks in this order
  if (l.bin.cols() != b.rows()) throw std::invalid_argument("gemm dimension mismatch");
  GemmProblem{l.bin.rows(), l.bin.cols(), b.cols()}.validate();
  check_threads(threads);
  if (l.residual.cols != b.rows()) throw std::invalid_argument("gemm dimension mismatch");
  DenseMatrix c(l.bin.rows(), b.cols());
  raise_on(bitmm_layer_forward_host(
      l.bin.rows(), l.bin.cols(), l.alpha, nullptr, l.bin.row_data(0),
      static_cast<std::int64_t>(l.bin.words_per_row()), l.residual.row_ptr.data(),
      l.residual.col_idx.data(), l.residual.vals.data(),
      static_cast<std::int64_t>(l.residual.nnz()), b.row_data(0), b.cols(), b.cols(),
      c.row_data(0), c.cols()));
  return c;
}

}  // namespace bitmm
