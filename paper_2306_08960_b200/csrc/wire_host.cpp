// Host half of the 16-bit output wire (wire_host.h / wire.cuh): a fixed worker pool and the
// widening of wire words into int32 units and fp32 values, bit-identical to the GEMM
// epilogue (tc_gemm.cuh: s = scale * row_scale[r]; s = s * col_scale[c]; C = s * float(u)).
//
// Widening is bound by the host's memory system: 2 B read, 4 B (or 8 B) written per cell.
// Outputs are written with streaming stores, which skip the read-for-ownership of the
// destination lines; 64-byte AVX-512 stores where the CPU has them, else 16-byte SSE2 ones
// (profiles/micro/host_bw.c measures both on the GPU box's host).
#include "wire_host.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace bitmm_dev {

namespace {

class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }

  void run(int n, const std::function<void(int)>& f) {
    if (n <= 0) return;
    if (workers_.empty() || n == 1) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);  // one batch at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      n_ = n;
      next_.store(0);
      pending_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

  // A batch the workers start at once while the caller goes on (it joins the batch later).
  // The pool stays reserved for this caller until join.
  void start(int n, std::function<void(int)> f) {
    std::unique_lock<std::mutex> call(call_mu_);  // one batch at a time, held until join
    owned_ = std::move(f);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &owned_;
      n_ = n;
      next_.store(0);
      pending_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    call_lk_ = std::move(call);
  }
  void join() {
    drain();
    {
      std::unique_lock<std::mutex> lk(mu_);
      done_cv_.wait(lk, [&] { return pending_ == 0; });
      job_ = nullptr;
    }
    owned_ = nullptr;
    call_lk_.unlock();
  }

 private:
  HostPool() {
    int n = static_cast<int>(std::thread::hardware_concurrency());
    if (const char* e = std::getenv("BITMM_HOST_THREADS")) n = std::atoi(e);
    n = std::max(1, std::min(n, 32));
    for (int i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void drain() {
    for (int i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*job_)(i);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      drain();
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }

  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::unique_lock<std::mutex> call_lk_;  // start() .. join(): the batch's hold on call_mu_
  std::function<void(int)> owned_;        // start()'s job
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0};
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

template <Wire MODE>
inline int32_t decode(uint16_t v, int k) {
  if constexpr (MODE == Wire::Popc) return k - 2 * static_cast<int32_t>(v);
  else if constexpr (MODE == Wire::Half) return 2 * static_cast<int32_t>(static_cast<int16_t>(v));
  else return 4 * static_cast<int32_t>(v);
}

// One output row: pointers already offset to the block's first column.
struct Row {
  const uint16_t* src;
  int32_t* du;      // int32 units or null
  float* dc;        // fp32 values or null
  const float* cs;  // column scales or null
  float s_r;        // scale * row_scale[r] (or scale)
  int k;
  int64_t cols;
};

template <Wire MODE>
inline void cell(const Row& w, int64_t j) {
  const int32_t u = decode<MODE>(w.src[j], w.k);
  if (w.du) w.du[j] = u;
  if (w.dc) w.dc[j] = (w.cs ? w.s_r * w.cs[j] : w.s_r) * static_cast<float>(u);
}

template <int ALIGN>
inline bool misaligned(const Row& w, int64_t j) {
  return (w.du && (reinterpret_cast<uintptr_t>(w.du + j) & (ALIGN - 1))) ||
         (w.dc && (reinterpret_cast<uintptr_t>(w.dc + j) & (ALIGN - 1)));
}

#if defined(__x86_64__)
// Sixteen words -> sixteen int32 units, 64-byte streaming stores.
template <Wire MODE>
__attribute__((target("avx512f,avx512bw"))) int64_t row_avx512(const Row& w, int64_t j) {
  const __m512i kk = _mm512_set1_epi32(w.k);
  const __m512 sr = _mm512_set1_ps(w.s_r);
  for (; j + 16 <= w.cols; j += 16) {
    const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(w.src + j));
    __m512i u;
    if constexpr (MODE == Wire::Popc) u = _mm512_sub_epi32(kk, _mm512_slli_epi32(_mm512_cvtepu16_epi32(v), 1));
    else if constexpr (MODE == Wire::Half) u = _mm512_slli_epi32(_mm512_cvtepi16_epi32(v), 1);
    else u = _mm512_slli_epi32(_mm512_cvtepu16_epi32(v), 2);
    if (w.du) _mm512_stream_si512(reinterpret_cast<__m512i*>(w.du + j), u);
    if (w.dc) {
      const __m512 s = w.cs ? _mm512_mul_ps(sr, _mm512_loadu_ps(w.cs + j)) : sr;  // (s_r * cs) first
      _mm512_stream_ps(w.dc + j, _mm512_mul_ps(s, _mm512_cvtepi32_ps(u)));
    }
  }
  return j;
}

// Eight words -> eight int32 units, 16-byte streaming stores (x86-64 baseline).
template <Wire MODE>
int64_t row_sse2(const Row& w, int64_t j) {
  const __m128i kk = _mm_set1_epi32(w.k), z = _mm_setzero_si128();
  const __m128 sr = _mm_set1_ps(w.s_r);
  for (; j + 8 <= w.cols; j += 8) {
    const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(w.src + j));
    __m128i lo, hi;
    if constexpr (MODE == Wire::Half) {  // sign-extend: interleave with itself, arithmetic shift
      lo = _mm_slli_epi32(_mm_srai_epi32(_mm_unpacklo_epi16(v, v), 16), 1);
      hi = _mm_slli_epi32(_mm_srai_epi32(_mm_unpackhi_epi16(v, v), 16), 1);
    } else if constexpr (MODE == Wire::Popc) {
      lo = _mm_sub_epi32(kk, _mm_slli_epi32(_mm_unpacklo_epi16(v, z), 1));
      hi = _mm_sub_epi32(kk, _mm_slli_epi32(_mm_unpackhi_epi16(v, z), 1));
    } else {
      lo = _mm_slli_epi32(_mm_unpacklo_epi16(v, z), 2);
      hi = _mm_slli_epi32(_mm_unpackhi_epi16(v, z), 2);
    }
    if (w.du) {
      _mm_stream_si128(reinterpret_cast<__m128i*>(w.du + j), lo);
      _mm_stream_si128(reinterpret_cast<__m128i*>(w.du + j + 4), hi);
    }
    if (w.dc) {
      __m128 s0 = sr, s1 = sr;
      if (w.cs) {
        s0 = _mm_mul_ps(sr, _mm_loadu_ps(w.cs + j));
        s1 = _mm_mul_ps(sr, _mm_loadu_ps(w.cs + j + 4));
      }
      _mm_stream_ps(w.dc + j, _mm_mul_ps(s0, _mm_cvtepi32_ps(lo)));
      _mm_stream_ps(w.dc + j + 4, _mm_mul_ps(s1, _mm_cvtepi32_ps(hi)));
    }
  }
  return j;
}

bool has_avx512() {
  static const bool cpu = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
  }();
  const char* e = std::getenv("BITMM_HOST_SIMD");  // "sse2" forces the baseline path (tests)
  return cpu && !(e && std::string(e) == "sse2");
}
#endif

// One output row r from its 16-bit words (cols of them, the block's columns from col0 on).
template <Wire MODE>
void widen_row(const WireOut& o, const uint16_t* src, int64_t r, int64_t col0, int64_t cols) {
#if defined(__x86_64__)
  const bool wide = has_avx512();
#endif
  {
    Row w;
    w.src = src;
    w.du = o.c_units ? o.c_units + r * o.ldc + col0 : nullptr;
    w.dc = o.c ? o.c + r * o.ldc + col0 : nullptr;
    w.cs = o.col_scale ? o.col_scale + col0 : nullptr;
    w.s_r = o.row_scale ? o.scale * o.row_scale[r] : o.scale;
    w.k = o.k;
    w.cols = cols;
    int64_t j = 0;
#if defined(__x86_64__)
    // a scalar head up to the first column where every output is aligned for the stores
    // (both outputs may never align together; then the narrower stores or scalar code run)
    auto head = [&](auto align, int64_t max_head) {
      int64_t h = 0;
      while (h < max_head && h < cols && misaligned<decltype(align)::value>(w, h)) ++h;
      return misaligned<decltype(align)::value>(w, h) ? int64_t{-1} : h;
    };
    const int64_t h64 = wide ? head(std::integral_constant<int, 64>{}, 16) : -1;
    const int64_t h16 = h64 < 0 ? head(std::integral_constant<int, 16>{}, 4) : -1;
    if (h64 >= 0) {
      for (; j < h64; ++j) cell<MODE>(w, j);
      j = row_avx512<MODE>(w, j);
    } else if (h16 >= 0) {
      for (; j < h16; ++j) cell<MODE>(w, j);
      j = row_sse2<MODE>(w, j);
    }
#endif
    for (; j < cols; ++j) cell<MODE>(w, j);
  }
}

template <Wire MODE>
void expand_rows(const WireOut& o, const uint16_t* words, int64_t row0, int64_t col0, int64_t cols,
                 int64_t r0, int64_t r1) {
  for (int64_t r = r0; r < r1; ++r) widen_row<MODE>(o, words + (r - row0) * cols, r, col0, cols);
#if defined(__x86_64__)
  _mm_sfence();  // streaming stores ordered before the pool reports the task done
#endif
}

// 12-bit fields (two cells per 3 bytes, wire.cuh) + base, modulo 2^16 -> the 16-bit words.
void unpack12_scalar(const uint8_t* p, uint16_t base, uint16_t* out, int64_t j, int64_t n) {
  for (; j < n; ++j) {
    const uint8_t* b = p + 3 * (j >> 1);
    const uint32_t v = (j & 1) ? ((b[1] >> 4) | (static_cast<uint32_t>(b[2]) << 4))
                               : (b[0] | ((static_cast<uint32_t>(b[1]) & 0xFu) << 8));
    out[j] = static_cast<uint16_t>(v + base);
  }
}

#if defined(__x86_64__)
// Sixteen cells (24 bytes) per step: each 128-bit half takes 12 bytes, a byte shuffle puts the
// two bytes of every cell in its 16-bit lane, even lanes keep their low 12 bits, odd lanes
// shift right by 4. Reads 4 bytes past the last group (the staging parts are padded).
__attribute__((target("avx2"))) void unpack12_avx2(const uint8_t* p, uint16_t base, uint16_t* out, int64_t n) {
  const __m256i shuf = _mm256_setr_epi8(0, 1, 1, 2, 3, 4, 4, 5, 6, 7, 7, 8, 9, 10, 10, 11,
                                        0, 1, 1, 2, 3, 4, 4, 5, 6, 7, 7, 8, 9, 10, 10, 11);
  const __m256i mask = _mm256_set1_epi16(0x0FFF);
  const __m256i b = _mm256_set1_epi16(static_cast<short>(base));
  int64_t j = 0;
  for (; j + 16 <= n; j += 16) {
    const uint8_t* q = p + 3 * (j >> 1);
    const __m128i lo = _mm_loadu_si128(reinterpret_cast<const __m128i*>(q));
    const __m128i hi = _mm_loadu_si128(reinterpret_cast<const __m128i*>(q + 12));
    __m256i v = _mm256_shuffle_epi8(_mm256_set_m128i(hi, lo), shuf);
    v = _mm256_blend_epi16(_mm256_and_si256(v, mask), _mm256_srli_epi16(v, 4), 0xAA);
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(out + j), _mm256_add_epi16(v, b));
  }
  unpack12_scalar(p, base, out, j, n);
}

bool has_avx2() {
  static const bool cpu = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx2") != 0;
  }();
  const char* e = std::getenv("BITMM_HOST_SIMD");
  return cpu && !(e && std::string(e) == "sse2");
}
#endif

template <Wire MODE>
void expand_rows12(const WireOut& o, const uint8_t* payload, uint16_t base, int64_t prow0, int64_t col0,
                   int64_t cols, int64_t r0, int64_t r1) {
  // each row's 12-bit fields go through a small per-thread buffer of 16-bit words (L1/L2
  // resident), then the 16-bit widening: the output stores are what costs
  thread_local std::vector<uint16_t> tmp;
  if (static_cast<int64_t>(tmp.size()) < cols) tmp.resize(cols);
  for (int64_t r = r0; r < r1; ++r) {
    const uint8_t* p = payload + (r - prow0) * cols / 2 * 3;
#if defined(__x86_64__)
    if (has_avx2())
      unpack12_avx2(p, base, tmp.data(), cols);
    else
#endif
      unpack12_scalar(p, base, tmp.data(), 0, cols);
    widen_row<MODE>(o, tmp.data(), r, col0, cols);
  }
#if defined(__x86_64__)
  _mm_sfence();
#endif
}

#if defined(__x86_64__)
__attribute__((target("avx512f"))) void copy_nt_avx512(uint8_t* d, const uint8_t* s, size_t bytes) {
  size_t i = 0;
  for (; i + 256 <= bytes; i += 256) {
    const __m512i a = _mm512_loadu_si512(s + i), b = _mm512_loadu_si512(s + i + 64);
    const __m512i c = _mm512_loadu_si512(s + i + 128), e = _mm512_loadu_si512(s + i + 192);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), a);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 64), b);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 128), c);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 192), e);
  }
  for (; i + 64 <= bytes; i += 64)
    _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), _mm512_loadu_si512(s + i));
  if (i < bytes) std::memcpy(d + i, s + i, bytes - i);
}
#endif

}  // namespace

void copy_streaming(void* dst, const void* src, size_t bytes) {
  auto* d = static_cast<uint8_t*>(dst);
  const auto* s = static_cast<const uint8_t*>(src);
#if defined(__x86_64__)
  if (has_avx512() && bytes >= 4096) {
    const size_t head = (64 - (reinterpret_cast<uintptr_t>(d) & 63)) & 63;
    std::memcpy(d, s, head);
    copy_nt_avx512(d + head, s + head, bytes - head);
    _mm_sfence();
    return;
  }
#endif
  std::memcpy(d, s, bytes);
}

void host_pool_run(int n, const std::function<void(int)>& f) { HostPool::get().run(n, f); }
void host_pool_start(int n, std::function<void(int)> f) { HostPool::get().start(n, std::move(f)); }
void host_pool_join() { HostPool::get().join(); }
int host_pool_size() { return HostPool::get().size(); }

void wire_expand_range(const WireOut& o, const uint16_t* words, int64_t row0, int64_t col0,
                       int64_t cols, int64_t r0, int64_t r1) {
  switch (o.mode) {
    case Wire::Popc: expand_rows<Wire::Popc>(o, words, row0, col0, cols, r0, r1); break;
    case Wire::Half: expand_rows<Wire::Half>(o, words, row0, col0, cols, r0, r1); break;
    default: expand_rows<Wire::Quarter>(o, words, row0, col0, cols, r0, r1); break;
  }
}

void wire_expand_range12(const WireOut& o, const uint8_t* payload, uint16_t base, int64_t prow0, int64_t col0,
                         int64_t cols, int64_t r0, int64_t r1) {
  switch (o.mode) {
    case Wire::Popc: expand_rows12<Wire::Popc>(o, payload, base, prow0, col0, cols, r0, r1); break;
    case Wire::Half: expand_rows12<Wire::Half>(o, payload, base, prow0, col0, cols, r0, r1); break;
    default: expand_rows12<Wire::Quarter>(o, payload, base, prow0, col0, cols, r0, r1); break;
  }
}

}  // namespace bitmm_dev
