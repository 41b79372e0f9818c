// Host half of the 16-bit output wire (wire.cuh has the format and the device half):
// the worker pool and the widening of wire words into the caller's int32 / fp32 outputs.
// Implemented in wire_host.cpp (plain C++, compiled by the host compiler).
#pragma once

#include <stddef.h>
#include <stdint.h>

#include <functional>

namespace bitmm_dev {

enum class Wire : int { None = 0, Popc = 1, Half = 2, Quarter = 3 };

// The wire word for a routine's units at this K, or Wire::None when they do not fit.
inline Wire wire_for(int routine, int64_t k) {
  switch (routine) {
    case 0: return k <= 65535 ? Wire::Popc : Wire::None;
    case 1: return k <= 10922 ? Wire::Half : Wire::None;
    case 2: return k <= 7281 ? Wire::Quarter : Wire::None;
    default: return Wire::None;
  }
}

// Where one routine's widened output goes: int32 units and/or fp32 values, row-major with
// leading dimension ldc, plus the epilogue's scale terms (host copies).
struct WireOut {
  Wire mode;
  int k;
  float scale;
  const float* row_scale;  // [rows of the output] or null
  const float* col_scale;  // [columns of the output] or null
  int32_t* c_units;
  float* c;
  int64_t ldc;
};

// Calls f(0..n-1) across the host pool (BITMM_HOST_THREADS threads, else the hardware
// concurrency capped at 32; the caller is one of them) and returns when all are done.
void host_pool_run(int n, const std::function<void(int)>& f);
int host_pool_size();
// The same batch, started on the workers while the caller keeps going (e.g. enqueueing the
// device work whose results the tasks wait for); host_pool_join() then takes tasks too and
// returns when all are done. One batch at a time per process (start blocks until the pool is free).
void host_pool_start(int n, std::function<void(int)> f);
void host_pool_join();

// memcpy with 64-byte streaming stores where the CPU has AVX-512 (no read-for-ownership of the
// destination lines), else memcpy.
void copy_streaming(void* dst, const void* src, size_t bytes);

// Widens rows [r0, r1) of the output block at (row0, col0) with `cols` columns whose words
// are packed row-major at `words` (row r at words + (r - row0) * cols) into o's buffers.
void wire_expand_range(const WireOut& o, const uint16_t* words, int64_t row0, int64_t col0,
                       int64_t cols, int64_t r0, int64_t r1);
// The same from a part packed in 12 bits (wire.cuh, wire12_pack_kernel): `payload` holds rows
// prow0.. of the block as (word - base) fields, two cells per 3 bytes, cols a multiple of 16.
void wire_expand_range12(const WireOut& o, const uint8_t* payload, uint16_t base, int64_t prow0, int64_t col0,
                         int64_t cols, int64_t r0, int64_t r1);

}  // namespace bitmm_dev
