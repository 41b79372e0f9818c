// 16-bit output wire of the host-flavour entry points (bitmm_gemm_*_host).
//
// A host call's time is the PCIe copy of its output: 4 B per cell, int32 units or fp32
// scaled values (kernels.cpp:171 returns a float DenseMatrix). The integer units of all
// three routines have a small, data-independent range, so the device narrows them to one
// 16-bit word per cell and the host widens them again, applying the same fp32 scale
// sequence as the GEMM epilogue (tc_gemm.cuh: s = scale * row_scale[r]; s = s * col_scale[c];
// C = s * float(units)). The bytes that cross PCIe halve; the host result is bit-identical
// to the device output.
//
//   1/1: units = K - 2x with x = popc(a ^ b) in [0, K]         -> x as uint16   (K <= 65535)
//   1/2: units = 2 * sum s*p in [-6K, 6K], always even        -> units/2 int16 (K <= 10922)
//   2/2: units = 4 * sum p_w*p_a in [0, 36K], multiple of 4   -> units/4 uint16 (K <= 7281)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "wire_host.h"

namespace bitmm_dev {

// src: rows x cols int32 units (leading dimension ld); dst: rows x cols words, packed.
// Four cells per thread when the rows allow 16-byte loads, else one.
__global__ void __launch_bounds__(256) narrow_units_kernel(const int32_t* __restrict__ src,
                                                           int64_t ld, uint16_t* __restrict__ dst,
                                                           int64_t rows, int64_t cols, int mode,
                                                           int k) {
  auto enc = [&](int32_t u) -> uint16_t {
    if (mode == static_cast<int>(Wire::Popc)) return static_cast<uint16_t>((k - u) >> 1);
    if (mode == static_cast<int>(Wire::Half)) return static_cast<uint16_t>(static_cast<int16_t>(u >> 1));
    return static_cast<uint16_t>(u >> 2);
  };
  const bool vec = (cols & 3) == 0 && (ld & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  if (vec) {
    const int64_t q = cols >> 2, total = rows * q;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
      const int64_t r = i / q, c = (i - r * q) << 2;
      const int4 u = __ldcs(reinterpret_cast<const int4*>(src + r * ld + c));
      ushort4 o;
      o.x = enc(u.x);
      o.y = enc(u.y);
      o.z = enc(u.z);
      o.w = enc(u.w);
      *reinterpret_cast<ushort4*>(dst + r * cols + c) = o;
    }
  } else {
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total; i += stride) {
      const int64_t r = i / cols, c = i - r * cols;
      dst[i] = enc(src[r * ld + c]);
    }
  }
}

// ---- 12-bit packing of the wire words (round 2) ----
// Within one copied part the 16-bit words of all three routines span far less than 4096 values
// for random data (1/1: popcounts around K/2, sigma = sqrt(K)/2; 1/2: sigma = sqrt(3.5 K);
// 2/2: sigma ~ 2.7 sqrt(K)). A part then crosses PCIe as a 16-byte header {min, max} of its
// words followed by (word - min) in 12 bits, two cells per 3 bytes: 3/4 of the 16-bit bytes.
// The host reads the header; a part whose max - min exceeds 4095 is fetched again as 16-bit
// words (they stay on the device until the call ends), so the output is exact for any data.
// Words are compared as the routine's integers (int16 for 1/2, uint16 otherwise); the host adds
// min back modulo 2^16, which restores the word bit for bit.
struct Wire12Part {
  const uint16_t* src;  // the part's 16-bit words (cells of them)
  uint8_t* dst;         // header (16 bytes) then the packed payload
  int64_t cells;        // a multiple of 16
};
constexpr int kWire12MaxParts = 8;  // the parts of one slice (run_wire_items: kWireMaxParts)
struct Wire12Set {
  Wire12Part p[kWire12MaxParts];
  int count;
};

// Headers of a slice's parts: {min, max} slots before the atomics of wire12_minmax_kernel.
__global__ void wire12_init_kernel(const __grid_constant__ Wire12Set S) {
  if (threadIdx.x < S.count) {
    int* h = reinterpret_cast<int*>(S.p[threadIdx.x].dst);
    h[0] = 0x7FFFFFFF;
    h[1] = -0x7FFFFFFF - 1;
  }
}

__device__ __forceinline__ int wire12_value(uint16_t w, int mode) {
  return mode == static_cast<int>(Wire::Half) ? static_cast<int>(static_cast<int16_t>(w)) : static_cast<int>(w);
}

// Pass 1: min and max of every part (blockIdx.y) into its header (atomics on the slots
// wire12_init_kernel preset).
__global__ void __launch_bounds__(256) wire12_minmax_kernel(const __grid_constant__ Wire12Set S, int mode) {
  const Wire12Part& q = S.p[blockIdx.y];
  int lo = 0x7FFFFFFF, hi = -0x7FFFFFFF - 1;
  const int64_t n8 = q.cells >> 3;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(q.src) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int a = wire12_value(static_cast<uint16_t>(w[e] & 0xFFFFu), mode);
      const int b = wire12_value(static_cast<uint16_t>(w[e] >> 16), mode);
      lo = min(lo, min(a, b));
      hi = max(hi, max(a, b));
    }
  }
  for (int off = 16; off > 0; off >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, off));
    hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(reinterpret_cast<int*>(q.dst), lo);
    atomicMax(reinterpret_cast<int*>(q.dst) + 1, hi);
  }
}

// Pass 2: eight cells per thread, (word - min) as 12-bit fields, two cells per 3 bytes (cell 2i
// in the low 12 bits of bytes 3i, 3i+1; cell 2i+1 in the high 12 bits of bytes 3i+1, 3i+2).
// Parts whose range does not fit 12 bits are left unpacked (the host fetches their words).
__global__ void __launch_bounds__(256) wire12_pack_kernel(const __grid_constant__ Wire12Set S, int mode) {
  const Wire12Part& q = S.p[blockIdx.y];
  const int lo = reinterpret_cast<const int*>(q.dst)[0], hi = reinterpret_cast<const int*>(q.dst)[1];
  if (hi - lo > 4095) return;
  const int64_t n8 = q.cells >> 3;
  uint32_t* out = reinterpret_cast<uint32_t*>(q.dst + 16);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(q.src) + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t c[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      c[2 * e] = static_cast<uint32_t>(wire12_value(static_cast<uint16_t>(w[e] & 0xFFFFu), mode) - lo);
      c[2 * e + 1] = static_cast<uint32_t>(wire12_value(static_cast<uint16_t>(w[e] >> 16), mode) - lo);
    }
    // 8 cells -> 96 bits -> three words (little-endian byte stream)
    out[3 * i] = c[0] | (c[1] << 12) | (c[2] << 24);
    out[3 * i + 1] = (c[2] >> 8) | (c[3] << 4) | (c[4] << 16) | (c[5] << 28);
    out[3 * i + 2] = (c[5] >> 4) | (c[6] << 8) | (c[7] << 20);
  }
}

}  // namespace bitmm_dev
