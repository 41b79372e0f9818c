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

}  // namespace bitmm_dev
