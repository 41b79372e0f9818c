// Cost of one residual product in the fused 2-bit APB epilogue: s_j += fl(v * d_p(j)) for the 32
// tokens j of a lane, p(j) = 2 hi_j + lo_j from two 32-bit code masks. Variants of the
// selection, timed as SMSP cycles per warp-entry (32 tokens per lane) (warps per SMSP as given).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sel_rate sel_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int V>
__global__ void k(const uint2* __restrict__ codes, const float* __restrict__ vals, float* out, int entries) {
  float s[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) s[j] = 0.f;
  const float d1 = 0.37f, d2 = 0.74f, d3 = 1.11f;
  for (int e = 0; e < entries; ++e) {
    const uint2 w = codes[(e * 37 + threadIdx.x) & 1023];
    const float v = vals[(e + threadIdx.x) & 1023];
    const float p0 = __fmul_rn(v, 0.f), p1 = __fmul_rn(v, d1), p2 = __fmul_rn(v, d2), p3 = __fmul_rn(v, d3);
    if (V == 0) {  // ternary select: 2 LOP3.P + 2 FSEL + FADD
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool lo = (w.x >> j) & 1u, hi = (w.y >> j) & 1u;
        s[j] = __fadd_rn(s[j], hi ? (lo ? p3 : p2) : (lo ? p1 : p0));
      }
    } else if (V == 1) {  // integer sign masks from shifted words, LOP3 muxes
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const unsigned ml = static_cast<unsigned>(static_cast<int>(w.x << (31 - j)) >> 31);
        const unsigned mh = static_cast<unsigned>(static_cast<int>(w.y << (31 - j)) >> 31);
        const unsigned a = (__float_as_uint(p1) & ml) | (__float_as_uint(p0) & ~ml);
        const unsigned b = (__float_as_uint(p3) & ml) | (__float_as_uint(p2) & ~ml);
        s[j] = __fadd_rn(s[j], __uint_as_float((b & mh) | (a & ~mh)));
      }
    } else if (V == 2) {  // lo as an integer through IMAD (fma pipe), FSEL on hi
      const unsigned D10 = __float_as_uint(p1) - __float_as_uint(p0);
      const unsigned D32 = __float_as_uint(p3) - __float_as_uint(p2);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const unsigned l = (w.x >> j) & 1u;
        const unsigned a = l * D10 + __float_as_uint(p0), b = l * D32 + __float_as_uint(p2);
        const bool hi = (w.y >> j) & 1u;
        s[j] = __fadd_rn(s[j], __uint_as_float(hi ? b : a));
      }
    } else if (V == 8) {  // three float selects, hi last
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool lo = (w.x >> j) & 1u, hi = (w.y >> j) & 1u;
        const float a = lo ? p1 : p0, b = lo ? p3 : p2;
        s[j] = __fadd_rn(s[j], hi ? b : a);
      }
    } else if (V == 9) {  // integer selects on the bit patterns
      const unsigned u0 = __float_as_uint(p0), u1 = __float_as_uint(p1), u2 = __float_as_uint(p2),
                     u3 = __float_as_uint(p3);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const bool lo = (w.x >> j) & 1u, hi = (w.y >> j) & 1u;
        unsigned q = lo ? u1 : u0;
        if (hi) q = lo ? u3 : u2;
        s[j] = __fadd_rn(s[j], __uint_as_float(q));
      }
    } else if (V == 10) {  // predicated moves: q = p0, then overwrite for levels 1, 2, 3
      const unsigned b3 = w.x & w.y;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float q = p0;
        if ((w.x >> j) & 1u) q = p1;
        if ((w.y >> j) & 1u) q = p2;
        if ((b3 >> j) & 1u) q = p3;
        s[j] = __fadd_rn(s[j], q);
      }
    } else if (V >= 4) {  // mixed: every (V-2)-th token as V0 (ALU selects), the rest as V2 (IMAD)
      const unsigned D10 = __float_as_uint(p1) - __float_as_uint(p0);
      const unsigned D32 = __float_as_uint(p3) - __float_as_uint(p2);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j % (V > 2 ? V - 2 : 1) == 0) {
          const bool lo = (w.x >> j) & 1u, hi = (w.y >> j) & 1u;
          s[j] = __fadd_rn(s[j], hi ? (lo ? p3 : p2) : (lo ? p1 : p0));
        } else {
          const unsigned l = (w.x >> j) & 1u;
          const unsigned a = l * D10 + __float_as_uint(p0), b = l * D32 + __float_as_uint(p2);
          const bool hi = (w.y >> j) & 1u;
          s[j] = __fadd_rn(s[j], __uint_as_float(hi ? b : a));
        }
      }
    } else if (V == 3) {  // packed pair adds after the scalar selects
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const bool lo0 = (w.x >> j) & 1u, hi0 = (w.y >> j) & 1u;
        const bool lo1 = (w.x >> (j + 1)) & 1u, hi1 = (w.y >> (j + 1)) & 1u;
        const float q0 = hi0 ? (lo0 ? p3 : p2) : (lo0 ? p1 : p0);
        const float q1 = hi1 ? (lo1 ? p3 : p2) : (lo1 ? p1 : p0);
        unsigned long long acc = (unsigned long long)__float_as_uint(s[j]) |
                                 ((unsigned long long)__float_as_uint(s[j + 1]) << 32);
        const unsigned long long q = (unsigned long long)__float_as_uint(q0) |
                                     ((unsigned long long)__float_as_uint(q1) << 32);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(q));
        s[j] = __uint_as_float(static_cast<unsigned>(acc));
        s[j + 1] = __uint_as_float(static_cast<unsigned>(acc >> 32));
      }
    }
  }
  float t = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) t += s[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  uint2* codes;
  float *vals, *out;
  cudaMalloc(&codes, 1024 * 8);
  cudaMalloc(&vals, 1024 * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMemset(codes, 0x5A, 1024 * 8);
  cudaMemset(vals, 0x3F, 1024 * 4);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int entries = 2048;
  const char* names[] = {"ternary FSEL", "sign-mask LOP3", "IMAD lo + FSEL hi", "FSEL + FADD2",
                         "mix 1/2 ternary", "mix 1/3 ternary", "mix 1/4 ternary", "mix 1/5 ternary",
                         "3 float selects", "int selects", "predicated moves"};
  for (int wps : {2, 4, 8}) {
    for (int v = 0; v < 11; ++v) {
      if (v == 1 || v == 3 || (v >= 4 && v <= 7)) continue;
      const int threads = wps * 4 * 32;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float ms = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (v == 0) k<0><<<148, threads>>>(codes, vals, out, entries);
        if (v == 1) k<1><<<148, threads>>>(codes, vals, out, entries);
        if (v == 2) k<2><<<148, threads>>>(codes, vals, out, entries);
        if (v == 3) k<3><<<148, threads>>>(codes, vals, out, entries);
        if (v == 4) k<4><<<148, threads>>>(codes, vals, out, entries);
        if (v == 5) k<5><<<148, threads>>>(codes, vals, out, entries);
        if (v == 6) k<6><<<148, threads>>>(codes, vals, out, entries);
        if (v == 7) k<7><<<148, threads>>>(codes, vals, out, entries);
        if (v == 8) k<8><<<148, threads>>>(codes, vals, out, entries);
        if (v == 9) k<9><<<148, threads>>>(codes, vals, out, entries);
        if (v == 10) k<10><<<148, threads>>>(codes, vals, out, entries);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double cycles = ms * 1e-3 * clk * 1e3;
      printf("warps/SMSP %d  %-18s %.2f cycles per warp-entry (32 tokens x 32 lanes) per SMSP\n", wps, names[v],
             cycles / (static_cast<double>(wps) * entries));
    }
  }
  return cudaGetLastError() != cudaSuccess;
}
