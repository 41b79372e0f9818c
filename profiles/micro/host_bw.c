// Host memory bandwidth probe for the 16-bit output wire (csrc/wire.cuh): how fast can the
// host CPUs widen uint16 words into int32 / fp32 outputs, with plain and streaming stores?
// gcc -O3 -march=native -fopenmp host_bw.c -o host_bw && ./host_bw
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static double now(void) { return omp_get_wtime(); }

int main(void) {
  const size_t n = (size_t)64 << 20;  // 64 Mi cells: 128 MiB in, 256 MiB out
  uint16_t* src = aligned_alloc(64, n * 2);
  int32_t* dst = aligned_alloc(64, n * 4);
  for (size_t i = 0; i < n; ++i) src[i] = (uint16_t)(i * 2654435761u);
  memset(dst, 0, n * 4);
  int nt = omp_get_max_threads();
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) dst[i] = 4096 - 2 * (int32_t)src[i];
    double t1 = now();
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; i += 16) {
      __m256i v = _mm256_loadu_si256((const __m256i*)(src + i));
      __m512i w = _mm512_cvtepu16_epi32(v);
      w = _mm512_sub_epi32(_mm512_set1_epi32(4096), _mm512_slli_epi32(w, 1));
      _mm512_stream_si512((__m512i*)(dst + i), w);
    }
    _mm_sfence();
    double t2 = now();
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; i += 16) _mm512_stream_si512((__m512i*)(dst + i), _mm512_set1_epi32(rep));
    _mm_sfence();
    double t3 = now();
    printf("threads %d: plain widen %.1f GB/s out, stream widen %.1f GB/s out, stream fill %.1f GB/s\n", nt,
           n * 4 / (t1 - t0) / 1e9, n * 4 / (t2 - t1) / 1e9, n * 4 / (t3 - t2) / 1e9);
  }
  return 0;
}
