// Does a device->host copy into pinned memory leave the data in the host's last-level cache
// (Intel DDIO), so that reading it right after the copy is cheaper than reading cold memory?
// Decides whether the 16-bit output wire should widen from a small reused ring of staging
// parts (reads hit the LLC) instead of one staging buffer as large as the output.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -mavx2 ddio_probe.cu -o ddio_probe
#include <cuda_runtime.h>
#include <immintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static uint64_t read_sum(const uint8_t* p, size_t bytes) {
  __m256i acc = _mm256_setzero_si256();
  for (size_t i = 0; i < bytes; i += 32) acc = _mm256_add_epi64(acc, _mm256_load_si256(reinterpret_cast<const __m256i*>(p + i)));
  uint64_t o[4];
  _mm256_storeu_si256(reinterpret_cast<__m256i*>(o), acc);
  return o[0] + o[1] + o[2] + o[3];
}

int main() {
  const size_t part = 2u << 20, big = 512u << 20;
  uint8_t *dev, *ring, *cold;
  cudaMalloc(&dev, part);
  cudaMemset(dev, 1, part);
  cudaHostAlloc(&ring, 16 * part, cudaHostAllocDefault);
  cudaHostAlloc(&cold, big, cudaHostAllocDefault);
  memset(ring, 0, 16 * part);
  memset(cold, 0, big);
  std::vector<uint8_t> evict(big);
  uint64_t sink = 0;
  for (int rep = 0; rep < 3; ++rep) {
    // (a) copy then read at once, cycling through a 16-part ring
    double t_copy = 0, t_read = 0;
    for (int i = 0; i < 64; ++i) {
      uint8_t* slot = ring + (i % 16) * part;
      double t0 = now_us();
      cudaMemcpy(slot, dev, part, cudaMemcpyDeviceToHost);
      double t1 = now_us();
      sink += read_sum(slot, part);
      double t2 = now_us();
      t_copy += t1 - t0;
      t_read += t2 - t1;
    }
    // (b) read parts of a large buffer that was written long ago (evicted by a 512 MB sweep)
    memset(evict.data(), rep, big);
    double t_cold = 0;
    for (int i = 0; i < 64; ++i) {
      double t0 = now_us();
      sink += read_sum(cold + (size_t)i * part, part);
      t_cold += now_us() - t0;
    }
    // (c) copy into the large buffer's parts, read each right after its copy (what the wire does now)
    double t_read_big = 0;
    for (int i = 0; i < 64; ++i) {
      uint8_t* slot = cold + (size_t)((i * 37) % 256) * part;
      cudaMemcpy(slot, dev, part, cudaMemcpyDeviceToHost);
      double t1 = now_us();
      sink += read_sum(slot, part);
      t_read_big += now_us() - t1;
    }
    printf("2 MiB part: D2H %.1f us; read right after its copy %.1f us (%.1f GB/s); big-buffer part read after copy %.1f us; cold read %.1f us (%.1f GB/s)\n",
           t_copy / 64, t_read / 64, part / (t_read / 64) / 1e3, t_read_big / 64, t_cold / 64, part / (t_cold / 64) / 1e3);
  }
  printf("sink %llu\n", (unsigned long long)sink);
  return 0;
}
