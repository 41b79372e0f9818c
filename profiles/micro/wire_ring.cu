// The 16-bit output wire's host side, isolated: D2H copies of 2 MiB wire parts into pinned
// staging (one copy stream, an event per part) while T host threads widen each landed part into
// a 4 MiB int32 slice of a 256 MiB output with streaming stores. Staging is either one buffer
// as large as the wire (what run_pipelined_wire does) or a ring of R parts reused in order (a
// part's copy is issued only after the widening of the part R earlier finished), so that the
// staged lines may stay in the last-level cache (DDIO) instead of being written back to DRAM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -mavx2,-pthread wire_ring.cu -o wire_ring
#include <cuda_runtime.h>
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

static std::atomic<int> g_task_done[64];  // tasks finished per part
static std::atomic<int> g_issued[64];     // the part's copy and event are enqueued

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void widen(const uint16_t* src, int32_t* dst, size_t n) {
  const __m256i k = _mm256_set1_epi32(4096);
  for (size_t i = 0; i < n; i += 8) {
    __m256i v = _mm256_cvtepu16_epi32(_mm_load_si128(reinterpret_cast<const __m128i*>(src + i)));
    v = _mm256_sub_epi32(k, _mm256_slli_epi32(v, 1));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), v);
  }
}

int main(int argc, char** argv) {
  const int threads = argc > 1 ? atoi(argv[1]) : 15;
  const size_t part = 2u << 20, nparts = 64;            // 128 MiB of wire words per step
  const size_t words = part / 2;
  uint16_t* dev;
  cudaMalloc(&dev, nparts * part);
  cudaMemset(dev, 1, nparts * part);
  uint8_t* stage;
  cudaHostAlloc(&stage, nparts * part, cudaHostAllocDefault);
  memset(stage, 0, nparts * part);
  std::vector<int32_t> out_v(nparts * words + 16);
  int32_t* out = reinterpret_cast<int32_t*>((reinterpret_cast<uintptr_t>(out_v.data()) + 63) & ~uintptr_t(63));
  memset(out, 0, nparts * words * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  std::vector<cudaEvent_t> ev(nparts);
  for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  for (int ring : {64, 16, 8, 4, 2}) {
    double best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      std::atomic<int> next{0};
      std::vector<std::atomic<int>> done(nparts);
      for (auto& d : done) d.store(0);
      const double t0 = now_ms();
      std::thread issuer([&] {
        for (size_t p = 0; p < nparts; ++p) {
          if ((int)p >= ring)
            while (!done[p - ring].load(std::memory_order_acquire)) _mm_pause();
          cudaMemcpyAsync(stage + (p % ring) * part, reinterpret_cast<uint8_t*>(dev) + p * part, part,
                          cudaMemcpyDeviceToHost, st);
          cudaEventRecord(ev[p], st);
          g_issued[p].store(1, std::memory_order_release);
        }
      });
      std::vector<std::thread> ws;
      for (int t = 0; t < threads; ++t)
        ws.emplace_back([&] {
          // a part in 4 tasks of 512 KiB
          for (int i = next.fetch_add(1); i < (int)nparts * 4; i = next.fetch_add(1)) {
            const int p = i / 4, q = i % 4;
            while (!g_issued[p].load(std::memory_order_acquire)) _mm_pause();
            while (cudaEventQuery(ev[p]) != cudaSuccess) _mm_pause();
            const size_t n = words / 4;
            widen(reinterpret_cast<const uint16_t*>(stage + (p % ring) * part) + q * n, out + p * words + q * n, n);
            // count tasks
            _mm_sfence();
            if (g_task_done[p].fetch_add(1) == 3) done[p].store(1, std::memory_order_release);
          }
        });
      issuer.join();
      for (auto& w : ws) w.join();
      const double ms = now_ms() - t0;
      for (auto& c : g_task_done) c.store(0);
      for (auto& c : g_issued) c.store(0);
      if (ms < best) best = ms;
    }
    printf("ring %2d parts (%3d MiB staging), %d threads: %.2f ms per 128 MiB wire -> 256 MiB int32 (%.1f GB/s of output)\n",
           ring, ring * 2, threads, best, 256.0 * 1.048576 / best);
  }
  return 0;
}
