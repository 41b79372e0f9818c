// STS.128 throughput of the fx_gemm expander store pattern (profiles/micro/README.md).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sts_rate sts_rate.cu && ./sts_rate
// Per variant: cycles per warp-level STS.128 with W warps of one CTA storing into a 28 KB
// stage, pattern 0 = fx_gemm (8 lanes per 128-byte row, chunk j at j ^ (r & 7)),
// 1 = linear (lane t writes bytes 16t..16t+15 of a 512-byte run), 2 = fx pattern + fence.
#include <cstdio>
#include <cstdint>

__global__ void sts_kernel(int pattern, int warps, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= warps) return;
  const int tid = threadIdx.x;
  const int r0 = tid >> 3, j = tid & 7;
  const int T = warps * 32, step = T / 8;
  uint4 v = make_uint4(tid, tid * 3, tid * 5, tid * 7);
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint8_t* st = smem + (it & 3) * 28672;
    if (pattern == 1) {
#pragma unroll
      for (int i = 0; i < 7; ++i) *reinterpret_cast<uint4*>(st + (i * T + tid) * 16) = v;
    } else {
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        const int r = r0 + i * step;
        *reinterpret_cast<uint4*>(st + r * 128 + ((j ^ (r & 7)) << 4)) = v;
      }
      if (pattern == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    v.x += 1;
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) out[warp] = t1 - t0;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(sts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 28672);
  const int iters = 4096;
  for (int pattern = 0; pattern < 3; ++pattern)
    for (int warps : {1, 4, 8}) {
      sts_kernel<<<1, 512, 4 * 28672>>>(pattern, warps, iters, d);
      unsigned long long h[16];
      cudaMemcpy(h, d, warps * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
      // warp-level STS.128 per iteration per warp: 7 (the fx expander's per-stage count at 8 warps)
      printf("pattern %d warps %d: %.2f cycles per warp STS.128 (CTA-wide %.1f B/clk)\n", pattern, warps,
             double(mx) / (iters * 7.0), warps * 7.0 * 512 * iters / double(mx));
    }
  return 0;
}
