// Issue rate of the fp32 pair instructions (FADD2 / FMUL2) against FADD / FMUL / LOP3 / PRMT on
// sm_100a: each thread runs 8 independent chains of 4096 dependent ops; 4 warps per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f32x2_rate f32x2_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(unsigned long long* out, int iters, unsigned seed) {
  unsigned long long a[8];
  for (int i = 0; i < 8; ++i) a[i] = (0x3F8000013F800001ull + i + threadIdx.x) ^ seed;
  const unsigned long long b = 0x3F8000003F800000ull ^ (seed & 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(b));
      if (OP == 1) asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(b));
      if (OP == 2) {  // two scalar FADDs on the halves
        float x = __uint_as_float((unsigned)a[i]), y = __uint_as_float((unsigned)(a[i] >> 32));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x) : "f"(__uint_as_float((unsigned)b)));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(y) : "f"(__uint_as_float((unsigned)b)));
        a[i] = (unsigned long long)__float_as_uint(x) | ((unsigned long long)__float_as_uint(y) << 32);
      }
      if (OP == 3) {  // PRMT + LOP3 (bf16 pair -> two fp32)
        unsigned lo = (unsigned)a[i], hi = (unsigned)(a[i] >> 32);
        asm volatile("prmt.b32 %0, %0, 0, 0x1054;" : "+r"(lo));
        asm volatile("and.b32 %0, %0, 0xFFFF0000;" : "+r"(hi));
        a[i] = (unsigned long long)lo | ((unsigned long long)hi << 32);
      }
    }
  }
  unsigned long long s = 0;
  for (int i = 0; i < 8; ++i) s ^= a[i];
  if (s == 0x1234) out[0] = s;
}

int main() {
  unsigned long long* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096, threads = 512;
  const char* names[] = {"FADD2 (64-bit)", "FMUL2 (64-bit)", "2x FADD (32-bit)", "PRMT+AND"};
  for (int op = 0; op < 4; ++op) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) k<0><<<sms, threads>>>(out, iters, 0);
      if (op == 1) k<1><<<sms, threads>>>(out, iters, 0);
      if (op == 2) k<2><<<sms, threads>>>(out, iters, 0);
      if (op == 3) k<3><<<sms, threads>>>(out, iters, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    // instructions per SMSP: warps per SMSP * iters * 8 (op 2, 3: two instructions each)
    const double warp_instr = (threads / 32 / 4.0) * iters * 8 * (op >= 2 ? 2 : 1);
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-18s %.3f ms  %.2f cycles per warp instruction per SMSP (at %d MHz max)\n", names[op], ms,
           cycles / warp_instr, clk / 1000);
  }
  return 0;
}
