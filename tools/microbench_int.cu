// microbench_int.cu -- measured INT32 issue roof on this B200 ("measure it with an
// IMAD/LOP3-chain microbenchmark and record it beside the HBM peak").
// Three loops, 8 independent dependency chains per thread, 8 warps per SMSP:
//   lop3   : LOP3 only           -> the ALU pipe alone
//   imad   : IMAD only           -> the FMA pipe alone
//   mixed  : LOP3 and IMAD interleaved 1:1 -> both pipes, bounded by issue (1 warp-instr/clk/SMSP)
// Prints one JSON line: thread-ops/s per loop and the SM clock read around it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbint tools/microbench_int.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <int MODE>
__global__ void __launch_bounds__(1024) int_kernel(uint32_t* out, uint32_t seed) {
  uint32_t a[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) a[c] = seed * (threadIdx.x + 7u * c) + blockIdx.x;
  const uint32_t k1 = seed | 1u, k2 = seed ^ 0x9e3779b9u;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if (MODE == 0 || MODE == 2)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(k1), "r"(k2));
      if (MODE == 1 || MODE == 2)
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(k1), "r"(k2));
      if (MODE == 3) {   // immediate forms: fewer register-file reads per instruction
        asm volatile("xor.b32 %0, %0, 0x5bd1e995;" : "+r"(a[c]));
        asm volatile("mad.lo.u32 %0, %0, 0x27d4eb2d, 0x165667b1;" : "+r"(a[c]));
      }
      if (MODE == 4) {   // two-operand ALU + immediate IMAD
        asm volatile("add.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(k1));
        asm volatile("mad.lo.u32 %0, %0, 0x27d4eb2d, 0x165667b1;" : "+r"(a[c]));
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) r ^= a[c];
  if (r == 0x12345678u) out[0] = r;
}

template <int MODE>
static double run(int sms, uint32_t* out) {
  const int threads = 1024, blocks = sms * 2;   // 64 warps per SM = 16 per SMSP
  int_kernel<MODE><<<blocks, threads>>>(out, 3u);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 400;
  for (int r = 0; r < reps; ++r) int_kernel<MODE><<<blocks, threads>>>(out, 3u + r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = (double)reps * blocks * threads * kIters * kChains * (MODE >= 2 ? 2 : 1);
  return ops / (ms * 1e-3);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  uint32_t* out;
  cudaMalloc(&out, 4);
  const double lop3 = run<0>(p.multiProcessorCount, out);
  const double imad = run<1>(p.multiProcessorCount, out);
  const double mixed = run<2>(p.multiProcessorCount, out);
  const double mixed_imm = run<3>(p.multiProcessorCount, out);
  const double mixed_2op = run<4>(p.multiProcessorCount, out);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"lop3_tops\": %.3f, \"imad_tops\": %.3f, \"mixed_tops\": %.3f, "
         "\"mixed_imm_tops\": %.3f, \"mixed_2op_tops\": %.3f, \"max_clock_mhz\": %.0f, "
         "\"lanes_per_clk_per_sm\": {\"lop3\": %.1f, \"imad\": %.1f, \"mixed\": %.1f, \"mixed_imm\": %.1f, "
         "\"mixed_2op\": %.1f}}\n",
         p.multiProcessorCount, lop3 * 1e-12, imad * 1e-12, mixed * 1e-12, mixed_imm * 1e-12, mixed_2op * 1e-12,
         clk * 1e-3, lop3 / (p.multiProcessorCount * clk * 1e3), imad / (p.multiProcessorCount * clk * 1e3),
         mixed / (p.multiProcessorCount * clk * 1e3), mixed_imm / (p.multiProcessorCount * clk * 1e3),
         mixed_2op / (p.multiProcessorCount * clk * 1e3));
  return cudaGetLastError() != cudaSuccess;
}
