// microbench_atomics.cu -- global atomicAdd throughput on B200 (counters per (digit, 128K-entry chunk),
// random digits): the case for building radix histograms with per-record global atomics.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbatom tools/microbench_atomics.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(uint32_t* cnt, uint32_t ncnt, uint64_t n, uint32_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)(i * 2654435761u) ^ seed;
    h ^= h >> 15; h *= 0x2c1b3c6dU; h ^= h >> 12;
    // chunk-local: consecutive i share a chunk of 131072, digit random in 256
    const uint32_t c = (uint32_t)(i >> 17);
    const uint32_t d = h & 255;
    atomicAdd(&cnt[(uint64_t)d * ncnt + c], 1u);
  }
}
int main() {
  const uint64_t n = 558000000ull;
  const uint32_t ncnt = (uint32_t)(n >> 17) + 1;
  uint32_t* cnt;
  cudaMalloc(&cnt, sizeof(uint32_t) * 256 * ncnt);
  cudaMemset(cnt, 0, sizeof(uint32_t) * 256 * ncnt);
  k<<<148 * 8, 256>>>(cnt, ncnt, n, 1);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<148 * 8, 256>>>(cnt, ncnt, n, r);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%.3f ms per %llu atomics = %.1f G/s\n", ms / 5, (unsigned long long)n, n / (ms / 5 * 1e-3) / 1e9);
  return 0;
}
