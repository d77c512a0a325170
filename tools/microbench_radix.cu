// microbench_radix.cu -- design probes for the seed-table scatter (K7), run on B200:
//   1. L2 write combining: every CTA writes `run` contiguous u64 per digit (the scatter of one
//      LSD pass with 4096/run digits), runs start at unaligned offsets so neighbouring CTAs
//      share 32 B sectors.  ncu's dram__bytes_write.sum vs the 8 B/item algorithmic bytes says
//      whether L2 merges partial sectors written by different CTAs.
//   2. warp multi-split cost: MATCH.ANY vs an nbits-ballot multi-split, items/clk per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mb tools/microbench_radix.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void scatter_runs(uint64_t* out, uint64_t ntiles, int run, int skew) {
  const uint64_t c = blockIdx.x;
  const int T = 4096, D = T / run;
  const uint64_t region = ntiles * run + 8;  // per-digit region (+8: room for the skew)
  for (int q = threadIdx.x; q < T; q += blockDim.x) {
    const int d = q / run, r = q % run;
    const uint64_t idx = (uint64_t)d * region + (skew ? (d % 7) : 0) + c * run + r;
    out[idx] = idx ^ c;
  }
  (void)D;
}

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

template <int MODE, int NBITS>
__global__ void multisplit(uint32_t* sink, int iters) {
  const unsigned lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
  uint32_t acc = 0, s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    const uint32_t d = mix(s + i * 0x9E3779B9u) & ((1u << NBITS) - 1u);
    unsigned peers;
    if (MODE == 0) {
      peers = __match_any_sync(0xffffffffu, d);
    } else if (MODE == 1) {
      peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < NBITS; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
      }
    } else {
      peers = 1u;  // hash only: the cost floor of the loop
    }
    acc += __popc(peers & lt) + (peers >> 31);
  }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  // ---- 1. write combining
  const uint64_t ntiles = 65536;  // 2^28 items, 2 GiB
  uint64_t* out;
  cudaMalloc(&out, (ntiles * 4096 + 4096 * 8 + 64) * sizeof(uint64_t) + (1u << 20));
  const int runs[] = {1, 2, 4, 8, 16, 32, 4096};
  for (int skew = 0; skew < 2; ++skew)
    for (int run : runs) {
      for (int rep = 0; rep < 2; ++rep) scatter_runs<<<ntiles, 512>>>(out, ntiles, run, skew);
      cudaEventRecord(a);
      const int R = 5;
      for (int rep = 0; rep < R; ++rep) scatter_runs<<<ntiles, 512>>>(out, ntiles, run, skew);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= R;
      const double bytes = ntiles * 4096.0 * 8;
      printf("scatter run=%2d skew=%d: %.3f ms  %.0f GB/s (algorithmic 8 B/item)\n", run, skew, ms, bytes / ms / 1e6);
    }
  // ---- 2. multisplit cost
  uint32_t* sink;
  cudaMalloc(&sink, sms * 2048 * sizeof(uint32_t));
  const int iters = 4096;
  auto run_ms = [&](void (*kern)(uint32_t*, int), const char* name) {
    kern<<<sms * 2, 1024>>>(sink, iters);
    cudaEventRecord(a);
    kern<<<sms * 2, 1024>>>(sink, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double items = (double)sms * 2048 * iters;
    printf("%-24s %.3f ms  %.1f G items/s  %.2f items/clk/SM (at %d MHz)\n", name, ms, items / ms / 1e6,
           items / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1000);
  };
  run_ms(multisplit<2, 8>, "floor (hash only)");
  run_ms(multisplit<0, 8>, "MATCH.ANY 8-bit");
  run_ms(multisplit<1, 8>, "ballot 8-bit");
  run_ms(multisplit<0, 12>, "MATCH.ANY 12-bit");
  run_ms(multisplit<1, 12>, "ballot 12-bit");
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
