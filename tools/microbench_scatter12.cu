// microbench_scatter12.cu -- design probe for a 2-pass (12-bit digit) seed-table sort:
// can B200 scatter one item per (tile, digit) run at HBM speed?  Every CTA of a persistent grid
// owns one contiguous chunk of the input and, for each digit, one contiguous slice of that
// digit's output region (slices of consecutive CTAs are adjacent, as in a reduce-then-scan
// pass).  Tiles of 4096 items are read coalesced; each item takes an (unstable) slot in its
// digit's slice from a shared counter and is stored straight from registers.  With 4096 digits
// the runs of one tile are ~1 item long, so a 32 B sector is completed by ~4 successive tiles of
// the same CTA: the probe says whether L2 merges those partial sectors (ncu dram__bytes_write)
// and what the scattered stores cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mbs tools/microbench_scatter12.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill(uint64_t* a, uint64_t m) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = mix64(i);
}

// OUT: 0 = one u64 per item, 1 = u32 + u64 (the last pass: fp + position), 2 = u32 + u32
template <int DBITS, int OUT, int IPT>
__global__ void __launch_bounds__(256) scat(const uint64_t* __restrict__ in, uint64_t chunk, uint64_t rpc,
                                            uint64_t* __restrict__ o64, uint32_t* __restrict__ o32) {
  constexpr int D = 1 << DBITS, T = 256 * IPT;
  __shared__ uint32_t cnt[D];
  for (int i = threadIdx.x; i < D; i += 256) cnt[i] = 0;
  __syncthreads();
  const uint64_t c = blockIdx.x, G = gridDim.x;
  const uint64_t base0 = c * chunk;
  for (uint64_t t = 0; t < chunk; t += T) {
    uint64_t v[IPT];
#pragma unroll
    for (int u = 0; u < IPT; ++u) v[u] = in[base0 + t + u * 256 + threadIdx.x];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
      const uint32_t d = (uint32_t)(v[u] >> 40) & (D - 1);
      const uint32_t r = atomicAdd(&cnt[d], 1u);
      const uint64_t idx = ((uint64_t)d * G + c) * rpc + r;
      if (OUT == 0) {
        o64[idx] = v[u];
      } else if (OUT == 1) {
        o32[idx] = (uint32_t)(v[u] >> 32);
        o64[idx] = v[u] & 0xffffffffull;
      } else {
        o32[idx] = (uint32_t)(v[u] >> 32);
        reinterpret_cast<uint32_t*>(o64)[idx] = (uint32_t)v[u];
      }
    }
  }
}

template <int DBITS, int OUT, int IPT>
void run(const char* name, const uint64_t* in, uint64_t m, int G, uint64_t* o64, uint32_t* o32, uint64_t cap) {
  const uint64_t T = 256 * IPT;
  const uint64_t chunk = (m / G) / T * T;
  const uint64_t D = 1ull << DBITS;
  const uint64_t rpc = chunk / D + chunk / D / 4 + 64;  // slack for the per-(CTA, digit) count
  if (rpc * D * G > cap) { printf("%s: cap too small\n", name); return; }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  scat<DBITS, OUT, IPT><<<G, 256>>>(in, chunk, rpc, o64, o32);
  cudaEventRecord(a);
  const int R = 5;
  for (int i = 0; i < R; ++i) scat<DBITS, OUT, IPT><<<G, 256>>>(in, chunk, rpc, o64, o32);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= R;
  const double items = (double)chunk * G;
  const double bpi = 8 + (OUT == 0 ? 8 : OUT == 1 ? 12 : 8);
  printf("%-28s G=%d items=%.3g  %.3f ms  %.1f G items/s  %.0f GB/s algorithmic (%.0f B/item)\n", name, G, items, ms,
         items / ms / 1e6, items * bpi / ms / 1e6, bpi);
}

int main(int argc, char** argv) {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const uint64_t m = argc > 1 ? strtoull(argv[1], 0, 10) : 558000000ull;
  uint64_t *in, *o64;
  uint32_t* o32;
  const uint64_t cap = m + m / 2 + (1u << 24);
  cudaMalloc(&in, m * 8);
  cudaMalloc(&o64, cap * 8);
  cudaMalloc(&o32, cap * 4);
  fill<<<sms * 8, 256>>>(in, m);
  for (int occ : {2, 4}) {
    const int G = sms * occ;
    run<8, 0, 16>("8-bit u64", in, m, G, o64, o32, cap);
    run<12, 0, 16>("12-bit u64", in, m, G, o64, o32, cap);
    run<12, 1, 16>("12-bit u32+u64", in, m, G, o64, o32, cap);
    run<12, 2, 16>("12-bit u32+u32", in, m, G, o64, o32, cap);
    run<12, 0, 8>("12-bit u64 ipt8", in, m, G, o64, o32, cap);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
