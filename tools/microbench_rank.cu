// microbench_rank.cu -- cost of the warp/CTA ranking primitives a radix downsweep can be built
// from, on B200 (design probe for DESIGN.md 5, K7).  Each kernel ranks ITERS*32 random 8-bit
// digits per warp and reports items/clk/SM.  The HBM roof of one LSD pass on 8-byte items
// (16 B/item) is 6.5 TB/s / 16 B / (148 SMs * 1.965 GHz) = 0.93 items/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mr tools/microbench_rank.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

// MODE 0: hash only (floor).  1: 8 VOTEs only (no peer logic).  2: ballot multi-split (peers).
// 3: ballot multi-split with the bit predicate from one LOP3 and the select folded into one LOP3.
// 4: smem atomicAdd with return on a per-warp 256-counter histogram (unstable rank).
// 5: per-thread private counters [digit][thread] (u16 pairs), sequential within the thread.
// 6: red (no return) smem atomics per warp histogram.
template <int MODE>
__global__ void __launch_bounds__(256) rank_kernel(uint32_t* sink, int iters) {
  extern __shared__ uint32_t dyn[];
  uint32_t (*wh)[256] = reinterpret_cast<uint32_t (*)[256]>(dyn);          // [8][256]
  uint32_t (*tc)[256] = reinterpret_cast<uint32_t (*)[256]>(dyn + 2048);   // [128][256] (mode 5)
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5, lt = (1u << lane) - 1u;
  if (MODE == 4 || MODE == 6)
    for (int i = lane; i < 256; i += 32) wh[wid][i] = 0;
  if (MODE == 5)
    for (int i = 0; i < 128; ++i) tc[i][threadIdx.x] = 0;
  __syncthreads();
  uint32_t acc = 0, s = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    const uint32_t d = mix(s * 0x2545F491u + i) & 255u;
    if (MODE == 0) {
      acc += d;
    } else if (MODE == 1) {
#pragma unroll
      for (int b = 0; b < 8; ++b) acc += __ballot_sync(0xffffffffu, (d >> b) & 1u);
    } else if (MODE == 2) {
      unsigned peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const bool bit = (d >> b) & 1u;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
      }
      acc += __popc(peers & lt);
    } else if (MODE == 3) {
      unsigned peers = 0xffffffffu;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        unsigned m;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\tvote.sync.ballot.b32 %0, p, 0xffffffff;\n\t}"
                     : "=r"(m) : "r"(0), "r"(d & (1u << b)));
        const unsigned sx = 0u - ((d >> b) & 1u);
        peers &= ~(m ^ sx);
      }
      acc += __popc(peers & lt);
    } else if (MODE == 4) {
      acc += atomicAdd(&wh[wid][d], 1u);
    } else if (MODE == 5) {
      const uint32_t r = d & 127u, sh = (d >> 7) << 4;
      const uint32_t old = tc[r][threadIdx.x];
      tc[r][threadIdx.x] = old + (1u << sh);
      acc += (old >> sh) & 0xffffu;
    } else if (MODE == 6) {
      atomicAdd(&wh[wid][d], 1u);
    }
  }
  if (MODE == 6 || MODE == 4) { __syncwarp(); acc += wh[wid][lane]; }
  if (MODE == 5) acc += tc[lane][threadIdx.x];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  uint32_t* sink;
  const int maxb = sms * 8;
  cudaMalloc(&sink, (size_t)maxb * 256 * sizeof(uint32_t));
  const int iters = 2048;
  auto run = [&](void (*kern)(uint32_t*, int), const char* name, int smem) {
    for (int bps : {1, 2, 4, 8}) {  // CTAs of 256 threads per SM: occupancy sweep
      const int grid = sms * bps;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<grid, 256, smem>>>(sink, iters);
      cudaEventRecord(a);
      kern<<<grid, 256, smem>>>(sink, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double items = (double)grid * 256 * iters;
      printf("%-34s CTAs/SM=%d  %.3f ms  %.2f items/clk/SM\n", name, bps, ms,
             items / (ms * 1e-3) / sms / (p.clockRate * 1e3));
    }
  };
  run(rank_kernel<0>, "0 floor (hash)", 8192);
  run(rank_kernel<1>, "1 8 x VOTE", 8192);
  run(rank_kernel<2>, "2 ballot multi-split", 8192);
  run(rank_kernel<3>, "3 ballot multi-split (lop3)", 8192);
  run(rank_kernel<4>, "4 ATOMS with return", 8192);
  run(rank_kernel<5>, "5 per-thread counters", 8192 + 131072);
  run(rank_kernel<6>, "6 ATOMS no return (RED)", 8192);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
