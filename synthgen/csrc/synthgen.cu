// synthgen.cu -- device twin of synthgen/host.py (same counter-based SplitMix64 streams,
// bit-identical output; tests/test_gpu_synthgen.py checks it).  Input generation only:
// no k-mer, hash, window or seed-table arithmetic lives here.
#include <cuda_runtime.h>
#include <stdint.h>

#define SG_API extern "C" __attribute__((visibility("default")))

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __constant__ uint8_t kACGT[4] = {'A', 'C', 'G', 'T'};

__global__ void uniform_ascii_kernel(uint8_t* out, uint64_t lo, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = kACGT[mix64(seed, lo + i) >> 62];
}

__global__ void gc_ascii_kernel(uint8_t* out, uint64_t lo, uint64_t n, uint64_t seed, uint32_t ta, uint32_t tc,
                                uint32_t tg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = (uint32_t)(mix64(seed, lo + i) >> 32);
    out[i] = kACGT[(u >= ta) + (u >= tc) + (u >= tg)];
  }
}

// one block per interval [s, e) (global coordinates), clipped to [lo, lo+n)
__global__ void fill_n_kernel(uint8_t* out, uint64_t lo, uint64_t n, const int64_t* iv) {
  const int64_t s = iv[2 * blockIdx.x], e = iv[2 * blockIdx.x + 1];
  const int64_t a = s > (int64_t)lo ? s : (int64_t)lo;
  const int64_t b = e < (int64_t)(lo + n) ? e : (int64_t)(lo + n);
  for (int64_t g = a + threadIdx.x; g < b; g += blockDim.x) out[g - lo] = 'N';
}

// one block per read: base t of read r = template[start_r + t], 10 % substituted
__global__ void reads_ascii_kernel(uint8_t* out, const int64_t* read_off, const int64_t* starts, uint64_t nreads,
                                   uint64_t seed_t, uint64_t seed_sub, uint32_t sub_t) {
  for (uint64_t r = blockIdx.x; r < nreads; r += gridDim.x) {
    const int64_t o = read_off[r], len = read_off[r + 1] - o, st = starts[r];
    for (int64_t t = threadIdx.x; t < len; t += blockDim.x) {
      uint32_t b = (uint32_t)(mix64(seed_t, (uint64_t)(st + t)) >> 62);
      const uint64_t v = mix64(seed_sub, (uint64_t)(o + t));
      if ((uint32_t)(v >> 32) < sub_t) b = (b + 1 + (uint32_t)((v & 0xffffffffull) % 3)) & 3;
      out[o + t] = kACGT[b];
    }
  }
}

__global__ void u32_kernel(uint32_t* out, uint64_t lo, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = lo + i;
    out[i] = (uint32_t)(mix64(seed, g >> 1) >> ((g & 1) * 32));
  }
}

__global__ void f32_table_kernel(float* out, uint64_t lo, uint64_t n, uint64_t seed, const float* table) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = table[mix64(seed, lo + i) >> 48];
}

unsigned grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return (unsigned)(b < 148 * 32 ? (b ? b : 1) : 148 * 32);
}

}  // namespace

SG_API int sg_uniform_ascii(uint8_t* out, uint64_t lo, uint64_t n, uint64_t seed, void* stream) {
  uniform_ascii_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, lo, n, seed);
  return (int)cudaPeekAtLastError();
}

SG_API int sg_gc_ascii(uint8_t* out, uint64_t lo, uint64_t n, uint64_t seed, uint32_t ta, uint32_t tc, uint32_t tg,
                       const int64_t* iv, uint64_t niv, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  gc_ascii_kernel<<<grid_for(n), 256, 0, st>>>(out, lo, n, seed, ta, tc, tg);
  if (niv) fill_n_kernel<<<(unsigned)niv, 256, 0, st>>>(out, lo, n, iv);
  return (int)cudaPeekAtLastError();
}

SG_API int sg_reads_ascii(uint8_t* out, const int64_t* read_off, const int64_t* starts, uint64_t nreads,
                          uint64_t seed_t, uint64_t seed_sub, uint32_t sub_t, void* stream) {
  const unsigned g = (unsigned)(nreads < 148 * 64 ? (nreads ? nreads : 1) : 148 * 64);
  reads_ascii_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(out, read_off, starts, nreads, seed_t, seed_sub, sub_t);
  return (int)cudaPeekAtLastError();
}

SG_API int sg_u32(uint32_t* out, uint64_t lo, uint64_t n, uint64_t seed, void* stream) {
  u32_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, lo, n, seed);
  return (int)cudaPeekAtLastError();
}

SG_API int sg_f32_table(float* out, uint64_t lo, uint64_t n, uint64_t seed, const float* table, void* stream) {
  f32_table_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(out, lo, n, seed, table);
  return (int)cudaPeekAtLastError();
}
