// common.cuh -- shared device/host helpers of libmzslsum (sm_100a).
//
// Nothing in here is part of the oracle (oracle/ shares no code with csrc/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/mzslsum.h"

#define MZS_API extern "C" __attribute__((visibility("default")))

namespace mzs {

// ---------------------------------------------------------------- host helpers
void set_cuda_error(cudaError_t e);

#define MZS_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) {                             \
      ::mzs::set_cuda_error(e_);                         \
      return SLSUM_ECUDA;                                \
    }                                                    \
  } while (0)

#define MZS_LAUNCHED() MZS_CUDA(cudaPeekAtLastError())

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

// Carves typed sub-buffers out of a caller-provided workspace.
struct Carve {
  char* base;
  size_t cap;
  size_t used = 0;
  bool ok = true;
  Carve(void* p, size_t c) : base(static_cast<char*>(p)), cap(c) {}
  template <class T>
  T* take(size_t n) {
    size_t bytes = align_up(n * sizeof(T));
    if (used + bytes > cap) { ok = false; return nullptr; }
    T* r = reinterpret_cast<T*>(base + used);
    used += bytes;
    return r;
  }
};

// Sizes a workspace the same way Carve consumes it.
struct Sizer {
  size_t used = 0;
  template <class T>
  void take(size_t n) { used += align_up(n * sizeof(T)); }
};

// Owns a temporary workspace when the caller passed ws == NULL.
struct TempWs {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~TempWs() { if (p) cudaFreeAsync(p, s); }
};

// ---------------------------------------------------------------- radix chunk layout
// The seed-table radix passes cut their m entries into chunks (one downsweep CTA each): at
// most 131072 entries, at least 4096, and about m/296 in between so that small tables still
// spread over the SMs.  A pass's digit counts are laid out counts[digit * nchunks + chunk]
// with nchunks = ceil(m / chunk).  mz_extract_ex's first-pass histogram (mz_out.hist) uses the
// same layout with m = its capacity, so seedtable_build_items_ex can start from it.
constexpr uint32_t kRadixChunkMax = 131072;
constexpr uint32_t kRadixChunkMin = 4096;
inline uint32_t radix_chunk_for(uint64_t m) {
  const uint64_t want = (m + 295) / 296;
  const uint64_t c = (want + kRadixChunkMin - 1) / kRadixChunkMin * kRadixChunkMin;
  return (uint32_t)(c < kRadixChunkMin ? kRadixChunkMin : (c > kRadixChunkMax ? kRadixChunkMax : c));
}
inline uint64_t radix_nchunks(uint64_t m) { return (m + radix_chunk_for(m) - 1) / radix_chunk_for(m); }

// ---------------------------------------------------------------- shared host entry points
// (seedtable.cu) stable sort of (u32 fingerprint, u64 index) pairs by fingerprint bits
// [lo_bit, 32), used by the sorted seed lookup
size_t sort_fp_idx_workspace_bytes(uint64_t m, int lo_bit);
// (seedtable.cu) stable sort of packed u64 items by bits [lo_bit, hi_bit) of their high 32 bits
size_t sort_items_workspace_bytes(uint64_t m, int lo_bit, int hi_bit);
int sort_items(const uint64_t* items, uint64_t m, int lo_bit, int hi_bit, uint64_t* out, void* ws, size_t ws_bytes,
               cudaStream_t st);
int sort_fp_idx(const uint32_t* fp, const uint64_t* idx, uint64_t m, int lo_bit, uint32_t* fp_out, uint64_t* idx_out,
                void* ws, size_t ws_bytes, cudaStream_t st);

// ---------------------------------------------------------------- device self-checks
// MZS_DCHECK: bounds / invariant checks inside the kernels, compiled in only by a debug build
// (-DMZS_DEBUG_CHECKS=1, tools/variant_lib.sh); a violated check traps, which fails the launch.
// compute-sanitizer is not available on this pool, so a test run against the checked build
// stands in for memcheck on the indices the kernels compute themselves.
#if defined(MZS_DEBUG_CHECKS) && MZS_DEBUG_CHECKS
#define MZS_DCHECK(cond) \
  do {                   \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define MZS_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned warp_id() { return threadIdx.x >> 5; }

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t* p) {
  return *reinterpret_cast<const volatile uint64_t*>(p);
}
__device__ __forceinline__ void st_volatile_u64(uint64_t* p, uint64_t v) {
  *reinterpret_cast<volatile uint64_t*>(p) = v;
}

// Decoupled look-back tile status words: (flag << 62) | value.
constexpr uint64_t kLbAgg = 1ull << 62;      // tile aggregate published
constexpr uint64_t kLbInc = 2ull << 62;      // inclusive prefix published
constexpr uint64_t kLbVal = (1ull << 62) - 1;

// Decoupled look-back, split in two so a tile can publish its aggregate as soon as it is
// known and resolve its prefix later (after doing other work).
// publish: one thread.  Tile 0's aggregate is its inclusive prefix.
__device__ __forceinline__ void lookback_publish(uint64_t* status, uint64_t tile, uint64_t agg) {
  st_volatile_u64(&status[tile], (tile == 0 ? kLbInc : kLbAgg) | agg);
}
// resolve: ALL 32 lanes of ONE warp.  Walks back over predecessors 32 at a time, returns
// the exclusive prefix and publishes this tile's inclusive prefix.  Tiles are numbered in
// claim order and every claimed tile publishes its aggregate without waiting, so the walk
// always terminates.
__device__ __forceinline__ uint64_t lookback_resolve(uint64_t* status, uint64_t tile, uint64_t agg) {
  const unsigned lane = lane_id();
  if (tile == 0) return 0;
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    int64_t idx = base - (int64_t)lane;
    uint64_t v = idx >= 0 ? ld_volatile_u64(&status[idx]) : (kLbInc | 0);
    while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
      if ((v >> 62) == 0) v = ld_volatile_u64(&status[idx]);
    }
    unsigned inc_mask = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    uint64_t val = v & kLbVal;
    if (inc_mask) {
      int first = __ffs(inc_mask) - 1;  // closest predecessor with an inclusive prefix
      uint64_t part = lane <= (unsigned)first ? val : 0;
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      excl += part;
      break;
    }
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    excl += val;
    base -= 32;
  }
  if (lane == 0) st_volatile_u64(&status[tile], kLbInc | (excl + agg));
  return excl;
}

// Both steps at once (ALL 32 lanes of ONE warp).
__device__ __forceinline__ uint64_t lookback_exclusive(uint64_t* status, uint64_t tile, uint64_t agg) {
  if (lane_id() == 0) lookback_publish(status, tile, agg);
  __syncwarp();
  return lookback_resolve(status, tile, agg);
}

// Block-wide exclusive sum of one value per thread (TPB threads, multiple of 32).
// `warp_sums` must hold TPB/32 entries of shared memory.  Returns the exclusive prefix
// of this thread; *total receives the block total (valid in every thread).
template <int TPB, class T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* warp_sums, T* total) {
  constexpr int NW = TPB / 32;
  const unsigned lane = lane_id(), wid = warp_id();
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (unsigned)o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T s = lane < (unsigned)NW ? warp_sums[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= (unsigned)o) s += y;
    }
    if (lane < (unsigned)NW) warp_sums[lane] = s;  // inclusive warp prefix
  }
  __syncthreads();
  T wpre = wid ? warp_sums[wid - 1] : T(0);
  *total = warp_sums[NW - 1];
  __syncthreads();
  return wpre + x - v;
}

}  // namespace mzs
