// seedtable.cu -- seed pointer table + seed position table (Sec. 2.4, Fig. 1)
// for hashed minimizers, bucketed on the top `bits` bits of the 2k-bit key (R21).
//
// The build is a bucket histogram + a STABLE scatter into bucket order.  The scatter is
// done as an LSD radix sort on the bucket bits with 8-bit digits (one pass per digit):
// every pass ranks a tile of 4096 entries per digit with warp match_any (stable), gets the
// tile's per-digit global offset from a per-digit decoupled look-back over tiles, and
// scatters.  Stability makes the positions inside a bucket ascending (the input minimizer
// list is ascending by position), for any bucket-size distribution.  The pointer table
// is then read off the sorted fingerprints (first index of every bucket).
//
// Multi-GPU phases: count (histogram for the all-reduce), partition (one stable pass on
// the owner digit), finalize (stable passes on the remaining bucket bits of the owner).
#include <algorithm>

#include "common.cuh"

namespace mzs {
namespace {

constexpr int kTPB = 256;
constexpr int kIPT = 16;                     // items per thread per pass
constexpr int kTile = kTPB * kIPT;           // 4096 entries per tile
constexpr int kNW = kTPB / 32;

__device__ __forceinline__ uint32_t fingerprint(uint64_t key, int k) {
  const int b = 2 * k;
  return b >= 32 ? (uint32_t)(key >> (b - 32)) : (uint32_t)(key << (32 - b));
}

__device__ __forceinline__ uint64_t count_of(const uint64_t* d_m, uint64_t m) { return d_m ? *d_m : m; }

// ---------------------------------------------------------------- digit histograms
// hist[p*256 + d] += number of entries whose pass-p digit is d
template <bool FROM_HASH>
__global__ void __launch_bounds__(kTPB) hist_kernel(const void* keys, const uint64_t* d_m, uint64_t m_cap, int k,
                                                    int lo_bit, int hi_bit, unsigned long long* hist) {
  __shared__ uint32_t h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += kTPB) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t m = min(count_of(d_m, m_cap), m_cap);
  const int npass = (hi_bit - lo_bit + 7) / 8;
  for (uint64_t i = (uint64_t)blockIdx.x * kTPB + threadIdx.x; i < m; i += (uint64_t)gridDim.x * kTPB) {
    const uint32_t f = FROM_HASH ? fingerprint(static_cast<const uint64_t*>(keys)[i], k)
                                 : static_cast<const uint32_t*>(keys)[i];
    for (int p = 0; p < npass; ++p) {
      const int sh = lo_bit + 8 * p;
      const int nb = min(8, hi_bit - sh);
      atomicAdd(&h[p][(f >> sh) & ((1u << nb) - 1u)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += kTPB) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(&hist[i], (unsigned long long)v);
  }
}

// exclusive scan of each pass's 256 bins (one block of 256 threads)
__global__ void digit_scan_kernel(const unsigned long long* hist, unsigned long long* base, int npass) {
  __shared__ unsigned long long ws[kNW];
  for (int p = 0; p < npass; ++p) {
    unsigned long long tot;
    const unsigned long long v = hist[p * 256 + threadIdx.x];
    const unsigned long long ex = block_exclusive_sum<256, unsigned long long>(v, ws, &tot);
    base[p * 256 + threadIdx.x] = ex;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- one stable radix pass
template <bool FROM_HASH>
__global__ void __launch_bounds__(kTPB) radix_pass_kernel(const void* keys_in, const uint64_t* __restrict__ pos_in,
                                                          uint32_t* __restrict__ fp_out, uint64_t* __restrict__ pos_out,
                                                          const uint64_t* d_m, uint64_t m_cap, int k, int shift,
                                                          int dbits, const unsigned long long* __restrict__ dbase,
                                                          uint64_t* status, uint32_t* tile_counter) {
  __shared__ uint32_t wcnt[kNW][256];
  __shared__ uint64_t doff[256];
  __shared__ uint32_t s_tile;
  const unsigned lane = lane_id(), wid = warp_id();
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = lane; i < 256; i += 32) wcnt[wid][i] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t m = min(count_of(d_m, m_cap), m_cap);
  const uint64_t base = tile * (uint64_t)kTile;
  if (base >= m) return;  // no later tile has entries either
  const uint32_t dmask = (1u << dbits) - 1u;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t key[kIPT], rank[kIPT];
  uint64_t pos[kIPT];
#pragma unroll
  for (int it = 0; it < kIPT; ++it) {
    const uint64_t idx = base + (uint64_t)wid * (kIPT * 32) + (uint64_t)it * 32 + lane;
    const bool valid = idx < m;
    uint32_t f = 0;
    uint64_t p = 0;
    if (valid) {
      f = FROM_HASH ? fingerprint(static_cast<const uint64_t*>(keys_in)[idx], k)
                    : static_cast<const uint32_t*>(keys_in)[idx];
      p = pos_in[idx];
    }
    const uint32_t d = valid ? ((f >> shift) & dmask) : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = __popc(peers & lt);
    const uint32_t c = (d < 256u) ? wcnt[wid][d] : 0u;
    __syncwarp();
    if (d < 256u && before == 0) wcnt[wid][d] = c + __popc(peers);
    __syncwarp();
    key[it] = f;
    pos[it] = p;
    rank[it] = (d < 256u) ? c + before : 0xffffffffu;
  }
  __syncthreads();
  // per digit: exclusive prefix over warps, tile total, look-back over tiles
  {
    const uint32_t d = threadIdx.x;  // kTPB == 256 digits
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kNW; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    uint64_t* st = status + d;
    const uint64_t total = run;
    uint64_t excl = 0;
    if (tile == 0) {
      st_volatile_u64(st, kLbInc | total);
    } else {
      st_volatile_u64(st + tile * 256, kLbAgg | total);
      int64_t t = (int64_t)tile - 1;
      while (t >= 0) {
        uint64_t v;
        do { v = ld_volatile_u64(st + (uint64_t)t * 256); } while ((v >> 62) == 0);
        excl += v & kLbVal;
        if ((v >> 62) == 2) break;
        --t;
      }
      st_volatile_u64(st + tile * 256, kLbInc | (excl + total));
    }
    doff[d] = dbase[d] + excl;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kIPT; ++it) {
    if (rank[it] != 0xffffffffu) {
      const uint32_t d = (key[it] >> shift) & dmask;
      const uint64_t dst = doff[d] + wcnt[wid][d] + rank[it];
      fp_out[dst] = key[it];
      pos_out[dst] = pos[it];
    }
  }
}

// offsets[b] = first index whose bucket >= b (b in [0, nb]); fp sorted by bucket.
// bucket(f) = (f >> shift) & bmask
__global__ void offsets_kernel(const uint32_t* __restrict__ fp, const uint64_t* d_m, uint64_t m_cap, int shift,
                               uint32_t bmask, uint64_t nb, uint64_t* __restrict__ offsets) {
  const uint64_t m = min(count_of(d_m, m_cap), m_cap);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += stride) {
    const int64_t prev = i == 0 ? -1 : (int64_t)((fp[i - 1] >> shift) & bmask);
    const int64_t cur = i == m ? (int64_t)nb : (int64_t)((fp[i] >> shift) & bmask);
    for (int64_t b = prev + 1; b <= cur; ++b) offsets[b] = i;
  }
}

// counts[bucket] += 1 (global atomics; the 2^bits counters stay L2-resident)
__global__ void __launch_bounds__(kTPB) count_kernel(const uint64_t* __restrict__ hash, const uint64_t* d_m,
                                                     uint64_t m_cap, int k, int bits, uint32_t* counts) {
  const uint64_t m = min(count_of(d_m, m_cap), m_cap);
  for (uint64_t i = (uint64_t)blockIdx.x * kTPB + threadIdx.x; i < m; i += (uint64_t)gridDim.x * kTPB)
    atomicAdd(&counts[fingerprint(hash[i], k) >> (32 - bits)], 1u);
}

// offsets_local from the owner's slice of the all-reduced counts (one block, chained scan)
__global__ void counts_scan_kernel(const uint32_t* counts, uint64_t b0, uint64_t nb, uint64_t* offsets) {
  __shared__ unsigned long long ws[kNW];
  __shared__ unsigned long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint64_t per = (nb + kTPB - 1) / kTPB;
  // thread t scans its contiguous chunk serially, then a block scan of chunk totals
  const uint64_t c0 = threadIdx.x * per, c1 = min(nb, c0 + per);
  unsigned long long s = 0;
  for (uint64_t b = c0; b < c1; ++b) s += counts[b0 + b];
  unsigned long long tot;
  unsigned long long ex = block_exclusive_sum<kTPB, unsigned long long>(s, ws, &tot);
  for (uint64_t b = c0; b < c1; ++b) {
    offsets[b] = ex;
    ex += counts[b0 + b];
  }
  if (threadIdx.x == kTPB - 1) offsets[nb] = tot;
}

// identity partition (one rank): fingerprints + positions in input order, count = m
__global__ void fp_copy_kernel(const uint64_t* __restrict__ hash, const uint64_t* __restrict__ pos, const uint64_t* d_m,
                               uint64_t m_cap, int k, uint32_t* __restrict__ fp, uint64_t* __restrict__ pos_out,
                               uint64_t* send_counts) {
  const uint64_t m = min(count_of(d_m, m_cap), m_cap);
  const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i0 == 0) send_counts[0] = m;
  for (uint64_t i = i0; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    fp[i] = fingerprint(hash[i], k);
    pos_out[i] = pos[i];
  }
}

__global__ void u32_to_u64_kernel(const unsigned long long* in, uint64_t* out, int n) {
  if ((int)threadIdx.x < n) out[threadIdx.x] = in[threadIdx.x];
}

// ---------------------------------------------------------------- host helpers
struct SortWs {
  unsigned long long* hist;   // [npass*256]
  unsigned long long* dbase;  // [npass*256]
  uint32_t* counters;         // [npass]
  uint64_t* status;           // [ntiles*256]
  uint32_t* fpA;
  uint64_t* posA;
  uint32_t* fpB;
  uint64_t* posB;
  uint32_t* fpF;              // final fingerprints when the caller gave none
};

uint64_t tiles_for(uint64_t m) { return (m + kTile - 1) / kTile + 1; }

template <class C>
void size_sort_ws(C& c, uint64_t m, int npass, bool need_fp) {
  c.template take<unsigned long long>(4 * 256);
  c.template take<unsigned long long>(4 * 256);
  c.template take<uint32_t>(4);
  c.template take<uint64_t>(tiles_for(m) * 256);
  if (npass >= 2) {
    c.template take<uint32_t>(m + 1);
    c.template take<uint64_t>(m + 1);
  }
  if (npass >= 3) {
    c.template take<uint32_t>(m + 1);
    c.template take<uint64_t>(m + 1);
  }
  if (need_fp) c.template take<uint32_t>(m + 1);
}

bool carve_sort_ws(Carve& c, uint64_t m, int npass, bool need_fp, SortWs& s) {
  s = SortWs{};
  s.hist = c.take<unsigned long long>(4 * 256);
  s.dbase = c.take<unsigned long long>(4 * 256);
  s.counters = c.take<uint32_t>(4);
  s.status = c.take<uint64_t>(tiles_for(m) * 256);
  if (npass >= 2) { s.fpA = c.take<uint32_t>(m + 1); s.posA = c.take<uint64_t>(m + 1); }
  if (npass >= 3) { s.fpB = c.take<uint32_t>(m + 1); s.posB = c.take<uint64_t>(m + 1); }
  if (need_fp) s.fpF = c.take<uint32_t>(m + 1);
  return c.ok;
}

int grid_stride_blocks(uint64_t m) {
  const uint64_t want = (m + kTPB - 1) / kTPB;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  return (int)std::max<uint64_t>(1, std::min(want, cap));
}

// Stable LSD sort of m entries by fp bits [lo_bit, hi_bit) into (fp_dst, pos_dst).
int stable_sort(bool from_hash, const void* keys, const uint64_t* pos, const uint64_t* d_m, uint64_t m, int k,
                int lo_bit, int hi_bit, uint32_t* fp_dst, uint64_t* pos_dst, SortWs& s, cudaStream_t st) {
  const int npass = (hi_bit - lo_bit + 7) / 8;
  if (npass > 4 || npass < 1) return SLSUM_EINVAL;
  MZS_CUDA(cudaMemsetAsync(s.hist, 0, sizeof(unsigned long long) * 256 * npass, st));
  MZS_CUDA(cudaMemsetAsync(s.counters, 0, sizeof(uint32_t) * npass, st));
  const int hb = grid_stride_blocks(m);
  if (from_hash)
    hist_kernel<true><<<hb, kTPB, 0, st>>>(keys, d_m, m, k, lo_bit, hi_bit, s.hist);
  else
    hist_kernel<false><<<hb, kTPB, 0, st>>>(keys, d_m, m, k, lo_bit, hi_bit, s.hist);
  MZS_LAUNCHED();
  digit_scan_kernel<<<1, 256, 0, st>>>(s.hist, s.dbase, npass);
  MZS_LAUNCHED();
  const uint64_t ntiles = (m + kTile - 1) / kTile;
  const void* kin = keys;
  const uint64_t* pin = pos;
  bool kin_hash = from_hash;
  for (int p = 0; p < npass; ++p) {
    uint32_t* fo;
    uint64_t* po;
    if (p == npass - 1) { fo = fp_dst; po = pos_dst; }
    else if (p % 2 == 0) { fo = s.fpA; po = s.posA; }
    else { fo = s.fpB; po = s.posB; }
    const int sh = lo_bit + 8 * p;
    const int nb = std::min(8, hi_bit - sh);
    MZS_CUDA(cudaMemsetAsync(s.status, 0, sizeof(uint64_t) * 256 * std::max<uint64_t>(ntiles, 1), st));
    if (ntiles) {
      if (kin_hash)
        radix_pass_kernel<true><<<(unsigned)ntiles, kTPB, 0, st>>>(kin, pin, fo, po, d_m, m, k, sh, nb,
                                                                   s.dbase + 256 * p, s.status, s.counters + p);
      else
        radix_pass_kernel<false><<<(unsigned)ntiles, kTPB, 0, st>>>(kin, pin, fo, po, d_m, m, k, sh, nb,
                                                                    s.dbase + 256 * p, s.status, s.counters + p);
      MZS_LAUNCHED();
    }
    kin = fo;
    pin = po;
    kin_hash = false;
  }
  return SLSUM_OK;
}

int offsets_launch(const uint32_t* fp, const uint64_t* d_m, uint64_t m, int shift, uint32_t bmask, uint64_t nb,
                   uint64_t* offsets, cudaStream_t st) {
  const int blocks = grid_stride_blocks(m + 1);
  offsets_kernel<<<blocks, kTPB, 0, st>>>(fp, d_m, m, shift, bmask, nb, offsets);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }
int log2i(int x) { int r = 0; while ((1 << r) < x) ++r; return r; }

}  // namespace
}  // namespace mzs

using namespace mzs;

MZS_API size_t seedtable_workspace_bytes(uint64_t m, int bucket_bits) {
  Sizer z;
  const int npass = (bucket_bits + 7) / 8;
  size_sort_ws(z, m, npass, true);
  return z.used;
}

MZS_API int seedtable_build(const uint64_t* hash, const uint64_t* pos, uint64_t m, const uint64_t* d_m, int k,
                            int bucket_bits, uint64_t* offsets, uint32_t* fp_out, uint64_t* pos_out, void* ws,
                            size_t ws_bytes, void* stream) {
  if (k < 1 || k > 31 || bucket_bits < 1 || bucket_bits > 30 || bucket_bits > 2 * k) return SLSUM_EINVAL;
  if (!offsets || (m && (!hash || !pos || !pos_out))) return SLSUM_EINVAL;
  cudaStream_t st = as_stream(stream);
  const uint64_t nb = 1ull << bucket_bits;
  if (m == 0) {
    MZS_CUDA(cudaMemsetAsync(offsets, 0, sizeof(uint64_t) * (nb + 1), st));
    return SLSUM_OK;
  }
  TempWs tmp;
  const size_t need = seedtable_workspace_bytes(m, bucket_bits);
  if (!ws) {
    MZS_CUDA(cudaMallocAsync(&tmp.p, need, st));
    tmp.s = st;
    ws = tmp.p;
    ws_bytes = need;
  }
  if (ws_bytes < need) return SLSUM_ENOMEM;
  Carve c(ws, ws_bytes);
  const int npass = (bucket_bits + 7) / 8;
  SortWs s;
  if (!carve_sort_ws(c, m, npass, true, s)) return SLSUM_ENOMEM;
  uint32_t* fp_final = fp_out ? fp_out : s.fpF;
  const int lo = 32 - bucket_bits;
  int rc = stable_sort(true, hash, pos, d_m, m, k, lo, 32, fp_final, pos_out, s, st);
  if (rc) return rc;
  return offsets_launch(fp_final, d_m, m, lo, (uint32_t)(nb - 1), nb, offsets, st);
}

MZS_API int seedtable_count(const uint64_t* hash, uint64_t m, const uint64_t* d_m, int k, int bucket_bits,
                            uint32_t* counts, void* stream) {
  if (k < 1 || k > 31 || bucket_bits < 1 || bucket_bits > 30 || bucket_bits > 2 * k || !counts) return SLSUM_EINVAL;
  cudaStream_t st = as_stream(stream);
  MZS_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) << bucket_bits, st));
  if (m == 0) return SLSUM_OK;
  if (!hash) return SLSUM_EINVAL;
  count_kernel<<<grid_stride_blocks(m), kTPB, 0, st>>>(hash, d_m, m, k, bucket_bits, counts);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

MZS_API size_t seedtable_partition_workspace_bytes(uint64_t m, int nranks) {
  (void)nranks;
  Sizer z;
  size_sort_ws(z, m, 1, false);
  return z.used;
}

MZS_API int seedtable_partition(const uint64_t* hash, const uint64_t* pos, uint64_t m, const uint64_t* d_m, int k,
                                int bucket_bits, int nranks, uint32_t* send_fp, uint64_t* send_pos,
                                uint64_t* send_counts, void* ws, size_t ws_bytes, void* stream) {
  if (k < 1 || k > 31 || bucket_bits < 1 || bucket_bits > 30 || bucket_bits > 2 * k) return SLSUM_EINVAL;
  if (!is_pow2(nranks) || nranks > 256 || log2i(nranks) > bucket_bits || !send_counts) return SLSUM_EINVAL;
  cudaStream_t st = as_stream(stream);
  if (m == 0) {
    MZS_CUDA(cudaMemsetAsync(send_counts, 0, sizeof(uint64_t) * nranks, st));
    return SLSUM_OK;
  }
  if (!hash || !pos || !send_fp || !send_pos) return SLSUM_EINVAL;
  TempWs tmp;
  const size_t need = seedtable_partition_workspace_bytes(m, nranks);
  if (!ws) {
    MZS_CUDA(cudaMallocAsync(&tmp.p, need, st));
    tmp.s = st;
    ws = tmp.p;
    ws_bytes = need;
  }
  if (ws_bytes < need) return SLSUM_ENOMEM;
  Carve c(ws, ws_bytes);
  SortWs s;
  if (!carve_sort_ws(c, m, 1, false, s)) return SLSUM_ENOMEM;
  const int g = log2i(nranks);
  if (g == 0) {
    // one owner: the stable partition is the identity
    fp_copy_kernel<<<grid_stride_blocks(m), kTPB, 0, st>>>(hash, pos, d_m, m, k, send_fp, send_pos, send_counts);
    MZS_LAUNCHED();
    return SLSUM_OK;
  }
  int rc = stable_sort(true, hash, pos, d_m, m, k, 32 - g, 32, send_fp, send_pos, s, st);
  if (rc) return rc;
  u32_to_u64_kernel<<<1, 256, 0, st>>>(s.hist, send_counts, nranks);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

MZS_API size_t seedtable_finalize_workspace_bytes(uint64_t m_recv, int bucket_bits, int nranks) {
  Sizer z;
  const int npass = std::max(1, (bucket_bits - log2i(nranks) + 7) / 8);
  size_sort_ws(z, m_recv, npass, true);
  return z.used;
}

MZS_API int seedtable_finalize(const uint32_t* recv_fp, const uint64_t* recv_pos, uint64_t m_recv,
                               const uint32_t* global_counts, int bucket_bits, int rank, int nranks,
                               uint64_t* offsets_local, uint64_t* pos_out, uint32_t* fp_out, void* ws,
                               size_t ws_bytes, void* stream) {
  if (bucket_bits < 1 || bucket_bits > 30 || !is_pow2(nranks) || rank < 0 || rank >= nranks) return SLSUM_EINVAL;
  const int g = log2i(nranks);
  if (g > bucket_bits || !offsets_local) return SLSUM_EINVAL;
  cudaStream_t st = as_stream(stream);
  const int lbits = bucket_bits - g;
  const uint64_t nbl = 1ull << lbits;
  if (global_counts) {
    counts_scan_kernel<<<1, kTPB, 0, st>>>(global_counts, (uint64_t)rank * nbl, nbl, offsets_local);
    MZS_LAUNCHED();
  }
  if (m_recv == 0) {
    if (!global_counts) MZS_CUDA(cudaMemsetAsync(offsets_local, 0, sizeof(uint64_t) * (nbl + 1), st));
    return SLSUM_OK;
  }
  if (!recv_fp || !recv_pos || !pos_out) return SLSUM_EINVAL;
  TempWs tmp;
  const size_t need = seedtable_finalize_workspace_bytes(m_recv, bucket_bits, nranks);
  if (!ws) {
    MZS_CUDA(cudaMallocAsync(&tmp.p, need, st));
    tmp.s = st;
    ws = tmp.p;
    ws_bytes = need;
  }
  if (ws_bytes < need) return SLSUM_ENOMEM;
  Carve c(ws, ws_bytes);
  const int npass = std::max(1, (lbits + 7) / 8);
  SortWs s;
  if (!carve_sort_ws(c, m_recv, npass, true, s)) return SLSUM_ENOMEM;
  uint32_t* fp_final = fp_out ? fp_out : s.fpF;
  const int lo = 32 - bucket_bits;
  const int hi = lbits > 0 ? 32 - g : lo + 1;  // lbits == 0: one bucket per owner; a 1-bit no-op pass
  int rc = stable_sort(false, recv_fp, recv_pos, nullptr, m_recv, 0, lo, hi, fp_final, pos_out, s, st);
  if (rc) return rc;
  if (!global_counts)
    return offsets_launch(fp_final, nullptr, m_recv, lo, (uint32_t)(nbl - 1), nbl, offsets_local, st);
  return SLSUM_OK;
}
