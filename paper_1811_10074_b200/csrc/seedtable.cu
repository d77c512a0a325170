// seedtable.cu -- seed pointer table + seed position table (Sec. 2.4, Fig. 1)
// for hashed minimizers, bucketed on the top `bits` bits of the 2k-bit key (R21).
//
// The build is a bucket histogram + a STABLE scatter into bucket order.  The scatter is
// done as an LSD radix sort on the bucket bits with 8-bit digits (one pass per digit,
// reduce-then-scan: per-chunk digit counts, a scan over chunks, then a stable ranked
// scatter; see the pass kernels below).  Stability makes the positions inside a bucket ascending (the input minimizer
// list is ascending by position), for any bucket-size distribution.  The pointer table
// is then read off the sorted fingerprints (first index of every bucket).
//
// Multi-GPU phases: count (histogram for the all-reduce), partition (one stable pass on
// the owner digit), finalize (stable passes on the remaining bucket bits of the owner).
#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "tma.cuh"

namespace mzs {
namespace {

#ifndef MZS_RANK_SYNCWARP
#define MZS_RANK_SYNCWARP 1
#endif
#ifndef MZS_RANK_BALLOT
#define MZS_RANK_BALLOT 0
#endif
constexpr int kTPB = 256;
constexpr int kNW = kTPB / 32;

__device__ __forceinline__ uint32_t fingerprint(uint64_t key, int k) {
  const int b = 2 * k;
  return b >= 32 ? (uint32_t)(key >> (b - 32)) : (uint32_t)(key << (32 - b));
}

__device__ __forceinline__ uint64_t count_of(const uint64_t* d_m, uint64_t m) { return d_m ? *d_m : m; }

// min(*d_m, m_cap), read ONCE per block (a per-thread read of one word from every SM is an
// L2 hot spot).  Must be called by all threads of the block.
__device__ __forceinline__ uint64_t block_count(const uint64_t* d_m, uint64_t m_cap) {
  __shared__ uint64_t s_m;
  if (threadIdx.x == 0) s_m = min(count_of(d_m, m_cap), m_cap);
  __syncthreads();
  return s_m;
}

// ---------------------------------------------------------------- stable LSD radix pass
// Reduce-then-scan (no serial look-back chains): the m entries are cut into chunks of
// kChunk; (U) counts per (digit, chunk); (S) exclusive scan over chunks per digit, then
// over digits; (D) every chunk re-reads its entries tile by tile, ranks them stably
// (per-warp peer bit tables + per-warp counters, nsweep_kernel), stages them in digit order
// in shared memory and writes each digit run contiguously.
constexpr int kStages = 2;                  // TMA ring depth (sub-tiles in flight per CTA)
constexpr int kChunk = kRadixChunkMax;      // entries per chunk (at most; see chunk_for)
constexpr int kMinChunk = kRadixChunkMin;   // and at least: whole tiles of every kernel

// Path gate: the narrow (packed u64) and wide (u32 fp + u64 pos) passes are both enqueued;
// each kernel runs only if ctl[0] selects its path (ctl == nullptr: always run).  ctl[0] is
// only changed by the first narrow downsweep, never while a gated kernel is running.
__device__ __forceinline__ bool gate_off(const uint64_t* ctl, int want) {
  return ctl != nullptr && ld_volatile_u64(ctl) != (uint64_t)want;
}

// IN: 0 = u64 hashes (fingerprint taken here), 1 = u32 fingerprints, 2 = packed u64 items
// (fingerprint in the high half).
template <int IN>
__device__ __forceinline__ uint32_t load_key(const void* keys, uint64_t i, int k) {
  if (IN == 0) return fingerprint(static_cast<const uint64_t*>(keys)[i], k);
  if (IN == 1) return static_cast<const uint32_t*>(keys)[i];
  return (uint32_t)(static_cast<const uint64_t*>(keys)[i] >> 32);
}

template <int IN>
__global__ void __launch_bounds__(kTPB) upsweep_kernel(const void* keys, const uint64_t* d_m, uint64_t m_cap, int k,
                                                       int shift, int dbits, uint32_t* counts, uint64_t nchunks,
                                                       const uint64_t* ctl, int want, uint32_t chunk) {
  if (gate_off(ctl, want)) return;
  __shared__ uint32_t h[kNW][256];
  const unsigned lane = lane_id(), wid = warp_id();
  const uint64_t m = block_count(d_m, m_cap);
  const uint32_t dmask = (1u << dbits) - 1u;
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {  // grid-stride over chunks
    for (int i = lane; i < 256; i += 32) h[wid][i] = 0;
    __syncthreads();
    const uint64_t base = c * (uint64_t)chunk;
    const uint64_t end = min(m, base + chunk);
    {
      uint64_t i = base + threadIdx.x;
      for (; i + 3 * kTPB < end; i += 4 * kTPB) {  // 4 loads in flight per thread
        uint32_t f[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) f[u] = load_key<IN>(keys, i + u * kTPB, k);
#pragma unroll
        for (int u = 0; u < 4; ++u) atomicAdd(&h[wid][(f[u] >> shift) & dmask], 1u);
      }
      for (; i < end; i += kTPB) atomicAdd(&h[wid][(load_key<IN>(keys, i, k) >> shift) & dmask], 1u);
    }
    __syncthreads();
    const uint32_t d = threadIdx.x;
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < kNW; ++w) t += h[w][d];
    counts[(uint64_t)d * nchunks + c] = t;
    __syncthreads();
  }
}

// block d: offsets[d][c] = exclusive scan over chunks; totals[d] = digit total
__global__ void __launch_bounds__(kTPB) chunk_scan_kernel(const uint32_t* counts, uint64_t nchunks,
                                                          uint64_t* offsets, unsigned long long* totals,
                                                          const uint64_t* ctl, int want) {
  if (gate_off(ctl, want)) return;
  __shared__ unsigned long long ws[kNW];
  const uint64_t d = blockIdx.x;
  const uint32_t* cn = counts + d * nchunks;
  uint64_t* of = offsets + d * nchunks;
  const uint64_t per = (nchunks + kTPB - 1) / kTPB;
  const uint64_t c0 = threadIdx.x * per, c1 = min(nchunks, c0 + per);
  unsigned long long s = 0;
  for (uint64_t c = c0; c < c1; ++c) s += cn[c];
  unsigned long long tot;
  unsigned long long ex = block_exclusive_sum<kTPB, unsigned long long>(s, ws, &tot);
  for (uint64_t c = c0; c < c1; ++c) {
    of[c] = ex;
    ex += cn[c];
  }
  if (threadIdx.x == 0) totals[d] = tot;
}

// exclusive scan of the 256 digit totals (one block of 256 threads)
__global__ void digit_scan_kernel(const unsigned long long* totals, unsigned long long* base, const uint64_t* ctl,
                                  int want) {
  if (gate_off(ctl, want)) return;
  __shared__ unsigned long long ws[kNW];
  unsigned long long tot;
  base[threadIdx.x] = block_exclusive_sum<256, unsigned long long>(totals[threadIdx.x], ws, &tot);
}



// Optional per-phase cycle counters of the narrow downsweep (build with -DMZS_PROF; read via
// seedtable_prof_read).  Thread 0 of every CTA adds each phase's clock64 delta.
#ifdef MZS_PROF
__device__ unsigned long long g_prof[8];
#define MZS_PROF_DECL() long long prof_t = clock64()
#define MZS_PROF_MARK(i)                                                  \
  do {                                                                    \
    if (threadIdx.x == 0) {                                               \
      const long long now_ = clock64();                                   \
      if ((i) > 0) atomicAdd(&g_prof[(i) - 1], (unsigned long long)(now_ - prof_t)); \
      prof_t = now_;                                                      \
    }                                                                     \
  } while (0)
#else
#define MZS_PROF_DECL() (void)0
#define MZS_PROF_MARK(i) (void)0
#endif

// ---------------------------------------------------------------- narrow passes (packed items)
// When every position of the call lies in [pos0, pos0 + 2^32), pos0 = pos[0] (one
// mz_extract_ex call on < 2^32 bases always qualifies), an entry travels between passes as
// ONE u64 item = (fp << 32) | (pos mod 2^32): 8 B per entry per pass instead of 12, one load
// and one store; the last pass restores pos = pos0 + ((lo - pos0) mod 2^32), exact because
// pos - pos0 < 2^32 (so items written elsewhere, e.g. by mz_extract_ex, need no common base).  ctl_kernel makes the decision from pos[0] and pos[m-1]; the first narrow
// downsweep re-checks every entry and, on any violation (unsorted input), switches ctl[0]
// to the wide path, whose kernels are enqueued behind it and then redo the sort.
//
// Ranking (per-pass cost floor on B200, tools/microbench_rank.cu): a bitwise ballot
// multi-split gives each item its peers (same digit) among the 32 items of a warp step;
// the lowest peer adds the peer count to the warp's counter with one shared atomic and
// broadcasts the old value (no __syncwarp round trips, no MATCH.ANY, which runs at half
// the rate of 8 ballots on sm_100).  Items are numbered warp-major, so rank order = input
// order (stable).  Writes go out per digit run from a digit-sorted staging copy; partial
// 32 B sectors at run edges are merged in L2 (tools/microbench_radix.cu: DRAM writes stay
// at the algorithmic bytes for runs >= 4 items).
enum { kInHashPos = 0, kInFpPos = 1, kInPk = 2 };
enum { kOutPk = 0, kOutFpPos = 1, kOutFpPos32 = 2 };  // kOutFpPos32: positions mod 2^32 (u32)
// items ranked per round of __syncwarp (their shared-memory round trips overlap): 4 for big
// tiles, 2 where the smaller footprint lets a third CTA fit on the SM
template <int TPB, int IPT> constexpr int peer_tables() { return TPB >= 512 ? 1 : (IPT >= 16 ? 4 : 2); }

__global__ void ctl_kernel(const uint64_t* pos, const uint64_t* d_m, uint64_t m_cap, uint64_t* ctl) {
  if (threadIdx.x != 0) return;
  const uint64_t m = min(count_of(d_m, m_cap), m_cap);
  uint64_t narrow = 1, p0 = 0;
  if (m) {
    p0 = pos[0];
    const uint64_t p1 = pos[m - 1];
    narrow = (p1 >= p0 && p1 - p0 <= 0xffffffffull) ? 1 : 0;
  }
  ctl[0] = narrow;
  ctl[1] = p0;
}

template <int IN> struct NInA { using T = uint64_t; };
template <> struct NInA<kInFpPos> { using T = uint32_t; };

template <int IN, int T> struct NIn;
template <int T> struct NIn<kInHashPos, T> { uint64_t a[T]; uint64_t p[T]; };
template <int T> struct NIn<kInFpPos, T> { uint32_t a[T]; uint64_t p[T]; };
template <int T> struct NIn<kInPk, T> { uint64_t a[T]; };

template <int IN, int T>
__device__ __forceinline__ uint64_t* stage_of(NIn<IN, T>& r) {
  if constexpr (IN == kInPk) return r.a;
  else return r.p;
}

template <int IN, int TPB, int T>
struct NSmem {
  static constexpr int NW = TPB / 32;
  NIn<IN, T> ring[kStages];
  uint64_t mbar[kStages];
  uint64_t run_off[256];     // next output index of digit d (global)
  uint64_t gbase[256];       // staged entry j of digit d goes to gbase[d] + j
  uint32_t wcnt[NW][256];    // per-warp digit counters -> per-warp exclusive offsets
  uint32_t dummy[NW][32];    // atomic targets of non-leader lanes (branch-free ranking)
  uint32_t pm[NW][MZS_RANK_BALLOT ? 1 : peer_tables<TPB, T / TPB>()][MZS_RANK_BALLOT ? 1 : 256];  // per-warp peer bit tables
  uint32_t ws2[NW > 8 ? NW : 8];  // per-warp digit-scan totals
};

template <int IN, int T>
__device__ __forceinline__ uint64_t make_item(const NIn<IN, T>& r, uint32_t j, int k, uint64_t p0, bool& bad) {
  if constexpr (IN == kInPk) {
    return r.a[j];
  } else {
    uint32_t f;
    if constexpr (IN == kInHashPos) f = fingerprint(r.a[j], k);
    else f = r.a[j];
    const uint64_t pj = r.p[j];
    bad |= ((pj - p0) >> 32) != 0;
    return ((uint64_t)f << 32) | (uint32_t)pj;  // the low 32 bits of the position (see put)
  }
}


template <int IN, int OUT, int TPB, int IPT, bool WD = false>
__global__ void __launch_bounds__(TPB) nsweep_kernel(const void* a_in, const uint64_t* __restrict__ p_in,
                                                       void* a_out, uint64_t* __restrict__ p_out, const uint64_t* d_m,
                                                       uint64_t m_cap, int k, int shift, int dbits,
                                                       const uint64_t* __restrict__ offsets,
                                                       const unsigned long long* __restrict__ dbase, uint64_t nchunks,
                                                       uint64_t* ctl, int use_tma, uint32_t chunk, int gate,
                                                       uint32_t* const* __restrict__ dfp = nullptr,
                                                       uint64_t* const* __restrict__ dpos = nullptr) {
  // dfp/dpos (OUT == kOutFpPos only): per-digit destination arrays, e.g. the peer-mapped receive
  // buffers of the owner ranks (seedtable_partition_p2p); digit d's entries go to dfp[d][g]
  constexpr int T = TPB * IPT;
  constexpr int NW = TPB / 32;
  static_assert(kChunk % T == 0 && kMinChunk % T == 0, "chunks hold whole tiles");
  // WD: the wide path (positions spanning >= 2^32, or unsorted): an entry stays (fp, full
  // position) in registers -- `item` carries fp in its high word for the ranking, `ipos` the
  // position -- and is staged as two arrays (fp over the ring's key array, positions over
  // its position array), written as u32 fp + u64 position
  static_assert(!WD || (IN != kInPk && OUT == kOutFpPos), "wide passes read and write fp + pos");
  static_assert(TPB >= 256, "digit threads");
  using SM = NSmem<IN, TPB, T>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SM& S = *reinterpret_cast<SM*>(smem_raw);
  __shared__ uint64_t s_m, s_p0;
  __shared__ int s_go;
  const uint32_t td = threadIdx.x;
  if (td == 0) {
    s_go = ld_volatile_u64(ctl) == (uint64_t)gate;  // 1: packed items, 0: WD (the wide path)
    s_m = min(count_of(d_m, m_cap), m_cap);
    s_p0 = ctl[1];
  }
  __syncthreads();
  if (!s_go) return;
  const uint64_t m = s_m, p0 = s_p0;
  const unsigned lane = lane_id(), wid = warp_id(), lt = (1u << lane) - 1u;
  const uint32_t dmask = (1u << dbits) - 1u;
  const int dsh = 32 + shift;
  const uint64_t c = blockIdx.x, cbase = c * (uint64_t)chunk;
  if (cbase >= m) return;
  if (td < 256) S.run_off[td] = dbase[td] + offsets[(uint64_t)td * nchunks + c];
  for (uint32_t i = td; i < NW * 256; i += TPB) (&S.wcnt[0][0])[i] = 0;
  constexpr int kPeerTables = peer_tables<TPB, IPT>();
  if (!MZS_RANK_BALLOT)
    for (uint32_t i = td; i < NW * kPeerTables * 256; i += TPB) (&S.pm[0][0][0])[i] = 0;
  if (td == 0) {
    for (int b = 0; b < kStages; ++b) mbar_init(&S.mbar[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int nsubs = (int)min((uint64_t)(chunk / T), (m - cbase + T - 1) / T);
  auto tma_ok = [&](int sub) { return use_tma && cbase + (uint64_t)(sub + 1) * T <= m; };
  auto issue = [&](int sub) {
    if (td == 0 && sub < nsubs && tma_ok(sub)) {
      const int b = sub % kStages;
      const uint64_t base = cbase + (uint64_t)sub * T;
      constexpr uint32_t abytes = sizeof(S.ring[0].a);
      if constexpr (IN == kInPk) {
        mbar_arrive_expect_tx(&S.mbar[b], abytes);
        bulk_g2s(S.ring[b].a, static_cast<const uint64_t*>(a_in) + base, abytes, &S.mbar[b]);
      } else {
        constexpr uint32_t pbytes = sizeof(S.ring[0].p);
        mbar_arrive_expect_tx(&S.mbar[b], abytes + pbytes);
        bulk_g2s(S.ring[b].a, static_cast<const typename NInA<IN>::T*>(a_in) + base, abytes, &S.mbar[b]);
        bulk_g2s(S.ring[b].p, p_in + base, pbytes, &S.mbar[b]);
      }
    }
  };
  for (int p = 0; p < kStages - 1; ++p) issue(p);
  uint32_t parity = 0;
  bool bad = false;
  MZS_PROF_DECL();
  for (int sub = 0; sub < nsubs; ++sub) {
    const int b = sub % kStages;
    const uint64_t base = cbase + (uint64_t)sub * T;
    const uint32_t nvalid = (uint32_t)min((uint64_t)T, m - base);
    MZS_PROF_MARK(0);
    issue(sub + kStages - 1);
    if (tma_ok(sub)) {
      mbar_wait(&S.mbar[b], (parity >> b) & 1u);
      parity ^= 1u << b;
    } else {
      for (uint32_t j = td; j < (uint32_t)T; j += TPB) {
        const bool v = j < nvalid;
        if constexpr (IN == kInPk) {
          S.ring[b].a[j] = v ? static_cast<const uint64_t*>(a_in)[base + j] : 0ull;
        } else {
          S.ring[b].a[j] = v ? static_cast<const typename NInA<IN>::T*>(a_in)[base + j] : 0;
          S.ring[b].p[j] = v ? p_in[base + j] : p0;
        }
      }
      __syncthreads();
    }
    MZS_PROF_MARK(1);
    // ---- stable rank of every item within its digit (warp-major item order)
    uint64_t item[IPT];
    uint64_t ipos[WD ? IPT : 1];
    uint32_t rank[IPT];
    auto rank_tile = [&](auto whole_tag) {
      constexpr bool kWhole = decltype(whole_tag)::value;
      // Peers (lanes with the same digit) through per-warp shared bit tables: every lane ORs
      // its lane bit into pm[u][d], and after a __syncwarp reads its digit's word; after a
      // second __syncwarp it XORs its bit back out.  Each lane only flips its own bit, so the
      // atomics of different lanes commute.  kPeerTables items share one round of syncwarps
      // (one table each), so their shared-memory round trips overlap.  ~20 SASS per item
      // instead of ~60 for an 8-ballot multi-split (tools/microbench_rank.cu).
      unsigned peers[IPT];
#if MZS_RANK_BALLOT
#pragma unroll
      for (int it = 0; it < IPT; ++it) {
        const uint32_t j = wid * (IPT * 32) + it * 32 + lane;
        if constexpr (WD) {
          uint32_t f;
          if constexpr (IN == kInHashPos) f = fingerprint(S.ring[b].a[j], k);
          else f = S.ring[b].a[j];
          item[it] = (uint64_t)f << 32;
          ipos[it] = S.ring[b].p[j];
        } else {
          item[it] = make_item<IN, T>(S.ring[b], j, k, p0, bad);
        }
        const bool valid = kWhole || j < nvalid;
        const uint32_t d = (uint32_t)(item[it] >> dsh) & dmask;
        unsigned p = kWhole ? 0xffffffffu : __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) {
          const bool bit = (d >> bb) & 1u;
          const unsigned mm = __ballot_sync(0xffffffffu, bit);
          p &= bit ? mm : ~mm;
        }
        peers[it] = valid ? p : (1u << lane);
      }
#else
      uint32_t (*pm)[256] = S.pm[wid];
#pragma unroll
      for (int g = 0; g < IPT; g += kPeerTables) {
#pragma unroll
        for (int u = 0; u < kPeerTables; ++u) {
          const int it = g + u;
          const uint32_t j = wid * (IPT * 32) + it * 32 + lane;
          if constexpr (WD) {
            uint32_t f;
            if constexpr (IN == kInHashPos) f = fingerprint(S.ring[b].a[j], k);
            else f = S.ring[b].a[j];
            item[it] = (uint64_t)f << 32;
            ipos[it] = S.ring[b].p[j];
          } else {
            item[it] = make_item<IN, T>(S.ring[b], j, k, p0, bad);
          }
          if (kWhole || j < nvalid) atomicOr(&pm[u][(uint32_t)(item[it] >> dsh) & dmask], 1u << lane);
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kPeerTables; ++u) {
          const int it = g + u;
          const bool valid = kWhole || wid * (IPT * 32) + it * 32 + lane < nvalid;
          peers[it] = valid ? pm[u][(uint32_t)(item[it] >> dsh) & dmask] : (1u << lane);
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < kPeerTables; ++u) {
          const int it = g + u;
          if (kWhole || wid * (IPT * 32) + it * 32 + lane < nvalid)
            atomicXor(&pm[u][(uint32_t)(item[it] >> dsh) & dmask], 1u << lane);
        }
      }
#endif
      // per-warp digit counters, in item order: the lowest peer adds the peer count (every
      // other lane adds 0 to its own dummy word, so there is no branch); the old value is
      // broadcast to the peers.  The leaders of one digit in two item rounds can be different
      // lanes; MZS_RANK_SYNCWARP puts a __syncwarp between the rounds so that their atomics
      // are ordered by the memory model, not only by the warp's in-order issue.
      uint32_t old[IPT];
#pragma unroll
      for (int it = 0; it < IPT; ++it) {
        const bool valid = kWhole || wid * (IPT * 32) + it * 32 + lane < nvalid;
        const bool lead = valid && (peers[it] & lt) == 0u;
        uint32_t* tgt = lead ? &S.wcnt[wid][(uint32_t)(item[it] >> dsh) & dmask] : &S.dummy[wid][lane];
        old[it] = atomicAdd(tgt, lead ? (uint32_t)__popc(peers[it]) : 0u);
#if MZS_RANK_SYNCWARP
        if (it + 1 < IPT) __syncwarp();
#endif
      }
#pragma unroll
      for (int it = 0; it < IPT; ++it) {
        const bool valid = kWhole || wid * (IPT * 32) + it * 32 + lane < nvalid;
        const uint32_t o = __shfl_sync(0xffffffffu, old[it], __ffs(peers[it]) - 1);
        rank[it] = valid ? o + __popc(peers[it] & lt) : 0xffffffffu;
      }
    };
    if (nvalid == (uint32_t)T) rank_tile(std::true_type{});
    else rank_tile(std::false_type{});
    __syncthreads();
    MZS_PROF_MARK(2);
    // ---- offsets: digit totals over warps, block scan over digits, then every (warp, digit)
    // counter becomes its staging base (digit start + earlier warps' count)
    uint32_t cnt[NW];
    uint32_t run = 0;
    if (td < 256) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        cnt[w] = S.wcnt[w][td];
        run += cnt[w];
      }
    }
    // exclusive scan of the 256 digit totals with one barrier: warps 0..7 own 32 digits each
    uint32_t incl = run;
    if (td < 256) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
      }
      if (lane == 31) S.ws2[wid] = incl;
    }
    __syncthreads();
    if (td < 256) {
      uint32_t ex = incl - run;
#pragma unroll
      for (int v = 0; v < 8; ++v)
        if (v < (int)wid) ex += S.ws2[v];
      uint32_t acc = ex;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        S.wcnt[w][td] = acc;
        acc += cnt[w];
      }
      const uint64_t r0 = S.run_off[td];
      S.gbase[td] = r0 - ex;
      S.run_off[td] = r0 + run;
    }
    __syncthreads();
    MZS_PROF_MARK(3);
    // ---- stage in digit order (in place: every item of this tile is in registers)
    uint64_t* stage = stage_of<IN, T>(S.ring[b]);
    uint32_t* stage_f = reinterpret_cast<uint32_t*>(S.ring[b].a);  // (WD) fingerprints
    const uint32_t* wrow = S.wcnt[wid];
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
      if (rank[it] != 0xffffffffu) {
        const uint32_t sl = wrow[(uint32_t)(item[it] >> dsh) & dmask] + rank[it];
        MZS_DCHECK(sl < nvalid);
        if constexpr (WD) {
          stage_f[sl] = (uint32_t)(item[it] >> 32);
          stage[sl] = ipos[WD ? it : 0];
        } else {
          stage[sl] = item[it];
        }
      }
    }
    __syncthreads();
    for (uint32_t i = lane; i < 256; i += 32) S.wcnt[wid][i] = 0;  // own row: read only by this warp above
    MZS_PROF_MARK(4);
    // ---- write every digit run contiguously
    auto put = [&](uint32_t j) {
      if constexpr (WD) {
        const uint32_t f = stage_f[j];
        const uint64_t g = S.gbase[(f >> shift) & dmask] + j;
        static_cast<uint32_t*>(a_out)[g] = f;
        p_out[g] = stage[j];
        return;
      }
      const uint64_t v = stage[j];
      const uint64_t g = S.gbase[(uint32_t)(v >> dsh) & dmask] + j;
      MZS_DCHECK(dfp != nullptr || g < m);
      if constexpr (OUT == kOutPk) {
        static_cast<uint64_t*>(a_out)[g] = v;
      } else if constexpr (OUT == kOutFpPos32) {
        static_cast<uint32_t*>(a_out)[g] = (uint32_t)(v >> 32);
        reinterpret_cast<uint32_t*>(p_out)[g] = (uint32_t)v;  // the item carries pos mod 2^32
      } else if (dfp) {
        const uint32_t d = (uint32_t)(v >> dsh) & dmask;
        dfp[d][g] = (uint32_t)(v >> 32);  // a plain store: over NVLink when the buffer is a peer's
        dpos[d][g] = p0 + (uint32_t)((uint32_t)v - (uint32_t)p0);
      } else {
        static_cast<uint32_t*>(a_out)[g] = (uint32_t)(v >> 32);
        // the item holds pos mod 2^32; pos - p0 < 2^32 (the narrow precondition), so
        // pos = p0 + ((pos - p0) mod 2^32)
        p_out[g] = p0 + (uint32_t)((uint32_t)v - (uint32_t)p0);
      }
    };
    if (nvalid == (uint32_t)T) {
#pragma unroll
      for (int it = 0; it < IPT; ++it) put(td + it * TPB);
    } else {
      for (uint32_t j = td; j < nvalid; j += TPB) put(j);
    }
    fence_proxy_async();  // ring slot b is refilled by TMA in a later iteration
    __syncthreads();
    MZS_PROF_MARK(5);
  }
  if constexpr (IN != kInPk && !WD) {
    if (__syncthreads_or(bad) && td == 0) st_volatile_u64(ctl, 0);  // precondition broken: wide path redoes it
  }
}

template <int IN, int TPB, int IPT>
size_t nsweep_smem() { return sizeof(NSmem<IN, TPB, TPB * IPT>); }

// Pointer table from the bucket-sorted fingerprints, in three data-parallel steps (bucket
// sizes are very uneven: minimizer hashes are window minima, so high buckets are mostly
// empty and a "fill every empty bucket you see" loop serialises on a few threads):
//   1. offsets[*] = UINT64_MAX (memset); offsets[nb] = m
//   2. boundary scatter: offsets[bucket(i)] = i wherever bucket(i) != bucket(i-1)
//   3. suffix minimum over offsets[0..nb]: an empty bucket takes the start of the next
//      non-empty one.
// bucket(f) = (f >> shift) & bmask.
__global__ void __launch_bounds__(kTPB) offsets_scatter_kernel(const uint32_t* __restrict__ fp, const uint64_t* d_m,
                                                               uint64_t m_cap, int shift, uint32_t bmask, uint64_t nb,
                                                               uint64_t* __restrict__ offsets) {
  const uint64_t m = block_count(d_m, m_cap);
  const bool aligned = (reinterpret_cast<uintptr_t>(fp) & 15) == 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) offsets[nb] = m;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t * 16 < m;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = t * 16;
    uint32_t prev = i0 == 0 ? 0xffffffffu : ((fp[i0 - 1] >> shift) & bmask);
    uint32_t f[16];
    if (aligned && i0 + 16 <= m) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(fp + i0 + 4 * q);
        f[4 * q] = v.x; f[4 * q + 1] = v.y; f[4 * q + 2] = v.z; f[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) f[j] = i0 + j < m ? fp[i0 + j] : 0u;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (i0 + j >= m) break;
      const uint32_t cur = (f[j] >> shift) & bmask;
      if (cur != prev) offsets[cur] = i0 + j;
      prev = cur;
    }
  }
}

constexpr int kSminTile = kTPB * 16;  // 4096 entries per suffix-min tile

// per-tile minimum of offsets[] (tile t covers [t*4096, (t+1)*4096) of [0, n))
__global__ void __launch_bounds__(kTPB) smin_reduce_kernel(const uint64_t* __restrict__ v, uint64_t n,
                                                           uint64_t* __restrict__ tile_min) {
  __shared__ uint64_t ws[kNW];
  const uint64_t b0 = (uint64_t)blockIdx.x * kSminTile;
  uint64_t mn = ~0ull;
  for (uint64_t i = b0 + threadIdx.x; i < min(n, b0 + (uint64_t)kSminTile); i += kTPB) mn = min(mn, v[i]);
  for (int o = 16; o > 0; o >>= 1) mn = min(mn, (uint64_t)__shfl_xor_sync(0xffffffffu, mn, o));
  if (lane_id() == 0) ws[warp_id()] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t r = ~0ull;
    for (int w = 0; w < kNW; ++w) r = min(r, ws[w]);
    tile_min[blockIdx.x] = r;
  }
}

// suffix minimum of the per-tile minima (one block; a few thousand tiles): tile_min[t] <-
// min over tiles > t (the carry entering tile t from the right)
__global__ void __launch_bounds__(kTPB) smin_tiles_kernel(uint64_t* tile_min, uint64_t ntiles) {
  __shared__ uint64_t carry_s;
  __shared__ uint64_t buf[kTPB];
  if (threadIdx.x == 0) carry_s = ~0ull;
  __syncthreads();
  // process from the right in blocks of kTPB tiles
  for (int64_t hi = (int64_t)ntiles; hi > 0; hi -= kTPB) {
    const int64_t lo = max((int64_t)0, hi - kTPB);
    const int64_t i = lo + threadIdx.x;
    uint64_t x = i < hi ? tile_min[i] : ~0ull;
    buf[threadIdx.x] = x;
    __syncthreads();
    // inclusive suffix min within the block (Hillis-Steele, right to left)
    for (int o = 1; o < kTPB; o <<= 1) {
      const uint64_t y = threadIdx.x + o < kTPB ? buf[threadIdx.x + o] : ~0ull;
      __syncthreads();
      buf[threadIdx.x] = min(buf[threadIdx.x], y);
      __syncthreads();
    }
    const uint64_t carry = carry_s;
    const uint64_t excl = min((uint64_t)(threadIdx.x + 1 < kTPB ? buf[threadIdx.x + 1] : ~0ull), carry);
    __syncthreads();
    if (i < hi) tile_min[i] = excl;
    if (threadIdx.x == 0) carry_s = min(carry, buf[0]);
    __syncthreads();
  }
}

// offsets[i] <- min(offsets[i..end of tile], carry of the tile): serial per thread chunk of 16,
// then a right-to-left warp/block scan
__global__ void __launch_bounds__(kTPB) smin_apply_kernel(uint64_t* __restrict__ v, uint64_t n,
                                                          const uint64_t* __restrict__ tile_carry) {
  __shared__ uint64_t ws[kNW];
  const uint64_t b0 = (uint64_t)blockIdx.x * kSminTile + (uint64_t)threadIdx.x * 16;
  uint64_t x[16];
  const bool vec = b0 + 16 <= n && (reinterpret_cast<uintptr_t>(v) & 15) == 0;  // 16-byte accesses
  if (vec) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(v + b0 + j);
      x[j] = p.x;
      x[j + 1] = p.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = b0 + j < n ? v[b0 + j] : ~0ull;
  }
#pragma unroll
  for (int j = 14; j >= 0; --j) x[j] = min(x[j], x[j + 1]);
  // carry from threads to the right (their chunk minima), nearest first
  uint64_t c = x[0];
  const unsigned lane = lane_id(), wid = warp_id();
  uint64_t inc = c;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_down_sync(0xffffffffu, inc, o);
    if (lane + o < 32) inc = min(inc, y);
  }
  uint64_t right = __shfl_down_sync(0xffffffffu, inc, 1);
  if (lane == 31) right = ~0ull;
  if (lane == 0) ws[wid] = inc;
  __syncthreads();
  uint64_t wr = ~0ull;
  for (int w = wid + 1; w < kNW; ++w) wr = min(wr, ws[w]);
  const uint64_t carry = min(min(right, wr), tile_carry[blockIdx.x]);
  if (vec) {
#pragma unroll
    for (int j = 0; j < 16; j += 2)
      *reinterpret_cast<ulonglong2*>(v + b0 + j) = make_ulonglong2(min(x[j], carry), min(x[j + 1], carry));
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (b0 + j < n) v[b0 + j] = min(x[j], carry);
  }
}

// counts[bucket] += 1 (global atomics; the 2^bits counters stay L2-resident)
__global__ void __launch_bounds__(kTPB) count_kernel(const uint64_t* __restrict__ hash, const uint64_t* d_m,
                                                     uint64_t m_cap, int k, int bits, uint32_t* counts) {
  const uint64_t m = block_count(d_m, m_cap);
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

// (wide path, 32-bit position table) positions mod 2^32 from the wide path's u64 table; runs
// only when ctl[0] selects the wide path
__global__ void __launch_bounds__(kTPB) pos_to_u32_kernel(const uint64_t* __restrict__ p64, const uint64_t* d_m,
                                                          uint64_t m_cap, uint32_t* __restrict__ p32,
                                                          const uint64_t* ctl) {
  if (gate_off(ctl, 0)) return;
  const uint64_t m = block_count(d_m, m_cap);
  for (uint64_t i = (uint64_t)blockIdx.x * kTPB + threadIdx.x; i < m; i += (uint64_t)gridDim.x * kTPB)
    p32[i] = (uint32_t)p64[i];
}

// identity partition (one rank): fingerprints + positions in input order, count = m
__global__ void fp_copy_kernel(const uint64_t* __restrict__ hash, const uint64_t* __restrict__ pos, const uint64_t* d_m,
                               uint64_t m_cap, int k, uint32_t* __restrict__ fp, uint64_t* __restrict__ pos_out,
                               uint64_t* send_counts) {
  const uint64_t m = block_count(d_m, m_cap);
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
  uint32_t chunk;             // entries per chunk (chunk_for(m))
  uint32_t* counts;           // [256 * nchunks]
  uint64_t* offs;             // [256 * nchunks]
  unsigned long long* totals; // [256]
  unsigned long long* dbase;  // [256]
  uint64_t* ctl;              // [2]: path (1 narrow, 0 wide), pos0
  uint32_t* fpA;
  uint64_t* posA;             // also the narrow path's packed items (A)
  uint32_t* fpB;
  uint64_t* posB;             // also the narrow path's packed items (B)
  uint32_t* fpF;              // final fingerprints when the caller gave none
  uint64_t* posW;             // (32-bit position table) the wide path's u64 positions
};

// Chunk size: kChunk entries, but small inputs take smaller chunks (a multiple of 4096) so that
// about 296 CTAs (2 per SM) share the passes instead of a handful working through 128K
// entries each (C1's 1.9e5 entries were 2 chunks).  A function of m only (no device query), so
// the workspace size and the carve agree.
uint32_t chunk_for(uint64_t m) { return radix_chunk_for(m); }
uint64_t chunks_for(uint64_t m) { return (m + chunk_for(m) - 1) / chunk_for(m) + 1; }

template <class C>
void size_sort_ws(C& c, uint64_t m, int npass, bool need_fp) {
  c.template take<uint32_t>(256 * chunks_for(m));
  c.template take<uint64_t>(256 * chunks_for(m));
  c.template take<unsigned long long>(256);
  c.template take<unsigned long long>(256);
  c.template take<uint64_t>(2);
  if (npass >= 2) {
    c.template take<uint32_t>(m + 1);
    c.template take<uint64_t>(m + 1);
  }
  if (npass >= 3) {
    c.template take<uint32_t>(m + 1);
    c.template take<uint64_t>(m + 1);
  }
  if (need_fp) c.template take<uint32_t>(m + 1);
  if (npass != 3) c.template take<uint64_t>(m + 1);  // posW (with 3 passes the A buffer is free)
}

bool carve_sort_ws(Carve& c, uint64_t m, int npass, bool need_fp, SortWs& s) {
  s = SortWs{};
  s.chunk = chunk_for(m);
  s.counts = c.take<uint32_t>(256 * chunks_for(m));
  s.offs = c.take<uint64_t>(256 * chunks_for(m));
  s.totals = c.take<unsigned long long>(256);
  s.dbase = c.take<unsigned long long>(256);
  s.ctl = c.take<uint64_t>(2);
  if (npass >= 2) { s.fpA = c.take<uint32_t>(m + 1); s.posA = c.take<uint64_t>(m + 1); }
  if (npass >= 3) { s.fpB = c.take<uint32_t>(m + 1); s.posB = c.take<uint64_t>(m + 1); }
  if (need_fp) s.fpF = c.take<uint32_t>(m + 1);
  s.posW = npass != 3 ? c.take<uint64_t>(m + 1) : s.posA;
  return c.ok;
}

int grid_stride_blocks(uint64_t m) {
  const uint64_t want = (m + kTPB - 1) / kTPB;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  return (int)std::max<uint64_t>(1, std::min(want, cap));
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// One reduce-then-scan pass: upsweep (digit counts per chunk) + chunk scan + digit scan.
// counts_in: the pass's digit counts computed elsewhere (mz_extract_ex's fused histogram,
// mz_out.hist), in the upsweep's layout; the upsweep is then skipped.
template <int IN>
int count_pass(const void* kin, const uint64_t* d_m, uint64_t m, int k, int sh, int nb, uint64_t nch, SortWs& s,
               int want, cudaStream_t st, const uint32_t* counts_in = nullptr) {
  if (!counts_in) {
    const unsigned grid = (unsigned)std::min<uint64_t>(nch, (uint64_t)num_sms() * 8);
    upsweep_kernel<IN><<<grid, kTPB, 0, st>>>(kin, d_m, m, k, sh, nb, s.counts, nch, s.ctl, want, s.chunk);
    MZS_LAUNCHED();
  }
  chunk_scan_kernel<<<256, kTPB, 0, st>>>(counts_in ? counts_in : s.counts, nch, s.offs, s.totals, s.ctl, want);
  MZS_LAUNCHED();
  digit_scan_kernel<<<1, 256, 0, st>>>(s.totals, s.dbase, s.ctl, want);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

template <int IN, int OUT, int TPB, int IPT, bool WD = false>
int launch_nsweep(const void* a_in, const uint64_t* p_in, void* a_out, uint64_t* p_out, const uint64_t* d_m,
                  uint64_t m, int k, int sh, int nb, uint64_t nch, SortWs& s, int use_tma, cudaStream_t st) {
  auto kern = nsweep_kernel<IN, OUT, TPB, IPT, WD>;
  const size_t sm = nsweep_smem<IN, TPB, IPT>();
  MZS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  kern<<<(unsigned)nch, TPB, sm, st>>>(a_in, p_in, a_out, p_out, d_m, m, k, sh, nb, s.offs, s.dbase, nch, s.ctl,
                                       use_tma, s.chunk, WD ? 0 : 1, nullptr, nullptr);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

// cfg = TPB * 100 + IPT (tuning knob): 51208, 51204, 25616, 25608
template <int IN, int OUT>
int launch_nsweep_cfg(int cfg, const void* a_in, const uint64_t* p_in, void* a_out, uint64_t* p_out,
                      const uint64_t* d_m, uint64_t m, int k, int sh, int nb, uint64_t nch, SortWs& s, int use_tma,
                      cudaStream_t st) {
  switch (cfg) {
    case 51204: return launch_nsweep<IN, OUT, 512, 4>(a_in, p_in, a_out, p_out, d_m, m, k, sh, nb, nch, s, use_tma, st);
    case 25616: return launch_nsweep<IN, OUT, 256, 16>(a_in, p_in, a_out, p_out, d_m, m, k, sh, nb, nch, s, use_tma, st);
    case 25608: return launch_nsweep<IN, OUT, 256, 8>(a_in, p_in, a_out, p_out, d_m, m, k, sh, nb, nch, s, use_tma, st);
    default: return launch_nsweep<IN, OUT, 512, 8>(a_in, p_in, a_out, p_out, d_m, m, k, sh, nb, nch, s, use_tma, st);
  }
}

// Stable LSD sort of m entries by fp bits [lo_bit, hi_bit) into (fp_dst, pos_dst); input is
// (u64 hashes | u32 fingerprints) + u64 positions.  Both paths are enqueued: the narrow one
// (packed u64 items, ctl[0] == 1) and the wide one (u32 + u64 entries, ctl[0] == 0); see
// ctl_kernel.  After the call s.totals holds the digit totals of the LAST pass.
int stable_sort(bool from_hash, const void* keys, const uint64_t* pos, const uint64_t* d_m, uint64_t m, int k,
                int lo_bit, int hi_bit, uint32_t* fp_dst, uint64_t* pos_dst, SortWs& s, cudaStream_t st,
                const uint64_t* items = nullptr, uint32_t* pos32_dst = nullptr, const uint32_t* hist0 = nullptr) {
  // hist0 (with items): the first narrow pass's digit counts, from mz_extract_ex (mz_out.hist)
  // pos32_dst (packed items only): the final positions as u32 (pos mod 2^32) instead of pos_dst
  const int npass = (hi_bit - lo_bit + 7) / 8;
  if (npass > 4 || npass < 1) return SLSUM_EINVAL;
  const uint64_t nch = (m + s.chunk - 1) / s.chunk;
  if (nch == 0) return SLSUM_OK;
  int rc;
  static const int force = env_int("MZS_RADIX_PATH", -1);  // tests/tuning: 0 forces the wide path
  static const int ipt_first = env_int("MZS_NCFG_FIRST", 25608);
  static const int ipt_pk = env_int("MZS_NCFG", 25616);
  ctl_kernel<<<1, 32, 0, st>>>(pos, d_m, m, s.ctl);
  MZS_LAUNCHED();
  if (force == 0) MZS_CUDA(cudaMemsetAsync(s.ctl, 0, sizeof(uint64_t), st));
  const int tma_in = ((reinterpret_cast<uintptr_t>(keys) | reinterpret_cast<uintptr_t>(pos)) & 15) == 0;
  if (pos32_dst && !items) return SLSUM_EINVAL;
  auto pass_out = [&](int p, uint64_t*& pk, uint32_t*& fo, uint64_t*& po) {
    if (p == npass - 1) { fo = fp_dst; po = pos32_dst ? reinterpret_cast<uint64_t*>(pos32_dst) : pos_dst; pk = nullptr; }
    else if (p % 2 == 0) { fo = s.fpA; po = s.posA; pk = s.posA; }
    else { fo = s.fpB; po = s.posB; pk = s.posB; }
  };
  // ---- narrow pass 0 (reads the caller's arrays; re-checks the precondition)
  {
    uint64_t* pk; uint32_t* fo; uint64_t* po;
    pass_out(0, pk, fo, po);
    const int nb = std::min(8, hi_bit - lo_bit);
    if (items) {
      // pre-packed items (mz_extract_ex's out->items, positions ascending): pass 0 is an
      // ordinary 8-byte item pass; the hash/pos arrays serve only the wide path
      rc = count_pass<2>(items, d_m, m, k, lo_bit, nb, nch, s, 1, st, hist0);
      if (rc) return rc;
      const int tma_it = (reinterpret_cast<uintptr_t>(items) & 15) == 0;
      rc = npass != 1 ? launch_nsweep_cfg<kInPk, kOutPk>(ipt_pk, items, nullptr, pk, nullptr, d_m, m, k, lo_bit, nb, nch, s, tma_it, st)
           : pos32_dst ? launch_nsweep<kInPk, kOutFpPos32, 256, 16>(items, nullptr, fo, po, d_m, m, k, lo_bit, nb, nch, s, tma_it, st)
                       : launch_nsweep_cfg<kInPk, kOutFpPos>(ipt_pk, items, nullptr, fo, po, d_m, m, k, lo_bit, nb, nch, s, tma_it, st);
      if (rc) return rc;
    } else {
    rc = from_hash ? count_pass<0>(keys, d_m, m, k, lo_bit, nb, nch, s, 1, st)
                   : count_pass<1>(keys, d_m, m, k, lo_bit, nb, nch, s, 1, st);
    if (rc) return rc;
    if (from_hash) {
      rc = npass == 1 ? launch_nsweep_cfg<kInHashPos, kOutFpPos>(ipt_first, keys, pos, fo, po, d_m, m, k, lo_bit, nb, nch, s, tma_in, st)
                      : launch_nsweep_cfg<kInHashPos, kOutPk>(ipt_first, keys, pos, pk, nullptr, d_m, m, k, lo_bit, nb, nch, s, tma_in, st);
    } else {
      rc = npass == 1 ? launch_nsweep_cfg<kInFpPos, kOutFpPos>(ipt_first, keys, pos, fo, po, d_m, m, k, lo_bit, nb, nch, s, tma_in, st)
                      : launch_nsweep_cfg<kInFpPos, kOutPk>(ipt_first, keys, pos, pk, nullptr, d_m, m, k, lo_bit, nb, nch, s, tma_in, st);
    }
    if (rc) return rc;
    }
  }
  // ---- wide path: every pass (gated off when the narrow path holds); the same ranking and
  // staging as the narrow passes with (u32 fp, u64 position) entries (nsweep_kernel WD)
  {
    const void* kin = keys;
    const uint64_t* pin = pos;
    bool kin_hash = from_hash;
    for (int p = 0; p < npass; ++p) {
      uint64_t* pk; uint32_t* fo; uint64_t* po;
      pass_out(p, pk, fo, po);
      if (pos32_dst && p == npass - 1) po = s.posW;  // u64 here, narrowed below
      const int sh = lo_bit + 8 * p;
      const int nb = std::min(8, hi_bit - sh);
      rc = kin_hash ? count_pass<0>(kin, d_m, m, k, sh, nb, nch, s, 0, st) : count_pass<1>(kin, d_m, m, k, sh, nb, nch, s, 0, st);
      if (rc) return rc;
      const int tma = p == 0 ? tma_in : 1;
      rc = kin_hash ? launch_nsweep<kInHashPos, kOutFpPos, 256, 8, true>(kin, pin, fo, po, d_m, m, k, sh, nb, nch, s, tma, st)
                    : launch_nsweep<kInFpPos, kOutFpPos, 256, 8, true>(kin, pin, fo, po, d_m, m, k, sh, nb, nch, s, tma, st);
      if (rc) return rc;
      kin = fo;
      pin = po;
      kin_hash = false;
    }
    if (pos32_dst) {
      pos_to_u32_kernel<<<grid_stride_blocks(m), kTPB, 0, st>>>(s.posW, d_m, m, pos32_dst, s.ctl);
      MZS_LAUNCHED();
    }
  }
  // ---- narrow passes 1.. (packed items in, packed or final out)
  {
    const uint64_t* kin = nullptr;
    { uint64_t* pk; uint32_t* fo; uint64_t* po; pass_out(0, pk, fo, po); kin = pk; }
    for (int p = 1; p < npass; ++p) {
      uint64_t* pk; uint32_t* fo; uint64_t* po;
      pass_out(p, pk, fo, po);
      const int sh = lo_bit + 8 * p;
      const int nb = std::min(8, hi_bit - sh);
      rc = count_pass<2>(kin, d_m, m, k, sh, nb, nch, s, 1, st);
      if (rc) return rc;
      rc = p != npass - 1 ? launch_nsweep_cfg<kInPk, kOutPk>(ipt_pk, kin, nullptr, pk, nullptr, d_m, m, k, sh, nb, nch, s, 1, st)
           : pos32_dst ? launch_nsweep<kInPk, kOutFpPos32, 256, 16>(kin, nullptr, fo, po, d_m, m, k, sh, nb, nch, s, 1, st)
                       : launch_nsweep_cfg<kInPk, kOutFpPos>(ipt_pk, kin, nullptr, fo, po, d_m, m, k, sh, nb, nch, s, 1, st);
      if (rc) return rc;
      kin = pk;
    }
  }
  (void)force;
  return SLSUM_OK;
}

int offsets_launch(const uint32_t* fp, const uint64_t* d_m, uint64_t m, int shift, uint32_t bmask, uint64_t nb,
                   uint64_t* offsets, uint64_t* tile_min, cudaStream_t st) {
  MZS_CUDA(cudaMemsetAsync(offsets, 0xff, sizeof(uint64_t) * (nb + 1), st));
  const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((m / 16 + kTPB) / kTPB, (uint64_t)num_sms() * 8));
  offsets_scatter_kernel<<<(unsigned)blocks, kTPB, 0, st>>>(fp, d_m, m, shift, bmask, nb, offsets);
  MZS_LAUNCHED();
  const uint64_t n = nb + 1, nt = (n + kSminTile - 1) / kSminTile;
  smin_reduce_kernel<<<(unsigned)nt, kTPB, 0, st>>>(offsets, n, tile_min);
  MZS_LAUNCHED();
  smin_tiles_kernel<<<1, kTPB, 0, st>>>(tile_min, nt);
  MZS_LAUNCHED();
  smin_apply_kernel<<<(unsigned)nt, kTPB, 0, st>>>(offsets, n, tile_min);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

uint64_t smin_tiles_for(uint64_t nb) { return (nb + 1 + kSminTile - 1) / kSminTile + 1; }

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }
int log2i(int x) { int r = 0; while ((1 << r) < x) ++r; return r; }

}  // namespace

// Stable sort of m (fingerprint, index) pairs by fingerprint bits [lo_bit, 32), for other
// translation units (the sorted seed lookup, lookup.cu): the seed table's own radix passes.
size_t sort_fp_idx_workspace_bytes(uint64_t m, int lo_bit) {
  Sizer z;
  size_sort_ws(z, m, (32 - lo_bit + 7) / 8, false);
  return z.used;
}
int sort_fp_idx(const uint32_t* fp, const uint64_t* idx, uint64_t m, int lo_bit, uint32_t* fp_out, uint64_t* idx_out,
                void* ws, size_t ws_bytes, cudaStream_t st) {
  Carve c(ws, ws_bytes);
  SortWs s;
  if (!carve_sort_ws(c, m, (32 - lo_bit + 7) / 8, false, s)) return SLSUM_ENOMEM;
  return stable_sort(false, fp, idx, nullptr, m, 0, lo_bit, 32, fp_out, idx_out, s, st);
}

// Stable sort of m packed u64 items by bits [lo_bit, hi_bit) of their HIGH 32 bits (the rest
// of the item travels unchanged): the narrow passes alone, for other translation units (the
// sorted seed lookup puts its per-query results back into query order with it).
size_t sort_items_workspace_bytes(uint64_t m, int lo_bit, int hi_bit) {
  (void)lo_bit; (void)hi_bit;
  Sizer z;
  z.take<uint32_t>(256 * chunks_for(m));
  z.take<uint64_t>(256 * chunks_for(m));
  z.take<unsigned long long>(256);
  z.take<unsigned long long>(256);
  z.take<uint64_t>(2);
  z.take<uint64_t>(m + 1);
  z.take<uint64_t>(m + 1);
  return z.used;
}
int sort_items(const uint64_t* items, uint64_t m, int lo_bit, int hi_bit, uint64_t* out, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  if (m == 0) return SLSUM_OK;
  if (lo_bit < 0 || hi_bit > 32 || hi_bit <= lo_bit) return SLSUM_EINVAL;
  Carve c(ws, ws_bytes);
  SortWs s{};
  s.chunk = chunk_for(m);
  s.counts = c.take<uint32_t>(256 * chunks_for(m));
  s.offs = c.take<uint64_t>(256 * chunks_for(m));
  s.totals = c.take<unsigned long long>(256);
  s.dbase = c.take<unsigned long long>(256);
  s.ctl = c.take<uint64_t>(2);
  uint64_t* A = c.take<uint64_t>(m + 1);
  uint64_t* B = c.take<uint64_t>(m + 1);
  if (!c.ok) return SLSUM_ENOMEM;
  // ctl = {1 (the narrow path), 0}: every kernel runs, no wide fallback (the items are opaque)
  MZS_CUDA(cudaMemsetAsync(s.ctl, 0, 2 * sizeof(uint64_t), st));
  MZS_CUDA(cudaMemsetAsync(s.ctl, 1, 1, st));
  static const int ipt_pk = env_int("MZS_NCFG", 25616);
  const int npass = (hi_bit - lo_bit + 7) / 8;
  const uint64_t nch = (m + s.chunk - 1) / s.chunk;
  const uint64_t* kin = items;
  int tma = (reinterpret_cast<uintptr_t>(items) & 15) == 0;
  for (int p = 0; p < npass; ++p) {
    uint64_t* dst = p == npass - 1 ? out : ((p & 1) ? B : A);
    const int sh = lo_bit + 8 * p;
    const int nb = std::min(8, hi_bit - sh);
    int rc = count_pass<2>(kin, nullptr, m, 0, sh, nb, nch, s, 1, st);
    if (rc) return rc;
    rc = launch_nsweep_cfg<kInPk, kOutPk>(ipt_pk, kin, nullptr, dst, nullptr, nullptr, m, 0, sh, nb, nch, s, tma, st);
    if (rc) return rc;
    kin = dst;
    tma = 1;
  }
  return SLSUM_OK;
}

}  // namespace mzs

using namespace mzs;

#ifdef MZS_PROF
MZS_API int seedtable_prof_read(unsigned long long* out8, int reset) {
  MZS_CUDA(cudaMemcpyFromSymbol(out8, g_prof, sizeof(unsigned long long) * 8));
  if (reset) {
    static const unsigned long long z[8] = {0};
    MZS_CUDA(cudaMemcpyToSymbol(g_prof, z, sizeof(z)));
  }
  return SLSUM_OK;
}
#endif

MZS_API size_t seedtable_workspace_bytes(uint64_t m, int bucket_bits) {
  Sizer z;
  const int npass = (bucket_bits + 7) / 8;
  size_sort_ws(z, m, npass, true);
  z.take<uint64_t>(smin_tiles_for(1ull << bucket_bits));
  return z.used;
}

static int seedtable_build_impl(const uint64_t* items, const uint64_t* hash, const uint64_t* pos, uint64_t m,
                                const uint64_t* d_m, int k, int bucket_bits, uint64_t* offsets, uint32_t* fp_out,
                                uint64_t* pos_out, void* ws, size_t ws_bytes, void* stream,
                                uint32_t* pos32_out = nullptr, const uint32_t* hist0 = nullptr) {
  if (k < 1 || k > 31 || bucket_bits < 1 || bucket_bits > 30 || bucket_bits > 2 * k) return SLSUM_EINVAL;
  if (!offsets || (m && (!hash || !pos || (!pos_out && !pos32_out)))) return SLSUM_EINVAL;
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
  uint64_t* tile_min = c.take<uint64_t>(smin_tiles_for(nb));
  if (!c.ok) return SLSUM_ENOMEM;
  uint32_t* fp_final = fp_out ? fp_out : s.fpF;
  const int lo = 32 - bucket_bits;
  int rc = stable_sort(true, hash, pos, d_m, m, k, lo, 32, fp_final, pos_out, s, st, items, pos32_out,
                       items ? hist0 : nullptr);
  if (rc) return rc;
  return offsets_launch(fp_final, d_m, m, lo, (uint32_t)(nb - 1), nb, offsets, tile_min, st);
}

MZS_API int seedtable_build(const uint64_t* hash, const uint64_t* pos, uint64_t m, const uint64_t* d_m, int k,
                            int bucket_bits, uint64_t* offsets, uint32_t* fp_out, uint64_t* pos_out, void* ws,
                            size_t ws_bytes, void* stream) {
  return seedtable_build_impl(nullptr, hash, pos, m, d_m, k, bucket_bits, offsets, fp_out, pos_out, ws, ws_bytes,
                              stream);
}

MZS_API int seedtable_build_items(const uint64_t* items, const uint64_t* hash, const uint64_t* pos, uint64_t m,
                                  const uint64_t* d_m, int k, int bucket_bits, uint64_t* offsets, uint32_t* fp_out,
                                  uint64_t* pos_out, void* ws, size_t ws_bytes, void* stream) {
  if (m && !items) return SLSUM_EINVAL;
  return seedtable_build_impl(items, hash, pos, m, d_m, k, bucket_bits, offsets, fp_out, pos_out, ws, ws_bytes,
                              stream);
}

MZS_API int seedtable_build_items32(const uint64_t* items, const uint64_t* hash, const uint64_t* pos, uint64_t m,
                                    const uint64_t* d_m, int k, int bucket_bits, uint64_t* offsets, uint32_t* fp_out,
                                    uint32_t* pos32_out, void* ws, size_t ws_bytes, void* stream) {
  if (m && (!items || !pos32_out)) return SLSUM_EINVAL;
  return seedtable_build_impl(items, hash, pos, m, d_m, k, bucket_bits, offsets, fp_out, nullptr, ws, ws_bytes,
                              stream, pos32_out);
}

MZS_API size_t seedtable_hist_words(uint64_t capacity, int bucket_bits) {
  (void)bucket_bits;
  return capacity ? (size_t)256 * radix_nchunks(capacity) : 0;
}

MZS_API int seedtable_build_items_ex(const uint64_t* items, const uint64_t* hash, const uint64_t* pos, uint64_t m,
                                     const uint64_t* d_m, int k, int bucket_bits, const uint32_t* hist,
                                     uint64_t* offsets, uint32_t* fp_out, uint64_t* pos_out, uint32_t* pos32_out,
                                     void* ws, size_t ws_bytes, void* stream) {
  if ((pos_out != nullptr) == (pos32_out != nullptr)) return SLSUM_EINVAL;
  if (m && !items) return SLSUM_EINVAL;
  return seedtable_build_impl(items, hash, pos, m, d_m, k, bucket_bits, offsets, fp_out, pos_out, ws, ws_bytes,
                              stream, pos32_out, hist);
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
  u32_to_u64_kernel<<<1, 256, 0, st>>>(s.totals, send_counts, nranks);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

MZS_API size_t seedtable_partition_p2p_workspace_bytes(uint64_t m, int nranks) {
  Sizer z;
  size_sort_ws(z, m, 1, false);
  z.take<uint64_t>(2 * (size_t)nranks);  // device copies of the destination pointer tables
  return z.used;
}

// Partition fused with the all-to-all: the stable pass on the owner digit writes
// every entry straight into its owner's receive buffer (peer memory over NVLink), at the offset
// peer_base[o] this sender owns there.  Narrow path only (positions of the call within 2^32 of
// pos[0]); returns SLSUM_EUNSUPPORTED otherwise, and the caller uses partition + NCCL.
static int partition_p2p_impl(const uint64_t* items, const uint64_t* hash, const uint64_t* pos, uint64_t m,
                              const uint64_t* d_m, int k, int bucket_bits, int nranks, const uint64_t* peer_fp,
                              const uint64_t* peer_pos, const uint64_t* peer_base, void* ws, size_t ws_bytes,
                              void* stream) {
  if (k < 1 || k > 31 || bucket_bits < 1 || bucket_bits > 30 || bucket_bits > 2 * k) return SLSUM_EINVAL;
  if (!is_pow2(nranks) || nranks < 2 || nranks > 256 || log2i(nranks) > bucket_bits || !peer_fp || !peer_pos ||
      !peer_base)
    return SLSUM_EINVAL;
  if (m == 0) return SLSUM_OK;
  if ((!items && !hash) || !pos) return SLSUM_EINVAL;
  cudaStream_t st = as_stream(stream);
  TempWs tmp;
  const size_t need = seedtable_partition_p2p_workspace_bytes(m, nranks);
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
  uint64_t* dptr = c.take<uint64_t>(2 * (size_t)nranks);
  if (!c.ok) return SLSUM_ENOMEM;
  const int g = log2i(nranks);
  const uint64_t nch = (m + s.chunk - 1) / s.chunk;
  // the narrow precondition, decided here on the host (one small read)
  uint64_t h[3] = {m, 0, 0};
  if (d_m) MZS_CUDA(cudaMemcpyAsync(&h[0], d_m, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  MZS_CUDA(cudaStreamSynchronize(st));
  const uint64_t mm = std::min(h[0], m);
  if (mm == 0) return SLSUM_OK;
  MZS_CUDA(cudaMemcpy(&h[1], pos, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  MZS_CUDA(cudaMemcpy(&h[2], pos + mm - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (h[2] < h[1] || h[2] - h[1] > 0xffffffffull) return SLSUM_EUNSUPPORTED;
  ctl_kernel<<<1, 32, 0, st>>>(pos, d_m, m, s.ctl);
  MZS_LAUNCHED();
  const int nb = g;
  const int sh = 32 - nb;
  int rc = items ? count_pass<2>(items, d_m, m, k, sh, nb, nch, s, 1, st)
                 : count_pass<0>(hash, d_m, m, k, sh, nb, nch, s, 1, st);
  if (rc) return rc;
  // destinations: digit o -> owner o's buffers, from this sender's base there (replacing the
  // digit scan's bases; digits >= nranks carry no entries)
  std::vector<uint64_t> hp(2 * (size_t)nranks), hb(256, 0);
  for (int o = 0; o < nranks; ++o) {
    hp[o] = peer_fp[o];
    hp[nranks + o] = peer_pos[o];
    hb[o] = peer_base[o];
  }
  MZS_CUDA(cudaMemcpyAsync(dptr, hp.data(), sizeof(uint64_t) * 2 * nranks, cudaMemcpyHostToDevice, st));
  MZS_CUDA(cudaMemcpyAsync(s.dbase, hb.data(), sizeof(unsigned long long) * 256, cudaMemcpyHostToDevice, st));
  if (items) {
    // packed items (fp << 32 | pos mod 2^32): 8 B per entry in; the positions are restored from
    // pos[0] (ctl[1]) as in the last pass of seedtable_build_items
    const int tma_in = (reinterpret_cast<uintptr_t>(items) & 15) == 0;
    auto kern = nsweep_kernel<kInPk, kOutFpPos, 256, 8>;
    const size_t smem = nsweep_smem<kInPk, 256, 8>();
    MZS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nch, 256, smem, st>>>(items, nullptr, nullptr, nullptr, d_m, m, k, sh, nb, s.offs, s.dbase, nch,
                                           s.ctl, tma_in, s.chunk, 1, reinterpret_cast<uint32_t* const*>(dptr),
                                           reinterpret_cast<uint64_t* const*>(dptr + nranks));
  } else {
    const int tma_in = ((reinterpret_cast<uintptr_t>(hash) | reinterpret_cast<uintptr_t>(pos)) & 15) == 0;
    auto kern = nsweep_kernel<kInHashPos, kOutFpPos, 256, 8>;
    const size_t smem = nsweep_smem<kInHashPos, 256, 8>();
    MZS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)nch, 256, smem, st>>>(hash, pos, nullptr, nullptr, d_m, m, k, sh, nb, s.offs, s.dbase, nch, s.ctl,
                                           tma_in, s.chunk, 1, reinterpret_cast<uint32_t* const*>(dptr),
                                           reinterpret_cast<uint64_t* const*>(dptr + nranks));
  }
  MZS_LAUNCHED();
  // the host vectors above were read by the async copies; make them complete before returning.
  // The downsweep re-checks every entry against the narrow range and clears ctl[0] on a
  // violation (unsorted input): the peers' buffers then hold wrong entries, and the caller
  // must fall back to partition + NCCL (uniformly across ranks).
  uint64_t narrow = 0;
  MZS_CUDA(cudaMemcpyAsync(&narrow, s.ctl, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
  MZS_CUDA(cudaStreamSynchronize(st));
  return narrow ? SLSUM_OK : SLSUM_EUNSUPPORTED;
}

MZS_API int seedtable_partition_p2p(const uint64_t* hash, const uint64_t* pos, uint64_t m, const uint64_t* d_m, int k,
                                    int bucket_bits, int nranks, const uint64_t* peer_fp, const uint64_t* peer_pos,
                                    const uint64_t* peer_base, void* ws, size_t ws_bytes, void* stream) {
  return partition_p2p_impl(nullptr, hash, pos, m, d_m, k, bucket_bits, nranks, peer_fp, peer_pos, peer_base, ws,
                            ws_bytes, stream);
}

MZS_API int seedtable_partition_p2p_items(const uint64_t* items, const uint64_t* pos, uint64_t m, const uint64_t* d_m,
                                          int k, int bucket_bits, int nranks, const uint64_t* peer_fp,
                                          const uint64_t* peer_pos, const uint64_t* peer_base, void* ws,
                                          size_t ws_bytes, void* stream) {
  if (m && !items) return SLSUM_EINVAL;
  return partition_p2p_impl(items, nullptr, pos, m, d_m, k, bucket_bits, nranks, peer_fp, peer_pos, peer_base, ws,
                            ws_bytes, stream);
}

MZS_API size_t seedtable_finalize_workspace_bytes(uint64_t m_recv, int bucket_bits, int nranks) {
  Sizer z;
  const int npass = std::max(1, (bucket_bits - log2i(nranks) + 7) / 8);
  size_sort_ws(z, m_recv, npass, true);
  z.take<uint64_t>(smin_tiles_for(1ull << (bucket_bits - log2i(nranks))));
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
  uint64_t* tile_min = c.take<uint64_t>(smin_tiles_for(nbl));
  if (!c.ok) return SLSUM_ENOMEM;
  uint32_t* fp_final = fp_out ? fp_out : s.fpF;
  const int lo = 32 - bucket_bits;
  const int hi = lbits > 0 ? 32 - g : lo + 1;  // lbits == 0: one bucket per owner; a 1-bit no-op pass
  int rc = stable_sort(false, recv_fp, recv_pos, nullptr, m_recv, 0, lo, hi, fp_final, pos_out, s, st);
  if (rc) return rc;
  if (!global_counts)
    return offsets_launch(fp_final, nullptr, m_recv, lo, (uint32_t)(nbl - 1), nbl, offsets_local, tile_min, st);
  return SLSUM_OK;
}
