// lookup.cu -- batch seed lookup against the seed table (Sec. 2.4, Fig. 1:
// "The seed pointer table enables fast lookups to 'CG' and 'CT'").
//
// For query key q: f = fingerprint(q) (the top 32 bits of the 2k-bit key, R21),
// b = f >> (32 - bits); the hits are the entries of b's slice [offsets[b], offsets[b+1]) with
// fp == f, in table order (ascending position).  When 2k <= 32 the fingerprint is the whole
// key and the hits are exactly the stored positions of the seed (R30).
//
// Three steps: count (per query), exclusive scan of the counts (-> CSR offsets), emit.
// A group of kG lanes (8; one lane per query for short buckets, see lookup1_kernel) serves one query: the slice's fingerprints are read kG
// at a time, matches are counted with a group ballot, and in the emit step written in order
// (ballot prefix inside the group).  Minimizer hashes are skewed low, so queries land in the
// long buckets more often than the mean bucket length suggests.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace mzs {
namespace {

constexpr int kLTPB = 256;
#ifndef MZS_LOOKUP_EMIT_UNROLL
#define MZS_LOOKUP_EMIT_UNROLL 1
#endif

// POS1 paths: first[i] with this bit set is a table index to scan from (recounted queries with
// two or more hits); without it, a position (one hit) or a side-array index (2..14 hits)
constexpr uint64_t kScanFlag = 1ull << 63;

__device__ __forceinline__ uint32_t fp_of(uint64_t key, int k) {
  const int b = 2 * k;
  return b >= 32 ? (uint32_t)(key >> (b - 32)) : (uint32_t)(key << (32 - b));
}

__device__ __forceinline__ uint64_t query_count(const uint64_t* d_nq, uint64_t nq) {
  return d_nq ? min(*d_nq, nq) : nq;
}

// EMIT = false: hit_off[i] = number of hits of query i, first[i] = its first matching entry.
// EMIT = true: write them at hit_off[i] (exclusive offsets), scanning from first[i] until all
// hit_off[i+1] - hit_off[i] hits are found (hitless queries read nothing of the table).
template <bool EMIT, int kG>
__global__ void __launch_bounds__(kLTPB) lookup_kernel(const uint64_t* __restrict__ q, uint64_t nq_cap,
                                                       const uint64_t* d_nq, int k, int bits,
                                                       const uint64_t* __restrict__ offsets,
                                                       const uint32_t* __restrict__ fp,
                                                       const uint64_t* __restrict__ pos_tab, uint64_t* hit_off,
                                                       uint64_t* __restrict__ hit_pos, uint64_t hit_cap,
                                                       uint64_t* __restrict__ first) {
  const uint64_t nq = query_count(d_nq, nq_cap);
  const unsigned lane = lane_id();
  const unsigned gl = lane & (kG - 1);                   // lane inside the group
  const unsigned gshift = lane & ~(unsigned)(kG - 1);    // group's first lane
  const unsigned gmask = (kG == 32 ? 0xffffffffu : ((1u << kG) - 1u)) << gshift;
  const uint64_t groups = (uint64_t)gridDim.x * (kLTPB / kG);
  const uint64_t m_tab = EMIT ? offsets[(uint64_t)1 << bits] : 0;  // table entries (reads stay below)
  for (uint64_t i0 = ((uint64_t)blockIdx.x * kLTPB + threadIdx.x) / kG; i0 < ((nq + groups - 1) / groups) * groups;
       i0 += groups) {
    const bool live = i0 < nq;
    uint32_t f = 0;
    uint64_t lo = 0, hi = 0, o = 0, o_end = 0;
    if (live) {
      if (EMIT) {
        o = hit_off[i0];
        o_end = hit_off[i0 + 1];
        if (o < o_end) {
          f = fp_of(q[i0], k);
          lo = first[i0];
          hi = m_tab;
        }
      } else {
        f = fp_of(q[i0], k);
        const uint64_t b = f >> (32 - bits);
        lo = offsets[b];
        hi = offsets[b + 1];
      }
    }
    uint64_t cnt = 0, e0 = lo;
    // all groups of the warp iterate together (ballots need the full warp)
    if (EMIT) {
      for (uint64_t s = 0;; ++s) {
        const bool pending = o + cnt < o_end;
        if (!__any_sync(0xffffffffu, pending)) break;
        const uint64_t e = lo + s * kG + gl;
        const bool hit = pending && e < hi && fp[e] == f;
        const unsigned bal = __ballot_sync(0xffffffffu, hit) & gmask;
        if (hit) {
          const uint64_t r = o + cnt + __popc(bal & ((1u << lane) - 1u));
          if (r < o_end && r < hit_cap) hit_pos[r] = pos_tab[e];
        }
        cnt += __popc(bal);
      }
    } else {
      uint64_t len = hi - lo;
      uint64_t steps = (len + kG - 1) / kG;
      for (int o2 = kG; o2 < 32; o2 <<= 1) steps = max(steps, (uint64_t)__shfl_xor_sync(0xffffffffu, steps, o2));
      for (uint64_t s = 0; s < steps; ++s) {
        const uint64_t e = lo + s * kG + gl;
        const bool hit = e < hi && fp[e] == f;
        const unsigned bal = __ballot_sync(0xffffffffu, hit) & gmask;
        if (cnt == 0 && bal) e0 = lo + s * kG + (__ffs(bal >> gshift) - 1);
        cnt += __popc(bal);
      }
      if (live && gl == 0) {
        hit_off[i0] = cnt;
        first[i0] = e0;
      }
    }
  }
}

// One thread per query (no ballots): 32 independent random lookups in flight per warp, for
// tables whose buckets are short (the scan of a bucket is a serial loop in the thread).
// The count step also records each query's first matching entry (first[i]); the emit step
// then skips the queries without hits and starts at that entry -- no second pointer-table
// read and no second scan of the leading entries (one dependent random access fewer).
// POS1 (sorted lookup with the packed-item unsort): first[i] already holds the POSITION of a
// query's only hit (count 1; the count step read it while it walked the buckets in order), and
// the first match's table index otherwise.
template <bool EMIT, bool POS1 = false>
__global__ void __launch_bounds__(kLTPB) lookup1_kernel(const uint64_t* __restrict__ q, uint64_t nq_cap,
                                                        const uint64_t* d_nq, int k, int bits,
                                                        const uint64_t* __restrict__ offsets,
                                                        const uint32_t* __restrict__ fp,
                                                        const uint64_t* __restrict__ pos_tab, uint64_t* hit_off,
                                                        uint64_t* __restrict__ hit_pos, uint64_t hit_cap,
                                                        uint64_t* __restrict__ first,
                                                        const uint64_t* __restrict__ side = nullptr) {
  // side (POS1): first[i] of a query with 2..14 hits indexes its positions in side (count step)
  const uint64_t nq = query_count(d_nq, nq_cap);
  const uint64_t m_tab = EMIT && MZS_LOOKUP_EMIT_UNROLL ? offsets[(uint64_t)1 << bits] : 0;  // table entries
  for (uint64_t i = (uint64_t)blockIdx.x * kLTPB + threadIdx.x; i < nq; i += (uint64_t)gridDim.x * kLTPB) {
    if (EMIT) {
      uint64_t o = hit_off[i];
      const uint64_t o_end = hit_off[i + 1];
      if (o == o_end) continue;
      // the hits are the first o_end - o entries from first[i] on whose fingerprint is f;
      // first[i] itself is one (no need to read its fingerprint again)
      uint64_t e0 = first[i];
      if (POS1 && !(e0 & kScanFlag)) {
        if (o + 1 == o_end) {
          if (o < hit_cap) hit_pos[o] = e0;  // the position itself
          continue;
        }
        if (side) {  // 2..14 hits: their positions, copied from the count step's side array
          for (uint64_t r = 0; o + r < o_end; ++r)
            if (o + r < hit_cap) hit_pos[o + r] = side[e0 + r];
          continue;
        }
      }
      if (POS1) e0 &= ~kScanFlag;
      if (o < hit_cap) hit_pos[o] = pos_tab[e0];
      if (++o == o_end) continue;
      const uint32_t f = fp_of(q[i], k);
      uint64_t e = e0 + 1;
#if MZS_LOOKUP_EMIT_UNROLL
      // four fingerprints per step with independent loads (bounded by the table's last entry)
      for (; o < o_end && e + 4 <= m_tab; e += 4) {
        const uint32_t f0 = fp[e], f1 = fp[e + 1], f2 = fp[e + 2], f3 = fp[e + 3];
        const uint32_t mm = (uint32_t)(f0 == f) | ((uint32_t)(f1 == f) << 1) | ((uint32_t)(f2 == f) << 2) |
                            ((uint32_t)(f3 == f) << 3);
        for (uint32_t b = mm; b && o < o_end; b &= b - 1) {
          const uint64_t eh = e + (__ffs(b) - 1);
          if (o < hit_cap) hit_pos[o] = pos_tab[eh];
          ++o;
        }
      }
#endif
      for (; o < o_end; ++e) {
        if (fp[e] == f) {
          if (o < hit_cap) hit_pos[o] = pos_tab[e];
          ++o;
        }
      }
    } else {
      const uint32_t f = fp_of(q[i], k);
      const uint64_t b = f >> (32 - bits);
      const uint64_t lo = offsets[b], hi = offsets[b + 1];
      uint64_t cnt = 0, e0 = lo;
      for (uint64_t e = lo; e < hi; ++e) {
        if (fp[e] == f) {
          if (cnt == 0) e0 = e;
          ++cnt;
        }
      }
      hit_off[i] = cnt;
      first[i] = e0;
    }
  }
}

// Sorted lookup (large batches): the queries are first sorted by bucket (a stable radix sort
// of (fingerprint, query index), the seed table's own passes), so consecutive threads look up
// the same or neighbouring buckets -- the pointer table and the slices are then read nearly in
// order and mostly from L1/L2 instead of one random DRAM access chain per query.  Thread j
// serves the j-th query in bucket order; counts, first matches and hits go to the query's own
// index (the CSR stays in query order).  Same results as the unsorted kernels.
__global__ void __launch_bounds__(kLTPB) fp_idx_kernel(const uint64_t* __restrict__ q, uint64_t nq, int k,
                                                       uint32_t* __restrict__ fpq, uint64_t* __restrict__ idx) {
  for (uint64_t i = (uint64_t)blockIdx.x * kLTPB + threadIdx.x; i < nq; i += (uint64_t)gridDim.x * kLTPB) {
    fpq[i] = fp_of(q[i], k);
    idx[i] = i;
  }
}

template <bool EMIT>
__global__ void __launch_bounds__(kLTPB) lookup_sorted_kernel(const uint32_t* __restrict__ fps,
                                                              const uint64_t* __restrict__ ord, uint64_t nq, int bits,
                                                              const uint64_t* __restrict__ offsets,
                                                              const uint32_t* __restrict__ fp,
                                                              const uint64_t* __restrict__ pos_tab, uint64_t* hit_off,
                                                              uint64_t* __restrict__ hit_pos, uint64_t hit_cap,
                                                              uint64_t* __restrict__ first) {
  for (uint64_t j = (uint64_t)blockIdx.x * kLTPB + threadIdx.x; j < nq; j += (uint64_t)gridDim.x * kLTPB) {
    const uint64_t i = ord[j];
    const uint32_t f = fps[j];
    if (EMIT) {
      uint64_t o = hit_off[i];
      const uint64_t o_end = hit_off[i + 1];
      if (o == o_end) continue;
      const uint64_t e0 = first[j];                         // (kept in bucket order: coalesced)
      if (o < hit_cap) hit_pos[o] = pos_tab[e0];
      if (++o == o_end) continue;
      for (uint64_t e = e0 + 1; o < o_end; ++e) {
        if (fp[e] == f) {
          if (o < hit_cap) hit_pos[o] = pos_tab[e];
          ++o;
        }
      }
    } else {
      const uint64_t b = f >> (32 - bits);
      const uint64_t lo = offsets[b], hi = offsets[b + 1];
      uint64_t cnt = 0, e0 = lo;
      for (uint64_t e = lo; e < hi; ++e) {
        if (fp[e] == f) {
          if (cnt == 0) e0 = e;
          ++cnt;
        }
      }
      hit_off[i] = cnt;
      first[j] = e0;
    }
  }
}

// Sorted count (round 2b): thread j scans the slice of the j-th query in bucket order (the
// neighbouring threads mostly share the bucket, so the slice comes from L1/L2), four
// fingerprints per step with independent loads, and writes the count and first match to the
// query's OWN index -- so the emit step can run in query order (lookup1_kernel<true>): the CSR
// offsets and the hit positions are then read and written coalesced, and the only random
// accesses left are these two stores, the first hit's position and the scan of multi-hit
// queries.
template <bool FIRST_Q>
__global__ void __launch_bounds__(kLTPB) lookup_sorted_count_kernel(const uint32_t* __restrict__ fps,
                                                                    const uint64_t* __restrict__ ord, uint64_t nq,
                                                                    int bits, const uint64_t* __restrict__ offsets,
                                                                    const uint32_t* __restrict__ fp,
                                                                    uint64_t* __restrict__ hit_off,
                                                                    uint64_t* __restrict__ first) {
  for (uint64_t j = (uint64_t)blockIdx.x * kLTPB + threadIdx.x; j < nq; j += (uint64_t)gridDim.x * kLTPB) {
    const uint64_t i = ord[j];
    const uint32_t f = fps[j];
    const uint64_t b = f >> (32 - bits);
    const uint64_t lo = offsets[b], hi = offsets[b + 1];
    uint32_t cnt = 0;
    uint64_t e0 = hi;
    uint64_t e = lo;
    for (; e + 4 <= hi; e += 4) {
      const uint32_t f0 = fp[e], f1 = fp[e + 1], f2 = fp[e + 2], f3 = fp[e + 3];
      const uint32_t m = (uint32_t)(f0 == f) | ((uint32_t)(f1 == f) << 1) | ((uint32_t)(f2 == f) << 2) |
                         ((uint32_t)(f3 == f) << 3);
      if (m) {
        if (e0 == hi) e0 = e + (__ffs(m) - 1);
        cnt += __popc(m);
      }
    }
    for (; e < hi; ++e) {
      if (fp[e] == f) {
        if (e0 == hi) e0 = e;
        ++cnt;
      }
    }
    hit_off[i] = cnt;
    first[FIRST_Q ? i : j] = cnt ? e0 : lo;
  }
}

// Sorted lookup, round 2b (kSortedUnsort): the count step runs in bucket order and writes its
// result COALESCED as a packed item per query -- (query index << 4 | c) << 32 | first match,
// c = the hit count, or 15 when it is >= 15 or the first match does not fit 32 bits -- and a
// stable radix pass over the query index (sort_items) puts the items back into query order.
// The unpack step then writes the counts and first matches in query order (recounting the
// rare c = 15 queries), so the CSR scan and the emit (lookup1_kernel<true>) run in query order
// too: no random 8-byte store per query (which cost ~9 ms per 1.9e8 queries on B200).
__global__ void __launch_bounds__(kLTPB) lookup_sorted_count_pk_kernel(const uint32_t* __restrict__ fps,
                                                                       const uint64_t* __restrict__ ord, uint64_t nq,
                                                                       int bits, const uint64_t* __restrict__ offsets,
                                                                       const uint32_t* __restrict__ fp,
                                                                       uint64_t* __restrict__ items,
                                                                       const uint64_t* __restrict__ pos1_tab,
                                                                       uint64_t* __restrict__ side = nullptr) {
  // pos1_tab (the POS1 emit): a query with one hit carries that hit's POSITION in the item's low
  // word -- read here, where the slices are walked in bucket order and the reads nearly in order,
  // instead of by a random 8-byte read (~128 B of DRAM traffic) per hit in the query-order emit;
  // a position >= 2^32 forces c = 15 (recounted by the unpack).
  // side (with pos1_tab): a query with 2..14 hits writes their positions, in table order, to
  // side[s .. s + cnt) and carries s instead of its first match, so the emit copies them
  // instead of scanning the slice again in query order.  Every warp owns a private region of
  // qw = (its share of the queries, rounded up to 32) slots and a private fill counter (no
  // atomics: one global counter serialised the kernel at ~2x its time); a query that does not
  // fit its warp's region takes c = 15 (recount + scan).  The loop is warp-uniform (the slot
  // scan is a warp collective).  side holds nwarps * qw <= nq + 32 * nwarps entries.
  const unsigned lane = threadIdx.x & 31u;
  const uint64_t nwarps = (uint64_t)gridDim.x * (kLTPB / 32);
  const uint64_t qw = (nq + 32 * nwarps - 1) / (32 * nwarps) * 32;
  const uint64_t region = ((uint64_t)blockIdx.x * (kLTPB / 32) + (threadIdx.x >> 5)) * qw;
  uint64_t used = 0;  // warp-uniform
  for (uint64_t j0 = (uint64_t)blockIdx.x * kLTPB + (threadIdx.x & ~31u); j0 < nq; j0 += (uint64_t)gridDim.x * kLTPB) {
    const uint64_t j = j0 + lane;
    const bool valid = j < nq;
    uint64_t i = 0, lo = 0, e0 = 0, e1 = 0, e2 = 0, e3 = 0;  // the first four matches
    uint32_t f = 0, cnt = 0;
    if (valid) {
      i = ord[j];
      f = fps[j];
      const uint64_t b = f >> (32 - bits);
      lo = offsets[b];
      const uint64_t hi = offsets[b + 1];
      e0 = lo;
      auto record = [&](uint64_t eh) {
        if (cnt == 0) e0 = eh;
        else if (cnt == 1) e1 = eh;
        else if (cnt == 2) e2 = eh;
        else if (cnt == 3) e3 = eh;
        ++cnt;
      };
      // four independent fingerprint loads per step; the (rare) matches are recorded off the
      // main path, so the loop stays short and several loads stay in flight
      uint64_t e = lo;
      for (; e + 4 <= hi; e += 4) {
        const uint32_t f0 = fp[e], f1 = fp[e + 1], f2 = fp[e + 2], f3 = fp[e + 3];
        uint32_t mm = (uint32_t)(f0 == f) | ((uint32_t)(f1 == f) << 1) | ((uint32_t)(f2 == f) << 2) |
                      ((uint32_t)(f3 == f) << 3);
        while (mm) {
          record(e + (uint32_t)(__ffs(mm) - 1));
          mm &= mm - 1;
        }
      }
      for (; e < hi; ++e)
        if (fp[e] == f) record(e);
    }
    uint32_t c = (cnt >= 15 || (e0 >> 32) != 0) ? 15u : cnt;
    uint64_t lo32 = e0;
    if (pos1_tab && valid && c == 1) {
      lo32 = pos1_tab[e0];
      if (lo32 >> 32) c = 15;
    }
    if (side) {
      const uint32_t need = (valid && cnt >= 2 && cnt <= 14) ? cnt : 0u;  // (c may be 15 from e0 >= 2^32)
      uint32_t incl = need;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += y;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint64_t base = used;
      used += tot;
      if (need) {
        const uint64_t my = base + incl - need;
        if (my + need <= qw) {
          uint64_t* const sd = side + region + my;
          if (need <= 4) {  // the matches the scan kept (the common case: no second scan)
            sd[0] = pos1_tab[e0];
            sd[1] = pos1_tab[e1];
            if (need > 2) sd[2] = pos1_tab[e2];
            if (need > 3) sd[3] = pos1_tab[e3];
          } else {
            uint32_t r = 0;
            for (uint64_t e = e0; r < need; ++e) {
              if (fp[e] == f) sd[r++] = pos1_tab[e];
            }
          }
          c = cnt;
          lo32 = region + my;
        } else {
          c = 15;  // no room: recounted and scanned in query order
        }
      }
    }
    if (valid) items[j] = ((uint64_t)(((uint32_t)i << 4) | c) << 32) | (uint32_t)lo32;
  }
}

// query order: hit_off[i] = count, first[i] = first match (c = 15: counted again here)
__global__ void __launch_bounds__(kLTPB) lookup_unpack_kernel(const uint64_t* __restrict__ items, uint64_t nq,
                                                              const uint64_t* __restrict__ q, int k, int bits,
                                                              const uint64_t* __restrict__ offsets,
                                                              const uint32_t* __restrict__ fp,
                                                              uint64_t* __restrict__ hit_off,
                                                              uint64_t* __restrict__ first,
                                                              const uint64_t* __restrict__ pos1_tab) {
  for (uint64_t i = (uint64_t)blockIdx.x * kLTPB + threadIdx.x; i < nq; i += (uint64_t)gridDim.x * kLTPB) {
    const uint64_t it = items[i];
    MZS_DCHECK((it >> 36) == i);
    uint32_t c = (uint32_t)(it >> 32) & 15u;
    uint64_t e0 = (uint32_t)it;
    if (c == 15) {
      const uint32_t f = fp_of(q[i], k);
      const uint64_t b = f >> (32 - bits);
      const uint64_t lo = offsets[b], hi = offsets[b + 1];
      uint64_t cnt = 0;
      e0 = lo;
      for (uint64_t e = lo; e < hi; ++e) {
        if (fp[e] == f) {
          if (cnt == 0) e0 = e;
          ++cnt;
        }
      }
      if (pos1_tab && cnt == 1) e0 = pos1_tab[e0];  // (POS1) the only hit's position
      else if (pos1_tab && cnt >= 2) e0 |= kScanFlag;  // a table index: the emit scans from it
      hit_off[i] = cnt;
    } else {
      hit_off[i] = c;
    }
    first[i] = e0;
  }
}

// Unpack + CSR scan in one pass (query order): tiles of kUT queries, claimed in order through
// an atomic counter, each thread turning kUE consecutive packed items into counts and first
// matches (c = 15: counted again), a block scan, and the tile's prefix from a decoupled
// look-back over the tiles before it.  hit_off[i] = exclusive prefix, hit_off[nq] = total.
constexpr int kUE = 8;
constexpr int kUT = kLTPB * kUE;
__device__ __forceinline__ void unpack_one(uint64_t it, uint64_t i, const uint64_t* __restrict__ q, int k, int bits,
                                           const uint64_t* __restrict__ offsets, const uint32_t* __restrict__ fp,
                                           const uint64_t* __restrict__ pos1_tab, uint64_t& cnt, uint64_t& e0) {
  // pos1_tab: e0 of a count-1 query is its hit's position (from the item, or read here after a
  // recount); otherwise the first match's table index
  MZS_DCHECK((it >> 36) == i);
  const uint32_t c = (uint32_t)(it >> 32) & 15u;
  e0 = (uint32_t)it;
  cnt = c;
  if (c == 15) {
    const uint32_t f = fp_of(q[i], k);
    const uint64_t b = f >> (32 - bits);
    const uint64_t lo = offsets[b], hi = offsets[b + 1];
    cnt = 0;
    e0 = lo;
    for (uint64_t e = lo; e < hi; ++e) {
      if (fp[e] == f) {
        if (cnt == 0) e0 = e;
        ++cnt;
      }
    }
    if (pos1_tab && cnt == 1) e0 = pos1_tab[e0];
    else if (pos1_tab && cnt >= 2) e0 |= kScanFlag;  // a table index: the emit scans from it
  }
}
__global__ void __launch_bounds__(kLTPB) lookup_unpack_scan_kernel(const uint64_t* __restrict__ items, uint64_t nq,
                                                                   const uint64_t* __restrict__ q, int k, int bits,
                                                                   const uint64_t* __restrict__ offsets,
                                                                   const uint32_t* __restrict__ fp,
                                                                   uint64_t* __restrict__ hit_off,
                                                                   uint64_t* __restrict__ first, uint64_t* status,
                                                                   uint32_t* tile_counter, uint64_t* d_total,
                                                                   const uint64_t* __restrict__ pos1_tab) {
  __shared__ uint32_t s_tile;
  __shared__ uint64_t ws[kLTPB / 32];
  __shared__ uint64_t s_pre;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint64_t t = s_tile;
  const uint64_t ntiles = (nq + kUT - 1) / kUT;
  const uint64_t i0 = t * kUT + (uint64_t)threadIdx.x * kUE;
  uint64_t cnt[kUE], e0[kUE];
  uint64_t sum = 0;
  if (i0 + kUE <= nq) {
    uint64_t it[kUE];
#pragma unroll
    for (int u = 0; u < kUE; u += 2) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(items + i0 + u);
      it[u] = v.x;
      it[u + 1] = v.y;
    }
#pragma unroll
    for (int u = 0; u < kUE; ++u) {
      unpack_one(it[u], i0 + u, q, k, bits, offsets, fp, pos1_tab, cnt[u], e0[u]);
      sum += cnt[u];
    }
  } else {
#pragma unroll
    for (int u = 0; u < kUE; ++u) {
      cnt[u] = 0;
      e0[u] = 0;
      if (i0 + u < nq) unpack_one(items[i0 + u], i0 + u, q, k, bits, offsets, fp, pos1_tab, cnt[u], e0[u]);
      sum += cnt[u];
    }
  }
  uint64_t tot;
  uint64_t ex = block_exclusive_sum<kLTPB, uint64_t>(sum, ws, &tot);
  if (warp_id() == 0) {
    const uint64_t pre = lookback_exclusive(status, t, tot);
    if (lane_id() == 0) {
      s_pre = pre;
      if (t == ntiles - 1) {
        hit_off[nq] = pre + tot;
        if (d_total) *d_total = pre + tot;
      }
    }
  }
  __syncthreads();
  ex += s_pre;
  if (i0 + kUE <= nq) {
#pragma unroll
    for (int u = 0; u < kUE; u += 2) {
      const uint64_t a = ex;
      const uint64_t b = ex + cnt[u];
      ex = b + cnt[u + 1];
      *reinterpret_cast<ulonglong2*>(hit_off + i0 + u) = make_ulonglong2(a, b);
      *reinterpret_cast<ulonglong2*>(first + i0 + u) = make_ulonglong2(e0[u], e0[u + 1]);
    }
  } else {
#pragma unroll
    for (int u = 0; u < kUE; ++u) {
      if (i0 + u < nq) {
        hit_off[i0 + u] = ex;
        first[i0 + u] = e0[u];
      }
      ex += cnt[u];
    }
  }
}

// ---- exclusive scan of u64 counts in place (reduce, scan of block sums, add)
constexpr int kSE = 8;                   // elements per thread
constexpr int kSB = kLTPB * kSE;         // elements per block

__global__ void __launch_bounds__(kLTPB) scan_reduce_kernel(const uint64_t* x, uint64_t nq_cap, const uint64_t* d_nq,
                                                            uint64_t* bsum) {
  __shared__ uint64_t ws[kLTPB / 32];
  const uint64_t n = query_count(d_nq, nq_cap);
  const uint64_t b0 = (uint64_t)blockIdx.x * kSB;
  uint64_t s = 0;
  for (uint64_t i = b0 + threadIdx.x; i < min(n, b0 + kSB); i += kLTPB) s += x[i];
  uint64_t tot;
  block_exclusive_sum<kLTPB, uint64_t>(s, ws, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// one block: exclusive scan of the block sums; total -> x[n] and *d_total
__global__ void __launch_bounds__(kLTPB) scan_blocks_kernel(uint64_t* bsum, uint64_t nb, uint64_t* x, uint64_t nq_cap,
                                                            const uint64_t* d_nq, uint64_t* d_total) {
  __shared__ uint64_t ws[kLTPB / 32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint64_t c0 = 0; c0 < nb; c0 += kLTPB) {
    const uint64_t i = c0 + threadIdx.x;
    const uint64_t v = i < nb ? bsum[i] : 0;
    uint64_t tot;
    const uint64_t ex = block_exclusive_sum<kLTPB, uint64_t>(v, ws, &tot);
    if (i < nb) bsum[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint64_t n = query_count(d_nq, nq_cap);
    x[n] = carry;
    if (d_total) *d_total = carry;
  }
}

__global__ void __launch_bounds__(kLTPB) scan_apply_kernel(uint64_t* x, uint64_t nq_cap, const uint64_t* d_nq,
                                                           const uint64_t* bsum) {
  __shared__ uint64_t ws[kLTPB / 32];
  const uint64_t n = query_count(d_nq, nq_cap);
  const uint64_t i0 = (uint64_t)blockIdx.x * kSB + (uint64_t)threadIdx.x * kSE;
  uint64_t v[kSE];
  uint64_t s = 0;
#pragma unroll
  for (int j = 0; j < kSE; ++j) {
    v[j] = i0 + j < n ? x[i0 + j] : 0;
    s += v[j];
  }
  uint64_t tot;
  uint64_t ex = block_exclusive_sum<kLTPB, uint64_t>(s, ws, &tot) + bsum[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kSE; ++j) {
    if (i0 + j < n) x[i0 + j] = ex;
    ex += v[j];
  }
}

}  // namespace
}  // namespace mzs

using namespace mzs;

#ifndef MZS_LOOKUP_QEMIT
#define MZS_LOOKUP_QEMIT 0
#endif
// sorted lookup: count in bucket order, emit in query order (1) or both in bucket order (0)
constexpr bool kSortedQueryOrderEmit = MZS_LOOKUP_QEMIT != 0;
#ifndef MZS_LOOKUP_UNSORT
#define MZS_LOOKUP_UNSORT 1
#endif
// sorted lookup: per-query results put back into query order by a radix pass (round 2b)
constexpr bool kSortedUnsort = MZS_LOOKUP_UNSORT != 0;
#ifndef MZS_LOOKUP_EMIT_LANES
#define MZS_LOOKUP_EMIT_LANES 1
#endif
constexpr int kEmitLanes = MZS_LOOKUP_EMIT_LANES;
// queries from which the sorted lookup is used (MZS_LOOKUP_SORT=0/1 forces it off/on)
constexpr uint64_t kSortMin = 1u << 20;

// Long buckets only (< 2^26 buckets): there the unsorted kernels chase one random slice per
// query; with short buckets (2^28) the one-lane unsorted kernel is faster (10.2 against 4.6
// G queries/s: the sorted kernels' count and offset accesses become the random ones).
static bool use_sorted(uint64_t nq, int bits) {
  static const int env = [] {
    const char* e = getenv("MZS_LOOKUP_SORT");
    return e && *e ? atoi(e) : -1;
  }();
  return env >= 0 ? env == 1 : (nq >= kSortMin && bits < 26);
}

MZS_API size_t seedtable_lookup_workspace_bytes(uint64_t nq) {
  Sizer z;
  z.take<uint64_t>((nq + kSB - 1) / kSB + 1);
  z.take<uint64_t>(1);
  z.take<uint64_t>(nq);  // first matching entry per query
  z.take<uint64_t>(nq + (1u << 19));  // (sorted lookup) multi-hit positions from the count step (per-warp regions)
  // (sorted lookup) query fingerprints and indices, the sorted copies and the sort's scratch
  // (sized for the 4 passes of bucket_bits 25..30, enough for any bits)
  z.take<uint32_t>(nq + 1);
  z.take<uint64_t>(nq + 1);
  z.take<uint32_t>(nq + 1);
  z.take<uint64_t>(nq + 1);
  z.used += std::max(sort_fp_idx_workspace_bytes(std::max<uint64_t>(nq, 1), 2),
                     sort_items_workspace_bytes(std::max<uint64_t>(nq, 1), 4, 32)) + kAlign;
  return z.used;
}

MZS_API int seedtable_lookup(const uint64_t* qkey, uint64_t nq, const uint64_t* d_nq, int k, int bucket_bits,
                             const uint64_t* offsets, const uint32_t* fp, const uint64_t* pos_tab,
                             uint64_t* hit_off, uint64_t* hit_pos, uint64_t hit_cap, uint64_t* d_total, void* ws,
                             size_t ws_bytes, void* stream) {
  if (k < 1 || k > 31 || bucket_bits < 1 || bucket_bits > 30 || bucket_bits > 2 * k) return SLSUM_EINVAL;
  if (!hit_off) return SLSUM_EINVAL;
  cudaStream_t st = as_stream(stream);
  if (nq == 0) {
    MZS_CUDA(cudaMemsetAsync(hit_off, 0, sizeof(uint64_t), st));
    if (d_total) MZS_CUDA(cudaMemsetAsync(d_total, 0, sizeof(uint64_t), st));
    return SLSUM_OK;
  }
  if (!qkey || !offsets || !fp || (hit_cap && (!hit_pos || !pos_tab))) return SLSUM_EINVAL;
  TempWs tmp;
  const size_t need = seedtable_lookup_workspace_bytes(nq);
  if (!ws) {
    MZS_CUDA(cudaMallocAsync(&tmp.p, need, st));
    tmp.s = st;
    ws = tmp.p;
    ws_bytes = need;
  }
  if (ws_bytes < need) return SLSUM_ENOMEM;
  Carve c(ws, ws_bytes);
  const uint64_t nb = (nq + kSB - 1) / kSB;
  uint64_t* bsum = c.take<uint64_t>(nb + 1);
  c.take<uint64_t>(1);
  uint64_t* first = c.take<uint64_t>(nq);
  uint64_t* side = c.take<uint64_t>(nq + (1u << 19));
  uint32_t* fpq = c.take<uint32_t>(nq + 1);
  uint64_t* idx = c.take<uint64_t>(nq + 1);
  uint32_t* fps = c.take<uint32_t>(nq + 1);
  uint64_t* ord = c.take<uint64_t>(nq + 1);
  const size_t sort_ws = std::max(sort_fp_idx_workspace_bytes(std::max<uint64_t>(nq, 1), 2),
                                  sort_items_workspace_bytes(std::max<uint64_t>(nq, 1), 4, 32));
  void* sws = c.take<unsigned char>(sort_ws);
  if (!c.ok) return SLSUM_ENOMEM;
  if (!d_nq && use_sorted(nq, bucket_bits)) {
    // sorted lookup: queries in bucket order (the count is host-known: d_nq == NULL)
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nq + kLTPB - 1) / kLTPB,
                                                                          (uint64_t)num_sms() * 8));
    fp_idx_kernel<<<g, kLTPB, 0, st>>>(qkey, nq, k, fpq, idx);
    MZS_LAUNCHED();
    int rc = sort_fp_idx(fpq, idx, nq, 32 - bucket_bits, fps, ord, sws, sort_ws, st);
    if (rc) return rc;
    int qbits = 1;
    while (qbits < 28 && (1ull << qbits) < nq) ++qbits;
    if (kSortedUnsort && nq <= (1ull << 28)) {
      // count in bucket order -> packed items (into idx, free after the sort) -> back to query
      // order (into ord, free after the count) -> counts and first matches in query order
      uint64_t* pk = idx;
      uint64_t* pq = ord;
      // POS1: the count step carries a count-1 query's hit POSITION (read in bucket order) to the
      // emit, which then reads pos_tab only for multi-hit queries (MZS_LOOKUP_NO_POS1: off)
      static const bool pos1_env = getenv("MZS_LOOKUP_NO_POS1") == nullptr;
      const uint64_t* pos1_tab = (pos1_env && hit_cap && kEmitLanes == 1) ? pos_tab : nullptr;
      static const bool side_env = getenv("MZS_LOOKUP_NO_SIDE") == nullptr;
      const bool use_side = pos1_tab != nullptr && side_env;
      // per-warp side regions: g * 8 warps of qw slots <= nq + 32 * g * 8 <= nq + 2^19 (g <= 2048)
      const bool side_fits = (uint64_t)g * (kLTPB / 32) * 32 <= (1u << 19) && nq + (1u << 19) < (1ull << 32);
      const bool use_side2 = use_side && side_fits;
      lookup_sorted_count_pk_kernel<<<g, kLTPB, 0, st>>>(fps, ord, nq, bucket_bits, offsets, fp, pk, pos1_tab,
                                                         use_side2 ? side : nullptr);
      MZS_LAUNCHED();
      rc = sort_items(pk, nq, 4, 4 + qbits, pq, sws, sort_ws, st);
      if (rc) return rc;
      // unpack + scan in one pass; its tile status words and counter live in `fpq` (free
      // after the count: nq + 1 u32 >= 2 * ceil(nq / kUT) + 1 words)
      const uint64_t nt = (nq + kUT - 1) / kUT;
      uint64_t* status = reinterpret_cast<uint64_t*>(
          (reinterpret_cast<uintptr_t>(fpq) + 7) & ~static_cast<uintptr_t>(7));
      uint32_t* counter = reinterpret_cast<uint32_t*>(status + nt);
      MZS_CUDA(cudaMemsetAsync(status, 0, sizeof(uint64_t) * nt + sizeof(uint32_t), st));
      const bool aligned = ((reinterpret_cast<uintptr_t>(pq) | reinterpret_cast<uintptr_t>(hit_off) |
                             reinterpret_cast<uintptr_t>(first)) & 15) == 0;
      if (aligned) {
        lookup_unpack_scan_kernel<<<(unsigned)nt, kLTPB, 0, st>>>(pq, nq, qkey, k, bucket_bits, offsets, fp, hit_off,
                                                                  first, status, counter, d_total, pos1_tab);
        MZS_LAUNCHED();
      } else {
        lookup_unpack_kernel<<<g, kLTPB, 0, st>>>(pq, nq, qkey, k, bucket_bits, offsets, fp, hit_off, first,
                                                  pos1_tab);
        MZS_LAUNCHED();
        scan_reduce_kernel<<<(unsigned)nb, kLTPB, 0, st>>>(hit_off, nq, nullptr, bsum);
        MZS_LAUNCHED();
        scan_blocks_kernel<<<1, kLTPB, 0, st>>>(bsum, nb, hit_off, nq, nullptr, d_total);
        MZS_LAUNCHED();
        scan_apply_kernel<<<(unsigned)nb, kLTPB, 0, st>>>(hit_off, nq, nullptr, bsum);
        MZS_LAUNCHED();
      }
      if (hit_cap) {
        // the multi-hit queries scan their slice from the first match on: kEmitLanes lanes per
        // query (ballots) keep the scans short and the warp converged
        if (kEmitLanes == 1 && pos1_tab) {
          lookup1_kernel<true, true><<<g, kLTPB, 0, st>>>(qkey, nq, nullptr, k, bucket_bits, offsets, fp, pos_tab,
                                                          hit_off, hit_pos, hit_cap, first, use_side2 ? side : nullptr);
        } else if (kEmitLanes == 1) {
          lookup1_kernel<true><<<g, kLTPB, 0, st>>>(qkey, nq, nullptr, k, bucket_bits, offsets, fp, pos_tab, hit_off,
                                                    hit_pos, hit_cap, first);
        } else {
          const unsigned ge = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nq * kEmitLanes + kLTPB - 1) / kLTPB,
                                                                                 (uint64_t)num_sms() * 8));
          lookup_kernel<true, kEmitLanes><<<ge, kLTPB, 0, st>>>(qkey, nq, nullptr, k, bucket_bits, offsets, fp,
                                                               pos_tab, hit_off, hit_pos, hit_cap, first);
        }
        MZS_LAUNCHED();
      }
      return SLSUM_OK;
    }
    if (kSortedQueryOrderEmit)
      lookup_sorted_count_kernel<true><<<g, kLTPB, 0, st>>>(fps, ord, nq, bucket_bits, offsets, fp, hit_off, first);
    else
      lookup_sorted_count_kernel<false><<<g, kLTPB, 0, st>>>(fps, ord, nq, bucket_bits, offsets, fp, hit_off, first);
    MZS_LAUNCHED();
    scan_reduce_kernel<<<(unsigned)nb, kLTPB, 0, st>>>(hit_off, nq, nullptr, bsum);
    MZS_LAUNCHED();
    scan_blocks_kernel<<<1, kLTPB, 0, st>>>(bsum, nb, hit_off, nq, nullptr, d_total);
    MZS_LAUNCHED();
    scan_apply_kernel<<<(unsigned)nb, kLTPB, 0, st>>>(hit_off, nq, nullptr, bsum);
    MZS_LAUNCHED();
    if (hit_cap) {
      if (kSortedQueryOrderEmit)
        lookup1_kernel<true><<<g, kLTPB, 0, st>>>(qkey, nq, nullptr, k, bucket_bits, offsets, fp, pos_tab, hit_off,
                                                  hit_pos, hit_cap, first);
      else
        lookup_sorted_kernel<true><<<g, kLTPB, 0, st>>>(fps, ord, nq, bucket_bits, offsets, fp, pos_tab, hit_off,
                                                         hit_pos, hit_cap, first);
      MZS_LAUNCHED();
    }
    return SLSUM_OK;
  }
  // lanes per query: 1 (a thread per query, the most lookups in flight) when buckets are short
  // (>= 2^26 buckets for the tables measured), else 8; MZS_LOOKUP_LANES overrides (tuning)
  static const int lanes_env = [] {
    const char* e = getenv("MZS_LOOKUP_LANES");
    const int v = e && *e ? atoi(e) : 0;
    return (v == 1 || v == 8 || v == 16 || v == 32) ? v : 0;
  }();
  const int lanes = lanes_env ? lanes_env : (bucket_bits >= 26 ? 1 : 8);
  const uint64_t want = (nq * lanes + kLTPB - 1) / kLTPB;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)num_sms() * 8));
  auto launch = [&](auto emit_tag) -> int {
    constexpr bool E = decltype(emit_tag)::value;
    uint64_t* hp = E ? hit_pos : nullptr;
    const uint64_t hc = E ? hit_cap : 0;
    if (lanes == 1)
      lookup1_kernel<E><<<grid, kLTPB, 0, st>>>(qkey, nq, d_nq, k, bucket_bits, offsets, fp, pos_tab, hit_off, hp, hc,
                                               first);
    else if (lanes == 8)
      lookup_kernel<E, 8><<<grid, kLTPB, 0, st>>>(qkey, nq, d_nq, k, bucket_bits, offsets, fp, pos_tab, hit_off, hp, hc,
                                                   first);
    else if (lanes == 32)
      lookup_kernel<E, 32><<<grid, kLTPB, 0, st>>>(qkey, nq, d_nq, k, bucket_bits, offsets, fp, pos_tab, hit_off, hp, hc,
                                                   first);
    else
      lookup_kernel<E, 16><<<grid, kLTPB, 0, st>>>(qkey, nq, d_nq, k, bucket_bits, offsets, fp, pos_tab, hit_off, hp, hc,
                                                   first);
    MZS_LAUNCHED();
    return SLSUM_OK;
  };
  int rc = launch(std::false_type{});
  if (rc) return rc;
  scan_reduce_kernel<<<(unsigned)nb, kLTPB, 0, st>>>(hit_off, nq, d_nq, bsum);
  MZS_LAUNCHED();
  scan_blocks_kernel<<<1, kLTPB, 0, st>>>(bsum, nb, hit_off, nq, d_nq, d_total);
  MZS_LAUNCHED();
  scan_apply_kernel<<<(unsigned)nb, kLTPB, 0, st>>>(hit_off, nq, d_nq, bsum);
  MZS_LAUNCHED();
  if (hit_cap) return launch(std::true_type{});
  return SLSUM_OK;
}
