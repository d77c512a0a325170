// mz.cu -- minimizer extraction (Sec. 2.4, Fig. 2) on B200.
//
// One fused kernel per tile of TW consecutive windows (a window = w consecutive k-mers):
//   phase 1  rolling 2-bit k-mer codes from the packed words (L67: k-mers are a sliding
//            sum under string concatenation, realised as a shift register) and the
//            invertible hash H_2k (R5) -> packed keys (hash << 14 | slot) in
//            shared memory; hashes never round-trip HBM.
//   phase 2  the sliding window minimum with the paper's decomposition (Alg. 2):
//            blocks of w keys, suffix minima S (Y1) and prefix minima P (X1), window
//            argmin = S[i] (+) P[i+w-1]; keys compare as (hash, position) so the minimum
//            is the leftmost one (R2).  A window emits its argmin iff it is valid and its
//            predecessor is invalid or had a different argmin (change rule, R3); emitted
//            slots are marked in a shared bitmask.
//   phase 3  ordered compaction: popcounts -> block scan -> decoupled look-back over
//            tiles (single pass, deterministic) -> (hash, pos) records.
// Fast path: w in [1,16] as a compile-time block length (S/P in registers), k <= 25.
// Generic path: any w <= 1024 and any k <= 31, S/P by block-wide segmented scans.
#include <algorithm>
#include <type_traits>

#include "ops.cuh"

namespace mzs {
namespace {

constexpr int kSlotBits = 14;  // slot index inside a tile (< 16384)
#ifndef MZS_MZ_MARK32
#define MZS_MZ_MARK32 1
#endif
#ifndef MZS_MZ_MARKW
#define MZS_MZ_MARKW 1   // FULL-strip argmin marks from the key's low word (see fast_phase2)
#endif
#ifndef MZS_MZ_OUT_U
#define MZS_MZ_OUT_U 4   // records per thread per step of the fast path's output loop
#endif
constexpr uint64_t kSlotMask = (1ull << kSlotBits) - 1;

struct DKey;  // defined with the other key types below

// H_b (R5): the masked Wang/minimap2 integer mix, all arithmetic mod 2^b.
__device__ __forceinline__ uint32_t hash_b32(uint32_t x, uint32_t m) {
  x = (x * 0x1FFFFFu - 1u) & m;  // (2^21-1) x - 1
  x ^= x >> 24;
  x = (x * 265u) & m;
  x ^= x >> 14;
  x = (x * 21u) & m;
  x ^= x >> 28;
  x = (x * 0x80000001u) & m;     // (2^31+1) x
  return x;
}
__device__ __forceinline__ uint64_t hash_b64(uint64_t x, uint64_t m) {
  x = (x * 0x1FFFFFull - 1ull) & m;
  x ^= x >> 24;
  x = (x * 265ull) & m;
  x ^= x >> 14;
  x = (x * 21ull) & m;
  x ^= x >> 28;
  x = (x * 0x80000001ull) & m;
  return x;
}

// Reverse complement of a k-mer code (R32): complement every base (b -> 3 - b =
// bitwise not of its 2 bits) and reverse the order of the 2-bit groups.  Bit-reversal then a
// swap of the two bits of every group reverses the groups of a 64/32-bit word; the shift
// drops the complemented garbage above 2k bits.
__device__ __forceinline__ uint64_t revcomp64(uint64_t code, int k) {
  uint64_t x = __brevll(~code);
  x = ((x >> 1) & 0x5555555555555555ull) | ((x & 0x5555555555555555ull) << 1);
  return x >> (64 - 2 * k);
}
__device__ __forceinline__ uint32_t revcomp32(uint32_t code, int k) {
  uint32_t x = __brev(~code);
  x = ((x >> 1) & 0x55555555u) | ((x & 0x55555555u) << 1);
  return x >> (32 - 2 * k);
}

struct MzArgs {
  const uint64_t* words;     // packed bases (MSB-first, 32 per word)
  const uint32_t* invalid;   // invalid bitmap or nullptr
  uint64_t nwords;
  uint64_t n;                // bases
  uint64_t nwin;             // windows = n - (k+w-1) + 1
  const uint64_t* read_off;  // nreads+1 or nullptr
  uint64_t nreads;
  uint64_t pos_base, win_lo, win_hi;
  int k, w, raw, canon;      // key mode: raw code (R4) / canonical strand (R32)
  uint64_t* out_hash;
  uint64_t* out_pos;
  uint64_t* out_items;       // optional packed seed-table items (fp << 32 | pos mod 2^32)
  uint64_t capacity;
  uint64_t* d_count;
  uint64_t* status;          // look-back tile status [ntiles]
  uint32_t* tile_counter;
  uint64_t ntiles;
  uint32_t tw;               // windows per tile
  const uint64_t* ridx;      // coarse read index (kRidxShift), or nullptr
  // first radix pass digit counts of the seed table (mz_out.hist) or nullptr: record r adds 1
  // to hist[((fp >> hist_sh) & hist_mask) * hist_nch + r / hist_chunk]
  uint32_t* hist;
  uint64_t hist_nch;
  uint32_t hist_chunk;
  int hist_sh;
  uint32_t hist_mask;
};
// ridx[b] = first read r in [0, nreads+1] with read_off[r] >= b * 2^kRidxShift: brackets every
// read-start search to the reads of one 8 kbp block (a few loads instead of ~20 dependent ones)
constexpr int kRidxShift = 13;

// packed seed-table item of a record (seedtable_build_items): the fingerprint (the top 32 bits
// of the 2k-bit key, R21) over the position mod 2^32
__device__ __forceinline__ uint64_t item_of(uint64_t h, int k, uint64_t pos) {
  const int b = 2 * k;
  const uint32_t f = b >= 32 ? (uint32_t)(h >> (b - 32)) : (uint32_t)(h << (32 - b));
  return ((uint64_t)f << 32) | (uint32_t)pos;
}
__device__ __forceinline__ uint64_t ldw(const MzArgs& a, int64_t i) {
  return (i >= 0 && (uint64_t)i < a.nwords) ? __ldg(a.words + i) : 0ull;
}
__device__ __forceinline__ uint32_t ldi(const MzArgs& a, int64_t i) {
  return (a.invalid && i >= 0 && (uint64_t)i < a.nwords) ? __ldg(a.invalid + i) : 0u;
}
// bits for bases [lo, lo+64): bit j <-> base lo+j is invalid
__device__ __forceinline__ uint64_t inv_window64(const MzArgs& a, int64_t lo) {
  const int64_t wi = lo >> 5;
  const uint32_t sh = (uint32_t)(lo & 31);
  const uint64_t ab = (uint64_t)ldi(a, wi) | ((uint64_t)ldi(a, wi + 1) << 32);
  const uint64_t c = ldi(a, wi + 2);
  return sh ? (ab >> sh) | (c << (64 - sh)) : ab;
}
// first index r in [0, nreads+1] with read_off[r] > x  (read_off[nreads] = n)
__device__ __forceinline__ uint64_t upper_read(const MzArgs& a, int64_t x) {
  uint64_t lo = 0, hi = a.nreads + 1;
  if (a.ridx) {
    if (x < 0) {
      hi = __ldg(a.ridx);                 // reads starting at 0 .. : none <= x
    } else if ((uint64_t)x >= a.n) {
      lo = a.nreads + 1;                  // read_off[nreads] = n <= x
    } else {
      const uint64_t b = (uint64_t)x >> kRidxShift;
      lo = __ldg(a.ridx + b);             // read_off[r] < b 2^S <= x for r < lo
      hi = __ldg(a.ridx + b + 1);         // read_off[hi] >= (b+1) 2^S > x
    }
  }
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if ((int64_t)__ldg(a.read_off + mid) > x) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// ------------------------------------------------------------------ phase 1
// OR the bits of v into the shared bitmask m starting at bit s0
__device__ __forceinline__ void or_bits(uint32_t* m, uint32_t s0, uint64_t v) {
  const uint32_t w0 = s0 >> 5, sh = s0 & 31;
  const uint32_t lo = (uint32_t)(v << sh), mid = (uint32_t)(v >> (32 - sh));
  const uint32_t hi = sh ? (uint32_t)(v >> (64 - sh)) : 0u;
  if (lo) atomicOr(&m[w0], lo);
  if (mid) atomicOr(&m[w0 + 1], mid);
  if (hi) atomicOr(&m[w0 + 2], hi);
}

// Keys of k-mers q0 .. q0+Q-1 into slots s0 .. s0+Q-1.  If CHECK, bit `slot` of the shared
// bitmask wvb (zeroed by the caller) is set iff the window whose LAST k-mer is that slot's
// k-mer is valid (run of valid same-read bases ending at the k-mer's last base >= k+w-1).
// KK != 0: k is the compile-time constant KK (lets the compiler drop the masking and the
// xor-shift work on the always-zero high bits); KM bit 0 (RAW): keys are the codes themselves;
// KM bit 1 (CANON): the code is min(forward, reverse complement), the reverse complement
// rolled alongside (the entering base's complement enters at the top, R32).
template <class Key, int Q, bool H64, bool CHECK, int KK = 0, int KM = 0, int WC = 0>
__device__ __forceinline__ void phase1_keys(const MzArgs& a, int64_t q0, uint32_t s0, Key* keys, uint32_t* wvb,
                                            const uint64_t* pre = nullptr, const int64_t* rs = nullptr,
                                            int nrs = -1) {
  // rs[0 .. nrs): every read start the caller's tile range holds (shared memory), or nrs < 0
  static_assert(Q <= 33, "validity bits of one strip fit in a u64 shifted by < 32");
  uint64_t vbits = 0;
  const int k = KK ? KK : a.k;
  const int64_t wi = q0 >> 5;
  const uint32_t off = (uint32_t)(q0 & 31) * 2;
  // pre: the three packed words, already loaded by the caller (prefetched a phase earlier)
  const uint64_t A = pre ? pre[0] : ldw(a, wi), B = pre ? pre[1] : ldw(a, wi + 1), C = pre ? pre[2] : ldw(a, wi + 2);
  const uint64_t X = off ? (A << off) | (B >> (64 - off)) : A;
  const uint64_t Y = off ? (B << off) | (C >> (64 - off)) : B;
  // stream of the bases entering after the first k-mer: q0+k, q0+k+1, ...
  uint64_t Z = (X << (2 * k)) | (Y >> (64 - 2 * k));
  uint32_t run = 0;
  uint64_t iv = 0;
  int64_t next_rs = INT64_MAX;
  uint64_t ri = 0;
  const int span = k + (WC ? WC : a.w) - 1;  // compile-time with KK and WC (w) both given
  // BULK validity (the strip's windows and their bases fit one 64-bit mask): window s (last
  // k-mer q0+s) covers bases [L+s, L+s+span), L = q0-w+1.  It is invalid iff an invalid base
  // lies in that range -- the OR of the invalid bits over span positions, by doubling and one
  // overlapping OR (the idempotent-op trick of the sliding sums themselves) -- or a read
  // starts in (L+s, L+s+span).  Same result as the run counter below, without a walk.
  const bool bulk = CHECK && Q + span - 1 <= 64;
  if (bulk) {
    const int64_t L = q0 - (span - k);
    uint64_t T = inv_window64(a, L);  // bit j <-> base L+j invalid
    int p = 1;
    while (2 * p <= span) {
      T |= T >> p;
      p *= 2;
    }
    uint64_t bad = T | (T >> (span - p));
    if (a.read_off) {
      const int64_t last = L + Q + span - 2;  // last base of the strip's last window
      auto drop = [&](int64_t r) {            // windows with a read start in (first, last base]
        const int64_t hi = min(r - L - 1, (int64_t)63), lo = max(r - L - span + 1, (int64_t)0);
        if (hi >= lo) bad |= ((2ull << (hi - lo)) - 1ull) << lo;
      };
      if (nrs >= 0) {
        for (int i = 0; i < nrs; ++i) {
          const int64_t r = rs[i];
          if (r > L && r <= last) drop(r);
        }
      } else {
        for (uint64_t r_i = upper_read(a, L); r_i <= a.nreads; ++r_i) {
          const int64_t r = (int64_t)__ldg(a.read_off + r_i);  // > L
          if (r > last) break;
          drop(r);
        }
      }
    }
    vbits = ~bad & ((1ull << Q) - 1ull);
  } else if (CHECK) {
    // run length at base x0 = q0 + k - 2 (capped at span), then walk base by base
    const int64_t x0 = q0 + k - 2;
    // last invalid base in [x0-span+1, x0], scanning back 64 bases at a time (span may exceed 64)
    int64_t start = x0 - span + 1;
    for (int64_t hi = x0; hi >= x0 - span + 1; hi -= 64) {
      const int64_t lo = max(hi - 63, x0 - span + 1);
      const int cnt = (int)(hi - lo + 1);
      const uint64_t bits = inv_window64(a, lo) & (cnt >= 64 ? ~0ull : ((1ull << cnt) - 1));
      if (bits) {
        start = lo + (63 - __clzll(bits)) + 1;
        break;
      }
    }
    if (a.read_off) {
      ri = upper_read(a, x0);                 // first read start > x0
      const int64_t rs = ri ? (int64_t)__ldg(a.read_off + ri - 1) : 0;
      if (rs > start) start = rs;
      next_rs = ri <= a.nreads ? (int64_t)__ldg(a.read_off + ri) : INT64_MAX;
    }
    run = (uint32_t)max((int64_t)0, x0 - start + 1);
    iv = inv_window64(a, x0 + 1);  // bit s <-> base x0+1+s = last base of k-mer q0+s
  }
  const int kk = 2 * k;
  if (H64) {
    // 2k > 32: the low word of the mask is all ones (lets the compiler mask the high word only)
    const uint64_t km = ((uint64_t)((1u << (kk - 32)) - 1u) << 32) | 0xffffffffull;
    constexpr bool RAW = KM & 1, CANON = KM & 2;
    uint64_t code = X >> (64 - kk);
    uint64_t rc = CANON ? revcomp64(code, k) : 0;
    // DIRECT (compile-time k, hashed forward keys): every code is cut straight out of the
    // aligned 128-bit stream X:Y with two constant funnel shifts instead of rolling 2 bits per
    // base.  The high word keeps the stream bits above the code (garbage above bit 2k), which
    // the hash's first step, (x (2^21-1) - 1) mod 2^2k, discards.
    constexpr bool DIRECT = KK > 0 && KM == 0 && 2 * (Q - 1) + 2 * KK <= 128;
    const uint32_t sw[5] = {0u, (uint32_t)(X >> 32), (uint32_t)X, (uint32_t)(Y >> 32), (uint32_t)Y};
    // the 32 stream bits starting at stream bit b (b >= -32; bits before the stream read as 0)
    auto cut = [&](int b) -> uint32_t {
      const int j = (b + 32) >> 5, r = (b + 32) & 31;
      return r ? __funnelshift_l(sw[j + 1], sw[j], r) : sw[j];
    };
#pragma unroll
    for (int s = 0; s < Q; ++s) {
      if (DIRECT) {
        code = ((uint64_t)cut(2 * s + 2 * KK - 64) << 32) | cut(2 * s + 2 * KK - 32);
      } else if (s > 0) {
        if (CANON) rc = (rc >> 2) | ((uint64_t)(3u - (uint32_t)(Z >> 62)) << (kk - 2));
        code = ((code << 2) | (Z >> 62)) & km;
        Z <<= 2;
      }
      if (CHECK && !bulk) {
        const int64_t x = q0 + s + k - 1;
        const uint32_t inv = (uint32_t)(iv >> s) & 1u;
        if (x == next_rs) {
          run = 0;
          next_rs = (++ri <= a.nreads) ? (int64_t)__ldg(a.read_off + ri) : INT64_MAX;
          while (next_rs <= x) next_rs = (++ri <= a.nreads) ? (int64_t)__ldg(a.read_off + ri) : INT64_MAX;
        }
        run = inv ? 0u : run + 1u;
        vbits |= (uint64_t)(run >= (uint32_t)span) << s;
      }
      const uint64_t c = (CANON && rc < code) ? rc : code;
      const uint64_t h = RAW ? c : hash_b64(c, km);
      keys[s0 + s] = Key::make(h, s0 + s);
    }
  } else {
    const uint32_t km = (kk == 32) ? 0xffffffffu : ((1u << kk) - 1u);
    constexpr bool RAW = KM & 1, CANON = KM & 2;
    uint32_t code = (uint32_t)(X >> (64 - kk));
    uint32_t rc = CANON ? revcomp32(code, k) : 0u;
    // DIRECT as in the 64-bit branch: one constant funnel shift per code (garbage above bit
    // 2k is discarded by the hash's first step)
    constexpr bool DIRECT = KK > 0 && KM == 0 && 2 * (Q - 1) + 2 * KK <= 128;
    const uint32_t sw[5] = {0u, (uint32_t)(X >> 32), (uint32_t)X, (uint32_t)(Y >> 32), (uint32_t)Y};
    auto cut = [&](int b) -> uint32_t {
      const int j = (b + 32) >> 5, r = (b + 32) & 31;
      return r ? __funnelshift_l(sw[j + 1], sw[j], r) : sw[j];
    };
#pragma unroll
    for (int s = 0; s < Q; ++s) {
      if (DIRECT) {
        code = cut(2 * s + 2 * KK - 32);
      } else if (s > 0) {
        if (CANON) rc = (rc >> 2) | ((3u - (uint32_t)(Z >> 62)) << (kk - 2));
        code = ((code << 2) | (uint32_t)(Z >> 62)) & km;
        Z <<= 2;
      }
      if (CHECK && !bulk) {
        const int64_t x = q0 + s + k - 1;
        const uint32_t inv = (uint32_t)(iv >> s) & 1u;
        if (x == next_rs) {
          run = 0;
          next_rs = (++ri <= a.nreads) ? (int64_t)__ldg(a.read_off + ri) : INT64_MAX;
          while (next_rs <= x) next_rs = (++ri <= a.nreads) ? (int64_t)__ldg(a.read_off + ri) : INT64_MAX;
        }
        run = inv ? 0u : run + 1u;
        vbits |= (uint64_t)(run >= (uint32_t)span) << s;
      }
      const uint32_t c = (CANON && rc < code) ? rc : code;
      const uint32_t h = RAW ? c : hash_b32(c, km);
      if constexpr (std::is_same<Key, DKey>::value) {
        // h * 2^14 + slot as one 32x32->64 multiply-add (FMA pipe), then the exponent bits
        unsigned long long v;
        const unsigned long long c = (0x43300000ull << 32) | (s0 + s);
        asm("mad.wide.u32 %0, %1, 16384, %2;" : "=l"(v) : "r"(h), "l"(c));
        keys[s0 + s] = Key{v};
      } else {
        keys[s0 + s] = Key::make(h, s0 + s);
      }
    }
  }
  if (CHECK && vbits) or_bits(wvb, s0, vbits);
}

__device__ __forceinline__ bool wv_bit(const uint32_t* wvb, int s) { return (wvb[s >> 5] >> (s & 31)) & 1u; }
// bits b .. b+63 of a shared bitmask (the words up to (b >> 5) + 2 must exist)
__device__ __forceinline__ uint64_t bits64(const uint32_t* m, int b) {
  const int w0 = b >> 5, sh = b & 31;
  const uint64_t v = ((uint64_t)m[w0 + 1] << 32) | m[w0];
  return sh ? (v >> sh) | ((uint64_t)m[w0 + 2] << (64 - sh)) : v;
}

// Packed key: (hash << 14) | slot -- lexicographic (hash, position) order in one u64.
struct PackedKey {
  unsigned long long v;
  __device__ __forceinline__ static PackedKey make(uint64_t h, uint32_t slot) {
    return PackedKey{(h << kSlotBits) | slot};
  }
  __device__ __forceinline__ uint32_t slot() const { return (uint32_t)(v & kSlotMask); }
  __device__ __forceinline__ uint64_t hash() const { return v >> kSlotBits; }
  __device__ __forceinline__ bool operator!=(const PackedKey& o) const { return v != o.v; }
};
__device__ __forceinline__ PackedKey kmin(PackedKey a, PackedKey b) { return a.v <= b.v ? a : b; }

// The same packed key with the bit pattern of the double 2^52 + (hash << 14 | slot): for keys
// below 2^52 (2k <= 38) the IEEE order of these doubles is the integer order, so one FP64
// compare (DSETP, on the FP64 pipe) replaces the two 32-bit compares a 64-bit integer min
// needs on the ALU pipe -- the minimizer kernel is ALU-issue bound.
struct DKey {
  unsigned long long v;
  __device__ __forceinline__ static DKey make(uint64_t h, uint32_t slot) {
    // = 0x43300000'00000000 | h << 14 | slot, as two multiply-adds on the FMA pipe (the bit
    // fields do not overlap, so + is |): IMAD.WIDE.U32 of the low word with {slot, exponent}
    // as addend, then IMAD of the high word into the upper half.
    static_assert(kSlotBits == 14, "multiplier below assumes 14 slot bits");
    unsigned long long lo;
    uint32_t hi;
    const unsigned long long c = (0x43300000ull << 32) | slot;
    asm("mad.wide.u32 %0, %1, 16384, %2;" : "=l"(lo) : "r"((uint32_t)h), "l"(c));
    asm("mad.lo.u32 %0, %1, 16384, %2;" : "=r"(hi) : "r"((uint32_t)(h >> 32)), "r"((uint32_t)(lo >> 32)));
    return DKey{((unsigned long long)hi << 32) | (uint32_t)lo};
  }
  __device__ __forceinline__ uint32_t slot() const { return (uint32_t)(v & kSlotMask); }
  __device__ __forceinline__ uint64_t hash() const { return (v & 0x000FFFFFFFFFFFFFull) >> kSlotBits; }
  __device__ __forceinline__ bool operator!=(const DKey& o) const { return v != o.v; }
};
__device__ __forceinline__ DKey kmin(DKey a, DKey b) {
  unsigned long long r;
  asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, %2;\n\tselp.b64 %0, %3, %4, p;\n\t}"
      : "=l"(r)
      : "d"(__longlong_as_double((long long)a.v)), "d"(__longlong_as_double((long long)b.v)), "l"(a.v), "l"(b.v));
  return DKey{r};
}

// Wide key for 2k > 50: hash and slot kept apart (ties broken by the slot).
struct WideKey {
  unsigned long long h;
  uint32_t s;
  uint32_t pad;
  __device__ __forceinline__ static WideKey make(uint64_t h, uint32_t slot) { return WideKey{h, slot, 0}; }
  __device__ __forceinline__ uint32_t slot() const { return s; }
  __device__ __forceinline__ uint64_t hash() const { return h; }
  __device__ __forceinline__ bool operator!=(const WideKey& o) const { return h != o.h || s != o.s; }
};
__device__ __forceinline__ WideKey kmin(WideKey a, WideKey b) {
  return (a.h < b.h || (a.h == b.h && a.s <= b.s)) ? a : b;
}

template <class Key>
struct OpKeyMin {
  using T = Key;
  static constexpr bool kCommutative = true, kIdempotent = true;
  __device__ __forceinline__ static T id() { return T::make(~0ull >> kSlotBits, (uint32_t)kSlotMask); }
  __device__ __forceinline__ static T op(T a, T b) { return kmin(a, b); }
};
template <>
__device__ __forceinline__ WideKey OpKeyMin<WideKey>::id() { return WideKey{~0ull, 0xffffffffu, 0}; }

// shuffles of the key types (used by the generic path's segmented scans)
__device__ __forceinline__ PackedKey shfl_up(PackedKey v, int o) { return PackedKey{__shfl_up_sync(0xffffffffu, v.v, o)}; }
__device__ __forceinline__ PackedKey shfl_down(PackedKey v, int o) { return PackedKey{__shfl_down_sync(0xffffffffu, v.v, o)}; }
__device__ __forceinline__ WideKey shfl_up(WideKey v, int o) {
  return WideKey{__shfl_up_sync(0xffffffffu, v.h, o), __shfl_up_sync(0xffffffffu, v.s, o), 0};
}
__device__ __forceinline__ WideKey shfl_down(WideKey v, int o) {
  return WideKey{__shfl_down_sync(0xffffffffu, v.h, o), __shfl_down_sync(0xffffffffu, v.s, o), 0};
}

}  // namespace
// make the key shuffles visible to the segmented-scan templates in ops.cuh (ADL)
}  // namespace mzs

namespace mzs {
namespace {

// Tile cleanliness: no invalid base and no read start strictly inside the tile's bases.
template <int TPB>
__device__ __forceinline__ bool tile_is_clean(const MzArgs& a, int64_t b_lo, int64_t b_hi, const uint32_t* pre = nullptr) {
  int dirty = 0;
  if (a.invalid) {
    const int64_t w0 = max((int64_t)0, b_lo >> 5), w1 = min((int64_t)a.nwords - 1, (b_hi - 1) >> 5);
    for (int64_t wi = w0 + threadIdx.x; wi <= w1; wi += TPB) {
      // pre: this thread's first word, prefetched by the caller
      uint32_t m = (pre && wi == w0 + (int64_t)threadIdx.x) ? *pre : __ldg(a.invalid + wi);
      // restrict to [b_lo, b_hi)
      const int64_t base = wi << 5;
      if (base < b_lo) m &= 0xffffffffu << (uint32_t)(b_lo - base);
      if (base + 32 > b_hi) m &= (b_hi - base >= 32) ? 0xffffffffu : ((1u << (uint32_t)(b_hi - base)) - 1u);
      dirty |= (m != 0);
    }
  }
  if (a.read_off && threadIdx.x == 0) {
    const uint64_t r = upper_read(a, b_lo);  // first read start > b_lo
    if (r <= a.nreads && (int64_t)__ldg(a.read_off + r) < b_hi) dirty = 1;
  }
  return !__syncthreads_or(dirty);
}

// Sub-tile dirty map: bit u of dwm <-> packed word W0 + u (W0 = b_lo >> 5) holds an invalid
// base or a read start inside [b_lo, b_hi) (b_lo itself excluded for read starts, as a read
// may start at the first base).  Returns true iff the whole sub-tile is clean; warps of a
// dirty sub-tile test their own range of words (warp_dirty) and take the validity-free
// phase 1 when it is clean -- with ~1 read start per 10 kbp (C4) most warps are.
template <int TPB, int DW>
__device__ __forceinline__ bool subtile_dirty_map(const MzArgs& a, int64_t b_lo, int64_t b_hi, uint32_t* dwm,
                                                  const uint32_t* pre, const int64_t* rs, const int* p_nrs) {
  const int64_t W0 = b_lo >> 5;
  int dirty = 0;
  if (a.invalid) {
    const int64_t w0 = max((int64_t)0, W0), w1 = min((int64_t)a.nwords - 1, (b_hi - 1) >> 5);
    for (int64_t wi = w0 + threadIdx.x; wi <= w1; wi += TPB) {
      uint32_t m = (pre && wi == w0 + (int64_t)threadIdx.x) ? *pre : __ldg(a.invalid + wi);
      const int64_t base = wi << 5;
      if (base < b_lo) m &= 0xffffffffu << (uint32_t)(b_lo - base);
      if (base + 32 > b_hi) m &= (b_hi - base >= 32) ? 0xffffffffu : ((1u << (uint32_t)(b_hi - base)) - 1u);
      if (m) {
        dirty = 1;
        const uint32_t u = (uint32_t)(wi - W0);
        atomicOr(&dwm[u >> 5], 1u << (u & 31));
      }
    }
  }
  const int nrs = (a.read_off && p_nrs && threadIdx.x < 32) ? *p_nrs : -1;  // (warp 0 wrote it)
  if (a.read_off && threadIdx.x < 32 && nrs >= 0) {
    // the super-tile's read starts are in shared memory
    for (int i = threadIdx.x; i < nrs; i += 32) {
      const int64_t r = rs[i];
      if (r > b_lo && r < b_hi) {
        dirty = 1;
        const uint32_t u = (uint32_t)((r >> 5) - (b_lo >> 5));
        atomicOr(&dwm[u >> 5], 1u << (u & 31));
      }
    }
  } else if (a.read_off && threadIdx.x < 32) {
    // read starts r with b_lo < r < b_hi: warp 0 walks them 32 at a time
    uint64_t r0 = 0;
    if (threadIdx.x == 0) r0 = upper_read(a, b_lo);
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    for (uint64_t r = r0 + threadIdx.x;; r += 32) {
      const bool in = r <= a.nreads && (int64_t)__ldg(a.read_off + r) < b_hi;
      if (in) {
        dirty = 1;
        const uint32_t u = (uint32_t)(((int64_t)__ldg(a.read_off + r) >> 5) - W0);
        atomicOr(&dwm[u >> 5], 1u << (u & 31));
      }
      if (!__all_sync(0xffffffffu, in)) break;
    }
  }
  return !__syncthreads_or(dirty);
}

// Code + key of the k-mer at local position q, from scratch (phase 3 re-derives the hash
// of every emitted position instead of keeping all keys of a super-tile resident).
template <bool H64, int KK = 0, int CNM = -1>
__device__ __forceinline__ uint64_t key_from_words(const MzArgs& a, int64_t q, uint64_t A, uint64_t B) {
  const bool canon = CNM < 0 ? a.canon != 0 : CNM == 1;
  const uint32_t off = (uint32_t)(q & 31) * 2;
  const uint64_t X = off ? (A << off) | (B >> (64 - off)) : A;
  const int kk = 2 * (KK ? KK : a.k);
  if (H64) {
    uint64_t code = X >> (64 - kk);
    if (canon) code = min(code, revcomp64(code, kk / 2));
    const uint64_t km = ((uint64_t)((1u << (kk - 32)) - 1u) << 32) | 0xffffffffull;
    return a.raw ? code : hash_b64(code, km);
  } else {
    uint32_t code = (uint32_t)(X >> (64 - kk));
    if (canon) code = min(code, revcomp32(code, kk / 2));
    const uint32_t km = (kk == 32) ? 0xffffffffu : ((1u << kk) - 1u);
    return a.raw ? code : hash_b32(code, km);
  }
}
template <bool H64, int KK = 0, int CNM = -1>
__device__ __forceinline__ uint64_t key_at(const MzArgs& a, int64_t q) {
  return key_from_words<H64, KK, CNM>(a, q, ldw(a, q >> 5), ldw(a, (q >> 5) + 1));
}

// Phase 3: ordered output of the slots marked in `emit` (S sub-tiles x NS slots each; slot s
// of sub-tile u is the k-mer sub_lo(u) - 1 + s).  The set bits are first compacted, in order,
// into a shared list of super-tile slot indices (the keys' smem, no longer needed); one
// look-back per super-tile; then one thread per record re-derives the hash and writes.
template <int TPB, bool H64>
__device__ __forceinline__ void phase3_output(const MzArgs& a, uint64_t tile, int64_t super_lo, int NS, int nsub,
                                              const uint32_t* emit, uint16_t* list, uint64_t* warp_sums,
                                              uint64_t* bcast) {
  const int nsw = nsub * (NS / 32);
  const int wpt = (nsw + TPB - 1) / TPB;
  const int u0 = threadIdx.x * wpt;
  const int u1 = min(nsw, u0 + wpt);
  uint32_t cnt = 0;
  for (int u = u0; u < u1; ++u) cnt += __popc(emit[u]);
  uint64_t total;
  uint32_t o = (uint32_t)block_exclusive_sum<TPB, uint64_t>(cnt, warp_sums, &total);
  for (int u = u0; u < u1; ++u) {
    uint32_t bits = emit[u];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      list[o++] = (uint16_t)(u * 32 + b);
    }
  }
  if (warp_id() == 0) {
    const uint64_t off = lookback_exclusive(a.status, tile, total);
    if (lane_id() == 0) {
      *bcast = off;
      if (tile == a.ntiles - 1) *a.d_count = off + total;
    }
  }
  __syncthreads();
  const uint64_t base = *bcast;
  const uint32_t nrec = (uint32_t)total;
  for (uint32_t i = threadIdx.x; i < nrec; i += TPB) {
    const uint64_t oo = base + i;
    if (oo >= a.capacity) break;
    const int slot_all = list[i];
    const int sub = slot_all / NS, slot = slot_all - sub * NS;
    const int64_t q = super_lo + (int64_t)sub * a.tw - 1 + slot;
    const uint64_t h = key_at<H64>(a, q);
    a.out_hash[oo] = h;
    a.out_pos[oo] = a.pos_base + (uint64_t)q;
    const uint64_t it = item_of(h, a.k, a.pos_base + (uint64_t)q);
    if (a.out_items) a.out_items[oo] = it;
    if (a.hist) atomicAdd(&a.hist[(((uint32_t)(it >> 32) >> a.hist_sh) & a.hist_mask) * a.hist_nch + oo / a.hist_chunk], 1u);
  }
}

// ------------------------------------------------------------------ fast path kernel
template <int W>
struct FastGeom {
  static constexpr int TPB = 256;
  static constexpr int M0 = (32 / W) > 0 ? (32 / W) : 1;
  // R = M*W even so that Q = R + 1 is odd (conflict-free strided key stores), Q <= 33
  static constexpr int M = ((M0 * W) % 2 == 0) ? M0 : (M0 > 1 ? M0 - 1 : 2);
  static constexpr int R = M * W;
  static constexpr int Q = R + 1;
  static constexpr int TW = TPB * R;     // windows per sub-tile
  static constexpr int NS = TPB * Q;     // key slots per sub-tile
  static constexpr int NSW = NS / 32;
  static constexpr int SUBS = 4;         // sub-tiles per super-tile (one look-back each)
  static_assert(Q <= 33, "phase-1 rolling window holds 32 bases");
  static_assert(R + W <= 64, "per-thread emission mask");
  static_assert(NS < (1 << kSlotBits), "slot bits");
  static_assert(SUBS * NS * 2 <= NS * 8 && SUBS * NS < 65536, "phase-3 slot list fits in the keys smem");
  static_assert((SUBS - 1) * TW + NS <= 65536, "phase-3 list entries (k-mer offsets) fit 16 bits");
  static_assert(TPB >= W + 1, "halo slots");
};

// Phase 2 for one sub-tile: thread t owns windows jb .. jb+R-1 (window j = slots j+1 .. j+W).
// [vlo, vhi): windows that exist; [elo, ehi): windows allowed to emit (shard range).
// FULL: every window of the strip (and the one before it) is valid and may emit -- the
// common case -- so the per-window work is the 3 minima plus the change test.
template <int W, bool CHECK, bool FULL, class Key, bool MASKED = false>
__device__ __forceinline__ void fast_phase2(const Key* keys, const uint32_t* wvb, int vlo, int vhi, int elo,
                                            int ehi, uint32_t* emit, uint64_t vm = ~0ull) {
  // MASKED (with FULL): the strip lies inside the emission range but some of its windows are
  // invalid (a read start or an N nearby); vm bit i = window jb-1+i is valid.  The argmin of
  // every valid window is marked: the same set as the change rule, since the argmin of two
  // valid windows can only coincide when every window between them is valid (D3).
  using G = FastGeom<W>;
  const int jb = threadIdx.x * G::R;
  Key S[W], kb[W];
  uint32_t sprev;  // slot of the previous window's argmin
  uint32_t s_carry;  // argmin slot of window jb-1 (FULL strips)
  bool vprev;
  uint64_t em = 0;  // bit i <-> slot jb + 1 + i
  // FULL unmasked strips mark into a 32-bit mask per block of W windows (their argmins lie in
  // the block's slots + W - 1 more: < 2W <= 32 bits), folded into em once per block
  constexpr bool kM32 = FULL && MZS_MZ_MARK32;
  uint32_t m32 = 0, mbase = 0;
  uint32_t vmb = 0;  // (MASKED) validity of the block's windows: bit c <-> window jblk + c
  auto valid_of = [&](int j) -> bool {
    if (FULL) return true;
    const bool in = (unsigned)(j - vlo) < (unsigned)(vhi - vlo);
    return CHECK ? (in && wv_bit(wvb, j + W)) : in;
  };
  auto visit = [&](int j, Key y) {
    const uint32_t s = y.slot();
    if (FULL) {
      // every window's argmin is marked (argmins never decrease, so a repeat hits the same
      // bit); the carried-in argmin of window jb-1, owned by the strip on the left, is cleared
      // once after the strip (R3)
      if (kM32 && MASKED) {
        MZS_DCHECK(s - mbase < 32u);
#if MZS_MZ_MARKW
        m32 |= __funnelshift_l(0u, (vmb >> (uint32_t)(j - (int)mbase + 1)) & 1u, (uint32_t)y.v - mbase);
#else
        m32 |= ((vmb >> (uint32_t)(j - (int)mbase + 1)) & 1u) << (s - mbase);
#endif
      } else if (MASKED) {
        em |= (uint64_t)((vm >> (j - jb + 1)) & 1u) << (s - (uint32_t)(jb + 1));
      } else if (kM32) {
        MZS_DCHECK(s - mbase < 32u);
#if MZS_MZ_MARKW
        // (low key word - mbase) mod 32 = s - mbase: the slot is the key's low 14 bits and
        // s >= mbase, so the subtraction borrows nothing from above them; the wrapping funnel
        // shift uses only those 5 bits (no slot mask)
        m32 |= __funnelshift_l(0u, 1u, (uint32_t)y.v - mbase);
#else
        m32 |= 1u << (s - mbase);
#endif
      } else {
        MZS_DCHECK(s - (uint32_t)(jb + 1) < 64u);
        em |= 1ull << (s - (uint32_t)(jb + 1));
      }
    } else {
      const bool v = valid_of(j);
      const bool e = v && (!vprev || s != sprev) && ((unsigned)(j - elo) < (unsigned)(ehi - elo));
      em |= (uint64_t)e << (s - (uint32_t)(jb + 1));
      vprev = v;
    }
    sprev = s;
  };
  {
    const Key k0 = keys[jb];
#pragma unroll
    for (int q = 0; q < W; ++q) kb[q] = keys[jb + 1 + q];
    Key p = kb[0];
#pragma unroll
    for (int q = 1; q < W - 1; ++q) p = kmin(p, kb[q]);
    sprev = ((W == 1) ? k0 : kmin(k0, p)).slot();
    s_carry = sprev;
    vprev = valid_of(jb - 1);
    S[W - 1] = kb[W - 1];
#pragma unroll
    for (int q = W - 2; q >= 0; --q) S[q] = kmin(kb[q], S[q + 1]);
  }
#pragma unroll 1
  for (int b = 1; b <= G::M; ++b) {
    const int jblk = jb + (b - 1) * W;
    if (kM32) {
      m32 = 0;
      mbase = (uint32_t)(jblk + 1);
      if (MASKED) vmb = (uint32_t)(vm >> (jblk - jb + 1));
    }
    visit(jblk, S[0]);
    const int sb = jb + 1 + b * W;
#pragma unroll
    for (int q = 0; q < W; ++q) kb[q] = keys[sb + q];
    Key p = kb[0];
#pragma unroll
    for (int q = 0; q < W - 1; ++q) {
      if (q > 0) p = kmin(p, kb[q]);
      visit(jblk + q + 1, kmin(S[q + 1], p));
    }
    S[W - 1] = kb[W - 1];
#pragma unroll
    for (int q = W - 2; q >= 0; --q) S[q] = kmin(kb[q], S[q + 1]);
    if (kM32) em |= (uint64_t)m32 << (jblk - jb);
  }
  if (FULL && (!MASKED || (vm & 1u))) {  // (an invalid window jb-1 carries no record)
    const uint32_t rel = s_carry - (uint32_t)(jb + 1);  // wraps (large) when the carry is left of the strip
    if (rel < 64u) em &= ~(1ull << rel);
  }
  // OR the strip's mask into the shared bitmask (slots jb+1 .. jb+R+W)
  if (em) {
    const int s0 = jb + 1;
    const int w0 = s0 >> 5, sh = s0 & 31;
    const uint32_t lo = (uint32_t)(em << sh);
    const uint32_t mid = (uint32_t)(em >> (32 - sh));
    const uint32_t hi = sh ? (uint32_t)(em >> (64 - sh)) : 0u;
    if (lo) atomicOr(&emit[w0], lo);
    if (mid) atomicOr(&emit[w0 + 1], mid);
    if (hi) atomicOr(&emit[w0 + 2], hi);
  }
}

#define G_TPB_OF(W) (FastGeom<W>::TPB)
// Output of one finished super-tile (fast path): its emit bitmask -> ordered slot list in
// `list` -> prefix via look-back -> records.  Called one super-tile LATE (see the kernel), so
// the look-back finds its predecessors' aggregates already published.
template <int W, bool H64, int KK, bool CN>
__device__ __forceinline__ void fast_output(const MzArgs& a, uint64_t tile, const uint32_t* emit, uint32_t excl,
                                            uint32_t total, uint16_t* list, uint64_t* bcast, uint32_t* shist) {
  // shist[2][256]: this super-tile's first-radix-pass digit counts (a.hist) in the two radix
  // chunks its records can touch (c0 = base / chunk and c0 + 1), flushed with one global atomic
  // per non-zero counter; records past chunk c0 + 1 (only with chunks smaller than a
  // super-tile's records, i.e. small capacities) add to the global counts directly
  if (a.hist)
    for (int i = threadIdx.x; i < 512; i += G_TPB_OF(W)) shist[i] = 0;
  using G = FastGeom<W>;
  constexpr int NSWT = G::SUBS * G::NSW;
  constexpr int WPT = (NSWT + G::TPB - 1) / G::TPB;
  const int u0 = threadIdx.x * WPT;
  uint32_t o = excl;
#pragma unroll
  for (int uu = 0; uu < WPT; ++uu) {
    const int u = u0 + uu;
    if (u >= NSWT) break;
    uint32_t bits = emit[u];
    // list entries are k-mer offsets from the super-tile start minus one: slot s of sub-tile
    // `sub` is the k-mer super_lo + sub*TW - 1 + s (< SUBS*TW + NS <= 2^16; emitted s >= 1)
    const int sub = u / G::NSW;
    const uint32_t rel0 = (uint32_t)(sub * G::TW + (u - sub * G::NSW) * 32);
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      list[o++] = (uint16_t)(rel0 + b - 1);
    }
  }
  if (warp_id() == 0) {
    const uint64_t off = lookback_resolve(a.status, tile, total);
    if (lane_id() == 0) {
      *bcast = off;
      // chunks are multiples of 4096 entries and off < 2^44: a 32-bit division
      if (a.hist) bcast[1] = (uint32_t)(off >> 12) / (a.hist_chunk >> 12);
      if (tile == a.ntiles - 1) *a.d_count = off + total;
    }
  }
  __syncthreads();
  const uint64_t base = *bcast;
  const uint64_t hc0 = a.hist ? bcast[1] : 0;
  // record i of this super-tile lies in chunk c0 + 1 iff i >= i1 (i < total < 2^16)
  const uint32_t i1 = (uint32_t)min((hc0 + 1) * a.hist_chunk - base, (uint64_t)0xffffffffu);
  // records past chunk c0 + 1 exist only with chunks smaller than a super-tile's records
  const bool hist_far = a.hist && (uint64_t)i1 + a.hist_chunk < total;
  const int64_t super_lo = (int64_t)tile * (G::SUBS * G::TW);
  // four records per thread per step: their word loads are all in flight before the hashes
  const uint32_t lim = (uint32_t)min((uint64_t)total, a.capacity > base ? a.capacity - base : (uint64_t)0);
  constexpr int U = MZS_MZ_OUT_U;
  // super_lo is a multiple of 32 (TW = 256 R), so a record's k-mer offset `rel` from the
  // super-tile start gives its packed word (rel >> 5) and bit offset (rel & 31) relative to
  // word super_lo / 32: 32-bit index math per record, 64-bit bases once per super-tile
  static_assert((G::SUBS * G::TW) % 32 == 0, "super-tiles start on a packed word");
  const uint64_t* wp = a.words + (super_lo >> 5);
  // the word after an emitted k-mer's first is needed only when the k-mer crosses into it, so
  // clamping its index to the last word (instead of a bounds test) is safe
  const uint32_t wlast = (uint32_t)min(a.nwords - 1 - (uint64_t)(super_lo >> 5), (uint64_t)0xffffffffu);
  uint64_t* const oh = a.out_hash + base;
  uint64_t* const op = a.out_pos + base;
  uint64_t* const oi = a.out_items ? a.out_items + base : nullptr;
  const uint64_t p0 = a.pos_base + (uint64_t)super_lo;
  auto record = [&](uint32_t i, uint32_t rel, uint64_t A, uint64_t B) {
    const uint64_t h = key_from_words<H64, KK, CN ? 1 : 0>(a, (int64_t)rel, A, B);
    MZS_DCHECK(base + i < a.capacity && super_lo + rel < a.n);
    const uint64_t pos = p0 + rel;
    oh[i] = h;
    op[i] = pos;
    const uint64_t it = item_of(h, KK ? KK : a.k, pos);
    if (oi) oi[i] = it;
    if (a.hist) {
      const uint32_t d = ((uint32_t)(it >> 32) >> a.hist_sh) & a.hist_mask;
      if (!hist_far || i < i1 + a.hist_chunk) atomicAdd(&shist[(i >= i1 ? 256 : 0) + d], 1u);
      else atomicAdd(&a.hist[d * a.hist_nch + (base + i) / a.hist_chunk], 1u);
    }
  };
  uint32_t i0 = threadIdx.x;
  // full steps: all U records of the thread exist (no per-record guards), their word loads all
  // in flight before the hashes
  for (; i0 + (U - 1) * G::TPB < lim; i0 += U * G::TPB) {
    uint32_t rel[U];
    uint64_t A[U], B[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rel[u] = list[i0 + u * G::TPB];
      MZS_DCHECK(rel[u] < (uint32_t)(G::SUBS * G::TW + W));
      const uint32_t wr = rel[u] >> 5;
      A[u] = __ldg(wp + wr);
      B[u] = __ldg(wp + min(wr + 1, wlast));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) record(i0 + u * G::TPB, rel[u], A[u], B[u]);
  }
  for (; i0 < lim; i0 += G::TPB) {
    const uint32_t rel = list[i0];
    const uint32_t wr = rel >> 5;
    record(i0, rel, __ldg(wp + wr), __ldg(wp + min(wr + 1, wlast)));
  }
  __syncthreads();  // `list` and `emit` are reused next
  if (a.hist) {
    // each thread flushes the counters it zeroed (same indices: no barrier needed before the
    // next super-tile's zeroing)
    for (int i = threadIdx.x; i < 512; i += G::TPB) {
      const uint32_t v = shist[i];
      const uint64_t c = hc0 + (i >> 8);
      if (v && c < a.hist_nch) atomicAdd(&a.hist[(uint64_t)(i & 255) * a.hist_nch + c], v);
    }
  }
}

// Persistent: every CTA claims super-tiles in order (atomic counter), computes phases 1-2 of
// all SUBS sub-tiles into one of two emit bitmasks, publishes the super-tile's record count,
// and only then outputs its PREVIOUS super-tile -- one super-tile of slack for the
// predecessors' counts to arrive.
template <int W, bool H64, int KK, bool CN>
__global__ void __launch_bounds__(256, 3) mz_fast_kernel(MzArgs a) {
  using G = FastGeom<W>;
  constexpr int NSWT = G::SUBS * G::NSW;
  constexpr int WPT = (NSWT + G::TPB - 1) / G::TPB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 2k <= 38 with a compile-time k: FP64-compare keys (DKey); otherwise 64-bit integer keys
  using Key = typename std::conditional<(KK > 0 && 2 * KK + kSlotBits <= 52), DKey, PackedKey>::type;
  Key* keys = reinterpret_cast<Key*>(smem_raw);
  __shared__ uint32_t emit[2][NSWT + 2];
  __shared__ uint32_t wvb[G::NSW + 3];
  // dirty-word maps of the sub-tile's packed words (double-buffered: the next one is zeroed
  // while the current one is in use); DW words cover NS + k + 64 bases
  constexpr int DW = (G::NS + 64 + 64) / 1024 + 3;
  __shared__ uint32_t dwm[2][DW];
  __shared__ uint64_t warp_sums[G::TPB / 32];
  __shared__ uint64_t bcast[2];
  __shared__ uint32_t s_tile;
  __shared__ uint32_t shist[512];  // first radix pass digit counts of one super-tile (a.hist)
  // the read starts inside the current super-tile's bases (segmented input), found once per
  // super-tile by warp 0; s_nrs < 0: more than 31 (the sub-tiles search global memory)
  __shared__ int64_t s_rs[32];
  __shared__ int s_nrs;
  const int t = threadIdx.x;
  int64_t pend = -1;           // previous super-tile awaiting output
  uint32_t pend_excl = 0, pend_total = 0;
  int cur = 0;
  while (true) {
    if (t == 0) s_tile = atomicAdd(a.tile_counter, 1u);
    for (int u = t; u < NSWT + 2; u += G::TPB) emit[cur][u] = 0;
    if (t < 2 * DW) dwm[t / DW][t % DW] = 0;
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= a.ntiles) break;
    const int64_t super_lo = (int64_t)tile * (G::SUBS * G::TW);
    // the packed words and the first invalid-bitmap word a sub-tile needs are loaded one
    // sub-tile ahead (issued before phase 2 of the previous one), hiding their latency
    uint64_t pw[3];
    uint32_t pinv = 0;
    auto prefetch = [&](int64_t tlo) {
      const int64_t wi = (tlo - 1 + (int64_t)t * G::Q) >> 5;
      pw[0] = ldw(a, wi);
      pw[1] = ldw(a, wi + 1);
      pw[2] = ldw(a, wi + 2);
      const int64_t w0 = max((int64_t)0, (tlo - 1) >> 5) + t;
      pinv = ldi(a, w0);
    };
    prefetch(super_lo);
    if (a.read_off && t < 32) {
      const int64_t lo_b = super_lo - 1, hi_b = super_lo - 1 + (int64_t)(G::SUBS - 1) * G::TW + G::NS + a.k;
      uint64_t r0 = 0;
      if (t == 0) r0 = upper_read(a, lo_b);   // first read start > lo_b
      r0 = __shfl_sync(0xffffffffu, r0, 0);
      const uint64_t r = r0 + t;
      const int64_t v = r <= a.nreads ? (int64_t)__ldg(a.read_off + r) : INT64_MAX;
      const uint32_t in = __ballot_sync(0xffffffffu, v < hi_b);
      if (v < hi_b) s_rs[t] = v;
      if (t == 0) s_nrs = (in == 0xffffffffu) ? -1 : __popc(in);
      __syncwarp();
    }
    for (int sub = 0; sub < G::SUBS; ++sub) {
      const int64_t tile_lo = super_lo + (int64_t)sub * G::TW;
      if (tile_lo >= (int64_t)a.nwin) break;
      const int64_t b_lo = tile_lo - 1, b_hi = tile_lo - 1 + G::NS + a.k;  // bases touched
      for (int u = t; u < G::NSW + 3; u += G::TPB) wvb[u] = 0;
      const uint32_t inv0 = pinv;
      uint32_t* dm = dwm[sub & 1];
      const bool clean = subtile_dirty_map<G::TPB, DW>(a, b_lo, b_hi, dm, &inv0, s_rs, &s_nrs);  // (also the barrier for wvb)
      const int nrs = a.read_off ? s_nrs : 0;  // every warp reads the list after that barrier
      if (t < DW) dwm[(sub + 1) & 1][t] = 0;  // next sub-tile's map (unused until then)
      const int64_t q0 = tile_lo - 1 + (int64_t)t * G::Q;
      const uint32_t s0 = (uint32_t)(t * G::Q);
      // a warp whose windows touch no dirty word skips the validity walk: the windows with
      // their last k-mer in its slots cover bases [wq + 1 - W, wq + 32 Q + k - 2], wq = its first k-mer
      bool wclean = clean;
      if (!clean) {
        const int64_t wq = tile_lo - 1 + (int64_t)(t & ~31) * G::Q;
        const int64_t lo = max(b_lo, wq + 1 - W), hi = min(b_hi - 1, wq + 32 * G::Q + a.k - 2);
        const int u0 = (int)((lo >> 5) - (b_lo >> 5)), u1 = (int)((hi >> 5) - (b_lo >> 5));
        const int nb = u1 - u0 + 1;  // <= 64 (32 Q + k + W bases)
        const uint64_t m = bits64(dm, u0) & (nb >= 64 ? ~0ull : ((1ull << nb) - 1));
        wclean = m == 0;
      }
      const uint64_t w3[3] = {pw[0], pw[1], pw[2]};
      constexpr int KMC = CN ? 2 : 0;  // canonical keys: a separate kernel instantiation
      if (!a.raw) {
        if (wclean) phase1_keys<Key, G::Q, H64, false, KK, KMC, W>(a, q0, s0, keys, wvb, w3);
        else phase1_keys<Key, G::Q, H64, true, KK, KMC, W>(a, q0, s0, keys, wvb, w3, s_rs, nrs);
      } else {
        if (wclean) phase1_keys<Key, G::Q, H64, false, KK, KMC | 1, W>(a, q0, s0, keys, wvb, w3);
        else phase1_keys<Key, G::Q, H64, true, KK, KMC | 1, W>(a, q0, s0, keys, wvb, w3, s_rs, nrs);
      }
      if (!clean && wclean) or_bits(wvb, s0, (1ull << G::Q) - 1);  // every window ending here is valid
      if (sub + 1 < G::SUBS) prefetch(tile_lo + G::TW);
      __syncthreads();
      // window ranges relative to the sub-tile
      const int vlo = (int)max((int64_t)-1, -tile_lo);
      const int vhi = (int)min((int64_t)G::TW, (int64_t)a.nwin - tile_lo);
      // emitting windows: [win_lo, win_hi) and [0, vhi), clamped into [0, TW] with elo <= ehi
      const int64_t wl = min(max((int64_t)a.win_lo - tile_lo, (int64_t)0), (int64_t)G::TW);
      const int64_t wh = min((int64_t)min(a.win_hi, (uint64_t)INT64_MAX) - tile_lo, (int64_t)vhi);
      const int elo = (int)wl, ehi = (int)max(wh, wl);
      // vlo may be -1: the window before the sub-tile exists and feeds the change rule
      const int jb = t * G::R;
      // FULL: windows jb-1 .. jb+R-1 all valid (bits jb-1+W .. jb+R-1+W of wvb when the
      // sub-tile is dirty) and inside the emission range
      const bool inr = vlo <= jb - 1 && jb + G::R <= vhi && elo <= jb && jb + G::R <= ehi;
      uint32_t* em = emit[cur] + sub * G::NSW;
      if (clean) {
        if (inr) fast_phase2<W, false, true>(keys, wvb, vlo, vhi, elo, ehi, em);
        else fast_phase2<W, false, false>(keys, wvb, vlo, vhi, elo, ehi, em);
      } else {
        // dirty sub-tile: every in-range strip takes the masked FULL path (no divergence
        // between strips with and without invalid windows)
        const uint64_t vm = bits64(wvb, jb - 1 + W) & ((1ull << (G::R + 1)) - 1);
        if (inr) fast_phase2<W, false, true, Key, true>(keys, wvb, vlo, vhi, elo, ehi, em, vm);
        else fast_phase2<W, true, false>(keys, wvb, vlo, vhi, elo, ehi, em);
      }
      __syncthreads();
    }
    // count this super-tile's records and publish the count right away
    uint32_t cnt = 0;
#pragma unroll
    for (int uu = 0; uu < WPT; ++uu) {
      const int u = t * WPT + uu;
      if (u < NSWT) cnt += __popc(emit[cur][u]);
    }
    uint64_t total;
    const uint32_t excl = (uint32_t)block_exclusive_sum<G::TPB, uint64_t>(cnt, warp_sums, &total);
    if (t == 0) lookback_publish(a.status, tile, total);
    if (pend >= 0)
      fast_output<W, H64, KK, CN>(a, (uint64_t)pend, emit[cur ^ 1], pend_excl, pend_total,
                              reinterpret_cast<uint16_t*>(keys), bcast, shist);
    pend = (int64_t)tile;
    pend_excl = excl;
    pend_total = (uint32_t)total;
    cur ^= 1;
  }
  if (pend >= 0)
    fast_output<W, H64, KK, CN>(a, (uint64_t)pend, emit[cur ^ 1], pend_excl, pend_total,
                            reinterpret_cast<uint16_t*>(keys), bcast, shist);
}

// ------------------------------------------------------------------ generic path kernel
constexpr int kGenTPB = 256;
constexpr int kGenE = 16;                 // slots per thread
constexpr int kGenNS = kGenTPB * kGenE;   // 4096 slots per sub-tile
constexpr int kGenSubs = 4;

template <class Key, bool H64>
__global__ void __launch_bounds__(kGenTPB) mz_generic_kernel(MzArgs a) {
  using Op = OpKeyMin<Key>;
  constexpr int NSW = kGenNS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Key* keys = reinterpret_cast<Key*>(smem_raw);
  Key* sP = keys + kGenNS;
  Key* sS = sP + kGenNS;
  __shared__ uint32_t emit[kGenSubs * NSW];
  __shared__ uint32_t wvb[NSW + 3];
  __shared__ uint64_t warp_sums[kGenTPB / 32];
  __shared__ uint64_t bcast;
  __shared__ uint32_t s_tile;
  __shared__ SegScratch<Op, kGenTPB> sh;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
  for (int u = threadIdx.x; u < kGenSubs * NSW; u += kGenTPB) emit[u] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint32_t W = (uint32_t)a.w;
  const int64_t super_lo = (int64_t)tile * kGenSubs * a.tw;
  int nsub = 0;
  const int t = threadIdx.x;
  for (int sub = 0; sub < kGenSubs; ++sub) {
    const int64_t tile_lo = super_lo + (int64_t)sub * a.tw;
    if (tile_lo >= (int64_t)a.nwin) break;
    ++nsub;
    const int64_t b_lo = tile_lo - 1, b_hi = tile_lo - 1 + kGenNS + a.k;
    for (int u = t; u < NSW + 3; u += kGenTPB) wvb[u] = 0;
    const bool clean = tile_is_clean<kGenTPB>(a, b_lo, b_hi);
    const int64_t q0 = tile_lo - 1 + (int64_t)t * kGenE;
    auto p1 = [&](auto km_tag) {
      constexpr int KMV = decltype(km_tag)::value;
      if (clean) phase1_keys<Key, kGenE, H64, false, 0, KMV>(a, q0, t * kGenE, keys, wvb);
      else phase1_keys<Key, kGenE, H64, true, 0, KMV>(a, q0, t * kGenE, keys, wvb);
    };
    if (a.canon) {
      if (a.raw) p1(std::integral_constant<int, 3>{});
      else p1(std::integral_constant<int, 2>{});
    } else {
      if (a.raw) p1(std::integral_constant<int, 1>{});
      else p1(std::integral_constant<int, 0>{});
    }
    __syncthreads();
    // phase 2: block S/P over slots, blocks of W starting at slot 1 (slot s <-> k-mer tile_lo-1+s)
    {
      Key v[kGenE], P[kGenE], S[kGenE];
#pragma unroll
      for (int j = 0; j < kGenE; ++j) v[j] = keys[t * kGenE + j];
      block_prefix_suffix<Op, kGenTPB, kGenE>(v, P, S, W, 1u, sh);
#pragma unroll
      for (int j = 0; j < kGenE; ++j) {
        sP[t * kGenE + j] = P[j];
        sS[t * kGenE + j] = S[j];
      }
    }
    __syncthreads();
    {
      const uint32_t per = (a.tw + kGenTPB - 1) / kGenTPB;
      const int j0 = t * per;
      const int j1 = min((int)a.tw, j0 + (int)per);
      auto wmin = [&](int j) -> Key {
        if (j < 0) return W == 1 ? keys[0] : kmin(keys[0], sP[W - 1]);
        return (j % W == 0) ? sS[j + 1] : kmin(sS[j + 1], sP[j + W]);
      };
      auto valid_of = [&](int j) -> bool {
        const int64_t i = tile_lo + j;
        if (i < 0 || (uint64_t)i >= a.nwin) return false;
        return clean ? true : wv_bit(wvb, j + W);
      };
      uint32_t* em = emit + sub * NSW;
      if (j0 < j1) {
        Key yprev = wmin(j0 - 1);
        bool vprev = valid_of(j0 - 1);
        for (int j = j0; j < j1; ++j) {
          const Key y = wmin(j);
          const bool v = valid_of(j);
          const int64_t i = tile_lo + j;
          if (v && (!vprev || y != yprev) && (uint64_t)i >= a.win_lo && (uint64_t)i < a.win_hi) {
            const uint32_t s = y.slot();
            atomicOr(&em[s >> 5], 1u << (s & 31));
          }
          vprev = v;
          yprev = y;
        }
      }
    }
    __syncthreads();
  }
  phase3_output<kGenTPB, H64>(a, tile, super_lo, kGenNS, nsub, emit, reinterpret_cast<uint16_t*>(keys), warp_sums,
                              &bcast);
}

// ------------------------------------------------------------------ host side
__global__ void __launch_bounds__(256) ridx_kernel(const uint64_t* __restrict__ read_off, uint64_t nreads,
                                                   uint64_t* __restrict__ ridx, uint64_t nb) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const uint64_t x = b << kRidxShift;
  uint64_t lo = 0, hi = nreads + 1;   // first r with read_off[r] >= x
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (__ldg(read_off + mid) >= x) hi = mid; else lo = mid + 1;
  }
  ridx[b] = lo;
}
uint64_t ridx_entries(uint64_t n) { return (n >> kRidxShift) + 2; }

int launch_mz(MzArgs a, int path, cudaStream_t st) {
  const int k = a.k, w = a.w;
  const bool h64 = 2 * k > 32;
  const bool packed_ok = 2 * k + kSlotBits <= 64;
  // 0 = auto, 1 = force generic
  const bool fast = path == 0 && packed_ok && w >= 1 && w <= 16;
  if (fast) {
#define MZS_FAST_KK(WW, KKV, H64V)                                                                     \
  {                                                                                                    \
    using G = FastGeom<WW>;                                                                            \
    a.tw = G::TW;                                                                                      \
    a.ntiles = (a.nwin + (uint64_t)G::TW * G::SUBS - 1) / ((uint64_t)G::TW * G::SUBS);                 \
    const size_t smem = sizeof(PackedKey) * G::NS;                                                     \
    auto kern = a.canon ? mz_fast_kernel<WW, H64V, KKV, true> : mz_fast_kernel<WW, H64V, KKV, false>;   \
    MZS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
    MZS_CUDA(cudaMemsetAsync(a.tile_counter, 0, sizeof(uint32_t), st));                                \
    MZS_CUDA(cudaMemsetAsync(a.status, 0, sizeof(uint64_t) * a.ntiles, st));                           \
    int occ = 0;                                                                                       \
    MZS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, G::TPB, smem));                 \
    const uint64_t grid = std::min<uint64_t>(a.ntiles, (uint64_t)num_sms() * (uint64_t)std::max(occ, 1)); \
    kern<<<(unsigned)grid, G::TPB, smem, st>>>(a);                                                     \
    MZS_LAUNCHED();                                                                                    \
    return SLSUM_OK;                                                                                   \
  }
#define MZS_FAST(WW)                                                                                   \
  case WW:                                                                                             \
    if (h64) MZS_FAST_KK(WW, 0, true) else MZS_FAST_KK(WW, 0, false)
    // compile-time k for the configurations the paper and BASELINE measure
    if (w == 10 && k == 19) MZS_FAST_KK(10, 19, true)
    if (w == 10 && k == 15) MZS_FAST_KK(10, 15, false)
    switch (w) {
      MZS_FAST(1) MZS_FAST(2) MZS_FAST(3) MZS_FAST(4) MZS_FAST(5) MZS_FAST(6) MZS_FAST(7) MZS_FAST(8)
      MZS_FAST(9) MZS_FAST(10) MZS_FAST(11) MZS_FAST(12) MZS_FAST(13) MZS_FAST(14) MZS_FAST(15) MZS_FAST(16)
      default: break;
    }
#undef MZS_FAST
#undef MZS_FAST_KK
  }
  if (w > 1024) return SLSUM_EUNSUPPORTED;
  a.tw = (uint32_t)(kGenNS - w - 1);
  a.ntiles = (a.nwin + (uint64_t)a.tw * kGenSubs - 1) / ((uint64_t)a.tw * kGenSubs);
  MZS_CUDA(cudaMemsetAsync(a.tile_counter, 0, sizeof(uint32_t), st));
  MZS_CUDA(cudaMemsetAsync(a.status, 0, sizeof(uint64_t) * a.ntiles, st));
  if (packed_ok) {
    const size_t smem = 3 * sizeof(PackedKey) * kGenNS;
    auto kern = h64 ? mz_generic_kernel<PackedKey, true> : mz_generic_kernel<PackedKey, false>;
    MZS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)a.ntiles, kGenTPB, smem, st>>>(a);
  } else {
    const size_t smem = 3 * sizeof(WideKey) * kGenNS;
    auto kern = mz_generic_kernel<WideKey, true>;
    MZS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)a.ntiles, kGenTPB, smem, st>>>(a);
  }
  MZS_LAUNCHED();
  return SLSUM_OK;
}

// max tiles for n bases (the generic path has the smallest tiles: >= 4096-1025 windows)
uint64_t max_tiles(uint64_t n) { return n / 3000 + 2; }

}  // namespace

int encode_launch(const uint8_t* seq, uint64_t n, uint64_t* words, uint32_t* invalid, cudaStream_t st);

}  // namespace mzs

using namespace mzs;

MZS_API size_t mz_workspace_bytes(uint64_t n, int k, int w, int kind) {
  (void)k; (void)w;
  Sizer z;
  z.take<uint32_t>(1);                  // tile counter
  z.take<uint64_t>(max_tiles(n));       // look-back status
  z.take<uint64_t>(ridx_entries(n));    // coarse read index (segmented input)
  if (kind == MZ_IN_ASCII) {
    z.take<uint64_t>((n + 31) / 32 + 1);
    z.take<uint32_t>((n + 31) / 32 + 1);
  }
  return z.used;
}

// internal entry with a path selector (0 auto, 1 generic) for tests
MZS_API int mz_extract_path(const mz_in_t* in, int k, int w, int keymode, mz_out_t* out, void* ws,
                            size_t ws_bytes, void* stream, int path) {
  if (!in || !out || !out->d_count || k < 1 || k > 31 || w < 1) return SLSUM_EINVAL;
  if (in->kind != MZ_IN_ASCII && in->kind != MZ_IN_PACKED2) return SLSUM_EINVAL;
  if (keymode < MZ_KEY_HASH || keymode > MZ_KEY_CANON_RAW) return SLSUM_EINVAL;
  if (in->read_off && in->nreads == 0) return SLSUM_EINVAL;
  if (out->capacity && (!out->hash || !out->pos)) return SLSUM_EINVAL;
  cudaStream_t st = as_stream(stream);
  const uint64_t n = in->n;
  const uint64_t span = (uint64_t)k + (uint64_t)w - 1;
  if (n < span || in->win_lo >= in->win_hi) {
    MZS_CUDA(cudaMemsetAsync(out->d_count, 0, sizeof(uint64_t), st));
    if (out->hist && out->capacity)
      MZS_CUDA(cudaMemsetAsync(out->hist, 0, sizeof(uint32_t) * 256 * radix_nchunks(out->capacity), st));
    return SLSUM_OK;
  }
  if (!in->seq) return SLSUM_EINVAL;
  TempWs tmp;
  const size_t need = mz_workspace_bytes(n, k, w, in->kind);
  if (!ws) {
    MZS_CUDA(cudaMallocAsync(&tmp.p, need, st));
    tmp.s = st;
    ws = tmp.p;
    ws_bytes = need;
  }
  if (ws_bytes < need) return SLSUM_ENOMEM;
  Carve c(ws, ws_bytes);
  MzArgs a{};
  a.tile_counter = c.take<uint32_t>(1);
  a.status = c.take<uint64_t>(max_tiles(n));
  uint64_t* ridx = c.take<uint64_t>(ridx_entries(n));
  a.nwords = (n + 31) / 32;
  if (in->kind == MZ_IN_ASCII) {
    uint64_t* words = c.take<uint64_t>(a.nwords + 1);
    uint32_t* inval = c.take<uint32_t>(a.nwords + 1);
    int rc = encode_launch(static_cast<const uint8_t*>(in->seq), n, words, inval, st);
    if (rc) return rc;
    a.words = words;
    a.invalid = inval;
  } else {
    a.words = static_cast<const uint64_t*>(in->seq);
    a.invalid = in->invalid;
  }
  a.n = n;
  a.nwin = n - span + 1;
  a.read_off = in->read_off;
  a.nreads = in->read_off ? in->nreads : 0;
  if (in->read_off) {
    const uint64_t nb = ridx_entries(n);
    ridx_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(in->read_off, a.nreads, ridx, nb);
    MZS_LAUNCHED();
    a.ridx = ridx;
  }
  a.pos_base = in->pos_base;
  a.win_lo = in->win_lo;
  a.win_hi = in->win_hi;
  a.k = k;
  a.w = w;
  a.raw = keymode == MZ_KEY_RAW || keymode == MZ_KEY_CANON_RAW;
  a.canon = keymode == MZ_KEY_CANON || keymode == MZ_KEY_CANON_RAW;
  a.out_hash = out->hash;
  a.out_pos = out->pos;
  a.out_items = out->items;
  a.capacity = out->capacity;
  a.d_count = out->d_count;
  if (out->hist) {
    // the seed table's first radix pass: digit = the low 8 bits of the bucket (fp bits
    // [32 - bits, 40 - bits)), chunks as seedtable_build_items_ex lays them out for m = capacity
    const int bits = out->hist_bucket_bits;
    if (bits < 1 || bits > 30 || bits > 2 * k || out->capacity == 0) return SLSUM_EINVAL;
    a.hist = out->hist;
    a.hist_chunk = radix_chunk_for(out->capacity);
    a.hist_nch = radix_nchunks(out->capacity);
    a.hist_sh = 32 - bits;
    a.hist_mask = (1u << (bits < 8 ? bits : 8)) - 1u;
    MZS_CUDA(cudaMemsetAsync(out->hist, 0, sizeof(uint32_t) * 256 * a.hist_nch, st));
  }
  return launch_mz(a, path, st);
}

MZS_API int mz_extract_ex(const mz_in_t* in, int k, int w, int keymode, mz_out_t* out, void* ws, size_t ws_bytes,
                          void* stream) {
  return mz_extract_path(in, k, w, keymode, out, ws, ws_bytes, stream, 0);
}

MZS_API int mz_extract(const uint8_t* seq, uint64_t n, int k, int w, mz_out_t* out) {
  if (!out) return SLSUM_EINVAL;
  mz_in_t in{};
  in.kind = MZ_IN_ASCII;
  in.seq = seq;
  in.n = n;
  in.win_lo = 0;
  in.win_hi = UINT64_MAX;
  int rc = mz_extract_ex(&in, k, w, MZ_KEY_HASH, out, nullptr, 0, nullptr);
  if (rc) return rc;
  uint64_t cnt = 0;
  MZS_CUDA(cudaMemcpy(&cnt, out->d_count, sizeof(cnt), cudaMemcpyDeviceToHost));
  return cnt > out->capacity ? SLSUM_ECAPACITY : SLSUM_OK;
}

// ------------------------------------------------------------------ minimap2-compatible variant
// mz_extract_ties (R35): every tied minimum of every window, windows kept
// inside runs of present k-mers (a run shorter than w is one window), symmetric k-mers never
// selected.  Built from two sliding window sums of the paper (Eq. 2 with (+) = min, PAPER.md
// L38-41): with K_q = key+1 for a present k-mer (0 if absent, ~0 if symmetric),
//   m_j = min(K_j .. K_{j+w-1})            (0 iff window j leaves its run)
//   M_q = max(m_j : j in [q-w+1, q])        (= ~min(~m_j), the same min sum on a padded copy)
// k-mer q is selected iff K_q = M_q: the windows of its run containing q all have m_j <= K_q,
// and one has m_j = K_q iff q is a tied minimum of it.  M_q = 0 iff q's run is shorter than w;
// there the run's minimum is found by a scan of the (< w) run.
namespace mzs {
namespace {
constexpr uint64_t kTieSym = ~0ull;
constexpr int kTieTPB = 256;
constexpr int kTieBlk = kTieTPB * 32;  // positions per mark/write block (one bitmap word per thread)

// K_q = key + 1 for a present k-mer, 0 for an absent one (an N or a read start inside it),
// kTieSym for a symmetric one.  One packed word (32 k-mers) per thread: the word pair and the
// 64 validity bits are loaded once, the 32 keys are staged in shared memory (row t*33:
// conflict-free both ways) and written out coalesced.  8192 k-mers per CTA; KK != 0: the
// compile-time k (C1/C3/C4 values), masks and shifts fold.
template <int KK>
__global__ void __launch_bounds__(256) ties_key_tile_kernel(MzArgs a, uint64_t nk, uint64_t* __restrict__ K) {
  extern __shared__ uint64_t s_k[];
  const int k = KK ? KK : a.k;
  const uint64_t base = (uint64_t)blockIdx.x * kTieBlk;
  const int64_t wi = (int64_t)(base >> 5) + threadIdx.x;
  const uint64_t A = ldw(a, wi), B = ldw(a, wi + 1);
  const uint64_t inv = (uint64_t)ldi(a, wi) | ((uint64_t)ldi(a, wi + 1) << 32);
  const uint64_t kmask = (1ull << k) - 1ull;
#pragma unroll 4
  for (int r = 0; r < 32; ++r) {
    const uint64_t q = (uint64_t)wi * 32 + (uint64_t)r;
    bool ok = q < nk && ((inv >> r) & kmask) == 0;
    if (ok && a.read_off) {
      const uint64_t rr = upper_read(a, (int64_t)q);
      ok = !(rr <= a.nreads && __ldg(a.read_off + rr) <= q + (uint64_t)k - 1);
    }
    uint64_t v = 0;
    if (ok) {
      const uint32_t off = (uint32_t)r * 2;
      const uint64_t X = off ? (A << off) | (B >> (64 - off)) : A;
      const uint64_t code = X >> (64 - 2 * k);
      if (a.canon && revcomp64(code, k) == code) {
        v = kTieSym;
      } else {
        v = 1 + (2 * k > 32 ? key_from_words<true, (2 * KK > 32 ? KK : 0)>(a, (int64_t)q, A, B)
                            : key_from_words<false, (2 * KK > 32 ? 0 : KK)>(a, (int64_t)q, A, B));
      }
    }
    s_k[threadIdx.x * 33 + r] = v;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < kTieBlk; j += 256) {
    const uint64_t q = base + (uint64_t)j;
    if (q < nk) K[q] = s_k[(j >> 5) * 33 + (j & 31)];
  }
}

// c[t] = ~m[t - (w-1)] inside, ~0 (m = 0: no window) in the w-1 pads on each side
__global__ void __launch_bounds__(256) ties_pad_kernel(const uint64_t* __restrict__ m, uint64_t nw, uint32_t w,
                                                       uint64_t* __restrict__ c, uint64_t nc) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nc; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = t - (uint64_t)(w - 1);
    c[t] = (t >= (uint64_t)(w - 1) && j < nw) ? ~__ldg(m + j) : ~0ull;
  }
}

// selection bitmap (bit q & 31 of word q >> 5) and per-block counts.
// INLINE = false: z = ~M from the second sliding sum.  INLINE = true (w <= kTieInlineW): z = m,
// the window minima themselves; the block stages them in shared memory a quarter of its k-mers
// at a time (16.6 KB, so 8 CTAs fit per SM) and tests K_q against m_{q-w+1} .. m_q there (w
// equality tests per k-mer, no padded copy and no second sum in HBM).
constexpr int kTieInlineW = 32;
// k-mer q of a run shorter than w (no full window holds it): the whole run is the window
__device__ __forceinline__ bool tie_short_run(const uint64_t* __restrict__ K, uint64_t nk, uint64_t q, uint64_t kq) {
  uint64_t mn = kq;
  for (uint64_t j = q; j > 0;) {
    const uint64_t v = __ldg(K + --j);
    if (v == 0) break;
    mn = min(mn, v);
  }
  for (uint64_t j = q + 1; j < nk; ++j) {
    const uint64_t v = __ldg(K + j);
    if (v == 0) break;
    mn = min(mn, v);
  }
  return kq == mn;
}
constexpr int kTieQuarter = kTieBlk / 4;  // INLINE: the block stages m a quarter at a time
// the w equality tests of k-mer q against s[0 .. w-1] = m_{q-w+1} .. m_q.  W > 0: w = W at compile
// time (unrolled, immediate shared-memory offsets); W = 0: any w
template <int W>
__device__ __forceinline__ void tie_window_tests(const uint64_t* s, int w, uint64_t kq, bool& eq, uint32_t& nz) {
  const int ww = W ? W : w;
#pragma unroll
  for (int d = 0; d < ww; ++d) {
    const uint64_t v = s[d];
    eq |= v == kq;
    nz |= (uint32_t)v | (uint32_t)(v >> 32);
  }
}
template <bool INLINE>
__global__ void __launch_bounds__(kTieTPB) ties_mark_kernel(const uint64_t* __restrict__ K, const uint64_t* __restrict__ z,
                                                            uint64_t nk, uint64_t nw, int w, uint32_t* __restrict__ bits,
                                                            uint64_t* __restrict__ blkcnt) {
  extern __shared__ uint64_t s_m[];
  const uint64_t base = (uint64_t)blockIdx.x * kTieBlk;
  uint32_t cnt = 0;
  for (int r = 0; r < 32; ++r) {
    if (INLINE && r % (kTieQuarter / kTieTPB) == 0) {
      // stage m_{qb-w+1 .. qb+kTieQuarter-1} (0 outside [0, nw)) for this quarter's k-mers
      const uint64_t qb = base + (uint64_t)r * kTieTPB;
      __syncthreads();
      for (int t = threadIdx.x; t < kTieQuarter + w - 1; t += kTieTPB) {
        const uint64_t j = qb + (uint64_t)t - (uint64_t)(w - 1);  // wraps below 0: >= nw
        s_m[t] = j < nw ? __ldg(z + j) : 0ull;
      }
      __syncthreads();
    }
    const uint64_t q = base + (uint64_t)r * kTieTPB + threadIdx.x;
    bool f = false;
    if (q < nk) {
      const uint64_t kq = __ldg(K + q);
      if (kq != 0 && kq != kTieSym) {
        if (INLINE) {
          // every m_j of a window holding q is <= K_q, so K_q = max_j m_j iff some m_j = K_q;
          // all m_j = 0 iff q's run is shorter than w
          const int t0 = (r % (kTieQuarter / kTieTPB)) * kTieTPB + threadIdx.x;
          bool eq = false;
          uint32_t nz = 0;
          switch (w) {  // the usual window lengths unrolled (minimap2 presets: 5, 10, 11, 19)
            case 5: tie_window_tests<5>(s_m + t0, w, kq, eq, nz); break;
            case 10: tie_window_tests<10>(s_m + t0, w, kq, eq, nz); break;
            case 11: tie_window_tests<11>(s_m + t0, w, kq, eq, nz); break;
            case 19: tie_window_tests<19>(s_m + t0, w, kq, eq, nz); break;
            default: tie_window_tests<0>(s_m + t0, w, kq, eq, nz); break;
          }
          f = nz ? eq : tie_short_run(K, nk, q, kq);
        } else {
          const uint64_t M = ~__ldg(z + q);
          f = M ? kq == M : tie_short_run(K, nk, q, kq);
        }
      }
    }
    const uint32_t b = __ballot_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && base + (uint64_t)r * kTieTPB + threadIdx.x < nk)
      bits[(base + (uint64_t)r * kTieTPB + threadIdx.x) >> 5] = b;
    cnt += (threadIdx.x & 31) == 0 ? __popc(b) : 0u;
  }
  __shared__ uint32_t s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt, cnt);
  __syncthreads();
  if (threadIdx.x == 0) blkcnt[blockIdx.x] = s_cnt;
}

// exclusive scan of the block counts (one CTA); d_count = the total
__global__ void __launch_bounds__(1024) ties_scan_kernel(const uint64_t* __restrict__ blkcnt, uint64_t nblk,
                                                         uint64_t* __restrict__ blkoff, uint64_t* __restrict__ d_count) {
  __shared__ uint64_t s_warp[32];
  __shared__ uint64_t s_carry;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint64_t b0 = 0; b0 < nblk; b0 += 1024) {
    const uint64_t b = b0 + threadIdx.x;
    const uint64_t v = b < nblk ? blkcnt[b] : 0;
    uint64_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint64_t t = s_warp[lane];
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, t, d);
        if (lane >= d) t += y;
      }
      s_warp[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const uint64_t incl = x + (wid ? s_warp[wid - 1] : 0) + s_carry;
    if (b < nblk) blkoff[b] = incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *d_count = s_carry;
}

// ordered output: thread t of block b owns bitmap word b * 256 + t.  The block's records are
// first listed in order in shared memory (13-bit k-mer offsets within the block), then written
// by consecutive threads to consecutive outputs (coalesced stores, K read in order).
__global__ void __launch_bounds__(kTieTPB) ties_write_kernel(MzArgs a, const uint64_t* __restrict__ K, uint64_t nk,
                                                             const uint32_t* __restrict__ bits,
                                                             const uint64_t* __restrict__ blkoff) {
  __shared__ uint32_t s_warp[kTieTPB / 32];
  __shared__ uint16_t s_list[kTieBlk];
  const uint64_t wi = (uint64_t)blockIdx.x * kTieTPB + threadIdx.x;
  const uint64_t nwords = (nk + 31) / 32;
  uint32_t word = wi < nwords ? bits[wi] : 0u;
  const uint32_t c = __popc(word);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = c;
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  uint32_t pre = 0, total = 0;
  for (int i = 0; i < kTieTPB / 32; ++i) {
    if (i < wid) pre += s_warp[i];
    total += s_warp[i];
  }
  uint32_t lo = pre + x - c;  // block-local index of this word's first record
  while (word) {
    const int b = __ffs(word) - 1;
    word &= word - 1;
    s_list[lo++] = (uint16_t)(threadIdx.x * 32 + b);
  }
  __syncthreads();
  const uint64_t o0 = blkoff[blockIdx.x];
  const uint64_t qb = (uint64_t)blockIdx.x * kTieBlk;
  const int k = a.k;
  for (uint32_t i = threadIdx.x; i < total; i += kTieTPB) {
    const uint64_t o = o0 + i;
    if (o >= a.capacity) break;
    const uint64_t q = qb + s_list[i];
    const uint64_t h = __ldg(K + q) - 1;
    a.out_hash[o] = h;
    a.out_pos[o] = a.pos_base + q;
    if (a.out_items) a.out_items[o] = item_of(h, k, a.pos_base + q);
  }
}

uint64_t ties_grid(uint64_t n) { return std::min<uint64_t>((n + 255) / 256, 148ull * 16); }
}  // namespace
}  // namespace mzs

MZS_API size_t mz_ties_workspace_bytes(uint64_t n, int k, int w, int kind) {
  Sizer z;
  z.take<uint64_t>(ridx_entries(n));
  if (kind == MZ_IN_ASCII) {
    z.take<uint64_t>((n + 31) / 32 + 1);
    z.take<uint32_t>((n + 31) / 32 + 1);
  }
  const uint64_t nk = (k >= 1 && n >= (uint64_t)k) ? n - (uint64_t)k + 1 : 0;
  const uint64_t ww = w >= 1 ? (uint64_t)w : 1;
  const uint64_t nw = nk >= ww ? nk - ww + 1 : 0;
  const uint64_t nblk = (nk + kTieBlk - 1) / kTieBlk + 1;
  z.take<uint64_t>(nk + 1);           // K
  z.take<uint64_t>(nw + 1);           // m
  z.take<uint64_t>(nw + 2 * (ww - 1) + 1);  // padded ~m
  z.take<uint64_t>(nk + 1);           // z = ~M
  z.take<uint32_t>((nk + 31) / 32 + 1);
  z.take<uint64_t>(nblk);
  z.take<uint64_t>(nblk);
  return z.used;
}

MZS_API int mz_extract_ties(const mz_in_t* in, int k, int w, int keymode, mz_out_t* out, void* ws,
                            size_t ws_bytes, void* stream) {
  if (!in || !out || !out->d_count || k < 1 || k > 31 || w < 1) return SLSUM_EINVAL;
  if (in->kind != MZ_IN_ASCII && in->kind != MZ_IN_PACKED2) return SLSUM_EINVAL;
  if (keymode < MZ_KEY_HASH || keymode > MZ_KEY_CANON_RAW) return SLSUM_EINVAL;
  if (in->read_off && in->nreads == 0) return SLSUM_EINVAL;
  if (out->capacity && (!out->hash || !out->pos)) return SLSUM_EINVAL;
  if (out->hist) return SLSUM_EINVAL;
  if (in->win_lo != 0 || in->win_hi != UINT64_MAX) return SLSUM_EUNSUPPORTED;
  cudaStream_t st = as_stream(stream);
  const uint64_t n = in->n;
  if (n < (uint64_t)k) {
    MZS_CUDA(cudaMemsetAsync(out->d_count, 0, sizeof(uint64_t), st));
    return SLSUM_OK;
  }
  if (!in->seq) return SLSUM_EINVAL;
  TempWs tmp;
  const size_t need = mz_ties_workspace_bytes(n, k, w, in->kind);
  if (!ws) {
    MZS_CUDA(cudaMallocAsync(&tmp.p, need, st));
    tmp.s = st;
    ws = tmp.p;
    ws_bytes = need;
  }
  if (ws_bytes < need) return SLSUM_ENOMEM;
  Carve c(ws, ws_bytes);
  MzArgs a{};
  uint64_t* ridx = c.take<uint64_t>(ridx_entries(n));
  a.nwords = (n + 31) / 32;
  if (in->kind == MZ_IN_ASCII) {
    uint64_t* words = c.take<uint64_t>(a.nwords + 1);
    uint32_t* inval = c.take<uint32_t>(a.nwords + 1);
    int rc = encode_launch(static_cast<const uint8_t*>(in->seq), n, words, inval, st);
    if (rc) return rc;
    a.words = words;
    a.invalid = inval;
  } else {
    a.words = static_cast<const uint64_t*>(in->seq);
    a.invalid = in->invalid;
  }
  a.n = n;
  a.read_off = in->read_off;
  a.nreads = in->read_off ? in->nreads : 0;
  if (in->read_off) {
    const uint64_t nb = ridx_entries(n);
    ridx_kernel<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(in->read_off, a.nreads, ridx, nb);
    MZS_LAUNCHED();
    a.ridx = ridx;
  }
  a.pos_base = in->pos_base;
  a.k = k;
  a.w = w;
  a.raw = keymode == MZ_KEY_RAW || keymode == MZ_KEY_CANON_RAW;
  a.canon = keymode == MZ_KEY_CANON || keymode == MZ_KEY_CANON_RAW;
  a.out_hash = out->hash;
  a.out_pos = out->pos;
  a.out_items = out->items;
  a.capacity = out->capacity;
  a.d_count = out->d_count;
  const uint64_t nk = n - (uint64_t)k + 1, ww = (uint64_t)w;
  const uint64_t nw = nk >= ww ? nk - ww + 1 : 0;
  const uint64_t nblk = (nk + kTieBlk - 1) / kTieBlk;
  uint64_t* K = c.take<uint64_t>(nk + 1);
  uint64_t* m = c.take<uint64_t>(nw + 1);
  uint64_t* cp = c.take<uint64_t>(nw + 2 * (ww - 1) + 1);
  uint64_t* z = c.take<uint64_t>(nk + 1);
  uint32_t* bits = c.take<uint32_t>((nk + 31) / 32 + 1);
  uint64_t* blkcnt = c.take<uint64_t>(nblk + 1);
  uint64_t* blkoff = c.take<uint64_t>(nblk + 1);
  if (!c.ok) return SLSUM_ENOMEM;
  {
    const size_t ksm = sizeof(uint64_t) * 256 * 33;
    auto kfn = k == 19 ? ties_key_tile_kernel<19> : k == 15 ? ties_key_tile_kernel<15> : ties_key_tile_kernel<0>;
    MZS_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksm));
    kfn<<<(unsigned)nblk, 256, ksm, st>>>(a, nk, K);
    MZS_LAUNCHED();
  }
  if (nw > 0 && w <= kTieInlineW) {
    int rc = slsum_run_ex(SLSUM_MIN_U64, (uint32_t)w, K, m, nk, SLSUM_PATH_GENERIC, st);
    if (rc) return rc;
    const size_t smem = sizeof(uint64_t) * (kTieQuarter + kTieInlineW - 1);
    MZS_CUDA(cudaFuncSetAttribute(ties_mark_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ties_mark_kernel<true><<<(unsigned)nblk, kTieTPB, smem, st>>>(K, m, nk, nw, w, bits, blkcnt);
    MZS_LAUNCHED();
  } else if (nw > 0) {
    int rc = slsum_run_ex(SLSUM_MIN_U64, (uint32_t)w, K, m, nk, SLSUM_PATH_GENERIC, st);
    if (rc) return rc;
    const uint64_t nc = nw + 2 * (ww - 1);
    ties_pad_kernel<<<(unsigned)ties_grid(nc), 256, 0, st>>>(m, nw, (uint32_t)w, cp, nc);
    MZS_LAUNCHED();
    rc = slsum_run_ex(SLSUM_MIN_U64, (uint32_t)w, cp, z, nc, SLSUM_PATH_GENERIC, st);  // nc-w+1 = nk outputs
    if (rc) return rc;
    ties_mark_kernel<false><<<(unsigned)nblk, kTieTPB, 0, st>>>(K, z, nk, nw, w, bits, blkcnt);
    MZS_LAUNCHED();
  } else {
    MZS_CUDA(cudaMemsetAsync(z, 0xff, sizeof(uint64_t) * nk, st));  // no full window: M = 0
    ties_mark_kernel<false><<<(unsigned)nblk, kTieTPB, 0, st>>>(K, z, nk, nw, w, bits, blkcnt);
    MZS_LAUNCHED();
  }
  ties_scan_kernel<<<1, 1024, 0, st>>>(blkcnt, nblk, blkoff, out->d_count);
  MZS_LAUNCHED();
  ties_write_kernel<<<(unsigned)nblk, kTieTPB, 0, st>>>(a, K, nk, bits, blkoff);
  MZS_LAUNCHED();
  return SLSUM_OK;
}
