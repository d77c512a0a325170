// ops.cuh -- the operators (+) of Eq. 1 / Eq. 2 for the sliding-sum
// kernels, and the block-level suffix/prefix decomposition of Algorithm 2 (L123-150).
//
// Every Op::op(a, b) is called with `a` the fold of EARLIER elements and `b` of LATER ones,
// so the kernels never reorder operands (the AFFINE op proves it in the tests).
#pragma once

#include "common.cuh"

namespace mzs {

struct OpMinU32 {
  using T = uint32_t;
  static constexpr bool kCommutative = true, kIdempotent = true;
  __device__ __forceinline__ static T id() { return 0xffffffffu; }
  __device__ __forceinline__ static T op(T a, T b) { return a < b ? a : b; }
};
struct OpMaxU32 {
  using T = uint32_t;
  static constexpr bool kCommutative = true, kIdempotent = true;
  __device__ __forceinline__ static T id() { return 0u; }
  __device__ __forceinline__ static T op(T a, T b) { return a > b ? a : b; }
};
struct OpAddU32 {
  using T = uint32_t;
  static constexpr bool kCommutative = true, kIdempotent = false;
  __device__ __forceinline__ static T id() { return 0u; }
  __device__ __forceinline__ static T op(T a, T b) { return a + b; }
};
struct OpAddF32 {
  using T = float;
  static constexpr bool kCommutative = true, kIdempotent = false;
  __device__ __forceinline__ static T id() { return 0.0f; }
  __device__ __forceinline__ static T op(T a, T b) { return __fadd_rn(a, b); }
};
struct OpMinU64 {
  using T = unsigned long long;
  static constexpr bool kCommutative = true, kIdempotent = true;
  __device__ __forceinline__ static T id() { return ~0ull; }
  __device__ __forceinline__ static T op(T a, T b) { return a < b ? a : b; }
};
// t -> a t + b over Z/2^32; (a,b) (+) (c,d) = (a c, a d + b): apply the later map first.
struct OpAffine {
  using T = uint2;  // x = a, y = b
  static constexpr bool kCommutative = false, kIdempotent = false;
  __device__ __forceinline__ static T id() { return make_uint2(1u, 0u); }
  __device__ __forceinline__ static T op(T l, T r) { return make_uint2(l.x * r.x, l.x * r.y + l.y); }
};
// string concatenation of base-sigma numerals (L67: k-mers as a sliding sum under
// concatenation): (v1,s1) (+) (v2,s2) = (v1 s2 + v2, s1 s2) over Z/2^32; the empty string (0,1).
struct OpConcat {
  using T = uint2;  // x = value, y = weight sigma^length
  static constexpr bool kCommutative = false, kIdempotent = false;
  __device__ __forceinline__ static T id() { return make_uint2(0u, 1u); }
  __device__ __forceinline__ static T op(T l, T r) { return make_uint2(l.x * r.y + r.x, l.y * r.y); }
};

// ---------------------------------------------------------------- shuffles
__device__ __forceinline__ uint32_t shfl_up(uint32_t v, int o) { return __shfl_up_sync(0xffffffffu, v, o); }
__device__ __forceinline__ float shfl_up(float v, int o) { return __shfl_up_sync(0xffffffffu, v, o); }
__device__ __forceinline__ unsigned long long shfl_up(unsigned long long v, int o) { return __shfl_up_sync(0xffffffffu, v, o); }
__device__ __forceinline__ uint2 shfl_up(uint2 v, int o) {
  return make_uint2(__shfl_up_sync(0xffffffffu, v.x, o), __shfl_up_sync(0xffffffffu, v.y, o));
}
__device__ __forceinline__ uint32_t shfl_down(uint32_t v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ float shfl_down(float v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ unsigned long long shfl_down(unsigned long long v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ uint2 shfl_down(uint2 v, int o) {
  return make_uint2(__shfl_down_sync(0xffffffffu, v.x, o), __shfl_down_sync(0xffffffffu, v.y, o));
}

__device__ __forceinline__ uint32_t shfl_idx(uint32_t v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ float shfl_idx(float v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ unsigned long long shfl_idx(unsigned long long v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ uint2 shfl_idx(uint2 v, int l) {
  return make_uint2(__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l));
}

// ---------------------------------------------------------------- segmented scans
// A segment value: f = "a segment boundary lies inside", v = fold of the open part.
template <class T>
struct Seg {
  bool f;
  T v;
};

// Forward (left-to-right) combine: a is the earlier part.
template <class Op>
__device__ __forceinline__ Seg<typename Op::T> seg_fwd(Seg<typename Op::T> a, Seg<typename Op::T> b) {
  return {a.f || b.f, b.f ? b.v : Op::op(a.v, b.v)};
}
// Backward (right-to-left) combine: l is the nearer (earlier) part, r the farther one.
template <class Op>
__device__ __forceinline__ Seg<typename Op::T> seg_bwd(Seg<typename Op::T> l, Seg<typename Op::T> r) {
  return {l.f || r.f, l.f ? l.v : Op::op(l.v, r.v)};
}

// Shared scratch for the two block-wide segmented scans.
template <class Op, int TPB>
struct SegScratch {
  typename Op::T v[TPB / 32];
  bool f[TPB / 32];
};

// Exclusive forward segmented scan over the threads of the block (thread order).
template <class Op, int TPB>
__device__ __forceinline__ Seg<typename Op::T> block_seg_fwd_excl(Seg<typename Op::T> s, SegScratch<Op, TPB>& sh) {
  using T = typename Op::T;
  constexpr int NW = TPB / 32;
  const unsigned lane = lane_id(), wid = warp_id();
  Seg<T> x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg<T> y{(bool)__shfl_up_sync(0xffffffffu, (int)x.f, o), shfl_up(x.v, o)};
    if (lane >= (unsigned)o) x = seg_fwd<Op>(y, x);
  }
  Seg<T> ex{(bool)__shfl_up_sync(0xffffffffu, (int)x.f, 1), shfl_up(x.v, 1)};
  if (lane == 0) ex = Seg<T>{false, Op::id()};
  if (lane == 31) { sh.v[wid] = x.v; sh.f[wid] = x.f; }
  __syncthreads();
  if (wid == 0) {
    Seg<T> w = lane < (unsigned)NW ? Seg<T>{sh.f[lane], sh.v[lane]} : Seg<T>{false, Op::id()};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      Seg<T> y{(bool)__shfl_up_sync(0xffffffffu, (int)w.f, o), shfl_up(w.v, o)};
      if (lane >= (unsigned)o) w = seg_fwd<Op>(y, w);
    }
    Seg<T> we{(bool)__shfl_up_sync(0xffffffffu, (int)w.f, 1), shfl_up(w.v, 1)};
    if (lane == 0) we = Seg<T>{false, Op::id()};
    if (lane < (unsigned)NW) { sh.v[lane] = we.v; sh.f[lane] = we.f; }  // exclusive warp prefix
  }
  __syncthreads();
  Seg<T> wp{sh.f[wid], sh.v[wid]};
  __syncthreads();
  return seg_fwd<Op>(wp, ex);
}

// Exclusive backward segmented scan (fold of all LATER threads, nearest first).
template <class Op, int TPB>
__device__ __forceinline__ Seg<typename Op::T> block_seg_bwd_excl(Seg<typename Op::T> s, SegScratch<Op, TPB>& sh) {
  using T = typename Op::T;
  constexpr int NW = TPB / 32;
  const unsigned lane = lane_id(), wid = warp_id();
  Seg<T> x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    Seg<T> y{(bool)__shfl_down_sync(0xffffffffu, (int)x.f, o), shfl_down(x.v, o)};
    if (lane + o < 32u) x = seg_bwd<Op>(x, y);
  }
  Seg<T> ex{(bool)__shfl_down_sync(0xffffffffu, (int)x.f, 1), shfl_down(x.v, 1)};
  if (lane == 31) ex = Seg<T>{false, Op::id()};
  if (lane == 0) { sh.v[wid] = x.v; sh.f[wid] = x.f; }
  __syncthreads();
  if (wid == 0) {
    Seg<T> w = lane < (unsigned)NW ? Seg<T>{sh.f[lane], sh.v[lane]} : Seg<T>{false, Op::id()};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      Seg<T> y{(bool)__shfl_down_sync(0xffffffffu, (int)w.f, o), shfl_down(w.v, o)};
      if (lane + o < 32u) w = seg_bwd<Op>(w, y);
    }
    Seg<T> we{(bool)__shfl_down_sync(0xffffffffu, (int)w.f, 1), shfl_down(w.v, 1)};
    if (lane == 31) we = Seg<T>{false, Op::id()};
    if (lane < (unsigned)NW) { sh.v[lane] = we.v; sh.f[lane] = we.f; }
  }
  __syncthreads();
  Seg<T> wp{sh.f[wid], sh.v[wid]};
  __syncthreads();
  return seg_bwd<Op>(ex, wp);
}

// Algorithm 2's per-block prefix (X1) and suffix (Y1) folds, for a tile of TPB*E elements
// held "blocked" in registers (thread t owns tile elements tE .. tE+E-1).  Blocks have
// length w and start at tile indices congruent to `a` mod w; the tile's first element
// also starts a (partial) block and its last element ends one.
//   P[j] = fold of the elements from the start of j's block up to j      (prefix, X1)
//   S[j] = fold of the elements from j to the end of j's block           (suffix, Y1)
template <class Op, int TPB, int E>
__device__ __forceinline__ void block_prefix_suffix(const typename Op::T (&v)[E], typename Op::T (&P)[E],
                                                    typename Op::T (&S)[E], uint32_t w, uint32_t a,
                                                    SegScratch<Op, TPB>& sh) {
  static_assert(E <= 31, "head mask holds E+1 bits");
  using T = typename Op::T;
  const uint32_t e0 = threadIdx.x * E;
  // r0 = position of element e0 inside its block (0 = block start); 32-bit (e0 < 2^16, a < 2^32)
  uint32_t r0 = e0 % w;
  if (a) r0 = (r0 + w - a % w) % w;
  // heads bit j (0 <= j <= E): element e0+j starts a block; element j ends one iff bit j+1
  uint32_t heads = 0;
  for (uint32_t j = r0 ? w - r0 : 0u; j <= (uint32_t)E; j += w) heads |= 1u << j;
  constexpr uint32_t kMask = (1u << E) - 1u;
  // forward pass: P
  {
    T p = v[0];
    P[0] = p;
#pragma unroll
    for (int j = 1; j < E; ++j) {
      p = ((heads >> j) & 1u) ? v[j] : Op::op(p, v[j]);
      P[j] = p;
    }
    const bool has_head = (heads & kMask) != 0u;
    Seg<T> c = block_seg_fwd_excl<Op, TPB>(Seg<T>{has_head || threadIdx.x == 0, p}, sh);
    if (threadIdx.x > 0) {
      // elements before this thread's first head continue the block from the left
      const uint32_t open = (heads & kMask) ? ((heads & kMask) & (0u - (heads & kMask))) - 1u : kMask;
#pragma unroll
      for (int j = 0; j < E; ++j)
        if ((open >> j) & 1u) P[j] = Op::op(c.v, P[j]);
    }
  }
  // backward pass: S
  {
    const uint32_t tails = heads >> 1;  // bit j: element j ends a block (bit E-1: next thread starts one)
    T s = v[E - 1];
    S[E - 1] = s;
#pragma unroll
    for (int j = E - 2; j >= 0; --j) {
      s = ((tails >> j) & 1u) ? v[j] : Op::op(v[j], s);
      S[j] = s;
    }
    const bool has_tail = (tails & kMask) != 0u;
    Seg<T> c = block_seg_bwd_excl<Op, TPB>(Seg<T>{has_tail || threadIdx.x == TPB - 1, s}, sh);
    if (threadIdx.x < TPB - 1) {
      // elements after this thread's last tail continue into the block on the right
      const uint32_t tm = tails & kMask;
      const uint32_t open = tm ? (kMask & ~((2u << (31 - __clz(tm))) - 1u)) : kMask;
#pragma unroll
      for (int j = 0; j < E; ++j)
        if ((open >> j) & 1u) S[j] = Op::op(S[j], c.v);
    }
  }
}

// padded shared-memory index: one spare slot every 128 bytes (conflict-free blocked access)
template <class T>
__device__ __forceinline__ uint32_t pad_idx(uint32_t i) {
  return i + i / (128u / (uint32_t)sizeof(T));
}
template <class T>
__host__ __device__ constexpr uint32_t padded_len(uint32_t n) {
  return n + n / (128u / (uint32_t)sizeof(T)) + 1;
}

}  // namespace mzs
