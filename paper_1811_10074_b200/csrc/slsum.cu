// slsum.cu -- sliding window sums, Eq. 2:
//   y_i = x_i (+) x_{i+1} (+) ... (+) x_{i+w-1}
//
// GENERIC path: Algorithm 2 "VectorInput" (L123-150) re-planned for a CTA instead of a
// P-lane SIMD register.  A CTA tile of L = TPB*E inputs is split into blocks of length w;
// per block the prefix folds (Alg. 2's X1) and suffix folds (Alg. 2's Y1, the carry) are
// computed by a serial register strip per thread plus order-preserving segmented
// warp-shuffle scans across threads (Blelloch-style parallel scan, L150).  Then
//   y_i = S[i]                 if i starts a block
//   y_i = S[i] (+) P[i+w-1]    otherwise
// i.e. 3 (+) per output independent of w (L150: "for any operator (+)"; associativity
// only).  Consecutive tiles overlap by w-1 inputs (the carry of Alg. 2 becomes a halo).
//
// COMMUTATIVE path: ceil(log2 w) doubling rounds t_{r+1}[i] = t_r[i] (+) t_r[i+2^r] in
// shared memory (L44: "every sum ... is a prefix sum ... O(log(w))"; abstract L8), finished
// by the overlap t_m[i] (+) t_m[i+w-2^m] for idempotent ops or by the binary digits of w.
#include <algorithm>
#include <cstdlib>

#include "ops.cuh"

namespace mzs {
namespace {

// elements of one staged P or S array: L plus 16 B of padding per 128 B (and one spare vector)
inline bool env_flag(const char* name) {  // tests / A-B timing only
  const char* v = getenv(name);
  return v && v[0] == '1';
}

template <class T>
constexpr uint32_t slsum_smem_len(uint32_t L) {
  return L + (16 / sizeof(T)) * (L / (128 / sizeof(T)) + 1);
}

template <class T, uint32_t OV, uint32_t R>
__device__ __forceinline__ void take_shifted(const T (&lo)[OV], const T (&hi)[OV], T (&o)[OV]) {
#pragma unroll
  for (uint32_t q = 0; q < OV; ++q) o[q] = (R + q < OV) ? lo[R + q] : hi[R + q - OV];
}
// o[q] = A[b + sh + q] for A in the padded layout (sidx), b a multiple of OV, sh < OV uniform
// across the CTA: the two aligned 16-byte vectors around the run and a select (no divergence)
template <class T, uint32_t OV, class Idx>
__device__ __forceinline__ void ld_shifted_pad(const T* A, uint32_t b, uint32_t sh, Idx sidx, T (&o)[OV]) {
  T lo[OV], hi[OV];
  *reinterpret_cast<uint4*>(lo) = *reinterpret_cast<const uint4*>(A + sidx(b));
  if (sh == 0) {
#pragma unroll
    for (uint32_t q = 0; q < OV; ++q) o[q] = lo[q];
    return;
  }
  *reinterpret_cast<uint4*>(hi) = *reinterpret_cast<const uint4*>(A + sidx(b + OV));
  if constexpr (OV == 4) {
    if (sh == 1) take_shifted<T, OV, 1>(lo, hi, o);
    else if (sh == 2) take_shifted<T, OV, 2>(lo, hi, o);
    else take_shifted<T, OV, 3>(lo, hi, o);
  } else {
    take_shifted<T, OV, 1>(lo, hi, o);
  }
}

// One tile of L = TPB*E inputs per CTA (tout outputs + the w-1 halo).  P and S are staged in
// shared memory as 16-byte vectors with 16 B of padding every 128 B: the blocked 64-byte
// writes of 8 consecutive threads then hit 8 distinct bank groups, and the strided output
// reads stay conflict-free.  (A persistent variant with cp.async prefetch of the next tile
// measured slower on B200: 47 % vs 54 % of HBM at w = 4.)
template <class Op, int TPB, int E>
__global__ void __launch_bounds__(TPB) slsum_generic_kernel(const typename Op::T* __restrict__ x,
                                                           typename Op::T* __restrict__ y, uint64_t n,
                                                           uint32_t w, uint64_t nout, uint32_t tout) {
  using T = typename Op::T;
  constexpr uint32_t L = TPB * E;
  constexpr uint32_t OV = 16 / sizeof(T);   // elements per 16-byte vector
  constexpr uint32_t G = 128 / sizeof(T);   // elements per 128 bytes
  static_assert(E % OV == 0, "whole vectors per thread");
  auto sidx = [](uint32_t i) { return i + OV * (i / G); };
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sP = reinterpret_cast<T*>(smem_raw);
  T* sS = sP + slsum_smem_len<T>(L);
  __shared__ SegScratch<Op, TPB> sh;

  const uint64_t g0 = (uint64_t)blockIdx.x * tout;
  const uint32_t t = threadIdx.x;
  T v[E], P[E], S[E];
  {
    const uint64_t g = g0 + (uint64_t)t * E;
    if (g + E <= n && ((reinterpret_cast<uintptr_t>(x + g) & 15) == 0)) {
      const uint4* src = reinterpret_cast<const uint4*>(x + g);
#pragma unroll
      for (int q = 0; q < (int)(sizeof(T) * E / 16); ++q) {
        uint4 u = __ldg(src + q);
        *reinterpret_cast<uint4*>(reinterpret_cast<char*>(v) + 16 * q) = u;
      }
    } else {
#pragma unroll
      for (int j = 0; j < E; ++j) v[j] = (g + j < n) ? x[g + j] : Op::id();
    }
  }
  block_prefix_suffix<Op, TPB, E>(v, P, S, w, 0u, sh);
  {
    const uint32_t b0 = sidx(t * E);  // t*E is 64-byte aligned: no pad inside the thread's run
#pragma unroll
    for (int q = 0; q < E; q += OV) {
      *reinterpret_cast<uint4*>(sP + b0 + q) = *reinterpret_cast<const uint4*>(P + q);
      *reinterpret_cast<uint4*>(sS + b0 + q) = *reinterpret_cast<const uint4*>(S + q);
    }
  }
  __syncthreads();
  // outputs: y_i = S[i] if i starts a block, else S[i] (+) P[i+w-1]; OV consecutive outputs
  // per thread per step (one 16-byte store), e % w tracked incrementally
  const uint32_t e_end = (uint32_t)min((uint64_t)tout, nout - g0);
  uint32_t e_scalar = 0;
  if ((reinterpret_cast<uintptr_t>(y + g0) & 15) == 0) {
    const uint32_t step = (TPB * OV) % w;
    const uint32_t psh = (w - 1) % OV;        // P[e + w - 1 ..] starts psh past an aligned vector
    uint32_t e = t * OV;
    uint32_t r = e % w;
    for (; e + OV <= e_end; e += TPB * OV) {
      T s[OV], o[OV], pw[OV];
      *reinterpret_cast<uint4*>(s) = *reinterpret_cast<const uint4*>(sS + sidx(e));
      ld_shifted_pad<T, OV>(sP, e + w - 1 - psh, psh, sidx, pw);
      uint32_t rr = r;
#pragma unroll
      for (uint32_t q = 0; q < OV; ++q) {
        o[q] = (rr == 0) ? s[q] : Op::op(s[q], pw[q]);
        rr = (rr + 1 == w) ? 0u : rr + 1;
      }
      *reinterpret_cast<uint4*>(y + g0 + e) = *reinterpret_cast<const uint4*>(o);
      r += step;
      r -= (r >= w) ? w : 0u;
    }
    e_scalar = e_end / OV * OV;
  }
  for (uint32_t e = e_scalar + t; e < e_end; e += TPB) {  // unaligned y, or the last partial vector
    const T s = sS[sidx(e)];
    y[g0 + e] = (e % w == 0) ? s : Op::op(s, sP[sidx(e + w - 1)]);
  }
}

// Doubling rounds over a tile of L inputs held in two ping-pong shared buffers.  Every step of
// the rounds, loads and stores works on 16-byte vectors of OV = 16/sizeof(T) consecutive
// elements (one LDS.128 of A[e..], one of A[e+d..] when d is a multiple of OV, otherwise the
// shifted vector is assembled from two aligned ones; one STS.128), so a round costs a few
// instructions per element.  Interior tiles are loaded and stored with 16-byte global accesses.
// o[q] = A[e + d + q] for e a multiple of OV: one or two aligned 16-byte loads; the shift
// r = d mod OV is uniform across the CTA, so the switch does not diverge
template <class T, uint32_t OV>
__device__ __forceinline__ void ld_shifted(const T* A, uint32_t e, uint32_t d, T (&o)[OV]) {
  const uint32_t base = e + d, r = base % OV, a0 = base - r;
  T lo[OV], hi[OV];
  *reinterpret_cast<uint4*>(lo) = *reinterpret_cast<const uint4*>(A + a0);
  if (r == 0) {
#pragma unroll
    for (uint32_t q = 0; q < OV; ++q) o[q] = lo[q];
    return;
  }
  *reinterpret_cast<uint4*>(hi) = *reinterpret_cast<const uint4*>(A + a0 + OV);
  if constexpr (OV == 4) {
    if (r == 1) take_shifted<T, OV, 1>(lo, hi, o);
    else if (r == 2) take_shifted<T, OV, 2>(lo, hi, o);
    else take_shifted<T, OV, 3>(lo, hi, o);
  } else {
    take_shifted<T, OV, 1>(lo, hi, o);
  }
}

template <class Op, int TPB>
__global__ void __launch_bounds__(TPB) slsum_doubling_kernel(const typename Op::T* __restrict__ x,
                                                            typename Op::T* __restrict__ y, uint64_t n,
                                                            uint32_t w, uint64_t nout, uint32_t L,
                                                            uint32_t tout) {
  using T = typename Op::T;
  constexpr uint32_t OV = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* A = reinterpret_cast<T*>(smem_raw);
  T* B = A + L + 2 * OV;  // (+2 vectors: shifted reads past L stay inside the buffer)
  const uint64_t g0 = (uint64_t)blockIdx.x * tout;
  const uint32_t t = threadIdx.x;
  const bool vin = ((reinterpret_cast<uintptr_t>(x + g0) & 15) == 0) && g0 + L <= n;
  if (vin) {
    for (uint32_t e = t * OV; e < L; e += TPB * OV)
      *reinterpret_cast<uint4*>(A + e) = __ldg(reinterpret_cast<const uint4*>(x + g0 + e));
  } else {
    for (uint32_t e = t; e < L; e += TPB) A[e] = (g0 + e < n) ? x[g0 + e] : Op::id();
  }
  for (uint32_t e = L + t; e < L + 2 * OV; e += TPB) A[e] = Op::id();
  __syncthreads();
  // m = floor(log2 w)
  const int m = 31 - __clz(w);
  const uint32_t e_end = (uint32_t)min((uint64_t)tout, nout - g0);
  const bool vout = ((reinterpret_cast<uintptr_t>(y + g0) & 15) == 0) && e_end == tout;
  if (Op::kIdempotent) {
    for (int r = 0; r < m; ++r) {
      const uint32_t d = 1u << r;
      for (uint32_t e = t * OV; e + d < L; e += TPB * OV) {
        T a[OV], c[OV], o[OV];
        *reinterpret_cast<uint4*>(a) = *reinterpret_cast<const uint4*>(A + e);
        ld_shifted<T, OV>(A, e, d, c);
#pragma unroll
        for (uint32_t q = 0; q < OV; ++q) o[q] = Op::op(a[q], c[q]);
        *reinterpret_cast<uint4*>(B + e) = *reinterpret_cast<const uint4*>(o);
      }
      __syncthreads();
      T* tmp = A; A = B; B = tmp;
    }
    const uint32_t d = w - (1u << m);
    if (vout) {
      for (uint32_t e = t * OV; e < tout; e += TPB * OV) {
        T a[OV], c[OV], o[OV];
        *reinterpret_cast<uint4*>(a) = *reinterpret_cast<const uint4*>(A + e);
        ld_shifted<T, OV>(A, e, d, c);
#pragma unroll
        for (uint32_t q = 0; q < OV; ++q) o[q] = d ? Op::op(a[q], c[q]) : a[q];
        *reinterpret_cast<uint4*>(y + g0 + e) = *reinterpret_cast<const uint4*>(o);
      }
    } else {
      for (uint32_t e = t; e < e_end; e += TPB) y[g0 + e] = d ? Op::op(A[e], A[e + d]) : A[e];
    }
  } else {
    // binary digits of w, smallest piece leftmost: y_i = t_c0[i] (+) t_c1[i+2^c0] (+) ...
    constexpr int NV = 8 / (int)OV;  // output vectors per thread: 8 outputs (tout = 8*TPB, host-enforced)
    T acc[NV][OV];
#pragma unroll
    for (int j = 0; j < NV; ++j)
#pragma unroll
      for (uint32_t q = 0; q < OV; ++q) acc[j][q] = Op::id();
    uint32_t off = 0;
    for (int r = 0; r <= m; ++r) {
      if ((w >> r) & 1u) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const uint32_t e = (t + j * TPB) * OV;
          if (e < tout) {
            T c[OV];
            ld_shifted<T, OV>(A, e, off, c);
#pragma unroll
            for (uint32_t q = 0; q < OV; ++q) acc[j][q] = Op::op(acc[j][q], c[q]);
          }
        }
        off += 1u << r;
      }
      if (r < m) {
        const uint32_t d = 1u << r;
        for (uint32_t e = t * OV; e + d < L; e += TPB * OV) {
          T a[OV], c[OV], o[OV];
          *reinterpret_cast<uint4*>(a) = *reinterpret_cast<const uint4*>(A + e);
          ld_shifted<T, OV>(A, e, d, c);
#pragma unroll
          for (uint32_t q = 0; q < OV; ++q) o[q] = Op::op(a[q], c[q]);
          *reinterpret_cast<uint4*>(B + e) = *reinterpret_cast<const uint4*>(o);
        }
        __syncthreads();
        T* tmp = A; A = B; B = tmp;
      }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const uint32_t e = (t + j * TPB) * OV;
      if (vout) {
        if (e < tout) *reinterpret_cast<uint4*>(y + g0 + e) = *reinterpret_cast<const uint4*>(acc[j]);
      } else {
#pragma unroll
        for (uint32_t q = 0; q < OV; ++q)
          if (e + q < e_end) y[g0 + e + q] = acc[j][q];
      }
    }
  }
}


// GENERIC path for small power-of-two w (W | E): the same block decomposition (Alg. 2, blocks
// of W aligned at the warp tile), but a block never straddles two lanes, so P and S are pure
// register strips and the only exchange is the W-1 prefix values the last outputs of a lane
// need from the next lane (shuffles).  Each warp owns a tile of 32E inputs and emits the first
// 31E outputs (the last lane is the halo), so there is no shared memory and no barrier.
template <class Op, int W, int EE = 0>
__global__ void __launch_bounds__(256) slsum_generic_warp_kernel(const typename Op::T* __restrict__ x,
                                                                typename Op::T* __restrict__ y, uint64_t n,
                                                                uint64_t nout) {
  using T = typename Op::T;
  // EE: elements per lane when it is not the default 16 (8 for 8-byte types): a multiple of
  // both W and the 16-byte vector, so that small w which do not divide 16 (3, 5, 6, 7, 10,
  // 12, 14) also keep whole blocks inside a lane
  constexpr int E = EE ? EE : ((sizeof(T) == 4) ? 16 : 8);
  constexpr uint32_t OV = 16 / sizeof(T);
  static_assert(E % W == 0 && W <= E, "blocks inside a lane");
  constexpr uint64_t kOut = 31ull * E;  // outputs per warp
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t t0 = warp * kOut;            // first input (and output) of the warp's tile
  if (t0 >= nout) return;                     // uniform per warp
  const uint64_t g = t0 + (uint64_t)lane * E;
  T v[E];
  if (g + E <= n && ((reinterpret_cast<uintptr_t>(x + g) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(v + q) = __ldg(reinterpret_cast<const uint4*>(x + g + q));
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = (g + j < n) ? x[g + j] : Op::id();
  }
  // P: prefix fold from the start of the block; S: suffix fold to its end (blocks of W)
  T P[E], S[E];
#pragma unroll
  for (int j = 0; j < E; ++j) P[j] = (j % W == 0) ? v[j] : Op::op(P[j - (j % W == 0 ? 0 : 1)], v[j]);
#pragma unroll
  for (int j = E - 1; j >= 0; --j) S[j] = (j % W == W - 1) ? v[j] : Op::op(v[j], S[j + (j % W == W - 1 ? 0 : 1)]);
  // the next lane's first W-1 prefix values
  T Pn[W > 1 ? W - 1 : 1];
#pragma unroll
  for (int q = 0; q < W - 1; ++q) Pn[q] = shfl_down(P[q], 1);
  if (lane == 31) return;                     // the halo lane has no outputs of its own
  T o[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    if (j % W == 0) o[j] = S[j];
    else o[j] = Op::op(S[j], (j + W - 1 < E) ? P[(j + W - 1) % E] : Pn[(j + W - 1 - E) % (W > 1 ? W - 1 : 1)]);
  }
  if (g + E <= nout && ((reinterpret_cast<uintptr_t>(y + g) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(y + g + q) = *reinterpret_cast<const uint4*>(o + q);
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j)
      if (g + j < nout) y[g + j] = o[j];
  }
}

template <class Op, int W, int EE = 0>
int launch_generic_warp(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  constexpr int E = EE ? EE : ((sizeof(T) == 4) ? 16 : 8);
  const uint64_t nout = n - w + 1;
  const uint64_t warps = (nout + 31ull * E - 1) / (31ull * E);
  const uint64_t grid = (warps + 7) / 8;
  slsum_generic_warp_kernel<Op, W, EE><<<(unsigned)grid, 256, 0, st>>>(static_cast<const T*>(xv), static_cast<T*>(yv),
                                                                      n, nout);
  MZS_LAUNCHED();
  return SLSUM_OK;
}


// GENERIC path for w = M*E (M in {2,4,8} lanes per block): blocks span M aligned lanes of a
// warp.  P and S are in-lane prefix / suffix strips plus an M-lane exclusive scan across the
// block's lanes (order-preserving: the left operand is always the earlier part); the combine
// takes P[i+w-1] from lanes l+M and l+M-1 by shuffles.  A warp emits (32-M)*E outputs (the
// last M lanes are the halo); no shared memory, no barrier.
template <class Op, int M>
__global__ void __launch_bounds__(256) slsum_generic_warpm_kernel(const typename Op::T* __restrict__ x,
                                                                 typename Op::T* __restrict__ y, uint64_t n,
                                                                 uint64_t nout) {
  using T = typename Op::T;
  constexpr int E = (sizeof(T) == 4) ? 16 : 8;
  constexpr uint32_t OV = 16 / sizeof(T);
  static_assert(M >= 2 && M <= 16 && (M & (M - 1)) == 0, "M lanes per block");
  constexpr uint64_t kOut = (uint64_t)(32 - M) * E;  // outputs per warp
  const uint32_t lane = threadIdx.x & 31, gl = lane & (M - 1);  // lane inside its block
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t t0 = warp * kOut;
  if (t0 >= nout) return;  // uniform per warp
  const uint64_t g = t0 + (uint64_t)lane * E;
  T v[E];
  if (g + E <= n && ((reinterpret_cast<uintptr_t>(x + g) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(v + q) = __ldg(reinterpret_cast<const uint4*>(x + g + q));
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = (g + j < n) ? x[g + j] : Op::id();
  }
  T P[E], S[E];
  P[0] = v[0];
#pragma unroll
  for (int j = 1; j < E; ++j) P[j] = Op::op(P[j - 1], v[j]);
  S[E - 1] = v[E - 1];
#pragma unroll
  for (int j = E - 2; j >= 0; --j) S[j] = Op::op(v[j], S[j + 1]);
  // exclusive fold of the lanes to the left inside the block (forward), to the right (backward)
  T lt = P[E - 1], rt = S[0];   // running inclusive folds
#pragma unroll
  for (int o = 1; o < M; o <<= 1) {
    const T a = shfl_up(lt, o);
    const T b = shfl_down(rt, o);
    if (gl >= (uint32_t)o) lt = Op::op(a, lt);
    if (gl + o < (uint32_t)M) rt = Op::op(rt, b);
  }
  const T le = shfl_up(lt, 1), re = shfl_down(rt, 1);  // exclusive: the neighbour's inclusive fold
  if (gl > 0) {
#pragma unroll
    for (int j = 0; j < E; ++j) P[j] = Op::op(le, P[j]);
  }
  if (gl < (uint32_t)(M - 1)) {
#pragma unroll
    for (int j = 0; j < E; ++j) S[j] = Op::op(S[j], re);
  }
  // y_i = S[i] (+) P[i+w-1]: element j >= 1 takes lane l+M's P[j-1], element 0 lane l+M-1's P[E-1]
  T Pm[E];
#pragma unroll
  for (int j = 0; j < E - 1; ++j) Pm[j] = shfl_down(P[j], M);
  Pm[E - 1] = shfl_down(P[E - 1], M - 1);
  if (lane >= 32 - M) return;  // halo lanes
  T o[E];
  o[0] = (gl == 0) ? S[0] : Op::op(S[0], Pm[E - 1]);  // a block head is its own window start
#pragma unroll
  for (int j = 1; j < E; ++j) o[j] = Op::op(S[j], Pm[j - 1]);
  if (g + E <= nout && ((reinterpret_cast<uintptr_t>(y + g) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(y + g + q) = *reinterpret_cast<const uint4*>(o + q);
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j)
      if (g + j < nout) y[g + j] = o[j];
  }
}

template <class Op, int M>
int launch_generic_warpm(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  constexpr int E = (sizeof(T) == 4) ? 16 : 8;
  const uint64_t nout = n - w + 1;
  const uint64_t warps = (nout + (uint64_t)(32 - M) * E - 1) / ((uint64_t)(32 - M) * E);
  const uint64_t grid = (warps + 7) / 8;
  slsum_generic_warpm_kernel<Op, M><<<(unsigned)grid, 256, 0, st>>>(static_cast<const T*>(xv), static_cast<T*>(yv),
                                                                   n, nout);
  MZS_LAUNCHED();
  return SLSUM_OK;
}


// GENERIC path for w = M*E with M >= 16 lanes per block (w = 256 .. 2048 for 4-byte types):
// the warp-tiled decomposition at CTA scale.  In-lane P/S strips, shuffle scans across the
// block's lanes inside a warp, a shared-memory step across warps when a block spans several
// warps (M > 32); P is then staged in shared memory (16 B of padding per 128 B) so that every
// lane can read the P[i+w-1] of the block M lanes ahead.  A CTA of TPB lanes emits (TPB-M)*E
// outputs (the last M lanes are the halo).
template <class Op, int TPB, int M>
__global__ void __launch_bounds__(TPB) slsum_generic_cta_kernel(const typename Op::T* __restrict__ x,
                                                                typename Op::T* __restrict__ y, uint64_t n,
                                                                uint64_t nout) {
  using T = typename Op::T;
  constexpr int E = (sizeof(T) == 4) ? 16 : 8;
  constexpr uint32_t OV = 16 / sizeof(T);
  constexpr uint32_t G = 128 / sizeof(T);
  constexpr int L = TPB * E;
  constexpr int NW = TPB / 32;
  constexpr int MW = M < 32 ? M : 32;  // lanes of one block inside one warp
  static_assert(M >= 16 && (M & (M - 1)) == 0 && M < TPB, "M lanes per block");
  constexpr uint64_t kOut = (uint64_t)(TPB - M) * E;
  auto sidx = [](uint32_t i) { return i + OV * (i / G); };
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sP = reinterpret_cast<T*>(smem_raw);
  __shared__ T wl[NW], wr[NW];  // per-warp left / right folds of its part of a block
  const uint32_t t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint32_t gl = t & (M - 1);          // lane inside its block
  const uint32_t gw = lane & (MW - 1);      // lane inside its block's part of this warp
  const uint64_t t0 = (uint64_t)blockIdx.x * kOut;
  const uint64_t g = t0 + (uint64_t)t * E;
  T v[E];
  if (g + E <= n && ((reinterpret_cast<uintptr_t>(x + g) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(v + q) = __ldg(reinterpret_cast<const uint4*>(x + g + q));
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = (g + j < n) ? x[g + j] : Op::id();
  }
  T P[E], S[E];
  P[0] = v[0];
#pragma unroll
  for (int j = 1; j < E; ++j) P[j] = Op::op(P[j - 1], v[j]);
  S[E - 1] = v[E - 1];
#pragma unroll
  for (int j = E - 2; j >= 0; --j) S[j] = Op::op(v[j], S[j + 1]);
  T lt = P[E - 1], rt = S[0];  // inclusive folds across the block's lanes in this warp
#pragma unroll
  for (int o = 1; o < MW; o <<= 1) {
    const T a = shfl_up(lt, o);
    const T b = shfl_down(rt, o);
    if (gw >= (uint32_t)o) lt = Op::op(a, lt);
    if (gw + o < (uint32_t)MW) rt = Op::op(rt, b);
  }
  T le = shfl_up(lt, 1), re = shfl_down(rt, 1);  // exclusive, inside the warp
  bool has_le = gw > 0, has_re = gw + 1 < (uint32_t)MW;
  if (M > 32) {
    // blocks span M/32 warps: fold in the totals of the block's earlier / later warps
    if (lane == 31) wl[wid] = lt;
    if (lane == 0) wr[wid] = rt;
    __syncthreads();
    constexpr int BW = M > 32 ? M / 32 : 1;  // warps per block
    const int wb = (int)(wid & (BW - 1));     // warp index inside the block
    if (wb > 0) {
      T c = wl[wid - wb];
      for (int q = 1; q < wb; ++q) c = Op::op(c, wl[wid - wb + q]);
      le = has_le ? Op::op(c, le) : c;
      has_le = true;
    }
    if (wb < BW - 1) {
      T c = wr[wid + BW - 1 - wb];
      for (int q = BW - 2 - wb; q >= 1; --q) c = Op::op(wr[wid + q], c);
      re = has_re ? Op::op(re, c) : c;
      has_re = true;
    }
  }
  if (has_le) {
#pragma unroll
    for (int j = 0; j < E; ++j) P[j] = Op::op(le, P[j]);
  }
  if (has_re) {
#pragma unroll
    for (int j = 0; j < E; ++j) S[j] = Op::op(S[j], re);
  }
  {
    const uint32_t b0 = sidx(t * E);
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(sP + b0 + q) = *reinterpret_cast<const uint4*>(P + q);
  }
  __syncthreads();
  if (t >= (uint32_t)(TPB - M)) return;  // halo lanes
  // y_i = S[i] (+) P[i+w-1]; for this lane i+w-1 = (t+M)*E - 1 + j
  T Pw[E];
  Pw[0] = sP[sidx((t + M) * E - 1)];
  {
    T nx[E];
    const uint32_t b1 = sidx((t + M) * E);
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(nx + q) = *reinterpret_cast<const uint4*>(sP + b1 + q);
#pragma unroll
    for (int j = 1; j < E; ++j) Pw[j] = nx[j - 1];
  }
  T o[E];
  o[0] = (gl == 0) ? S[0] : Op::op(S[0], Pw[0]);
#pragma unroll
  for (int j = 1; j < E; ++j) o[j] = Op::op(S[j], Pw[j]);
  if (g + E <= nout && ((reinterpret_cast<uintptr_t>(y + g) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(y + g + q) = *reinterpret_cast<const uint4*>(o + q);
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j)
      if (g + j < nout) y[g + j] = o[j];
  }
}

template <class Op, int TPB, int M>
int launch_generic_cta(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  constexpr int E = (sizeof(T) == 4) ? 16 : 8;
  const uint64_t nout = n - w + 1;
  const uint64_t kOut = (uint64_t)(TPB - M) * E;
  const uint64_t grid = (nout + kOut - 1) / kOut;
  const size_t smem = sizeof(T) * slsum_smem_len<T>(TPB * E);
  auto k = slsum_generic_cta_kernel<Op, TPB, M>;
  MZS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)grid, TPB, smem, st>>>(static_cast<const T*>(xv), static_cast<T*>(yv), n, nout);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

// GENERIC path, a TEAM of NWT warps per block of w = 32*EL*NWT inputs (EL = 8 consecutive per
// lane), streaming: every team walks its own contiguous range of blocks and keeps the suffix
// folds S of the previous block in registers, so there is no halo except one block per team
// range, and the only synchronisation is a named barrier among the team's warps per block.
// Per block b+1 (warp k holds its part k):
//   in-lane prefix and suffix strips, warp shuffle scans -> the part's local P and S and its
//   left / right folds T_k, R_k (shared memory, two slots by parity) -> team barrier ->
//   carries C_k = T_0 (+) .. (+) T_{k-1}, D_k = R_{k+1} (+) .. (+) R_{NWT-1};
//   P = C_k (+) P_local, S = S_local (+) D_k;
//   outputs of block b: y_i = S_b[i] (+) P_{b+1}[i+w-1], the P one position to the left: the
//   same register, the previous lane's last, or (lane 0 of warp k > 0) C_k itself.
// Operand order is preserved (any associative op).  NWT = 1 needs no shared memory at all.
constexpr int kTeamEL = 8;

// RT (round 2b): any block length w with 256 (NWT-1) < w <= 256 NWT -- the block's slots past
// w hold the identity (they never reach an output: S folds them in as identities, P stops
// before them), blocks start at b * w (16-byte vector loads only for the blocks that start on
// a vector), so every w in (256, 2048] streams like the powers of two.
template <class Op, int NWT, bool RT = false>
__global__ void __launch_bounds__(256) slsum_generic_team_kernel(const typename Op::T* __restrict__ x,
                                                                typename Op::T* __restrict__ y, uint64_t n,
                                                                uint64_t nout, uint64_t blocks_per_team,
                                                                uint32_t w_rt = 0) {
  using T = typename Op::T;
  constexpr int EL = kTeamEL;
  constexpr uint32_t OV = 16 / sizeof(T);
  constexpr uint32_t PW = 32 * EL;                          // elements of one warp's part
  const uint32_t W = RT ? w_rt : PW * NWT;
  constexpr int NTEAM = 8 / NWT;                            // teams per 256-thread CTA
  static_assert(EL % OV == 0 && NWT >= 1 && NWT <= 8 && (RT || 8 % NWT == 0), "team shape");
  __shared__ T sT[2][NTEAM][NWT], sR[2][NTEAM][NWT];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t team = wid / NWT, k = wid % NWT;
  const uint64_t gteam = (uint64_t)blockIdx.x * NTEAM + team;
  const uint64_t nb = (n + W - 1) / W;
  const uint64_t nbo = (nout + W - 1) / W;
  const uint64_t b0 = gteam * blocks_per_team;
  if (b0 >= nbo) return;                                    // whole teams leave together
  const uint64_t b1 = min(nbo, b0 + blocks_per_team);
  const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  auto team_sync = [&]() {
    if (NWT > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(32 * NWT) : "memory");
  };
  const uint32_t loc0 = k * PW + lane * EL;                 // this lane's first slot in a block
  auto load = [&](uint64_t b, T (&v)[EL]) {
    const uint64_t g = b * W + loc0;
    if (aligned && b + 1 < nb && (!RT || (loc0 + EL <= W && ((b * W) % OV) == 0))) {
#pragma unroll
      for (int q = 0; q < EL; q += OV) *reinterpret_cast<uint4*>(v + q) = __ldg(reinterpret_cast<const uint4*>(x + g + q));
    } else {
#pragma unroll
      for (int j = 0; j < EL; ++j) v[j] = (g + j < n && (!RT || loc0 + j < W)) ? x[g + j] : Op::id();
    }
  };
  int par = 0;
  // block b's prefix folds into v (in place) and suffix folds into S (from v), both team-wide;
  // returns C_k (the fold of the parts left of k; unused for k == 0)
  auto folds = [&](T (&v)[EL], T (&S)[EL]) -> T {
    S[EL - 1] = v[EL - 1];
#pragma unroll
    for (int j = EL - 2; j >= 0; --j) S[j] = Op::op(v[j], S[j + 1]);
#pragma unroll
    for (int j = 1; j < EL; ++j) v[j] = Op::op(v[j - 1], v[j]);
    T lt = v[EL - 1], rt = S[0];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T a = shfl_up(lt, o);
      const T c = shfl_down(rt, o);
      if (lane >= (uint32_t)o) lt = Op::op(a, lt);
      if (lane + o < 32) rt = Op::op(rt, c);
    }
    const T le = shfl_up(lt, 1), re = shfl_down(rt, 1);
    if (lane > 0) {
#pragma unroll
      for (int j = 0; j < EL; ++j) v[j] = Op::op(le, v[j]);
    }
    if (lane < 31) {
#pragma unroll
      for (int j = 0; j < EL; ++j) S[j] = Op::op(S[j], re);
    }
    T C = Op::id();
    if (NWT > 1) {
      const T tot_l = shfl_idx(lt, 31);     // fold of the whole part
      const T tot_r = shfl_idx(rt, 0);
      if (lane == 0) {
        sT[par][team][k] = tot_l;
        sR[par][team][k] = tot_r;
      }
      team_sync();
      if (k > 0) {
        C = sT[par][team][0];
        for (uint32_t q = 1; q < k; ++q) C = Op::op(C, sT[par][team][q]);
#pragma unroll
        for (int j = 0; j < EL; ++j) v[j] = Op::op(C, v[j]);
      }
      if (k + 1 < (uint32_t)NWT) {
        T D = sR[par][team][NWT - 1];
        for (int q = NWT - 2; q > (int)k; --q) D = Op::op(sR[par][team][q], D);
#pragma unroll
        for (int j = 0; j < EL; ++j) S[j] = Op::op(S[j], D);
      }
      par ^= 1;
    }
    return C;
  };
  T Sp[EL];
  {
    T v[EL];
    load(b0, v);
    folds(v, Sp);
  }
  for (uint64_t b = b0; b < b1; ++b) {
    T v[EL], Sn[EL];
    load(b + 1, v);
    const T C = folds(v, Sn);                               // v: P of block b+1
    const T pl = shfl_up(v[EL - 1], 1);                     // the previous lane's last prefix
    T o[EL];
    if (lane > 0) o[0] = Op::op(Sp[0], pl);
    else o[0] = k == 0 ? Sp[0] : Op::op(Sp[0], C);
#pragma unroll
    for (int j = 1; j < EL; ++j) o[j] = Op::op(Sp[j], v[j - 1]);
    const uint64_t g = b * W + loc0;
    MZS_DCHECK(b < nb);
    if (aligned && g + EL <= nout && (!RT || (loc0 + EL <= W && ((b * W) % OV) == 0))) {
#pragma unroll
      for (int q = 0; q < EL; q += OV) *reinterpret_cast<uint4*>(y + g + q) = *reinterpret_cast<const uint4*>(o + q);
    } else {
#pragma unroll
      for (int j = 0; j < EL; ++j)
        if (g + j < nout && (!RT || loc0 + j < W)) y[g + j] = o[j];
    }
#pragma unroll
    for (int j = 0; j < EL; ++j) Sp[j] = Sn[j];
  }
}

template <class Op, int NWT, bool RT = false>
int launch_generic_team(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  const uint32_t W = RT ? w : 32 * kTeamEL * NWT;
  const uint64_t nout = n - w + 1;
  const uint64_t nbo = (nout + W - 1) / W;
  static int occ = 0;
  if (occ == 0) {
    MZS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slsum_generic_team_kernel<Op, NWT, RT>,
                                                           32 * NWT * (8 / NWT), 0));
    occ = std::max(occ, 1);
  }
  constexpr int NTEAM = 8 / NWT;                 // teams per CTA (CTA = 32 NWT NTEAM <= 256 threads)
  const uint64_t teams = (uint64_t)num_sms() * occ * NTEAM;
  const uint64_t per = std::max<uint64_t>(4, (nbo + teams - 1) / teams);
  const uint64_t nt = (nbo + per - 1) / per;
  const uint64_t grid = (nt + NTEAM - 1) / NTEAM;
  slsum_generic_team_kernel<Op, NWT, RT><<<(unsigned)grid, 32 * NWT * NTEAM, 0, st>>>(static_cast<const T*>(xv),
                                                                         static_cast<T*>(yv), n, nout, per, w);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

template <class Op>
int launch_generic(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  constexpr int E = (sizeof(T) == 4) ? 16 : 8;
  // small power-of-two w: the warp-tiled, shared-memory-free variant of the same decomposition
  if (!env_flag("MZS_SLSUM_NO_WARP")) {
    if (w == 2) return launch_generic_warp<Op, 2>(xv, yv, n, w, st);
    if (w == 4) return launch_generic_warp<Op, 4>(xv, yv, n, w, st);
    if (w == 8) return launch_generic_warp<Op, 8>(xv, yv, n, w, st);
    if (w == 16 && E >= 16) return launch_generic_warp<Op, E >= 16 ? 16 : 8>(xv, yv, n, w, st);
    // small w that do not divide E: lanes of a multiple of lcm(w, 16-byte vector) elements
    constexpr bool B4 = sizeof(T) == 4;
    if (w == 3) return launch_generic_warp<Op, 3, B4 ? 24 : 12>(xv, yv, n, w, st);
    if (w == 5) return launch_generic_warp<Op, 5, B4 ? 20 : 10>(xv, yv, n, w, st);
    if (w == 6) return launch_generic_warp<Op, 6, B4 ? 24 : 12>(xv, yv, n, w, st);
    if (w == 7) return launch_generic_warp<Op, 7, B4 ? 28 : 14>(xv, yv, n, w, st);
    if (w == 10) return launch_generic_warp<Op, 10, B4 ? 20 : 10>(xv, yv, n, w, st);
    if (w == 12) return launch_generic_warp<Op, 12, B4 ? 24 : 12>(xv, yv, n, w, st);
    if (w == 14) return launch_generic_warp<Op, 14, B4 ? 28 : 14>(xv, yv, n, w, st);
    if (w == 9) return launch_generic_warp<Op, 9, B4 ? 36 : 18>(xv, yv, n, w, st);
    if (w == 11) return launch_generic_warp<Op, 11, B4 ? 44 : 22>(xv, yv, n, w, st);
    if (w == 13) return launch_generic_warp<Op, 13, B4 ? 52 : 26>(xv, yv, n, w, st);
    if (w == 15) return launch_generic_warp<Op, 15, B4 ? 60 : 30>(xv, yv, n, w, st);
    if (w == 20) return launch_generic_warp<Op, 20, 20>(xv, yv, n, w, st);
    if (w == 24) return launch_generic_warp<Op, 24, 24>(xv, yv, n, w, st);
    if (w == 28) return launch_generic_warp<Op, 28, 28>(xv, yv, n, w, st);
    if (w == 18) return launch_generic_warp<Op, 18, B4 ? 36 : 18>(xv, yv, n, w, st);
    if (w == 22) return launch_generic_warp<Op, 22, B4 ? 44 : 22>(xv, yv, n, w, st);
    if (w == 26) return launch_generic_warp<Op, 26, B4 ? 52 : 26>(xv, yv, n, w, st);
    if (w == 30) return launch_generic_warp<Op, 30, B4 ? 60 : 30>(xv, yv, n, w, st);
    if (w == 2 * E) return launch_generic_warpm<Op, 2>(xv, yv, n, w, st);
    if (w == 4 * E) return launch_generic_warpm<Op, 4>(xv, yv, n, w, st);
    if (w == 8 * E) return launch_generic_warpm<Op, 8>(xv, yv, n, w, st);
    if (!env_flag("MZS_SLSUM_NO_TEAM")) {            // a team of warps per block, streaming
      if (w == 256) return launch_generic_team<Op, 1>(xv, yv, n, w, st);
      if (w == 512) return launch_generic_team<Op, 2>(xv, yv, n, w, st);
      if (w == 1024) return launch_generic_team<Op, 4>(xv, yv, n, w, st);
      if (w == 2048) return launch_generic_team<Op, 8>(xv, yv, n, w, st);
      // any other w in (256, 2048]: the same team kernel with a runtime block length
      // (NWT = ceil(w / 256) warps per team; taken when at most a quarter of the slots pad)
      const uint32_t nwt = (w + 255) / 256;
      if (w > 256 && w <= 2048 && 4 * w >= 3 * 256 * nwt && !env_flag("MZS_SLSUM_NO_TEAM_RT")) {
        switch (nwt) {
          case 2: return launch_generic_team<Op, 2, true>(xv, yv, n, w, st);
          case 3: return launch_generic_team<Op, 3, true>(xv, yv, n, w, st);
          case 4: return launch_generic_team<Op, 4, true>(xv, yv, n, w, st);
          case 5: return launch_generic_team<Op, 5, true>(xv, yv, n, w, st);
          case 6: return launch_generic_team<Op, 6, true>(xv, yv, n, w, st);
          case 7: return launch_generic_team<Op, 7, true>(xv, yv, n, w, st);
          default: return launch_generic_team<Op, 8, true>(xv, yv, n, w, st);
        }
      }
    }
    if (w == 16 * E) return launch_generic_cta<Op, 256, 16>(xv, yv, n, w, st);  // 256 > 512 lanes (75 vs 68 %)
    if (w == 32 * E) return launch_generic_cta<Op, 512, 32>(xv, yv, n, w, st);
    if (w == 64 * E) return launch_generic_cta<Op, 512, 64>(xv, yv, n, w, st);  // 512 > 1024 lanes (61 vs 54 %)
  }
  const uint64_t nout = n - w + 1;
  // smallest CTA whose tile keeps the halo (w-1) under 1/8 of it; 1024 threads max
  int tpb = 256;
  while (tpb < 1024 && (uint64_t)(w - 1) * 8 > (uint64_t)tpb * E) tpb *= 2;
  const uint32_t L = tpb * E;
  if (w - 1 >= L / 2) return SLSUM_EUNSUPPORTED;  // w > ~8192 (4-byte) / ~4096 (8-byte)
  uint32_t tout = (L - (w - 1)) & ~31u;
  if (tout == 0) tout = L - (w - 1);
  const uint64_t grid = (nout + tout - 1) / tout;
  const size_t smem = 2 * sizeof(T) * slsum_smem_len<T>(L);
  const T* x = static_cast<const T*>(xv);
  T* y = static_cast<T*>(yv);
#define MZS_GEN(TPB_)                                                                          \
  do {                                                                                         \
    auto k = slsum_generic_kernel<Op, TPB_, E>;                                                \
    MZS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k<<<(unsigned)grid, TPB_, smem, st>>>(x, y, n, w, nout, tout);                            \
  } while (0)
  if (tpb == 256) MZS_GEN(256);
  else if (tpb == 512) MZS_GEN(512);
  else MZS_GEN(1024);
#undef MZS_GEN
  MZS_LAUNCHED();
  return SLSUM_OK;
}


// COMMUTATIVE path for small w (powers of two up to 4E, and 3..15): the doubling rounds
// t_{r+1}[i] = t_r[i] (+) t_r[i + 2^r] on a warp tile held in registers (E consecutive values
// per lane).  A shift by s < E pulls the next lane's first s values by shuffles; a shift by
// s >= E pulls whole registers from lane + s/E.  For w = 2^m, t_m is the window fold itself.
// Otherwise, with m = floor(log2 w): an idempotent op finishes with t_m[i] (+) t_m[i+w-2^m]
// (the two halves overlap); add takes the binary digits of w, the smallest piece
// leftmost, t_{c0}[i] (+) t_{c1}[i+2^c0] (+) ... (every shift is a compile-time constant).
// Each warp emits the outputs whose windows fit in its 32E inputs; no shared memory, no barrier.
template <class T, int E, int SH>
__device__ __forceinline__ void shifted_regs(const T (&t)[E], T (&u)[E]) {
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int src = j + SH;
    if (src < E) u[j] = t[src];
    else u[j] = shfl_down(t[src % E], src / E);
  }
}
// EE: values per lane (default 16 for 4-byte types, 8 for 8-byte ones); EE = 32 for w = 128
// and 256 on 4-byte types (round 2b): every round in registers, the warp's 1024 inputs give
// 1024 - 32 * ceil((w-1)/32) outputs (75 % at w = 256) instead of shared-memory rounds.
template <class Op, int W, int EE = (sizeof(typename Op::T) == 4) ? 16 : 8>
__global__ void __launch_bounds__(256) slsum_doubling_warp_kernel(const typename Op::T* __restrict__ x,
                                                                 typename Op::T* __restrict__ y, uint64_t n,
                                                                 uint64_t nout) {
  using T = typename Op::T;
  constexpr int E = EE;
  constexpr uint32_t OV = 16 / sizeof(T);
  static_assert(W >= 2 && W <= 8 * E, "halo within a warp (at most 8 of its 32 lanes)");
  constexpr int M = 31 - __builtin_clz((unsigned)W);  // floor(log2 W)
  constexpr int P2 = 1 << M;
  constexpr int HL = (W - 1 + E - 1) / E;             // halo lanes
  constexpr uint64_t kOut = (uint64_t)(32 - HL) * E;  // outputs per warp
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t t0 = warp * kOut;
  if (t0 >= nout) return;  // uniform per warp
  const uint64_t g = t0 + (uint64_t)lane * E;
  T t[E];
  if (g + E <= n && ((reinterpret_cast<uintptr_t>(x + g) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(t + q) = __ldg(reinterpret_cast<const uint4*>(x + g + q));
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j) t[j] = (g + j < n) ? x[g + j] : Op::id();
  }
  // non-idempotent, w not a power of two: the binary-digit accumulation (acc, next offset)
  constexpr bool kDigits = !Op::kIdempotent && W != P2;
  T acc[E];
  int off = 0;
  bool have = false;
  auto take = [&](auto shift_tag) {  // acc (+)= t shifted left by the tag's value
    constexpr int SH = decltype(shift_tag)::value;
    T u[E];
    shifted_regs<T, E, SH>(t, u);
#pragma unroll
    for (int j = 0; j < E; ++j) acc[j] = have ? Op::op(acc[j], u[j]) : u[j];
    have = true;
  };
  auto digit = [&](auto r_tag) {
    constexpr int R = decltype(r_tag)::value;
    if constexpr (kDigits && ((W >> R) & 1)) {
      // offset of this piece = the sum of the smaller pieces = W mod 2^R
      take(std::integral_constant<int, (W & ((1 << R) - 1))>{});
    }
  };
  auto round = [&](auto r_tag) {   // t_r -> t_{r+1}
    constexpr int D = 1 << decltype(r_tag)::value;
    T u[E];
    shifted_regs<T, E, D>(t, u);
#pragma unroll
    for (int j = 0; j < E; ++j) t[j] = Op::op(t[j], u[j]);
  };
  auto level = [&](auto r_tag) {
    constexpr int R = decltype(r_tag)::value;
    if constexpr (R <= M) {
      digit(r_tag);
      if constexpr (R < M) round(r_tag);
    }
  };
  level(std::integral_constant<int, 0>{});
  level(std::integral_constant<int, 1>{});
  level(std::integral_constant<int, 2>{});
  level(std::integral_constant<int, 3>{});
  level(std::integral_constant<int, 4>{});
  level(std::integral_constant<int, 5>{});
  level(std::integral_constant<int, 6>{});
  level(std::integral_constant<int, 7>{});
  level(std::integral_constant<int, 8>{});
  static_assert(M <= 8, "levels unrolled above");
  T* out = t;
  if constexpr (kDigits) {
    out = acc;
  } else if constexpr (W != P2) {  // idempotent: overlap of two 2^M windows
    T u[E];
    shifted_regs<T, E, W - P2>(t, u);
#pragma unroll
    for (int j = 0; j < E; ++j) t[j] = Op::op(t[j], u[j]);
  }
  if (lane >= 32 - HL) return;  // halo lanes
  if (g + E <= nout && ((reinterpret_cast<uintptr_t>(y + g) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(y + g + q) = *reinterpret_cast<const uint4*>(out + q);
  } else {
#pragma unroll
    for (int j = 0; j < E; ++j)
      if (g + j < nout) y[g + j] = out[j];
  }
}

template <class Op, int W, int EE = (sizeof(typename Op::T) == 4) ? 16 : 8>
int launch_doubling_warp(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  constexpr int E = EE;
  constexpr int HL = (W - 1 + E - 1) / E;
  const uint64_t nout = n - w + 1;
  const uint64_t kOut = (uint64_t)(32 - HL) * E;
  const uint64_t warps = (nout + kOut - 1) / kOut;
  slsum_doubling_warp_kernel<Op, W, EE><<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(
      static_cast<const T*>(xv), static_cast<T*>(yv), n, nout);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

// COMMUTATIVE path for large w (>= 8E): the first RR rounds (shifts 1 .. 2E, < 4E) run in
// registers on warp spans of 32E consecutive inputs -- a shift below E moves values inside a
// lane plus the next lane's first d values by shuffles, a shift of E or 2E moves whole
// registers from lane + 1 or + 2 -- and only the rounds with shifts >= 4E go through the
// shared-memory ping-pong.  Warp spans overlap by 4E inputs so that every stored t_RR value
// saw its whole 2^RR-input window; a CTA tile of L = NW*28E + 4E inputs gives L - w outputs
// (rounded down to whole 16-byte vectors).  Power-of-two w for any commutative op; other w
// only for idempotent ops (overlap finish t_m[i] (+) t_m[i + w - 2^m]).
template <class Op, int TPB, int XR = 0>
__global__ void __launch_bounds__(TPB) slsum_doubling_rs_kernel(const typename Op::T* __restrict__ x,
                                                               typename Op::T* __restrict__ y, uint64_t n,
                                                               uint32_t w, uint64_t nout, uint32_t tout,
                                                               int four) {
  // XR extra register rounds: shifts up to 2E << XR, spans overlapping by 4E << XR
  // four (w = 2^m, m - 2 >= RR): the shared-memory rounds stop at t_{m-2} and the output takes
  // y[i] = t_{m-2}[i] (+) t_{m-2}[i+d] (+) t_{m-2}[i+2d] (+) t_{m-2}[i+3d], d = w/4: two
  // rounds' stores and barriers fewer for one more (+) per output (the four windows of d
  // partition the window of w, so any commutative op is exact)
  using T = typename Op::T;
  constexpr int E = (sizeof(T) == 4) ? 16 : 8;
  constexpr uint32_t OV = 16 / sizeof(T);
  constexpr int NWp = TPB / 32;
  constexpr int RR = ((E == 16) ? 6 : 5) + XR;    // 2^RR = 4E << XR
  constexpr uint32_t HALO = 4u * E << XR;
  constexpr uint32_t VS = 32 * E - HALO;          // valid positions per warp span after RR rounds
  constexpr uint32_t Lv = NWp * VS;               // valid t_RR positions of the tile
  constexpr uint32_t L = Lv + HALO;               // inputs of the tile
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* A = reinterpret_cast<T*>(smem_raw);
  T* B = A + L + 2 * OV;
  const uint64_t g0 = (uint64_t)blockIdx.x * tout;
  const uint32_t t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const bool vin = ((reinterpret_cast<uintptr_t>(x + g0) & 15) == 0) && g0 + L <= n;
  if (vin) {
    for (uint32_t e = t * OV; e < L; e += TPB * OV)
      *reinterpret_cast<uint4*>(A + e) = __ldg(reinterpret_cast<const uint4*>(x + g0 + e));
  } else {
    for (uint32_t e = t; e < L; e += TPB) A[e] = (g0 + e < n) ? x[g0 + e] : Op::id();
  }
  __syncthreads();
  {
    const uint32_t base = wid * VS + lane * E;
    T v[E];
#pragma unroll
    for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(v + q) = *reinterpret_cast<const uint4*>(A + base + q);
#pragma unroll
    for (int r = 0; r < RR; ++r) {
      const int d = 1 << r;
      T u[E];
      if (d < E) {
#pragma unroll
        for (int j = 0; j < E; ++j) u[j] = (j + d < E) ? v[j + d] : shfl_down(v[(j + d) % E], 1);
      } else {
#pragma unroll
        for (int j = 0; j < E; ++j) u[j] = shfl_down(v[j], d / E);
      }
#pragma unroll
      for (int j = 0; j < E; ++j) v[j] = Op::op(v[j], u[j]);
    }
    if (lane * E < VS) {
#pragma unroll
      for (int q = 0; q < E; q += OV) *reinterpret_cast<uint4*>(B + base + q) = *reinterpret_cast<const uint4*>(v + q);
    }
  }
  __syncthreads();
  T* cur = B;
  T* nxt = A;
  const int m = 31 - __clz(w);
  const int mend = four ? m - 2 : m;
  for (int r = RR; r < mend; ++r) {
    const uint32_t d = 1u << r;               // a multiple of OV
    for (uint32_t e = t * OV; e + d < Lv; e += TPB * OV) {
      T a[OV], c[OV], o[OV];
      *reinterpret_cast<uint4*>(a) = *reinterpret_cast<const uint4*>(cur + e);
      *reinterpret_cast<uint4*>(c) = *reinterpret_cast<const uint4*>(cur + e + d);
#pragma unroll
      for (uint32_t q = 0; q < OV; ++q) o[q] = Op::op(a[q], c[q]);
      *reinterpret_cast<uint4*>(nxt + e) = *reinterpret_cast<const uint4*>(o);
    }
    __syncthreads();
    T* tmp = cur; cur = nxt; nxt = tmp;
  }
  const uint32_t dd = w - (1u << m);          // 0 unless an idempotent op with w not a power of two
  const uint32_t e_end = (uint32_t)min((uint64_t)tout, nout - g0);
  const bool vout = ((reinterpret_cast<uintptr_t>(y + g0) & 15) == 0) && e_end == tout;
  if (four) {
    const uint32_t d = 1u << (m - 2);           // a multiple of OV
    for (uint32_t e = t * OV; e < e_end; e += TPB * OV) {
      MZS_DCHECK(e + 3 * d + OV <= L + 2 * OV);  // t_{m-2} reads stay inside the ping-pong buffer
      T a[OV], b[OV], c[OV], f[OV], o[OV];
      *reinterpret_cast<uint4*>(a) = *reinterpret_cast<const uint4*>(cur + e);
      *reinterpret_cast<uint4*>(b) = *reinterpret_cast<const uint4*>(cur + e + d);
      *reinterpret_cast<uint4*>(c) = *reinterpret_cast<const uint4*>(cur + e + 2 * d);
      *reinterpret_cast<uint4*>(f) = *reinterpret_cast<const uint4*>(cur + e + 3 * d);
#pragma unroll
      for (uint32_t q = 0; q < OV; ++q) o[q] = Op::op(Op::op(a[q], b[q]), Op::op(c[q], f[q]));
      if (vout) {
        *reinterpret_cast<uint4*>(y + g0 + e) = *reinterpret_cast<const uint4*>(o);
      } else {
#pragma unroll
        for (uint32_t q = 0; q < OV; ++q)
          if (e + q < e_end) y[g0 + e + q] = o[q];
      }
    }
  } else if (vout) {
    for (uint32_t e = t * OV; e < tout; e += TPB * OV) {
      T a[OV], c[OV], o[OV];
      *reinterpret_cast<uint4*>(a) = *reinterpret_cast<const uint4*>(cur + e);
      if (dd) {
        ld_shifted<T, OV>(cur, e, dd, c);
#pragma unroll
        for (uint32_t q = 0; q < OV; ++q) o[q] = Op::op(a[q], c[q]);
      } else {
#pragma unroll
        for (uint32_t q = 0; q < OV; ++q) o[q] = a[q];
      }
      *reinterpret_cast<uint4*>(y + g0 + e) = *reinterpret_cast<const uint4*>(o);
    }
  } else {
    for (uint32_t e = t; e < e_end; e += TPB) y[g0 + e] = dd ? Op::op(cur[e], cur[e + dd]) : cur[e];
  }
}

template <class Op, int TPB, int XR = 0>
int launch_doubling_rs(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  constexpr int E = (sizeof(T) == 4) ? 16 : 8;
  constexpr uint32_t OV = 16 / sizeof(T);
  constexpr uint32_t HALO = 4u * E << XR;
  constexpr uint32_t L = (TPB / 32) * (32 * E - HALO) + HALO;
  if (w + OV >= L) return SLSUM_EUNSUPPORTED;
  const uint32_t tout = (L - w) & ~(OV - 1);
  const uint64_t nout = n - w + 1;
  const uint64_t grid = (nout + tout - 1) / tout;
  const size_t smem = 2 * sizeof(T) * ((size_t)L + 2 * OV);
  auto k = slsum_doubling_rs_kernel<Op, TPB, XR>;
  MZS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  constexpr int RR = ((E == 16) ? 6 : 5) + XR;
  int m = 0;
  while ((2u << m) <= w) ++m;                   // 2^m <= w < 2^(m+1)
  const int four = (w & (w - 1)) == 0 && m - 2 >= RR && !env_flag("MZS_SLSUM_NO_RS4");
  k<<<(unsigned)grid, TPB, smem, st>>>(static_cast<const T*>(xv), static_cast<T*>(yv), n, w, nout, tout, four);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

template <class Op>
int launch_doubling(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  constexpr int TPB = 512;
  constexpr int E = (sizeof(T) == 4) ? 16 : 8;
  if (!env_flag("MZS_SLSUM_NO_WARP")) {  // power-of-two w <= 4E: registers and shuffles only
    if (w == 2) return launch_doubling_warp<Op, 2>(xv, yv, n, w, st);
    if (w == 4) return launch_doubling_warp<Op, 4>(xv, yv, n, w, st);
    if (w == 8) return launch_doubling_warp<Op, 8>(xv, yv, n, w, st);
    if (w == 16) return launch_doubling_warp<Op, 16>(xv, yv, n, w, st);
    if (w == 32) return launch_doubling_warp<Op, 32>(xv, yv, n, w, st);
    if (w == 4 * E) return launch_doubling_warp<Op, 4 * E>(xv, yv, n, w, st);
    // 4-byte types: 32 values per lane keep w = 128 and 256 in registers too
    if constexpr (sizeof(T) == 4) {
      if (w == 128 && n >= 4096 && !env_flag("MZS_SLSUM_NO_WARP32")) return launch_doubling_warp<Op, 128, 32>(xv, yv, n, w, st);
      // (w = 256 takes the register-start kernel below: its 4-way finish needs no shared-memory
      // round there, 393 against 353 Gelem/s)
      if (w == 256 && n >= 4096 && env_flag("MZS_SLSUM_WARP32_256")) return launch_doubling_warp<Op, 256, 32>(xv, yv, n, w, st);
    }
    // w = 3..15 outside the powers of two: finishing combine in registers too
    if (w == 3) return launch_doubling_warp<Op, 3>(xv, yv, n, w, st);
    if (w == 5) return launch_doubling_warp<Op, 5>(xv, yv, n, w, st);
    if (w == 6) return launch_doubling_warp<Op, 6>(xv, yv, n, w, st);
    if (w == 7) return launch_doubling_warp<Op, 7>(xv, yv, n, w, st);
    if (w == 9) return launch_doubling_warp<Op, 9>(xv, yv, n, w, st);
    if (w == 10) return launch_doubling_warp<Op, 10>(xv, yv, n, w, st);
    if (w == 11) return launch_doubling_warp<Op, 11>(xv, yv, n, w, st);
    if (w == 12) return launch_doubling_warp<Op, 12>(xv, yv, n, w, st);
    if (w == 13) return launch_doubling_warp<Op, 13>(xv, yv, n, w, st);
    if (w == 14) return launch_doubling_warp<Op, 14>(xv, yv, n, w, st);
    if (w == 15) return launch_doubling_warp<Op, 15>(xv, yv, n, w, st);
  }
  // w >= 8E: the first rounds in registers (power-of-two w, or any w for idempotent ops)
  if (!env_flag("MZS_SLSUM_NO_RS") && w >= 8u * E && ((w & (w - 1)) == 0 || Op::kIdempotent) &&
      n >= (uint64_t)w + 16 * 1024) {
    // one more register round (spans overlapping by 8E) below w = 4096: w=1024 264 -> 272,
    // w=2048 224 -> 230 Gelem/s; at 4096 the wider overlap costs more than the round saves
    if (w < 512) return launch_doubling_rs<Op, 512>(xv, yv, n, w, st);
    if (w < 4096) return launch_doubling_rs<Op, 1024, 1>(xv, yv, n, w, st);
    if (w < 8192) return launch_doubling_rs<Op, 1024, 0>(xv, yv, n, w, st);
  }
  const uint64_t nout = n - w + 1;
  // tile: tout = 8*TPB outputs (register accumulators) from L = tout + w - 1 inputs held in
  // two ping-pong shared-memory buffers (<= 200 KB)
  const uint32_t tout = 8 * TPB;
  const uint64_t Lw = ((uint64_t)tout + w - 1 + 31) & ~31ull;
  if (2 * sizeof(T) * Lw > 200 * 1024) return SLSUM_EUNSUPPORTED;  // w > ~21500 (4-byte)
  const uint32_t L = (uint32_t)Lw;
  const uint64_t grid = (nout + tout - 1) / tout;
  const size_t smem = 2 * sizeof(T) * ((size_t)L + 2 * (16 / sizeof(T)));
  auto k = slsum_doubling_kernel<Op, TPB>;
  MZS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)grid, TPB, smem, st>>>(static_cast<const typename Op::T*>(xv), static_cast<typename Op::T*>(yv),
                                       n, w, nout, L, tout);
  MZS_LAUNCHED();
  return SLSUM_OK;
}


// RECURRENT path (Conclusion: sums with a "recurrent interpretation" run at a
// speedup independent of w): for an invertible (+) -- here uint32 add, exact mod 2^32 --
//   y_i = PS[i+w-1] (-) PS[i-1],   PS = the prefix sums.
// The prefix sums are tile-local (the tile's first element starts them); the difference
// cancels the offset, so no cross-tile scan is needed.  One scan plus one subtraction per
// element, whatever w is.
template <int TPB, int E>
__global__ void __launch_bounds__(TPB) slsum_prefixdiff_kernel(const uint32_t* __restrict__ x, uint32_t* __restrict__ y,
                                                              uint64_t n, uint32_t w, uint64_t nout, uint32_t tout) {
  constexpr uint32_t L = TPB * E;
  constexpr uint32_t NW = TPB / 32;
  constexpr uint32_t OV = 4, G = 32;
  auto sidx = [](uint32_t i) { return i + OV * (i / G); };
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* sPS = reinterpret_cast<uint32_t*>(smem_raw);
  __shared__ uint32_t wsum[NW];
  const uint64_t g0 = (uint64_t)blockIdx.x * tout;
  const uint32_t t = threadIdx.x, lane = t & 31, wid = t >> 5;
  uint32_t v[E];
  {
    const uint64_t g = g0 + (uint64_t)t * E;
    if (g + E <= n && ((reinterpret_cast<uintptr_t>(x + g) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < E / 4; ++q) *reinterpret_cast<uint4*>(v + 4 * q) = __ldg(reinterpret_cast<const uint4*>(x + g) + q);
    } else {
#pragma unroll
      for (int j = 0; j < E; ++j) v[j] = (g + j < n) ? x[g + j] : 0u;
    }
  }
  // inclusive scan: serial in the thread, then warp shuffles, then over warps
#pragma unroll
  for (int j = 1; j < E; ++j) v[j] += v[j - 1];
  uint32_t s = v[E - 1];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= (unsigned)o) s += u;
  }
  if (lane == 31) wsum[wid] = s;
  __syncthreads();
  uint32_t base = s - v[E - 1];
#pragma unroll
  for (uint32_t q = 0; q < NW; ++q)
    if (q < wid) base += wsum[q];
  {
    const uint32_t b0 = sidx(t * E);
#pragma unroll
    for (int q = 0; q < E; q += 4) {
      uint4 o4 = make_uint4(v[q] + base, v[q + 1] + base, v[q + 2] + base, v[q + 3] + base);
      *reinterpret_cast<uint4*>(sPS + b0 + q) = o4;
    }
  }
  __syncthreads();
  const uint32_t e_end = (uint32_t)min((uint64_t)tout, nout - g0);
  uint32_t e_scalar = 0;
  if ((reinterpret_cast<uintptr_t>(y + g0) & 15) == 0) {
    for (uint32_t e = t * OV; e + OV <= e_end; e += TPB * OV) {
      uint32_t o[OV];
#pragma unroll
      for (uint32_t q = 0; q < OV; ++q) {
        const uint32_t i = e + q;
        o[q] = sPS[sidx(i + w - 1)] - (i ? sPS[sidx(i - 1)] : 0u);
      }
      *reinterpret_cast<uint4*>(y + g0 + e) = *reinterpret_cast<const uint4*>(o);
    }
    e_scalar = e_end / OV * OV;
  }
  for (uint32_t i = e_scalar + t; i < e_end; i += TPB) y[g0 + i] = sPS[sidx(i + w - 1)] - (i ? sPS[sidx(i - 1)] : 0u);
}

int launch_prefixdiff(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  constexpr int E = 16;
  const uint64_t nout = n - w + 1;
  int tpb = 256;
  while (tpb < 1024 && (uint64_t)(w - 1) * 8 > (uint64_t)tpb * E) tpb *= 2;
  const uint32_t L = tpb * E;
  if (w - 1 >= L / 2) return SLSUM_EUNSUPPORTED;
  uint32_t tout = (L - (w - 1)) & ~31u;
  if (tout == 0) tout = L - (w - 1);
  const uint64_t grid = (nout + tout - 1) / tout;
  const size_t smem = sizeof(uint32_t) * slsum_smem_len<uint32_t>(L);
  const uint32_t* x = static_cast<const uint32_t*>(xv);
  uint32_t* y = static_cast<uint32_t*>(yv);
#define MZS_PD(TPB_)                                                                           \
  do {                                                                                         \
    auto k = slsum_prefixdiff_kernel<TPB_, E>;                                                 \
    MZS_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k<<<(unsigned)grid, TPB_, smem, st>>>(x, y, n, w, nout, tout);                            \
  } while (0)
  if (tpb == 256) MZS_PD(256);
  else if (tpb == 512) MZS_PD(512);
  else MZS_PD(1024);
#undef MZS_PD
  MZS_LAUNCHED();
  return SLSUM_OK;
}

// SCALAR path: Algorithm 1 "ScalarInput".  A warp is the vector Y: lane l holds
// Y[l + 32 r] (r < K), the partial fold of the window that will complete r*32 + l steps later.
// Every input x_t is broadcast to the first w entries (Y <- Y (+) X), the newest window
// Y[w-1] starts with x_t itself, Y[0] is the finished window y_{t-w+1}, then Y <<< 1.  Each
// window is the strict left fold x_i (+) x_{i+1} (+) ... (+) x_{i+w-1}, with "no additional
// requirements on the operator": the outputs are bit-identical to the oracle's fold
// for every op, f32 add and the non-commutative affine maps included.  O(w) work per output;
// each warp runs a chunk of consecutive outputs (w-1 inputs of warm-up per chunk).
template <class Op, int K>
__global__ void __launch_bounds__(256) slsum_scalar_kernel(const typename Op::T* __restrict__ x,
                                                          typename Op::T* __restrict__ y, uint64_t n, uint32_t w,
                                                          uint64_t nout, uint32_t chunk) {
  using T = typename Op::T;
  const uint64_t warp = ((uint64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t c0 = warp * chunk;
  if (c0 >= nout) return;  // uniform per warp
  const uint64_t c1 = min(nout, c0 + chunk);
  const uint64_t t_end = c1 + w - 1;  // inputs [c0, c1 + w - 1) <= n
  T acc[K];
#pragma unroll
  for (int r = 0; r < K; ++r) acc[r] = Op::id();  // windows that started before c0: never output
  T stash = Op::id();
  uint64_t obase = c0;  // first output of the current stash
  uint32_t ocnt = 0;    // outputs in the stash (lane ocnt receives the next one)
  for (uint64_t tb = c0; tb < t_end; tb += 32) {
    const uint64_t ti = tb + lane;
    const T xv = ti < t_end ? x[ti] : Op::id();
    const uint32_t nb = (uint32_t)min((uint64_t)32, t_end - tb);
    for (uint32_t s = 0; s < nb; ++s) {
      const T xs = shfl_idx(xv, (int)s);
      // Y <- Y (+) X, X = x_t broadcast to the first w entries; the newest window starts at x_t
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const uint32_t j = lane + 32u * r;
        if (j < w) acc[r] = (j == w - 1) ? xs : Op::op(acc[r], xs);
      }
      // y_{t-w+1} <- Y[0]
      if (tb + s >= c0 + w - 1) {
        const T o = shfl_idx(acc[0], 0);
        if (lane == ocnt) stash = o;
        if (++ocnt == 32) {
          y[obase + lane] = stash;
          obase += 32;
          ocnt = 0;
        }
      }
      // Y <- Y <<< 1
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const T up = shfl_down(acc[r], 1);
        const T wrap = (r + 1 < K) ? shfl_idx(acc[r + 1 < K ? r + 1 : r], 0) : up;
        acc[r] = (lane == 31) ? wrap : up;
      }
    }
  }
  if (lane < ocnt) y[obase + lane] = stash;
}

template <class Op, int K>
int launch_scalar_k(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  using T = typename Op::T;
  const uint64_t nout = n - w + 1;
  const uint32_t chunk = std::max<uint32_t>(2048u, 32u * w);
  const uint64_t warps = (nout + chunk - 1) / chunk;
  const uint64_t grid = (warps + 7) / 8;
  slsum_scalar_kernel<Op, K><<<(unsigned)grid, 256, 0, st>>>(static_cast<const T*>(xv), static_cast<T*>(yv), n, w,
                                                            nout, chunk);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

template <class Op>
int launch_scalar(const void* xv, void* yv, uint64_t n, uint32_t w, cudaStream_t st) {
  if (w <= 32) return launch_scalar_k<Op, 1>(xv, yv, n, w, st);
  if (w <= 64) return launch_scalar_k<Op, 2>(xv, yv, n, w, st);
  if (w <= 128) return launch_scalar_k<Op, 4>(xv, yv, n, w, st);
  if (w <= 256) return launch_scalar_k<Op, 8>(xv, yv, n, w, st);
  if (w <= 512) return launch_scalar_k<Op, 16>(xv, yv, n, w, st);
  if (w <= 1024) return launch_scalar_k<Op, 32>(xv, yv, n, w, st);
  return SLSUM_EUNSUPPORTED;  // the shift register holds at most 1024 windows
}

}  // namespace
}  // namespace mzs

using namespace mzs;

MZS_API int slsum_run_ex(int op, uint32_t w, const void* x, void* y, uint64_t n, int path, void* stream) {
  if (w == 0 || op < SLSUM_MIN_U32 || op > SLSUM_CONCAT_U32X2) return SLSUM_EINVAL;
  if (path < SLSUM_PATH_GENERIC || path > SLSUM_PATH_SCALAR) return SLSUM_EINVAL;
  if (n < w) return SLSUM_OK;  // zero outputs (not an error)
  if (!x || !y) return SLSUM_EINVAL;
  cudaStream_t st = as_stream(stream);
  if (path == SLSUM_PATH_AUTO) path = SLSUM_PATH_GENERIC;
  if (path == SLSUM_PATH_SCALAR) {
    switch (op) {
      case SLSUM_MIN_U32: return launch_scalar<OpMinU32>(x, y, n, w, st);
      case SLSUM_MAX_U32: return launch_scalar<OpMaxU32>(x, y, n, w, st);
      case SLSUM_ADD_U32: return launch_scalar<OpAddU32>(x, y, n, w, st);
      case SLSUM_ADD_F32: return launch_scalar<OpAddF32>(x, y, n, w, st);
      case SLSUM_AFFINE_U32X2: return launch_scalar<OpAffine>(x, y, n, w, st);
      case SLSUM_CONCAT_U32X2: return launch_scalar<OpConcat>(x, y, n, w, st);
      case SLSUM_MIN_U64: return launch_scalar<OpMinU64>(x, y, n, w, st);
    }
    return SLSUM_EINVAL;
  }
  if (path == SLSUM_PATH_RECURRENT) {
    // invertible (+) only: uint32 add (exact).  min/max have no inverse; f32 add loses the
    // tolerance to cancellation (4-53x over); the affine maps are not all invertible.
    if (op != SLSUM_ADD_U32) return SLSUM_EUNSUPPORTED;
    return launch_prefixdiff(x, y, n, w, st);
  }
  if (path == SLSUM_PATH_GENERIC) {
    switch (op) {
      case SLSUM_MIN_U32: return launch_generic<OpMinU32>(x, y, n, w, st);
      case SLSUM_MAX_U32: return launch_generic<OpMaxU32>(x, y, n, w, st);
      case SLSUM_ADD_U32: return launch_generic<OpAddU32>(x, y, n, w, st);
      case SLSUM_ADD_F32: return launch_generic<OpAddF32>(x, y, n, w, st);
      case SLSUM_AFFINE_U32X2: return launch_generic<OpAffine>(x, y, n, w, st);
      case SLSUM_CONCAT_U32X2: return launch_generic<OpConcat>(x, y, n, w, st);
      case SLSUM_MIN_U64: return launch_generic<OpMinU64>(x, y, n, w, st);
    }
  } else {
    switch (op) {
      case SLSUM_MIN_U32: return launch_doubling<OpMinU32>(x, y, n, w, st);
      case SLSUM_MAX_U32: return launch_doubling<OpMaxU32>(x, y, n, w, st);
      case SLSUM_ADD_U32: return launch_doubling<OpAddU32>(x, y, n, w, st);
      case SLSUM_ADD_F32: return launch_doubling<OpAddF32>(x, y, n, w, st);
      case SLSUM_AFFINE_U32X2:
      case SLSUM_CONCAT_U32X2: return SLSUM_EUNSUPPORTED;  // not commutative (abstract L8, D15)
      case SLSUM_MIN_U64: return launch_doubling<OpMinU64>(x, y, n, w, st);
    }
  }
  return SLSUM_EINVAL;
}

MZS_API int slsum_run(int op, uint32_t w, const void* x, void* y, uint64_t n) {
  int rc = slsum_run_ex(op, w, x, y, n, SLSUM_PATH_GENERIC, nullptr);
  if (rc != SLSUM_OK) return rc;
  MZS_CUDA(cudaStreamSynchronize(nullptr));
  return SLSUM_OK;
}
