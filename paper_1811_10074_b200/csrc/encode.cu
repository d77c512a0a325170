// encode.cu -- 2-bit packing of DNA (Sec. 2.4, the sequence R = r_0 r_1 ...).
// A/a -> 0, C/c -> 1, G/g -> 2, T/t -> 3, MSB-first, 32 bases per uint64 word (R6);
// every other byte is invalid: code 0 plus a set bit in the invalid bitmap (R7).
// HBM-bound: 1 byte read + 0.375 byte written per base; one thread per 32-base word,
// two 128-bit loads per thread.
#include "common.cuh"

namespace mzs {
namespace {

// 4 ASCII bytes (little-endian in v) -> one byte of 4 MSB-first 2-bit codes and a 4-bit
// invalid mask (bit j <-> byte j).  SWAR, no per-byte branches:
//   u    = v & 0xDF..              upper case
//   c_j  = ((u>>1)&3) ^ ((u>>2)&1) A 0x41 -> 0, C 0x43 -> 1, G 0x47 -> 2, T 0x54 -> 3
//   e_j  = 0x41 + {0,2,6,19}[c_j]  the letter that code would come from
//   valid_j <=> u_j == e_j          exact per-byte zero test of u ^ e
__device__ __forceinline__ void enc4(uint32_t v, uint32_t& packed_byte, uint32_t& inv4) {
  const uint32_t u = v & 0xDFDFDFDFu;
  const uint32_t c = ((u >> 1) & 0x03030303u) ^ ((u >> 2) & 0x01010101u);
  const uint32_t c1 = (c >> 1) & 0x01010101u;                 // c >= 2
  const uint32_t c3 = c & c1;                                  // c == 3
  const uint32_t e = 0x41414141u + 2u * c + 2u * c1 + 11u * c3;
  const uint32_t x = u ^ e;
  // per byte: 0x80 iff the byte of x is zero (valid), exact (no borrow across bytes)
  const uint32_t z = ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
  const uint32_t cm = c & ((z >> 7) * 0xFFu);                 // invalid bases carry code 0
  // gather c_j (bits 8j) to bits 30-2j of the low word: byte = c0<<6|c1<<4|c2<<2|c3
  packed_byte = (cm * 0x40100401u) >> 24;
  // gather the invalid flags (bits 8j after >> 7) to bits 21..24
  inv4 = ((((~z & 0x80808080u) >> 7) * 0x00204081u) >> 21) & 0xFu;
}

// Encode the 32 bases of word t from its 8 little-endian 4-byte groups.
__device__ __forceinline__ void enc_word(const uint32_t (&v)[8], uint64_t b0, uint64_t n, uint64_t& word, uint32_t& inv) {
  word = 0;
  inv = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t pb, m;
    enc4(v[i], pb, m);
    // bases 4i..4i+3 -> bits (63-8i .. 56-8i)
    word |= (uint64_t)pb << (56 - 8 * i);
    inv |= m << (4 * i);
  }
  if (b0 + 32 > n) {  // bits past n are 0
    const uint32_t valid_bases = (uint32_t)(n - b0);
    word &= valid_bases ? ~0ull << (64 - 2 * valid_bases) : 0ull;
    inv &= valid_bases >= 32 ? 0xffffffffu : ((1u << valid_bases) - 1u);
  }
}

__device__ __forceinline__ void load_word_bytes(const uint8_t* __restrict__ seq, uint64_t b0, uint64_t n, bool al,
                                                uint32_t (&v)[8]) {
  if (al && b0 + 32 <= n) {
    const uint4 p = __ldg(reinterpret_cast<const uint4*>(seq + b0));
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(seq + b0 + 16));
    v[0] = p.x; v[1] = p.y; v[2] = p.z; v[3] = p.w; v[4] = q.x; v[5] = q.y; v[6] = q.z; v[7] = q.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t x = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t b = b0 + 4 * i + j;
        x |= (uint32_t)(b < n ? seq[b] : (uint8_t)'A') << (8 * j);
      }
      v[i] = x;
    }
  }
}

// Two words per thread (words t and t + nthreads): four 16-byte loads in flight before any
// arithmetic, so each thread covers more of the memory latency.
__global__ void __launch_bounds__(256) encode_kernel(const uint8_t* __restrict__ seq, uint64_t n,
                                                     uint64_t* __restrict__ words, uint32_t* __restrict__ invalid,
                                                     uint64_t nwords) {
  const uint64_t half = (nwords + 1) / 2;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= half) return;
  const bool al = (reinterpret_cast<uintptr_t>(seq) & 15) == 0;
  const uint64_t t2 = t + half;
  uint32_t v0[8], v1[8];
  load_word_bytes(seq, t * 32, n, al, v0);
  if (t2 < nwords) load_word_bytes(seq, t2 * 32, n, al, v1);
  uint64_t w;
  uint32_t m;
  enc_word(v0, t * 32, n, w, m);
  words[t] = w;
  invalid[t] = m;
  if (t2 < nwords) {
    enc_word(v1, t2 * 32, n, w, m);
    words[t2] = w;
    invalid[t2] = m;
  }
}

}  // namespace

int encode_launch(const uint8_t* seq, uint64_t n, uint64_t* words, uint32_t* invalid, cudaStream_t st) {
  const uint64_t nwords = (n + 31) / 32;
  if (nwords == 0) return SLSUM_OK;
  const unsigned grid = (unsigned)(((nwords + 1) / 2 + 255) / 256);
  encode_kernel<<<grid, 256, 0, st>>>(seq, n, words, invalid, nwords);
  MZS_LAUNCHED();
  return SLSUM_OK;
}

}  // namespace mzs

MZS_API int mz_encode(const uint8_t* seq, uint64_t n, uint64_t* words, uint32_t* invalid, void* stream) {
  if (n == 0) return SLSUM_OK;
  if (!seq || !words || !invalid) return SLSUM_EINVAL;
  return mzs::encode_launch(seq, n, words, invalid, mzs::as_stream(stream));
}
