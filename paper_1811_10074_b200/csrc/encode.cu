// encode.cu -- 2-bit packing of DNA (Sec. 2.4, the sequence R = r_0 r_1 ...).
// A/a -> 0, C/c -> 1, G/g -> 2, T/t -> 3, MSB-first, 32 bases per uint64 word (R6);
// every other byte is invalid: code 0 plus a set bit in the invalid bitmap (R7).
// HBM-bound: 1 byte read + 0.375 byte written per base; one thread per 32-base word,
// two 128-bit loads per thread.
#include "common.cuh"

namespace mzs {
namespace {

// 4 ASCII bytes (little-endian in v) -> 4 codes (byte lanes) and a 4-bit invalid mask
__device__ __forceinline__ void enc4(uint32_t v, uint32_t& codes, uint32_t& inv) {
  const uint32_t u = v & 0xDFDFDFDFu;  // upper case
  // code = ((c >> 1) & 3) ^ ((c >> 2) & 1): A 0x41 -> 0, C 0x43 -> 1, G 0x47 -> 2, T 0x54 -> 3
  codes = ((u >> 1) & 0x03030303u) ^ ((u >> 2) & 0x01010101u);
  const uint32_t ok = __vcmpeq4(u, 0x41414141u) | __vcmpeq4(u, 0x43434343u) | __vcmpeq4(u, 0x47474747u) |
                      __vcmpeq4(u, 0x54545454u);
  // ok has 0xFF in every valid byte lane
  const uint32_t bad = ~ok;
  inv = ((bad >> 7) & 1u) | ((bad >> 14) & 2u) | ((bad >> 21) & 4u) | ((bad >> 28) & 8u);
  codes &= ok;  // invalid bases carry code 0
}

__global__ void __launch_bounds__(256) encode_kernel(const uint8_t* __restrict__ seq, uint64_t n,
                                                     uint64_t* __restrict__ words, uint32_t* __restrict__ invalid,
                                                     uint64_t nwords) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nwords) return;
  const uint64_t b0 = t * 32;
  uint32_t v[8];
  if (b0 + 32 <= n && ((reinterpret_cast<uintptr_t>(seq) & 15) == 0)) {
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
  uint64_t word = 0;
  uint32_t inv = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t c, m;
    enc4(v[i], c, m);
    // bases 4i..4i+3 (byte lanes 0..3) -> bits (63-2j, 62-2j), j = 4i + lane
    const uint32_t packed = ((c & 0xFFu) << 6) | (((c >> 8) & 0xFFu) << 4) | (((c >> 16) & 0xFFu) << 2) | (c >> 24);
    word |= (uint64_t)packed << (56 - 8 * i);
    inv |= m << (4 * i);
  }
  if (b0 + 32 > n) {  // bits past n are 0
    const uint32_t valid_bases = (uint32_t)(n - b0);
    word &= valid_bases ? ~0ull << (64 - 2 * valid_bases) : 0ull;
    inv &= valid_bases >= 32 ? 0xffffffffu : ((1u << valid_bases) - 1u);
  }
  words[t] = word;
  invalid[t] = inv;
}

}  // namespace

int encode_launch(const uint8_t* seq, uint64_t n, uint64_t* words, uint32_t* invalid, cudaStream_t st) {
  const uint64_t nwords = (n + 31) / 32;
  if (nwords == 0) return SLSUM_OK;
  const unsigned grid = (unsigned)((nwords + 255) / 256);
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
