// rng.cuh -- counter-based randomness of the client side (R14, R26):
// Philox4x32-10 keyed by (seed_lo, seed_hi), counter (coef j, modulus index l, object,
// tag<<16 | sub); uniform residues, CBD(21) errors and ternary values derived from it.
#pragma once
#include "common.cuh"

enum {
  TAG_SECRET = 1, TAG_KEY_A = 2, TAG_KEY_E = 3, TAG_ENC_A = 4, TAG_ENC_E = 5,
  // encrypted-database mode (NEXT-1, R26)
  TAG_PK_A = 6, TAG_PK_E = 7, TAG_PKE_V = 8, TAG_PKE_E = 9, TAG_RLK_A = 10, TAG_RLK_E = 11
};

static __device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                              uint32_t k1, uint64_t &w0, uint64_t &w1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  w0 = (uint64_t)c0 | ((uint64_t)c1 << 32);
  w1 = (uint64_t)c2 | ((uint64_t)c3 << 32);
}
static __device__ __forceinline__ void draw(uint64_t seed, uint32_t j, uint32_t l, uint32_t obj, uint32_t tag, uint32_t sub,
                                     uint64_t &w0, uint64_t &w1) {
  philox4x32_10(j, l, obj, (tag << 16) | sub, (uint32_t)seed, (uint32_t)(seed >> 32), w0, w1);
}
static __device__ __forceinline__ int64_t cbd21(uint64_t w0) {
  return (int64_t)__popcll(w0 & 0x1FFFFFull) - (int64_t)__popcll((w0 >> 21) & 0x1FFFFFull);
}
static __device__ __forceinline__ uint64_t smod_dev(int64_t x, uint64_t q, uint64_t bar) {
  if (x >= 0) return reduce64((uint64_t)x, q, bar);
  uint64_t r = reduce64((uint64_t)(-x), q, bar);
  return r ? q - r : 0;
}

