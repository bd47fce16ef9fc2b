// Counter-seeded PRNG variants for neighbour selection (north_star: pcg32,
// sfc64, xoshiro256++).  The reference has only SplitMix64 keys
// (rng.py:28-62); these variants are defined here:
//
//   per frontier node v at step d with degree D > fanout F:
//     nk   = mix64((v+1)*GOLDEN ^ s_d)          (the reference's node key)
//     gen  = <variant> seeded from (nk, s_d)    (see seed() below)
//     take = F distinct positions by Floyd's algorithm: for j = D-F .. D-1,
//            t = bounded(gen, j+1); S += (t in S ? j : t)
//     edges = neighbours at the positions of S, ascending id
//   D <= F keeps the whole neighbourhood, as in the reference.
//
// bounded(n) is Lemire's multiply-shift with rejection (32-bit for pcg32,
// 64-bit for the 64-bit generators).  Everything is __host__ __device__ so
// the same code backs the device sampler and rg_prng_raw (host KATs).
#pragma once

#include <stdint.h>

namespace rg {

enum PrngKind : int { kSplitMix = 0, kPcg32 = 1, kSfc64 = 2, kXoshiro256pp = 3 };

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) {
  return (x << k) | (x >> (64 - k));
}

__host__ __device__ __forceinline__ uint64_t splitmix_next(uint64_t& x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// PCG-XSH-RR 64/32 (O'Neill, pcg_basic.c): srandom(initstate, initseq)
struct Pcg32 {
  uint64_t state, inc;
  __host__ __device__ void seed(uint64_t initstate, uint64_t initseq) {
    state = 0u;
    inc = (initseq << 1u) | 1u;
    next32();
    state += initstate;
    next32();
  }
  __host__ __device__ uint32_t next32() {
    const uint64_t old = state;
    state = old * 6364136223846793005ull + inc;
    const uint32_t xorshifted = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = (uint32_t)(old >> 59u);
    return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
  }
  // Lemire (32-bit) on [0, n)
  __host__ __device__ uint32_t bounded(uint32_t n) {
    uint64_t m = (uint64_t)next32() * n;
    uint32_t l = (uint32_t)m;
    if (l < n) {
      const uint32_t t = (0u - n) % n;
      while (l < t) {
        m = (uint64_t)next32() * n;
        l = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

__host__ __device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Lemire (64-bit) on [0, n) for a 64-bit generator G with next64()
template <typename G>
__host__ __device__ __forceinline__ uint64_t bounded64(G& g, uint64_t n) {
  uint64_t x = g.next64();
  uint64_t l = x * n;
  uint64_t h = mulhi64(x, n);
  if (l < n) {
    const uint64_t t = (0ull - n) % n;
    while (l < t) {
      x = g.next64();
      l = x * n;
      h = mulhi64(x, n);
    }
  }
  return h;
}

// SFC64 (Doty-Humphrey, as numpy.random.SFC64's generator step)
struct Sfc64 {
  uint64_t a, b, c, w;
  __host__ __device__ void seed(uint64_t k0, uint64_t k1) {
    uint64_t x = k0;
    a = splitmix_next(x);
    b = splitmix_next(x);
    c = k1;
    w = 1;
    for (int i = 0; i < 12; ++i) next64();
  }
  __host__ __device__ uint64_t next64() {
    const uint64_t tmp = a + b + w++;
    a = b ^ (b >> 11);
    b = c + (c << 3);
    c = rotl64(c, 24) + tmp;
    return tmp;
  }
  __host__ __device__ uint32_t bounded(uint32_t n) { return (uint32_t)bounded64(*this, n); }
};

// xoshiro256++ (Blackman & Vigna), state filled by splitmix64
struct Xoshiro256pp {
  uint64_t s[4];
  __host__ __device__ void seed(uint64_t k0, uint64_t k1) {
    uint64_t x = k0 ^ k1;
    for (int i = 0; i < 4; ++i) s[i] = splitmix_next(x);
  }
  __host__ __device__ uint64_t next64() {
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
  }
  __host__ __device__ uint32_t bounded(uint32_t n) { return (uint32_t)bounded64(*this, n); }
};

}  // namespace rg
