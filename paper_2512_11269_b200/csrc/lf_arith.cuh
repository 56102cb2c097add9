// Modular arithmetic for 28-bit NTT primes held in 32-bit words (sm_100a).
//
// Every prime q satisfies q < 2^28 (reference params.py:14-16), which leaves 4 bits of
// headroom in a uint32: values may be kept lazily in [0, 16q) and reduced only when
// needed.  Multiplication by a per-prime constant w uses Shoup's method with the
// precomputed companion w' = floor(w * 2^32 / q):
//     mul_shoup(x, w, w') = x*w - umulhi(x, w')*q   in [0, 2q)   for any x < 2^32.
// Products of two variables use a 64-bit product and a two-word Shoup fold.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef uint32_t u32;
typedef uint64_t u64;

#define LF_DEV __device__ __forceinline__

// x in [0, 2m) -> [0, m)   (unsigned wrap makes x - m huge when x < m)
LF_DEV u32 csub(u32 x, u32 m) { return min(x, x - m); }

LF_DEV u32 mul_shoup_lazy(u32 x, u32 w, u32 wp, u32 q) {
  u32 h = __umulhi(x, wp);
  return x * w - h * q;                 // [0, 2q)
}

LF_DEV u32 mul_shoup(u32 x, u32 w, u32 wp, u32 q) {
  return csub(mul_shoup_lazy(x, w, wp, q), q);
}

// Per-prime constants needed by the device code.
struct PrimeK {
  u32 q;
  u32 qbar;      // floor(2^32 / q): Shoup companion of w = 1 (x mod q for x < 2^32)
  u32 r32;       // 2^32 mod q
  u32 r32p;      // Shoup companion of r32
  u32 ninv;      // N^-1 mod q
  u32 ninvp;     // Shoup companion
  u32 pad0, pad1;
};

// x < 2^32 -> [0, 2q)
LF_DEV u32 reduce32_lazy(u32 x, const PrimeK& k) { return x - __umulhi(x, k.qbar) * k.q; }
LF_DEV u32 reduce32(u32 x, const PrimeK& k) { return csub(reduce32_lazy(x, k), k.q); }

// x < 2^64 -> [0, q): x = hi*2^32 + lo, hi*2^32 == hi*r32 (mod q)
LF_DEV u32 reduce64(u64 x, const PrimeK& k) {
  u32 hi = (u32)(x >> 32), lo = (u32)x;
  u32 a = mul_shoup_lazy(hi, k.r32, k.r32p, k.q);    // [0, 2q)
  u32 b = reduce32_lazy(lo, k);                      // [0, 2q)
  u32 s = a + b;                                     // [0, 4q) < 2^30
  s = csub(s, 2 * k.q);
  return csub(s, k.q);
}

// a*b mod q for a < 2^32, b < 2^32 (full 64-bit product)
LF_DEV u32 mulmod(u32 a, u32 b, const PrimeK& k) { return reduce64((u64)a * b, k); }

LF_DEV u32 addmod(u32 a, u32 b, u32 q) { return csub(a + b, q); }
LF_DEV u32 submod(u32 a, u32 b, u32 q) { return csub(a + q - b, q); }

// bit reversal of the low `bits` bits
LF_DEV u32 brev_bits(u32 x, int bits) { return __brev(x) >> (32 - bits); }

// automorphism X -> X^g in bit-reversed evaluation order (reference ntt.py:108-121):
//   perm[i] = brv(((2*brv(i)+1)*g mod 2N - 1)/2);  out[i] = in[perm[i]]
LF_DEV u32 auto_src_index(u32 i, u32 g, int logN) {
  u32 r = brev_bits(i, logN);
  u32 two_n_mask = (2u << logN) - 1u;
  u32 e = ((2u * r + 1u) * g) & two_n_mask;
  return brev_bits((e - 1u) >> 1, logN);
}

// For a line-local gather through a bit-reversed staging buffer (element k of a line of 2^lb
// stored at brev_lb(k)): the slot of auto_src_index(i) & (2^lb - 1), i.e. its bit reversal,
// which is the top lb bits of the pre-reversal index.  Reads of a warp then hit 32 distinct
// banks (the map is affine in the bit-reversed domain with an odd multiplier).
LF_DEV u32 auto_src_slot_brev(u32 i, u32 g, int logN, int lb) {
  u32 r = brev_bits(i, logN);
  u32 two_n_mask = (2u << logN) - 1u;
  u32 e = ((2u * r + 1u) * g) & two_n_mask;
  return ((e - 1u) >> 1) >> (logN - lb);
}
