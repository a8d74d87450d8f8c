// Word-level modular arithmetic for the RNS limbs of the HE ring.
//
// Two word widths:
//   u32 residues for primes p < 2^30  (the reference's default 30-bit chain,
//       he.py:135-165, and every auxiliary 30-bit NTT prime ring.py:498-513);
//   u64 residues for primes p < 2^62  (the 50-bit limbs of the N=8192 configs,
//       which the reference cannot express: ring.py:134-135).
//
// Harvey lazy reduction keeps butterfly values in [0, 4p), so 4p must fit the
// word: p < 2^30 for u32 and p < 2^62 for u64.
//
// Multiplication by a *known* constant w uses Shoup's trick with the
// precomputed quotient w' = floor(w * 2^W / p) (3 integer multiplies).
// Multiplication of two *data* operands uses Montgomery REDC with R = 2^W.
#pragma once
#include <cstdint>

namespace ctb {

template <typename T> struct WordTraits;
template <> struct WordTraits<uint32_t> {
  using Wide = uint64_t;
  static constexpr int BITS = 32;
  __device__ __forceinline__ static uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }
};
template <> struct WordTraits<uint64_t> {
  using Wide = unsigned __int128;
  static constexpr int BITS = 64;
  __device__ __forceinline__ static uint64_t mulhi(uint64_t a, uint64_t b) { return __umul64hi(a, b); }
};

// x - y if x >= y else x, branch-free for unsigned words: when x < y the
// subtraction wraps to a value larger than x, and min() keeps x.
template <typename T>
__device__ __forceinline__ T csub(T x, T y) {
  return min(x - y, x);  // IMNMX
}

// log2 of a power of two (the ring degree): index splits by shift and mask instead of a 64-bit
// division by a runtime value
__device__ __forceinline__ int pow2_shift(uint64_t n) { return __ffsll((long long)n) - 1; }

// Shoup: a * w mod p, lazily in [0, 2p), for any a < 2^W.
template <typename T>
__device__ __forceinline__ T shoup_mul(T a, T w, T wq, T p) {
  T q = WordTraits<T>::mulhi(a, wq);
  return a * w - q * p;
}

// 64-bit Shoup with an approximate high product: the lowest 32x32 partial
// product and the carries of the middle ones are dropped, so the quotient may
// be low by at most 2 and the result lies in [0, 4p) (p < 2^62, any a).  Three
// IMAD.WIDE instead of the exact __umul64hi sequence.
__device__ __forceinline__ uint64_t mulhi64_approx(uint64_t a, uint64_t b) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  const uint64_t m1 = (uint64_t)a1 * b0, m2 = (uint64_t)a0 * b1, hh = (uint64_t)a1 * b1;
  return hh + (m1 >> 32) + (m2 >> 32);
}
__device__ __forceinline__ uint64_t shoup_mul_lazy4(uint64_t a, uint64_t w, uint64_t wq, uint64_t p) {
  return a * w - mulhi64_approx(a, wq) * p;
}

// Montgomery REDC of a*b with R = 2^W: returns a*b*R^-1 mod p in [0, 2p)
// provided a*b < 2p * R (true for a < 4p, b < 2p, p < 2^(W-2)... see DESIGN.md).
// pinv = p^-1 mod 2^W.
template <typename T>
__device__ __forceinline__ T mont_mul(T a, T b, T p, T pinv) {
  T lo = a * b;
  T hi = WordTraits<T>::mulhi(a, b);
  T m = lo * pinv;                         // m*p == lo (mod 2^W)
  T r = hi - WordTraits<T>::mulhi(m, p);   // exact (a*b - m*p) / 2^W, may be negative
  return min(r + p, r);                    // add p back when r wrapped negative
}

// Full canonical reduction from [0, 4p) to [0, p).
template <typename T>
__device__ __forceinline__ T reduce4(T x, T p) {
  x = csub(x, p + p);
  return csub(x, p);
}

// (a + b) mod p for canonical inputs.
template <typename T>
__device__ __forceinline__ T add_mod(T a, T b, T p) { return csub(a + b, p); }
template <typename T>
__device__ __forceinline__ T sub_mod(T a, T b, T p) { return csub(a + p - b, p); }

}  // namespace ctb
