// Exact per-coefficient RNS <-> integer machinery (device side).
//
// Mixed-radix (Garner) conversion: residues r_i mod q_i (i < L) of an integer
// x in [0, Q) give digits a_i in [0, q_i) with
//     x = a_0 + a_1 q_0 + a_2 q_0 q_1 + ... + a_{L-1} q_0 ... q_{L-2},
// computed with L(L-1)/2 Shoup multiplications by the constants
// q_i^-1 mod q_j.  From the digits, Horner evaluation gives x mod any other
// modulus (exact base extension) or the positional words of x.  This is the
// exact replacement of the reference's big-integer CRT (ring.py:477-491) for
// everything that needs x as an integer: decryption's scale-and-round
// (he.py:347-348), relinearisation digits (he.py:420-424), tensoring's
// centred lifts and round(h t / q) (he.py:393-405), and the positional wire
// format (ring.py:592-615).
#pragma once
#include <cstdint>
#include "modarith.cuh"

namespace ctb {

constexpr int MAX_MRC = 24;  // primes per converted base

// Constant pair (w, w') for a Shoup multiplication by w mod p.
template <typename T>
struct ShoupC {
  T w, wq;
};

// Garner table of one base, in device memory.  inv[j*(j-1)/2 + i] =
// q_i^-1 mod q_j for i < j.
template <typename T>
struct MrcTab {
  int L;
  T q[MAX_MRC];
  T q2[MAX_MRC];           // 2 q_j
  T one_q[MAX_MRC];        // floor(2^W / q_j)  (Shoup reduction of arbitrary words)
  ShoupC<T> inv[MAX_MRC * (MAX_MRC - 1) / 2];
};

// Digits of x from its residues (canonical inputs; digits canonical).
// LC > 0 fixes the number of primes at compile time (loops unroll, the digit
// arrays stay in registers); LC = 0 reads it from the table.
template <typename T, int LC = 0>
__device__ __forceinline__ void mrc_digits(const MrcTab<T>& tab, const T* r, T* a) {
  a[0] = r[0];
  const int L = LC ? LC : tab.L;
#pragma unroll
  for (int j = 1; j < (LC ? LC : MAX_MRC); ++j) {
    if (!LC && j >= L) break;
    const T qj = tab.q[j], oq = tab.one_q[j];
    T t = r[j];
    const ShoupC<T>* iv = tab.inv + j * (j - 1) / 2;
#pragma unroll
    for (int i = 0; i < j; ++i) {
      // a_i mod q_j (a_i < q_i may exceed q_j): Shoup reduction then one csub
      const T ai = csub(shoup_mul<T>(a[i], (T)1, oq, qj), qj);
      t = sub_mod(t, ai, qj);
      t = csub(shoup_mul<T>(t, iv[i].w, iv[i].wq, qj), qj);
    }
    a[j] = t;
  }
}

// Horner evaluation of a mixed-radix number mod a word prime m:
// hc[k] = q_k mod m (Shoup pair), k < L-1.
template <typename T, typename TD>
__device__ __forceinline__ T mrc_eval(int L, const TD* a, const ShoupC<T>* hc, T m, T one_q) {
  T acc = csub(shoup_mul<T>((T)a[L - 1], (T)1, one_q, m), m);
  for (int k = L - 2; k >= 0; --k) {
    acc = csub(shoup_mul<T>(acc, hc[k].w, hc[k].wq, m), m);
    const T d = csub(shoup_mul<T>((T)a[k], (T)1, one_q, m), m);
    acc = add_mod(acc, d, m);
  }
  return acc;
}

// Horner into little-endian 32-bit positional words: X = sum a_k prod_{i<k} q_i.
// `words` must hold ceil(bits(Q)/32) + 1 words.
template <typename T>
__device__ __forceinline__ void mrc_positional(const MrcTab<T>& tab, const T* a, uint32_t* X, int words) {
  for (int w = 0; w < words; ++w) X[w] = 0;
  // X = a_{L-1}
  {
    const uint64_t v = (uint64_t)a[tab.L - 1];
    X[0] = (uint32_t)v;
    if (words > 1) X[1] = (uint32_t)(v >> 32);
  }
  for (int k = tab.L - 2; k >= 0; --k) {
    const uint64_t qk = (uint64_t)tab.q[k];
    const uint64_t ak = (uint64_t)a[k];
    unsigned __int128 carry = ak;
    for (int w = 0; w < words; ++w) {
      const unsigned __int128 t = (unsigned __int128)X[w] * qk + carry;
      X[w] = (uint32_t)t;
      carry = t >> 32;
    }
  }
}

}  // namespace ctb
