// CCMul on device: exact tensoring (K4) and relinearisation (K5).
//
// Reference semantics (he.py:384-432):
//   cc_mul_raw: centred lifts c0,c1,d0,d1 of the two ciphertexts; exact integer
//     negacyclic products h0 = c0 d0, h1 = c0 d1 + c1 d0, h2 = c1 d1
//     (ring.int_negacyclic_mul, ring.py:516-541); part_k = round(h_k t / q) mod q,
//     ties away from zero (he.py:527-531 -- ties cannot occur, q odd, gcd(t,q)=1).
//   relinearize: digits d_i = (c2 >> w i) & (2^w - 1) of c2 in [0,q);
//     (c0 + sum d_i b_i, c1 + sum d_i a_i) mod q.
//
// Device algorithm, all exact:
//  1 k_tensor_lift   per coefficient: Garner digits of x over Q (u32 limbs: 64-bit
//    accumulated, one reduction per digit); x > (Q-1)/2 is decided digit-wise against
//    the digits of (Q-1)/2; residues of the centred value over the auxiliary base A
//    (30-bit NTT primes, a superset of Q when Q's primes are 30-bit) as mixed-radix dot
//    products, minus Q mod p when negative.
//  2 k_tensor_product  per (ciphertext, aux prime) CTA: 4 forward NTTs, the
//    3 slotwise tensor products, 3 inverse NTTs -> h residues over A.
//  3 k_tensor_round  per coefficient, with z = h t + (Q-1)/2 (so the result is
//    floor(z / Q) for either sign of h): r = z mod Q from z's residues mod Q
//    (Garner), y = (z - r) Q^-1 modulo each prime of P2 (aux primes outside Q),
//    then y + floor(P2/2) is extended to Q by the float-assisted exact CRT
//    (crt_extend; P2 > 4(|y|max + 1)).  When Q's primes are not in A (50-bit limbs),
//    h + floor(M_A/2) is first extended the same way from A to Q.
//  4 k_relin_digits  w-bit digits of c2 from its Garner digits (limb dot products).
//  5 k_relin_accum   per (ciphertext, limb) CTA: sum over digits of
//    NTT(d_i) * prepared(b_i), NTT(d_i) * prepared(a_i) in registers, 2 INTT,
//    + (c0, c1).
//  6 ctb_ccmul_sum   the fused per-slot form of 1-5 (offline mask products).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "bigint.hpp"
#include "bulk.cuh"
#include "ctb200.h"
#include "kernels.hpp"
#include "rns.cuh"

namespace ctb {

// FP64-quotient butterflies (ntt.cuh F64Q_NE) in the tensoring / relinearisation transforms.
#ifndef CTB_TENSOR_QE
#define CTB_TENSOR_QE 0
#endif
constexpr int TENSOR_QE = CTB_TENSOR_QE;

constexpr int MAXA = 20;  // auxiliary primes
constexpr int MAXQ = 8;   // cipher primes on the tensoring path
constexpr int MAXDIG = 32;  // relinearisation digits on the lazy path

template <typename TQ>
struct TensorConsts {
  int L, K, K2, ext_h, relin_w, relin_d, qwords;
  MrcTab<TQ> mrcQ;
  TQ halfQ_dig[MAXQ];                 // Garner digits of (Q-1)/2 over Q
  int aux_is_q[MAXA];                 // aux k -> index in Q or -1
  int q_in_aux[MAXQ];                 // q_i -> aux index or -1
  uint32_t ap[MAXA], a_oneq[MAXA], a_r2[MAXA], a_r2q[MAXA];
  ShoupC<uint32_t> lift_hc[MAXA][MAXQ];  // q_j mod p_k
  uint32_t Q_aux[MAXA];               // Q mod p_k
  ShoupC<uint32_t> t_aux[MAXA];       // t mod p_k
  uint32_t hQ_aux[MAXA];              // (Q-1)/2 mod p_k
  ShoupC<TQ> t_q[MAXQ];               // t mod q_i
  TQ hQ_q[MAXQ];                      // (Q-1)/2 mod q_i
  int p2_idx[MAXA];                   // aux index of P2 prime k
  ShoupC<uint32_t> r_hc[MAXA][MAXQ];  // q_j mod p2_k
  ShoupC<uint32_t> Qinv_p2[MAXA];     // Q^-1 mod p2_k
  uint32_t Ky_p2[MAXA];               // floor(P2/2) mod p2_k
  TQ Ky_q[MAXQ];                      // floor(P2/2) mod q_i
  uint32_t Kh_aux[MAXA];              // floor(M_A/2) mod p_k
  TQ Kh_q[MAXQ];                      // floor(M_A/2) mod q_i
  // lazy (64-bit accumulated) forms, TQ = u32 only
  uint32_t q_r2[MAXQ], q_r2q[MAXQ];   // 2^32 mod q_i and its Shoup quotient (64-bit reduction)
  uint32_t gM[MAXQ][MAXQ];            // gM[j][i] = M_i mod q_j, M_i = q_0 ... q_{i-1}   (Garner)
  ShoupC<uint32_t> gMinv[MAXQ];       // M_j^-1 mod q_j
  uint32_t aM[MAXA][MAXQ];            // aM[k][i] = M_i mod p_k (mixed radix of Q -> aux prime)
  // float-assisted exact CRT extension of a value x' in [M/4, 3M/4) (M = P2, or M_A for ext_h):
  //   xi_k = x'_k (M/p_k)^-1 mod p_k ; v = floor(sum xi_k / p_k) ; x' = sum xi_k (M/p_k) - v M
  ShoupC<uint32_t> p2_hinv[MAXA];     // (P2/p_k)^-1 mod p_k (P2 index)
  float p2_rcp[MAXA];                 // 1/p_k
  ShoupC<TQ> p2_hat_q[MAXQ][MAXA];    // (P2/p_k) mod q_l (Shoup pair; the u32 path uses .w lazily)
  TQ p2_v_q[MAXQ][MAXA + 1];          // v * P2 mod q_l, v = 0..K2
  ShoupC<uint32_t> a_hinv[MAXA];      // (M_A/p_k)^-1 mod p_k
  float a_rcp[MAXA];
  ShoupC<TQ> a_hat_q[MAXQ][MAXA];     // (M_A/p_k) mod q_l
  TQ a_v_q[MAXQ][MAXA + 1];           // v * M_A mod q_l
  double q_d[MAXQ], q_dinv[MAXQ];     // q_i and 1/q_i (correctly rounded) as doubles (FP64 paths, 50-bit q)
  int lazy_digits;                    // u32 limbs and D <= MAXDIG: digits by limb dot products
  uint32_t dM[MAXQ][MAXDIG];          // dM[i][j] = j-th w-bit limb of M_i
};

struct TensorState {
  void* d_consts = nullptr;
  std::vector<unsigned char> host;  // the same constants, passed by value (constant bank) to the hot kernels
  int K = 0, K2 = 0, L = 0;
  bool q_lead = false;  // aux base = [Q primes in order] + [P2 primes in order] (index shortcuts valid)
  ~TensorState() {
    if (d_consts) cudaFree(d_consts);
  }
};

template <typename T>
__device__ __forceinline__ void load_consts(const T* src, T* dst) {
  const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
  uint32_t* d = reinterpret_cast<uint32_t*>(dst);
  for (int i = threadIdx.x; i < (int)(sizeof(T) / 4); i += blockDim.x) d[i] = s[i];
  __syncthreads();
}

__device__ __forceinline__ uint32_t red_u32(uint64_t v, uint32_t m, uint32_t oneq, uint32_t r2, uint32_t r2q) {
  const uint32_t a = shoup_mul<uint32_t>((uint32_t)(v >> 32), r2, r2q, m);
  const uint32_t b = shoup_mul<uint32_t>((uint32_t)v, 1u, oneq, m);
  return csub(csub(a + b, 2 * m), m);
}

// u32 value (< 2^32) into a TQ residue mod q
template <typename TQ>
__device__ __forceinline__ TQ small_to_q(uint32_t v, TQ q, TQ oneq) {
  if constexpr (sizeof(TQ) == 8) return (TQ)v;  // q > 2^32
  else return csub(shoup_mul<TQ>((TQ)v, (TQ)1, oneq, q), q);
}

// Horner of u32 digits dig[0..n) (radices r_k, constants hc[k] = r_k mod q) mod a TQ prime.
// NC > 0: n fixed at compile time.
template <typename TQ, int NC = 0>
__device__ __forceinline__ TQ horner_to_q(int n_rt, const uint32_t* dig, const ShoupC<TQ>* hc, TQ q, TQ oneq) {
  const int n = NC ? NC : n_rt;
  TQ acc = small_to_q<TQ>(dig[n - 1], q, oneq);
#pragma unroll
  for (int k = n - 2; k >= 0; --k) {
    acc = csub(shoup_mul<TQ>(acc, hc[k].w, hc[k].wq, q), q);
    acc = add_mod(acc, small_to_q<TQ>(dig[k], q, oneq), q);
  }
  return acc;
}

// Horner of TQ digits (Q mixed radix) mod an aux u32 prime.
template <typename TQ, int NC = 0>
__device__ __forceinline__ uint32_t horner_to_aux(int n_rt, const TQ* dig, const ShoupC<uint32_t>* hc, uint32_t p,
                                                  uint32_t oneq, uint32_t r2, uint32_t r2q) {
  const int n = NC ? NC : n_rt;
  uint32_t acc;
  if constexpr (sizeof(TQ) == 4) acc = csub(shoup_mul<uint32_t>((uint32_t)dig[n - 1], 1u, oneq, p), p);
  else acc = red_u32((uint64_t)dig[n - 1], p, oneq, r2, r2q);
#pragma unroll
  for (int k = n - 2; k >= 0; --k) {
    acc = csub(shoup_mul<uint32_t>(acc, hc[k].w, hc[k].wq, p), p);
    uint32_t dk;
    if constexpr (sizeof(TQ) == 4) dk = csub(shoup_mul<uint32_t>((uint32_t)dig[k], 1u, oneq, p), p);
    else dk = red_u32((uint64_t)dig[k], p, oneq, r2, r2q);
    acc = add_mod(acc, dk, p);
  }
  return acc;
}

// ----------------------------------------------------------------------------- lazy RNS helpers
// Dot products of 30-bit digits with 30-bit constants accumulate exactly in 64 bits
// (< 2^60 per term, folded every 8 terms) and are reduced once.

// Garner digits over Q (u32 limbs): a_j = (r_j - sum_{i<j} a_i M_i) M_j^-1 mod q_j.
template <int LC>
__device__ __forceinline__ void garner_lazy(const TensorConsts<uint32_t>& c, int L, const uint32_t* r, uint32_t* a) {
  a[0] = r[0];
#pragma unroll
  for (int j = 1; j < (LC ? LC : MAXQ); ++j) {
    if (!LC && j >= L) break;
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < j; ++i) s += (uint64_t)a[i] * c.gM[j][i];
    const uint32_t q = c.mrcQ.q[j];
    const uint32_t sj = red_u32(s, q, c.mrcQ.one_q[j], c.q_r2[j], c.q_r2q[j]);
    a[j] = csub(shoup_mul<uint32_t>(sub_mod(r[j], sj, q), c.gMinv[j].w, c.gMinv[j].wq, q), q);
  }
}

// x mod aux prime k from the Q mixed-radix digits of x (u32 digits).
template <typename TQ, int LC>
__device__ __forceinline__ uint32_t digits_to_aux(const TensorConsts<TQ>& c, int L, int k, const uint32_t* a) {
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < (LC ? LC : MAXQ); ++i) {
    if (!LC && i >= L) break;
    s += (uint64_t)a[i] * c.aM[k][i];
  }
  return red_u32(s, c.ap[k], c.a_oneq[k], c.a_r2[k], c.a_r2q[k]);
}

// Float-assisted exact CRT: x' in [M/4, 3M/4) given by residues xs[k] modulo n primes
// p_{idx(k)}; returns x' mod q_l for every l (then minus `shift`).  xi_k = x'_k (M/p_k)^-1,
// v = floor(sum xi_k / p_k) (the fractional part x'/M is at least 1/4 away from an integer,
// the float error is < 2^-17), x' = sum xi_k (M/p_k) - v M.
template <typename TQ, int NC, int LC>
__device__ __forceinline__ void crt_extend(const TensorConsts<TQ>& c, int n_rt, int L, const uint32_t* xs,
                                           const ShoupC<uint32_t>* hinv, const float* rcp, const uint32_t* pmod,
                                           const ShoupC<TQ> (*hat_q)[MAXA], const TQ (*v_q)[MAXA + 1],
                                           const TQ* shift, TQ* out) {
  const int n = NC ? NC : n_rt;
  uint32_t xi[MAXA];
  float S = 0.f;
#pragma unroll
  for (int k = 0; k < (NC ? NC : MAXA); ++k) {
    if (!NC && k >= n) break;
    const uint32_t p = pmod[k];
    xi[k] = csub(shoup_mul<uint32_t>(xs[k], hinv[k].w, hinv[k].wq, p), p);
    S = fmaf((float)xi[k], rcp[k], S);
  }
  const int v = (int)S;
#pragma unroll
  for (int l = 0; l < (LC ? LC : MAXQ); ++l) {
    if (!LC && l >= L) break;
    const TQ q = c.mrcQ.q[l];
    TQ x;
    if constexpr (sizeof(TQ) == 4) {
      uint64_t acc = 0;
#pragma unroll
      for (int k = 0; k < (NC ? NC : MAXA); ++k) {
        if (!NC && k >= n) break;
        acc += (uint64_t)xi[k] * hat_q[l][k].w;
        if ((k & 7) == 7) acc = red_u32(acc, q, c.mrcQ.one_q[l], c.q_r2[l], c.q_r2q[l]);
      }
      x = red_u32(acc, q, c.mrcQ.one_q[l], c.q_r2[l], c.q_r2q[l]);
    } else {
      // 50-bit q_l: FP64 products (ntt.cuh f64_mulmod; constants as (c, c/q) doubles), each in
      // (-q, q), the running sum re-centred every 4 terms
      // (q, 1/q precomputed on the host; xi converted by exponent splicing, not I2F)
      const F64Prime P{c.q_d[l], c.q_dinv[l]};
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < (NC ? NC : MAXA); ++k) {
        if (!NC && k >= n) break;
        acc = __dadd_rn(acc, f64_mulmod(f64_from_u64(xi[k]), __longlong_as_double((long long)hat_q[l][k].w),
                                        __longlong_as_double((long long)hat_q[l][k].wq), P.p));
        if ((k & 3) == 3) acc = f64_center(acc, P);
      }
      x = (TQ)f64_to_canon(acc, P);
    }
    x = sub_mod(x, v_q[l][v], q);
    out[l] = sub_mod(x, shift[l], q);
  }
}

// ----------------------------------------------------------------------------- 1 lift
// k_tensor_lift keeps the division form of its index split: with the shift form ptxas allocates 65
// registers (3 CTAs per SM instead of 4) and the kernel runs 19% slower (4.26 vs 5.07 ms per cfg4 batch)
#ifndef CTB_LIFT_DIV
#define CTB_LIFT_DIV 1
#endif
// in: [B][2][L][N] (TQ) -> out: [B][2][K][N] (u32), centred lifts over the aux base.
// LC / KC > 0: limb / aux counts fixed at compile time (register-resident digits).
template <typename TQ, int LC, int KC>
__global__ void __launch_bounds__(256, 3) k_tensor_lift(const TQ* in, uint32_t* out,
                                                     const __grid_constant__ TensorConsts<TQ> c, uint32_t n,
                                                     uint64_t total) {
  const int L = LC ? LC : c.L, K = KC ? KC : c.K;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
#if CTB_LIFT_DIV
    const uint64_t poly = g / n, i = g % n;   // poly = b * 2 + part
#else
    const uint64_t poly = g >> pow2_shift(n), i = g & (n - 1);   // poly = b * 2 + part
#endif
    TQ r[MAXQ], a[MAXQ];
#pragma unroll
    for (int l = 0; l < (LC ? LC : MAXQ); ++l) {
      if (!LC && l >= L) break;
      r[l] = in[(poly * L + l) * n + i];
    }
    if constexpr (sizeof(TQ) == 4) garner_lazy<LC>(c, L, r, a);
    else mrc_digits<TQ, LC>(c.mrcQ, r, a);
    // x > (Q-1)/2 ?  lexicographic from the most significant digit
    bool neg = false, decided = false;
#pragma unroll
    for (int l = (LC ? LC : MAXQ) - 1; l >= 0; --l) {
      if (!LC && l >= L) continue;
      if (!decided && a[l] != c.halfQ_dig[l]) { neg = a[l] > c.halfQ_dig[l]; decided = true; }
    }
#pragma unroll
    for (int k = 0; k < (KC ? KC : MAXA); ++k) {
      if (!KC && k >= K) break;
      uint32_t v;
      const int qi = c.aux_is_q[k];
      // 64-bit limbs: no cipher prime is an aux prime (build_tensor), so r[] is never indexed by a
      // runtime value there (it would live in local memory)
      if (sizeof(TQ) == 4 && qi >= 0) {
        v = (uint32_t)r[KC && LC && sizeof(TQ) == 4 && k < LC ? k : qi];  // x == centred value (mod q_i)
      } else {
        if constexpr (sizeof(TQ) == 4) v = digits_to_aux<TQ, LC>(c, L, k, a);
        else v = horner_to_aux<TQ, LC>(L, a, c.lift_hc[k], c.ap[k], c.a_oneq[k], c.a_r2[k], c.a_r2q[k]);
        if (neg) v = sub_mod(v, c.Q_aux[k], c.ap[k]);
      }
      out[(poly * K + k) * n + i] = v;
    }
  }
}

// ----------------------------------------------------------------------------- 2 products
// A, Bt: [B][2][K][N] lifted operands -> H: [B][3][K][N].  Persistent and
// prime-stationary: CTA k serves aux prime k % K for ciphertext pairs
// k / K, k / K + n_k, ...; the prime's twiddle table lives in shared memory.
template <int LOGN, bool SMEM_TW>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS, NttShape<LOGN>::MINB)
k_tensor_product(const uint32_t* A, const uint32_t* Bt, uint32_t* H, const PrimeTab<uint32_t>* __restrict__ tabs,
                 int K, uint32_t batch) {
  using Sh = NttShape<LOGN>;
  using T = uint32_t;
  constexpr int TW_WORDS = SMEM_TW ? tw_words<T>(LOGN) : 0;
  using Ex = Exchanger<T, LOGN, 1, 1>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* tw_sm = reinterpret_cast<T*>(smem_raw);
  Ex ex{tw_sm + TW_WORDS};
  T* strip = tw_sm + TW_WORDS + Ex::WORDS + threadIdx.x;  // 3 thread-private polys
  const int k = blockIdx.x % K;
  const uint32_t slot = blockIdx.x / K;
  const uint32_t nslots = (gridDim.x - k + K - 1) / K;
  PrimeRegs<T> pr(tabs + k);
  const T* twp = pr.fwd;
  if constexpr (SMEM_TW) {
    stage_twiddles(pr.fwd, tw_sm, TW_WORDS, Sh::THREADS);
    __syncthreads();
    twp = tw_sm;
  }
  const TwSrc<T, SMEM_TW> tw{twp};
  const size_t N = Sh::N;
  T x[Sh::E], y[Sh::E];
#pragma unroll 1
  for (uint32_t b = slot; b < batch; b += nslots) {
    auto src = [&](const T* base, int part) { return base + ((b * 2 + part) * K + k) * N + coef_base<LOGN>(); };
    // NTT(a0) -> strip 0, NTT(a1) -> strip 1 (Montgomery form, N^-1 folded), NTT(b0) -> strip 2
#pragma unroll 1
    for (int s = 0; s < 3; ++s) {
      const T* p = s < 2 ? src(A, s) : src(Bt, 0);
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) x[j] = __ldg(p + coef_off<LOGN>(j));
      ntt_fwd_regs<T, LOGN, 0, SMEM_TW, 1, 1, TENSOR_QE>(x, ex, tw, pr.p, pr.p2);
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) {
        T v = x[j];
        if (s < 2) v = shoup_mul(v, pr.ninvr, pr.ninvr_q, pr.p);  // [0,2p)
        strip[(s * Sh::E + j) * Sh::THREADS] = v;
      }
    }
    {  // NTT(b1) in registers
      const T* p = src(Bt, 1);
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) x[j] = __ldg(p + coef_off<LOGN>(j));
      ntt_fwd_regs<T, LOGN, 0, SMEM_TW, 1, 1, TENSOR_QE>(x, ex, tw, pr.p, pr.p2);
    }
    // h2 = a1 b1 ; h1 = a0 b1 + a1 b0 ; h0 = a0 b0
#pragma unroll 1
    for (int part = 2; part >= 0; --part) {
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) {
        const T a0 = strip[(0 * Sh::E + j) * Sh::THREADS];
        const T a1 = strip[(1 * Sh::E + j) * Sh::THREADS];
        const T b0 = strip[(2 * Sh::E + j) * Sh::THREADS];
        T v;
        if (part == 2) v = mont_mul(x[j], a1, pr.p, pr.pinv);
        else if (part == 1) v = csub(mont_mul(x[j], a0, pr.p, pr.pinv) + mont_mul(b0, a1, pr.p, pr.pinv), pr.p2);
        else v = mont_mul(b0, a0, pr.p, pr.pinv);
        y[j] = v;
      }
      ntt_inv_regs<T, LOGN, Sh::NPASS - 1, SMEM_TW, 1, 1, TENSOR_QE>(y, ex, tw, pr.p, pr.p2);
      T* dst = H + ((b * 3 + part) * K + k) * N + coef_base<LOGN>();
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) dst[coef_off<LOGN>(j)] = csub(y[j], pr.p);
    }
  }
}

template <int LOGN>
static cudaError_t launch_tensor_product(const Ctx* c, const uint32_t* a, const uint32_t* b, uint32_t* h,
                                         uint64_t batch, cudaStream_t s) {
  using Sh = NttShape<LOGN>;
  const Base& B = c->base[BASE_B];
  using T = uint32_t;
  constexpr size_t tw_bytes = (size_t)tw_words<T>(LOGN) * sizeof(T);
  constexpr size_t base_bytes = ((size_t)Exchanger<T, LOGN, 1, 1>::WORDS + 3 * (size_t)Sh::N) * sizeof(T);
  constexpr bool SMEM_TW = LOGN >= 9 && tw_bytes + base_bytes <= 200 * 1024;
  auto kern = k_tensor_product<LOGN, SMEM_TW>;
  const size_t smem = base_bytes + (SMEM_TW ? tw_bytes : 0);
  const int K = B.size();
  if (batch == 0) return cudaSuccess;
  uint32_t grid = persistent_grid((const void*)kern, Sh::THREADS, smem);
  grid = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(grid / K * K, (uint64_t)K), batch * (uint64_t)K);
  return launch_kernel_grid(kern, grid, Sh::THREADS, smem, s, a, b, h, (const PrimeTab<T>*)B.d_tabs, K,
                            (uint32_t)batch);
}

// ----------------------------------------------------------------------------- 3 round
// H: [B][3][K][N] -> out [B][3][L][N] (TQ): round(h t / Q) mod Q.
template <typename TQ, int LC, int KC, int K2C>
#ifndef CTB_ROUND64_MINB
#define CTB_ROUND64_MINB 4
#endif
__global__ void __launch_bounds__(256, sizeof(TQ) == 8 ? CTB_ROUND64_MINB : 3) k_tensor_round(const uint32_t* H, TQ* out,
                                                      const __grid_constant__ TensorConsts<TQ> c, uint32_t n,
                                                      uint64_t total) {
  const int L = LC ? LC : c.L, K = KC ? KC : c.K, K2 = K2C ? K2C : c.K2;
  // The K aux residues of the NEXT grid-stride item are copied into this thread's slots of a
  // double-buffered shared tile (cp.async) while the current item computes: the 11-17 strided
  // loads per coefficient were the kernel's top stall (long scoreboard) at its register-capped
  // occupancy.  Each thread reads only what it copied, so no block barrier is needed.
  extern __shared__ uint32_t hbuf[];   // [2][K][blockDim.x]
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  auto issue = [&](uint64_t gg, int slot) {
    if (gg < total) {
      const uint64_t poly = gg >> pow2_shift(n), i = gg & (n - 1);
#pragma unroll
      for (int k = 0; k < (KC ? KC : MAXA); ++k) {
        if (!KC && k >= K) break;
        cp_async4(hbuf + ((size_t)slot * K + k) * blockDim.x + threadIdx.x, H + (poly * K + k) * n + i);
      }
    }
    cp_async_commit();
  };
  uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  issue(g, 0);
  int slot = 0;
  for (; g < total; g += stride, slot ^= 1) {
    issue(g + stride, slot ^ 1);
    cp_async_wait<1>();
    const uint64_t poly = g >> pow2_shift(n), i = g & (n - 1);   // poly = b * 3 + part
    uint32_t h[MAXA];
#pragma unroll
    for (int k = 0; k < (KC ? KC : MAXA); ++k) {
      if (!KC && k >= K) break;
      h[k] = hbuf[((size_t)slot * K + k) * blockDim.x + threadIdx.x];
    }
    // h mod q_i
    TQ hq[MAXQ];
    if (c.ext_h) {
      // exact extension A -> Q of h + floor(M_A/2) (in [M_A/4, 3 M_A/4)), then minus floor(M_A/2)
      uint32_t hs[MAXA];
#pragma unroll
      for (int k = 0; k < (KC ? KC : MAXA); ++k) {
        if (!KC && k >= K) break;
        hs[k] = add_mod(h[k], c.Kh_aux[k], c.ap[k]);
      }
      crt_extend<TQ, KC, LC>(c, K, L, hs, c.a_hinv, c.a_rcp, c.ap, c.a_hat_q, c.a_v_q, c.Kh_q, hq);
    } else {
#pragma unroll
      for (int l = 0; l < (LC ? LC : MAXQ); ++l) {
        if (!LC && l >= L) break;
        hq[l] = (TQ)h[LC ? l : c.q_in_aux[l]];   // Q primes lead the aux base (build_tensor)
      }
    }
    // z = h t + (Q-1)/2 mod q_i ; r = z mod Q (Garner digits)
    TQ z[MAXQ], rd[MAXQ];
#pragma unroll
    for (int l = 0; l < (LC ? LC : MAXQ); ++l) {
      if (!LC && l >= L) break;
      const TQ q = c.mrcQ.q[l];
      z[l] = add_mod(csub(shoup_mul<TQ>(hq[l], c.t_q[l].w, c.t_q[l].wq, q), q), c.hQ_q[l], q);
    }
    if constexpr (sizeof(TQ) == 4) garner_lazy<LC>(c, L, z, rd);
    else mrc_digits<TQ, LC>(c.mrcQ, z, rd);
    // y' = (z - r) Q^-1 + floor(P2/2) mod each P2 prime
    uint32_t ys[MAXA], p2p[MAXA];
#pragma unroll
    for (int k = 0; k < (K2C ? K2C : MAXA); ++k) {
      if (!K2C && k >= K2) break;
      // P2 primes are the leading non-Q auxiliary primes (build_tensor; the launcher checks it
      // before picking the compile-time form), so the index stays static and h[] in registers
      const int ai = (KC && LC) ? (sizeof(TQ) == 4 ? LC + k : k) : c.p2_idx[k];
      const uint32_t p = c.ap[ai];
      p2p[k] = p;
      const uint32_t zk = add_mod(csub(shoup_mul<uint32_t>(h[ai], c.t_aux[ai].w, c.t_aux[ai].wq, p), p), c.hQ_aux[ai], p);
      uint32_t rk;
      if constexpr (sizeof(TQ) == 4) rk = digits_to_aux<TQ, LC>(c, L, ai, rd);
      else rk = horner_to_aux<TQ, LC>(L, rd, c.r_hc[k], p, c.a_oneq[ai], c.a_r2[ai], c.a_r2q[ai]);
      const uint32_t yk = csub(shoup_mul<uint32_t>(sub_mod(zk, rk, p), c.Qinv_p2[k].w, c.Qinv_p2[k].wq, p), p);
      ys[k] = add_mod(yk, c.Ky_p2[k], p);
    }
    // exact extension P2 -> Q of y' (in [P2/4, 3 P2/4)), minus floor(P2/2)
    TQ o[MAXQ];
    crt_extend<TQ, K2C, LC>(c, K2, L, ys, c.p2_hinv, c.p2_rcp, p2p, c.p2_hat_q, c.p2_v_q, c.Ky_q, o);
#pragma unroll
    for (int l = 0; l < (LC ? LC : MAXQ); ++l) {
      if (!LC && l >= L) break;
      out[(poly * L + l) * n + i] = o[l];
    }
  }
}

// ----------------------------------------------------------------------------- 4 relin digits
// w-bit digits of x in [0, Q) given by residues r (he.py:420-424 on the integer c2).
// u32 limbs: Garner digits a_i, then X = sum a_i M_i limb by limb with M_i cut into w-bit
// limbs (64-bit accumulators, carry between limbs); DC / WC > 0 fix D / w at compile time
// (limbs of M_i above 2^(30 i) are zero and skipped).  ACC: add into dig[] instead of store.
template <typename TQ, int LC, int DC, int WC, bool ACC>
__device__ __forceinline__ void value_digits(const TensorConsts<TQ>& c, const TQ* r, uint32_t* dig) {
  const int L = LC ? LC : c.L, D = DC ? DC : c.relin_d, w = WC ? WC : c.relin_w;
  const uint32_t mask = (w >= 32) ? 0xffffffffu : ((1u << w) - 1u);
  if constexpr (sizeof(TQ) == 4) {
    if (c.lazy_digits) {
      uint32_t a[MAXQ];
      garner_lazy<LC>(c, L, r, a);
      uint64_t carry = 0;
#pragma unroll
      for (int j = 0; j < (DC ? DC : MAXDIG); ++j) {
        if (!DC && j >= D) break;
        uint64_t acc = carry;
#pragma unroll
        for (int i = 0; i < (LC ? LC : MAXQ); ++i) {
          if (!LC && i >= L) break;
          if (WC && LC && j * WC >= (i ? 30 * i : 1)) continue;  // M_i < 2^(30 i), M_0 = 1: limb j is zero
          acc += (uint64_t)a[i] * c.dM[i][j];
        }
        const uint32_t d = (uint32_t)acc & mask;
        carry = acc >> w;
        if (ACC) dig[j] += d; else dig[j] = d;
      }
      return;
    }
  }
  if constexpr (sizeof(TQ) == 8 && LC > 0 && DC > 0 && WC > 0) {
    // 64-bit limbs with compile-time shape: mixed-radix digits, then X = sum a_k prod_{i<k} q_i in
    // 2 LC + 1 32-bit words with fully unrolled loops (registers, no local memory)
    TQ a[LC];
    mrc_digits<TQ, LC>(c.mrcQ, r, a);
    constexpr int NW = 2 * LC + 1;
    uint32_t X[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) X[w] = 0;
    X[0] = (uint32_t)a[LC - 1];
    X[1] = (uint32_t)((uint64_t)a[LC - 1] >> 32);
#pragma unroll
    for (int k = LC - 2; k >= 0; --k) {
      const uint64_t qk = (uint64_t)c.mrcQ.q[k];
      const uint32_t q0 = (uint32_t)qk, q1 = (uint32_t)(qk >> 32);
      // X = X * qk + a_k, word by word with a 64-bit carry (q_k < 2^50: two 32-bit halves)
      uint64_t carry = (uint64_t)a[k];
      uint32_t prev = 0;  // X[w-1], the word multiplied by the high half q1
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t xw = X[w];
        const unsigned __int128 t = (unsigned __int128)xw * q0 + (unsigned __int128)prev * q1 + carry;
        X[w] = (uint32_t)t;
        carry = (uint64_t)(t >> 32);
        prev = xw;
      }
    }
#pragma unroll
    for (int j = 0; j < DC; ++j) {
      const int bit = j * WC, wi = bit >> 5, sh = bit & 31;
      uint64_t v = (uint64_t)X[wi] >> sh;
      if (sh + WC > 32 && wi + 1 < NW) v |= (uint64_t)X[wi + 1] << (32 - sh);
      if (ACC) dig[j] += (uint32_t)v & mask; else dig[j] = (uint32_t)v & mask;
    }
    return;
  }
  TQ a[MAXQ];
  mrc_digits<TQ>(c.mrcQ, r, a);
  uint32_t X[20];
  mrc_positional(c.mrcQ, a, X, c.qwords);
  for (int j = 0; j < D; ++j) {
    const int bit = j * w, wi = bit >> 5, sh = bit & 31;
    uint64_t v = (uint64_t)X[wi] >> sh;
    if (sh + w > 32 && wi + 1 < c.qwords) v |= (uint64_t)X[wi + 1] << (32 - sh);
    if (ACC) dig[j] += (uint32_t)v & mask; else dig[j] = (uint32_t)v & mask;
  }
}

// ct3: [B][3][L][N] -> digits [B][D][N] (u32 < 2^w), d_j = (c2 >> w j) & (2^w - 1).
template <typename TQ, int LC, int DC, int WC>
__global__ void __launch_bounds__(256) k_relin_digits(const TQ* ct3, uint32_t* digits,
                                                      const __grid_constant__ TensorConsts<TQ> c, uint32_t n,
                                                      uint64_t total) {
  const int L = LC ? LC : c.L, D = DC ? DC : c.relin_d;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = g >> pow2_shift(n), i = g & (n - 1);
    TQ r[MAXQ];
#pragma unroll
    for (int l = 0; l < (LC ? LC : MAXQ); ++l) {
      if (!LC && l >= L) break;
      r[l] = ct3[((b * 3 + 2) * L + l) * n + i];
    }
    uint32_t d[MAXDIG];
    value_digits<TQ, LC, DC, WC, false>(c, r, d);
#pragma unroll
    for (int j = 0; j < (DC ? DC : MAXDIG); ++j) {
      if (!DC && j >= D) break;
      digits[(b * D + j) * n + i] = d[j];
    }
  }
}

// ----------------------------------------------------------------------------- 5 relin accumulate
// out [B][2][L][N] = (c0, c1) + sum_j NTT^-1(NTT(d_j) * keyprep[j][0|1]).  Persistent and
// limb-stationary (CTA k serves limb k % L), the limb's twiddle table staged in shared
// memory; both accumulators stay in registers across the D digit transforms.
// Relinearisation keys through the exchange image (ntt.cuh eval_xpose_*): off by default -- with
// the digit transform and both accumulators live it spills (232 B per thread at 64-bit limbs).
#ifndef CTB_RELIN_XPOSE
#define CTB_RELIN_XPOSE 0
#endif
// 32-bit limbs: key products with FP64-pipe quotients (ntt.cuh f64_pointwise), keys converted out
// of the Montgomery domain with the thread-major layout
#ifndef CTB_RELIN_F64_POINTWISE
#define CTB_RELIN_F64_POINTWISE 1
#endif
template <typename T, bool KSTRIP>
__host__ __device__ constexpr bool RELIN_F64PW() { return CTB_RELIN_F64_POINTWISE && sizeof(T) == 4 && KSTRIP && !CTB_RELIN_XPOSE; }
// L2 prefetch of the next digit polynomial while the current one transforms
#ifndef CTB_RELIN_L2PF
#define CTB_RELIN_L2PF 1
#endif
template <typename T, int LOGN>
struct RelinCfg {
  using Sh = NttShape<LOGN>;
  using Ex = Exchanger<T, LOGN, 1, 1>;
  static constexpr size_t TW_BYTES = (size_t)tw_words<T>(LOGN) * sizeof(T);
  static constexpr size_t EX_BYTES = ((size_t)Ex::WORDS * sizeof(T) + 15) / 16 * 16;
  static constexpr bool SMEM_TW = sizeof(T) == 4 && LOGN >= 9 && TW_BYTES + EX_BYTES <= 110 * 1024;  // u64: measured slower
  // digits (u32 [N]) staged by TMA one transform ahead: measured slower here (an extra CTA
  // barrier per digit, keys dominate the traffic), kept switchable
  static constexpr bool PF = false;
  static constexpr size_t SMEM = (SMEM_TW ? TW_BYTES : 0) + EX_BYTES + (PF ? Sh::N * 4 + 16 : 0);
  static constexpr int MINB = (Sh::THREADS == 256 && sizeof(T) == 4) ? 3 : Sh::MINB;
};

// 64-bit limbs with key strips: relinearisation in the FP64 domain (keys as centred doubles)
template <typename T, int LOGN, bool KSTRIP>
__host__ __device__ constexpr bool relin_f64() {
  return sizeof(T) == 8 && KSTRIP && !RelinCfg<T, LOGN>::PF;
}

template <typename T, int LOGN, bool SMEM_TW, bool KSTRIP = false>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS, RelinCfg<T, LOGN>::MINB)
k_relin_accum(const T* ct3, int ct_parts, const uint32_t* digits, const T* keyprep, T* out,
              const PrimeTab<T>* __restrict__ tabs, int L, int D, uint32_t batch) {
  using Sh = NttShape<LOGN>;
  using C = RelinCfg<T, LOGN>;
  constexpr bool PF = C::PF;
  constexpr int TW_WORDS = SMEM_TW ? tw_words<T>(LOGN) : 0;
  using Ex = typename C::Ex;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* tw_sm = reinterpret_cast<T*>(smem_raw);
  Ex ex{tw_sm + TW_WORDS};
  uint32_t* stg = reinterpret_cast<uint32_t*>(smem_raw + (SMEM_TW ? C::TW_BYTES : 0) + C::EX_BYTES);
  uint64_t* bar = reinterpret_cast<uint64_t*>(stg + Sh::N);
  const int limb = blockIdx.x % L;
  const uint32_t slot = blockIdx.x / L;
  const uint32_t nslots = (gridDim.x - limb + L - 1) / L;
  const size_t N = Sh::N;
  PrimeRegs<T> pr(tabs + limb);
  const T* twp = pr.fwd;
  if constexpr (SMEM_TW) {
    stage_twiddles(pr.fwd, tw_sm, TW_WORDS, Sh::THREADS);
    twp = tw_sm;
  }
  uint32_t phase = 0;
  if constexpr (PF) {
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      mbar_init_fence();
      if (slot < batch) bulk_load(stg, digits + (size_t)slot * D * N, (uint32_t)(N * 4), bar);
    }
  }
  if constexpr (SMEM_TW || PF) __syncthreads();
  const TwSrc<T, SMEM_TW> tw{twp};
  const int cb = coef_base<LOGN>();
  using EV = EvalVec<T, LOGN>;
  if constexpr (relin_f64<T, LOGN, KSTRIP>()) {
    // 64-bit limbs: digit transforms, the key products and the sums in the FP64 domain (keys as
    // centred doubles NTT(key) N^-1 in the thread-major strip, launch_relin_accum); the sums are
    // re-centred every 4 digits (|acc| <= 4 x 0.6 p + p/2 stays exact and a valid product input)
    const F64Prime P{(double)pr.p, __drcp_rn((double)pr.p)};
    double a0[Sh::E], a1[Sh::E], dx[Sh::E];
#pragma unroll 1
    for (uint32_t b = slot; b < batch; b += nslots) {
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) a0[j] = a1[j] = 0.0;
#pragma unroll 1
      for (int d = 0; d < D; ++d) {
        const uint32_t* src = digits + ((size_t)b * D + d) * N + cb;
#pragma unroll
        for (int j = 0; j < Sh::E; ++j) dx[j] = (double)__ldg(src + coef_off<LOGN>(j));   // digit sums < 2^32
        ntt_fwd_f64<T, LOGN, 0, SMEM_TW, 1, 1>(dx, ex, tw, P);
        const uint4* kb = reinterpret_cast<const uint4*>(keyprep + (((size_t)d * 2 + 0) * L + limb) * N);
        const uint4* ka = reinterpret_cast<const uint4*>(keyprep + (((size_t)d * 2 + 1) * L + limb) * N);
#pragma unroll
        for (int i = 0; i < EV::CHUNKS; ++i) {
          T vb[EV::VEC], va[EV::VEC];
          unpack_chunk<T>(__ldg(kb + i * Sh::THREADS + threadIdx.x), vb);
          unpack_chunk<T>(__ldg(ka + i * Sh::THREADS + threadIdx.x), va);
#pragma unroll
          for (int c = 0; c < EV::VEC; ++c) {
            const int j = i * EV::VEC + c;
            const double xc = f64_center(dx[j], P);
            const double kbd = __longlong_as_double((long long)vb[c]), kad = __longlong_as_double((long long)va[c]);
            a0[j] = __dadd_rn(a0[j], f64_mulmod(xc, kbd, __dmul_rn(kbd, P.pinv), P.p));
            a1[j] = __dadd_rn(a1[j], f64_mulmod(xc, kad, __dmul_rn(kad, P.pinv), P.p));
          }
        }
        if ((d & 3) == 3) {
#pragma unroll
          for (int j = 0; j < Sh::E; ++j) a0[j] = f64_center(a0[j], P), a1[j] = f64_center(a1[j], P);
        }
      }
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
#pragma unroll
        for (int j = 0; j < Sh::E; ++j) dx[j] = f64_center(part == 0 ? a0[j] : a1[j], P);   // < p: inverse input
        ntt_inv_f64<T, LOGN, Sh::NPASS - 1, SMEM_TW, 1, 1>(dx, ex, tw, P);
        const size_t off = (((size_t)b * ct_parts + part) * L + limb) * N + cb;
        const size_t oo = ((b * 2 + part) * L + limb) * N + cb;
#pragma unroll
        for (int j = 0; j < Sh::E; ++j)
          out[oo + coef_off<LOGN>(j)] = add_mod((T)f64_to_canon(dx[j], P), ct3[off + coef_off<LOGN>(j)], pr.p);
      }
    }
    return;
  }
  T acc0[Sh::E], acc1[Sh::E], x[Sh::E];
  const double pinv_d = __drcp_rn((double)pr.p);
  const uint32_t pn32 = 0u - (uint32_t)pr.p;
#pragma unroll 1
  for (uint32_t b = slot; b < batch; b += nslots) {
#pragma unroll
    for (int j = 0; j < Sh::E; ++j) acc0[j] = acc1[j] = 0;
#pragma unroll 1
    for (int d = 0; d < D; ++d) {
      if constexpr (PF) {
        mbar_wait(bar, phase);
        phase ^= 1;
#pragma unroll
        for (int j = 0; j < Sh::E; ++j) x[j] = pr.reduce_digit(stg[cb + coef_off<LOGN>(j)]);
        __syncthreads();  // staging consumed
        if (threadIdx.x == 0) {
          // next digit of this item, else the first digit of the next item
          const uint32_t nb = d + 1 < D ? b : b + nslots;
          const int nd = d + 1 < D ? d + 1 : 0;
          if (nb < batch) {
            fence_proxy_async_smem();
            bulk_load(stg, digits + ((size_t)nb * D + nd) * N, (uint32_t)(N * 4), bar);
          }
        }
      } else {
        const uint32_t* src = digits + ((size_t)b * D + d) * N + cb;
        // the next digit (or the next item's first) towards L2: 32-bit limbs -3.5% (13.49 -> 13.01 ms per
        // cfg4 batch); neutral-to-slower at 64-bit limbs
        if (CTB_RELIN_L2PF && sizeof(T) == 4 && threadIdx.x == 0) {
          const uint32_t nb = d + 1 < D ? b : b + nslots;
          const int nd = d + 1 < D ? d + 1 : 0;
          if (nb < batch) bulk_prefetch_l2(digits + ((size_t)nb * D + nd) * N, (uint32_t)(N * 4));
        }
#pragma unroll
        for (int j = 0; j < Sh::E; ++j) x[j] = pr.reduce_digit(__ldg(src + coef_off<LOGN>(j)));  // any u32 -> [0,p)
      }
      ntt_fwd_regs<T, LOGN, 0, SMEM_TW, 1, 1, TENSOR_QE>(x, ex, tw, pr.p, pr.p2);
      const T* kb = keyprep + (((size_t)d * 2 + 0) * L + limb) * N;
      const T* ka = keyprep + (((size_t)d * 2 + 1) * L + limb) * N;
      if constexpr (CTB_RELIN_XPOSE && eval_xpose_ok<T, LOGN>(Ex::WORDS)) {
        // keys read with contiguous 16-byte accesses through the exchange image (ntt.cuh)
        eval_xpose_stage<T, LOGN, 1>(kb, ex.buf);
#pragma unroll
        for (int i = 0; i < EV::CHUNKS; ++i) {
          T v[EV::VEC];
          eval_xpose_chunk<T, LOGN>(ex.buf, i, v);
#pragma unroll
          for (int c = 0; c < EV::VEC; ++c) {
            const int j = i * EV::VEC + c;
            acc0[j] = csub(acc0[j] + mont_mul(x[j], v[c], pr.p, pr.pinv), pr.p2);
          }
        }
        eval_xpose_stage<T, LOGN, 1>(ka, ex.buf);
#pragma unroll
        for (int i = 0; i < EV::CHUNKS; ++i) {
          T v[EV::VEC];
          eval_xpose_chunk<T, LOGN>(ex.buf, i, v);
#pragma unroll
          for (int c = 0; c < EV::VEC; ++c) {
            const int j = i * EV::VEC + c;
            acc1[j] = csub(acc1[j] + mont_mul(x[j], v[c], pr.p, pr.pinv), pr.p2);
          }
        }
      } else
#pragma unroll
      for (int i = 0; i < EV::CHUNKS; ++i) {
        T vb[EV::VEC], va[EV::VEC];
        if constexpr (KSTRIP) {  // thread-major chunk layout (k_eval_to_strip): contiguous warp loads
          unpack_chunk<T>(__ldg(reinterpret_cast<const uint4*>(kb) + i * Sh::THREADS + threadIdx.x), vb);
          unpack_chunk<T>(__ldg(reinterpret_cast<const uint4*>(ka) + i * Sh::THREADS + threadIdx.x), va);
        } else {
          EV::load(kb, i, vb);
          EV::load(ka, i, va);
        }
#pragma unroll
        for (int c = 0; c < EV::VEC; ++c) {
          const int j = i * EV::VEC + c;
          if constexpr (RELIN_F64PW<T, KSTRIP>()) {   // keys out of the Montgomery domain (k_eval_to_strip)
            const double xd = __uint2double_rn((uint32_t)x[j]);
            acc0[j] = csub(acc0[j] + (T)f64_pointwise2((uint32_t)x[j], (uint32_t)vb[c], xd, __uint2double_rn((uint32_t)vb[c]), pinv_d, (uint32_t)pr.p, pn32), pr.p2);
            acc1[j] = csub(acc1[j] + (T)f64_pointwise2((uint32_t)x[j], (uint32_t)va[c], xd, __uint2double_rn((uint32_t)va[c]), pinv_d, (uint32_t)pr.p, pn32), pr.p2);
          } else {
          acc0[j] = csub(acc0[j] + mont_mul(x[j], vb[c], pr.p, pr.pinv), pr.p2);
          acc1[j] = csub(acc1[j] + mont_mul(x[j], va[c], pr.p, pr.pinv), pr.p2);
          }
        }
      }
    }
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) x[j] = part == 0 ? acc0[j] : acc1[j];
      ntt_inv_regs<T, LOGN, Sh::NPASS - 1, SMEM_TW, 1, 1, TENSOR_QE>(x, ex, tw, pr.p, pr.p2);
      const size_t off = (((size_t)b * ct_parts + part) * L + limb) * N + cb;
      const size_t oo = ((b * 2 + part) * L + limb) * N + cb;
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) out[oo + coef_off<LOGN>(j)] = add_mod(csub(x[j], pr.p), ct3[off + coef_off<LOGN>(j)], pr.p);
    }
  }
}

// Relinearisation keys in the thread-major layout (per call: a stream-ordered temporary, D x 2 x L
// polynomials, negligible beside the D x L digit transforms per slot).  -DCTB_RELIN_KSTRIP=0: direct.
#ifndef CTB_RELIN_KSTRIP
#define CTB_RELIN_KSTRIP 1
#endif

template <typename T, int LOGN>
static cudaError_t launch_relin_accum(const Ctx* c, const void* ct3, int ct_parts, const uint32_t* digits,
                                      const void* keyprep, void* out, uint64_t batch, int D, cudaStream_t s) {
  using Sh = NttShape<LOGN>;
  using C = RelinCfg<T, LOGN>;
  using EV = EvalVec<T, LOGN>;
  constexpr bool KS = CTB_RELIN_KSTRIP && EV::CONTIG && EV::VEC * (int)sizeof(T) == 16 && !C::PF;
  const Base& B = c->base[BASE_Q];
  auto kern = k_relin_accum<T, LOGN, C::SMEM_TW, KS>;
  const int L = B.size();
  if (batch == 0) return cudaSuccess;
  const void* keys = keyprep;
  void* tmp = nullptr;
  if constexpr (KS) {
    const size_t npoly = (size_t)D * 2 * L;
    cudaError_t e = c->pool ? cudaMallocFromPoolAsync(&tmp, npoly * Sh::N * sizeof(T), c->pool, s)
                            : cudaMallocAsync(&tmp, npoly * Sh::N * sizeof(T), s);
    if (e != cudaSuccess) return e;
    k_eval_to_strip<T, LOGN, relin_f64<T, LOGN, KS>() || RELIN_F64PW<T, KS>()><<<(unsigned)npoly, Sh::THREADS, 0, s>>>(
        (const T*)keyprep, (T*)tmp, (const PrimeTab<T>*)B.d_tabs, L);
    if ((e = cudaGetLastError()) != cudaSuccess) { cudaFreeAsync(tmp, s); return e; }
    keys = tmp;
  }
  uint32_t grid = persistent_grid((const void*)kern, Sh::THREADS, C::SMEM);
  grid = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(grid / L * L, (uint64_t)L), batch * (uint64_t)L);
  cudaError_t e = launch_kernel_grid(kern, grid, Sh::THREADS, C::SMEM, s, (const T*)ct3, ct_parts, digits, (const T*)keys,
                                     (T*)out, (const PrimeTab<T>*)B.d_tabs, L, D, (uint32_t)batch);
  if (tmp) {
    const cudaError_t f = cudaFreeAsync(tmp, s);
    if (e == cudaSuccess) e = f;
  }
  return e;
}

// ----------------------------------------------------------------------------- 6 fused site sums
// Offline mask products / protocol-b slots (linprot.py:407-427, :371-379): for every output
// slot o, sum over its sites s of relinearize(cc_mul_raw(x[xs], w[ws])).  Exact reorganisation:
//  * each distinct ciphertext is lifted to the aux base and forward-transformed ONCE
//    (x prepared, w canonical), not once per site;
//  * per site only the three eval-domain tensor products and three inverse transforms
//    (k_site_product) and the exact rounding (k_tensor_round) remain;
//  * relinearisation is linear in the digits: sum_s relin(c_s) = (sum c0_s + sum_i (sum_s d_i,s) b_i,
//    sum c1_s + sum_i (sum_s d_i,s) a_i) mod q, so the digits and (c0, c1) are summed per slot
//    (k_slot_digits) and relinearised once per SLOT (k_relin_accum).

// AX [*][2][K][N] prepared eval, AW [*][2][K][N] canonical eval (aux base) -> H [nsite][3][K][N].
// -DCTB_SITE_G2=1: at N = 8192 two sites per 1024-thread CTA (one transform group each, named
// barriers) sharing the prime's twiddle table, 32 instead of 16 resident warps per SM -- measured
// 27% SLOWER (57.4 -> 72.7 ms per 4 cfg5 images): the 64-register cap of a 1024-thread CTA spills
// 128 B per thread, and the spills miss the ~20 KB of L1 the shared memory leaves.
#ifndef CTB_SITE_G2
#define CTB_SITE_G2 0
#endif
// site products keep h0 in a second strip up to this ring degree (above it, h0 is recomputed from
// re-read operands -- cheap since the operands are read in the thread-major layout)
#ifndef CTB_SITE_TWO_MAXLOGN
#define CTB_SITE_TWO_MAXLOGN 11  // N = 4096: one strip, 3 CTAs per SM (-3.3% vs two strips, 2 CTAs)
#endif
template <int LOGN>
__host__ __device__ constexpr int site_groups() { return CTB_SITE_G2 && LOGN == 13 ? 2 : 1; }
template <int LOGN>
__host__ __device__ constexpr int site_strips() { return LOGN <= CTB_SITE_TWO_MAXLOGN ? 2 : 1; }
// resident CTAs per SM the site-product registers are capped for (one strip: 3 CTAs of 256 threads fit
// the shared memory at N = 4096)
template <int LOGN>
__host__ __device__ constexpr int site_minb() {
  return site_groups<LOGN>() == 2 ? 1 : (site_strips<LOGN>() == 1 && NttShape<LOGN>::THREADS == 256 ? 3 : NttShape<LOGN>::MINB);
}
// 32-bit words per site group (exchange image + strips), rounded to 16 bytes
template <int LOGN, int GROUPS>
__host__ __device__ constexpr int site_group_words() {
  return (Exchanger<uint32_t, LOGN, 1, GROUPS>::WORDS + site_strips<LOGN>() * (1 << LOGN) + 3) / 4 * 4;
}

// SITE_STRIP: AX / AW in the thread-major chunk layout (stream_forward strip_out): contiguous warp
// loads instead of one 128-byte line per lane.  -DCTB_SITE_STRIP=0: eval layout.
#ifndef CTB_SITE_STRIP
#define CTB_SITE_STRIP 1
#endif
template <int LOGN>
__host__ __device__ constexpr bool site_strip() {
  return CTB_SITE_STRIP && EvalVec<uint32_t, LOGN>::CONTIG && EvalVec<uint32_t, LOGN>::VEC == 4;
}

template <int LOGN, bool SMEM_TW>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS * site_groups<LOGN>(), site_minb<LOGN>())
k_site_product(const uint32_t* AX, const uint32_t* AW, const int32_t* __restrict__ sx,
               const int32_t* __restrict__ sw, uint32_t* H, const PrimeTab<uint32_t>* __restrict__ tabs, int K,
               uint32_t nsite) {
  using Sh = NttShape<LOGN>;
  using T = uint32_t;
  constexpr int GROUPS = site_groups<LOGN>();
  constexpr int TW_WORDS = SMEM_TW ? tw_words<T>(LOGN) : 0;
  using Ex = Exchanger<T, LOGN, 1, GROUPS>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* tw_sm = reinterpret_cast<T*>(smem_raw);
  const int group = (int)(threadIdx.x / Sh::THREADS);
  T* gsm = tw_sm + TW_WORDS + group * site_group_words<LOGN, GROUPS>();
  Ex ex{gsm};
  // thread-private strips: h1 (and h0 when two strips: N <= 4096; at N = 8192 h0 is
  // recomputed from re-read operands, which measured faster than a second strip)
  constexpr bool TWO = site_strips<LOGN>() == 2;
  T* strip = gsm + Ex::WORDS + ntt_tid<LOGN>();
  // Work units are (aux prime, site) pairs in prime-major order; CTA b takes the contiguous range
  // [b U / G, (b + 1) U / G) of the U = K * nsite units, so every SM gets the same number of
  // products whatever gcd(K, SM count) is (K = 17 on 148 SMs left 12 SMs idle with one CTA per
  // prime), and a CTA switches prime -- restaging its twiddle table -- at most a few times.
  const uint64_t U = (uint64_t)K * nsite;
  const uint64_t u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
  const size_t N = Sh::N, KN = (size_t)K * N;
  using EV = EvalVec<T, LOGN>;
  auto ld = [&](const T* base, int i, T (&v)[EV::VEC]) {
    if constexpr (site_strip<LOGN>()) unpack_chunk<T>(__ldg(reinterpret_cast<const uint4*>(base) + i * Sh::THREADS + ntt_tid<LOGN>()), v);
    else EV::load(base, i, v);
  };
  T y[Sh::E];
#pragma unroll 1
  for (uint64_t seg = u0; seg < u1;) {
    const int k = (int)(seg / nsite);
    const uint32_t s_lo = (uint32_t)(seg - (uint64_t)k * nsite);
    const uint32_t s_hi = (uint32_t)(std::min<uint64_t>(u1, (uint64_t)(k + 1) * nsite) - (uint64_t)k * nsite);
    seg = (uint64_t)k * nsite + s_hi;
    PrimeRegs<T> pr(tabs + k);
    const T* twp = pr.fwd;
    if constexpr (SMEM_TW) {
      __syncthreads();  // every group is done with the previous prime's table
      stage_twiddles(pr.fwd, tw_sm, TW_WORDS, Sh::THREADS * GROUPS);
      __syncthreads();
      twp = tw_sm;
    }
    const TwSrc<T, SMEM_TW> tw{twp};
    auto store = [&](uint32_t s, int part) {
      T* dst = H + ((size_t)s * 3 + part) * KN + k * N + coef_base<LOGN>();
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) dst[coef_off<LOGN>(j)] = csub(y[j], pr.p);
    };
    constexpr uint32_t step = GROUPS;
#pragma unroll 1
    for (uint32_t s = s_lo + group; s < s_hi; s += step) {
      const T* a0p = AX + (size_t)sx[s] * 2 * KN + k * N;
      const T* b0p = AW + (size_t)sw[s] * 2 * KN + k * N;
      if (ntt_tid<LOGN>() == 0 && s + step < s_hi) {  // next item's operands towards L2
        const T* na = AX + (size_t)sx[s + step] * 2 * KN + k * N;
        const T* nb = AW + (size_t)sw[s + step] * 2 * KN + k * N;
        bulk_prefetch_l2(na, (uint32_t)(N * 4));
        bulk_prefetch_l2(na + KN, (uint32_t)(N * 4));
        bulk_prefetch_l2(nb, (uint32_t)(N * 4));
        bulk_prefetch_l2(nb + KN, (uint32_t)(N * 4));
      }
      // h2 = a1 b1 (registers), h1 = a0 b1 + a1 b0 (strip)
#pragma unroll
      for (int i = 0; i < EV::CHUNKS; ++i) {
        T a0[EV::VEC], a1[EV::VEC], b0[EV::VEC], b1[EV::VEC];
        ld(a0p, i, a0);
        ld(a0p + KN, i, a1);
        ld(b0p, i, b0);
        ld(b0p + KN, i, b1);
#pragma unroll
        for (int c = 0; c < EV::VEC; ++c) {
          const int j = i * EV::VEC + c;
          y[j] = mont_mul(a1[c], b1[c], pr.p, pr.pinv);
          strip[j * Sh::THREADS] =
              csub(mont_mul(a0[c], b1[c], pr.p, pr.pinv) + mont_mul(a1[c], b0[c], pr.p, pr.pinv), pr.p2);
          if constexpr (TWO) strip[(Sh::E + j) * Sh::THREADS] = mont_mul(a0[c], b0[c], pr.p, pr.pinv);
        }
      }
      ntt_inv_regs<T, LOGN, Sh::NPASS - 1, SMEM_TW, 1, GROUPS, TENSOR_QE>(y, ex, tw, pr.p, pr.p2);
      store(s, 2);
#pragma unroll
      for (int j = 0; j < Sh::E; ++j) y[j] = strip[j * Sh::THREADS];
      ntt_inv_regs<T, LOGN, Sh::NPASS - 1, SMEM_TW, 1, GROUPS, TENSOR_QE>(y, ex, tw, pr.p, pr.p2);
      store(s, 1);
      if constexpr (TWO) {
#pragma unroll
        for (int j = 0; j < Sh::E; ++j) y[j] = strip[(Sh::E + j) * Sh::THREADS];
      } else {
        // h0 = a0 b0 (operands re-read: L1/L2 hits)
#pragma unroll
        for (int i = 0; i < EV::CHUNKS; ++i) {
          T a0[EV::VEC], b0[EV::VEC];
          ld(a0p, i, a0);
          ld(b0p, i, b0);
#pragma unroll
          for (int c = 0; c < EV::VEC; ++c) y[i * EV::VEC + c] = mont_mul(a0[c], b0[c], pr.p, pr.pinv);
        }
      }
      ntt_inv_regs<T, LOGN, Sh::NPASS - 1, SMEM_TW, 1, GROUPS, TENSOR_QE>(y, ex, tw, pr.p, pr.p2);
      store(s, 0);
    }
  }
}

template <int LOGN>
static cudaError_t launch_site_product(const Ctx* c, const uint32_t* ax, const uint32_t* aw, const int32_t* sx,
                                       const int32_t* sw, uint32_t* h, uint64_t nsite, cudaStream_t s) {
  using Sh = NttShape<LOGN>;
  const Base& B = c->base[BASE_B];
  using T = uint32_t;
  constexpr size_t tw_bytes = (size_t)tw_words<T>(LOGN) * sizeof(T);
  constexpr int GROUPS = site_groups<LOGN>();
  constexpr size_t base_bytes = (size_t)site_group_words<LOGN, GROUPS>() * sizeof(T);
  constexpr bool SMEM_TW = LOGN >= 9 && tw_bytes + GROUPS * base_bytes <= (GROUPS == 2 ? 224 : 200) * 1024;
  static_assert(GROUPS == 1 || SMEM_TW, "two site groups need the shared twiddle table");
  auto kern = k_site_product<LOGN, SMEM_TW>;
  const size_t smem = GROUPS * base_bytes + (SMEM_TW ? tw_bytes : 0);
  const int K = B.size();
  if (nsite == 0) return cudaSuccess;
  const int threads = Sh::THREADS * GROUPS;
  uint32_t grid = persistent_grid((const void*)kern, threads, smem);   // all SMs (units balance per CTA)
  grid = (uint32_t)std::min<uint64_t>(grid, (nsite + GROUPS - 1) / GROUPS * (uint64_t)K);
  return launch_kernel_grid(kern, grid, threads, smem, s, ax, aw, sx, sw, h, (const PrimeTab<T>*)B.d_tabs, K,
                            (uint32_t)nsite);
}

// Per (slot, coefficient): over the slot's sites (contiguous in ct3, rows ptr[o]-base ..
// ptr[o+1]-base): C01[o] = sum (c0, c1) mod q_i, DS[o][j] = sum of the w-bit digits of c2
// (plain u32 sums: fewer than 2^(32-w) sites per slot, checked by the host).
template <typename TQ, int LC, int DC, int WC>
__global__ void __launch_bounds__(256) k_slot_digits(const TQ* ct3, const int32_t* __restrict__ ptr, int32_t base,
                                                     TQ* c01, uint32_t* ds, const __grid_constant__ TensorConsts<TQ> c,
                                                     uint32_t n, uint64_t total) {
  const int L = LC ? LC : c.L, D = DC ? DC : c.relin_d;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t o = g >> pow2_shift(n), i = g & (n - 1);
    const int s0 = ptr[o] - base, s1 = ptr[o + 1] - base;
    TQ acc0[MAXQ], acc1[MAXQ];
    uint32_t dsum[MAXDIG];
#pragma unroll
    for (int l = 0; l < (LC ? LC : MAXQ); ++l) acc0[l] = acc1[l] = 0;
#pragma unroll
    for (int j = 0; j < (DC ? DC : MAXDIG); ++j) dsum[j] = 0;
    for (int s = s0; s < s1; ++s) {
      TQ r[MAXQ];
#pragma unroll
      for (int l = 0; l < (LC ? LC : MAXQ); ++l) {
        if (!LC && l >= L) break;
        const TQ q = c.mrcQ.q[l];
        acc0[l] = add_mod(acc0[l], ct3[(((uint64_t)s * 3 + 0) * L + l) * n + i], q);
        acc1[l] = add_mod(acc1[l], ct3[(((uint64_t)s * 3 + 1) * L + l) * n + i], q);
        r[l] = ct3[(((uint64_t)s * 3 + 2) * L + l) * n + i];
      }
      value_digits<TQ, LC, DC, WC, true>(c, r, dsum);
    }
#pragma unroll
    for (int l = 0; l < (LC ? LC : MAXQ); ++l) {
      if (!LC && l >= L) break;
      c01[((o * 2 + 0) * L + l) * n + i] = acc0[l];
      c01[((o * 2 + 1) * L + l) * n + i] = acc1[l];
    }
#pragma unroll
    for (int j = 0; j < (DC ? DC : MAXDIG); ++j) {
      if (!DC && j >= D) break;
      ds[(o * D + j) * n + i] = dsum[j];
    }
  }
}

// ----------------------------------------------------------------------------- host constants
template <typename T>
static ShoupC<T> spair(uint64_t w, uint64_t p) {
  constexpr int W = 8 * sizeof(T);
  return ShoupC<T>{(T)w, (T)(((unsigned __int128)w << W) / p)};
}

template <typename T>
static void fill_mrc_tab(MrcTab<T>& m, const std::vector<uint64_t>& q) {
  constexpr int W = 8 * sizeof(T);
  m.L = (int)q.size();
  for (int j = 0; j < m.L; ++j) {
    m.q[j] = (T)q[j];
    m.q2[j] = (T)(2 * q[j]);
    m.one_q[j] = (T)(((unsigned __int128)1 << W) / q[j]);
    for (int i = 0; i < j; ++i) m.inv[j * (j - 1) / 2 + i] = spair<T>(invmod(q[i] % q[j], q[j]), q[j]);
  }
}

static bool is_prime_u64(uint64_t n) {
  if (n < 2) return false;
  for (uint64_t p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
    if (n % p == 0) return n == p;
  }
  uint64_t d = n - 1;
  int s = 0;
  while (!(d & 1)) { d >>= 1; ++s; }
  for (uint64_t a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
    uint64_t x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; ++r) {
      x = mulmod(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}

template <typename TQ>
static int build_tensor(Ctx* c, std::string& err) {
  const std::vector<uint64_t>& q = c->base[BASE_Q].primes;
  const int L = (int)q.size();
  if (L > MAXQ) { err = "tensoring supports at most 8 cipher primes"; return -3; }
  if (!c->t) { err = "tensoring needs the plain modulus"; return -1; }
  const uint64_t n = c->n;
  BigU Q(1);
  for (uint64_t p : q) Q.mul_small(p);
  BigU hQ = BigU::sub(Q, BigU(1));
  hQ.shr1();                                     // (Q-1)/2
  // |h| <= 2 N ((Q+1)/2)^2 ; |y| <= |h| t / Q + 1
  BigU half1 = Q; half1.add_small(1); half1.shr1();
  BigU hmax = BigU::mul(half1, half1); hmax.mul_small(2 * n);
  BigU ymax = hmax; ymax.mul_small(c->t);
  ymax = big_div(ymax, Q); ymax.add_small(2);
  // P2 > 4 (ymax + 1), M_A > 4 (hmax + 1): exactness needs 2x+1; the float-assisted CRT
  // extensions need the shifted value inside [M/4, 3M/4)
  BigU need_y = ymax; need_y.add_small(1); need_y.mul_small(4);
  BigU need_h = hmax; need_h.add_small(1); need_h.mul_small(4);
  const bool q_in = sizeof(TQ) == 4;             // 30-bit cipher primes are themselves aux primes
  std::vector<uint64_t> aux, p2;
  if (q_in) aux = q;
  // candidate 30-bit NTT primes, descending, skipping Q
  const uint64_t step = 2 * n;
  uint64_t cand = ((1ull << 30) - 2) / step * step + 1;
  BigU P2(1), MA(1);
  for (uint64_t p : aux) MA.mul_small(p);
  while (BigU::cmp(P2, need_y) <= 0 || (!q_in && BigU::cmp(MA, need_h) <= 0)) {
    if (cand <= step) { err = "ran out of 30-bit auxiliary primes"; return -3; }
    if (is_prime_u64(cand) && std::find(q.begin(), q.end(), cand) == q.end()) {
      aux.push_back(cand);
      MA.mul_small(cand);
      if (BigU::cmp(P2, need_y) <= 0) { p2.push_back(cand); P2.mul_small(cand); }
    }
    cand -= step;
  }
  if ((int)aux.size() > MAXA) { err = "tensoring needs more than 20 auxiliary primes"; return -3; }
  std::string e2;
  int rc = build_base(c->base[BASE_B], aux.data(), (int)aux.size(), c->logn, e2);
  if (rc) { err = "aux base: " + e2; return rc; }

  auto* h = new TensorConsts<TQ>();
  std::memset((void*)h, 0, sizeof(TensorConsts<TQ>));
  h->L = L; h->K = (int)aux.size(); h->K2 = (int)p2.size(); h->ext_h = q_in ? 0 : 1;
  h->relin_w = (int)c->relin_base_bits;
  h->relin_d = (int)((Q.bit_length() + c->relin_base_bits - 1) / c->relin_base_bits);
  h->qwords = (int)((Q.bit_length() + 31) / 32) + 2;
  if (h->qwords > 20) { delete h; err = "cipher modulus too wide for relinearisation digits"; return -3; }
  fill_mrc_tab(h->mrcQ, q);
  // digits of (Q-1)/2 over Q
  {
    BigU x = hQ;
    for (int l = 0; l < L; ++l) h->halfQ_dig[l] = (TQ)x.divmod_small(q[l]);
  }
  for (int l = 0; l < L; ++l) h->q_in_aux[l] = -1;
  for (int k = 0; k < h->K; ++k) {
    const uint64_t p = aux[k];
    h->aux_is_q[k] = -1;
    for (int l = 0; l < L; ++l)
      if (q[l] == p) { h->aux_is_q[k] = l; h->q_in_aux[l] = k; }
    h->ap[k] = (uint32_t)p;
    h->a_oneq[k] = (uint32_t)((1ull << 32) / p);
    const uint64_t r2 = (1ull << 32) % p;
    h->a_r2[k] = (uint32_t)r2;
    h->a_r2q[k] = (uint32_t)((r2 << 32) / p);
    for (int j = 0; j + 1 < L; ++j) h->lift_hc[k][j] = spair<uint32_t>(q[j] % p, p);
    h->Q_aux[k] = (uint32_t)Q.mod_small(p);
    h->t_aux[k] = spair<uint32_t>(c->t % p, p);
    h->hQ_aux[k] = (uint32_t)hQ.mod_small(p);
  }
  for (int l = 0; l < L; ++l) {
    h->q_d[l] = (double)q[l];
    h->q_dinv[l] = 1.0 / (double)q[l];  // IEEE division: the same value __drcp_rn gives on the device
    h->t_q[l] = spair<TQ>(c->t % q[l], q[l]);
    h->hQ_q[l] = (TQ)hQ.mod_small(q[l]);
  }
  BigU Ky = P2; Ky.shr1();
  for (int k = 0; k < h->K2; ++k) {
    const uint64_t p = p2[k];
    h->p2_idx[k] = (int)(std::find(aux.begin(), aux.end(), p) - aux.begin());
    for (int j = 0; j + 1 < L; ++j) h->r_hc[k][j] = spair<uint32_t>(q[j] % p, p);
    h->Qinv_p2[k] = spair<uint32_t>(invmod(Q.mod_small(p), p), p);
    h->Ky_p2[k] = (uint32_t)Ky.mod_small(p);
  }
  for (int l = 0; l < L; ++l) h->Ky_q[l] = (TQ)Ky.mod_small(q[l]);
  if (h->ext_h) {
    BigU Kh = MA; Kh.shr1();
    for (int k = 0; k < h->K; ++k) h->Kh_aux[k] = (uint32_t)Kh.mod_small(aux[k]);
    for (int l = 0; l < L; ++l) h->Kh_q[l] = (TQ)Kh.mod_small(q[l]);
  }
  // lazy forms
  {
    std::vector<BigU> M(L + 1, BigU(1));
    for (int i = 1; i <= L; ++i) { M[i] = M[i - 1]; M[i].mul_small(q[i - 1]); }
    for (int j = 0; j < L; ++j) {
      if (sizeof(TQ) == 4) {
        const uint64_t r2 = (1ull << 32) % q[j];
        h->q_r2[j] = (uint32_t)r2;
        h->q_r2q[j] = (uint32_t)((r2 << 32) / q[j]);
        for (int i = 0; i < j; ++i) h->gM[j][i] = (uint32_t)M[i].mod_small(q[j]);
        h->gMinv[j] = spair<uint32_t>(invmod(M[j].mod_small(q[j]), q[j]), q[j]);
      }
    }
    for (int k = 0; k < h->K; ++k)
      for (int i = 0; i < L; ++i) h->aM[k][i] = (uint32_t)M[i].mod_small(aux[k]);
    auto crt = [&](const std::vector<uint64_t>& ps, const BigU& MM, ShoupC<uint32_t>* hinv, float* rcp,
                   ShoupC<TQ> (*hat_q)[MAXA], TQ (*v_q)[MAXA + 1]) {
      for (size_t k = 0; k < ps.size(); ++k) {
        BigU hat = big_div(MM, BigU(ps[k]));
        hinv[k] = spair<uint32_t>(invmod(hat.mod_small(ps[k]), ps[k]), ps[k]);
        rcp[k] = (float)(1.0 / (double)ps[k]);
        for (int l = 0; l < L; ++l) {
          const uint64_t c = hat.mod_small(q[l]);
          if (sizeof(TQ) == 4) {
            hat_q[l][k] = spair<TQ>(c, q[l]);
          } else {  // 50-bit limbs: the bits of (double c, double c/q) for the FP64 products
            const double cd = (double)c, cq = (double)c / (double)q[l];
            uint64_t bc, bq;
            std::memcpy(&bc, &cd, 8);
            std::memcpy(&bq, &cq, 8);
            hat_q[l][k] = ShoupC<TQ>{(TQ)bc, (TQ)bq};
          }
        }
      }
      for (int l = 0; l < L; ++l) {
        const uint64_t mq = MM.mod_small(q[l]);
        for (size_t v = 0; v <= ps.size(); ++v) v_q[l][v] = (TQ)mulmod(v % q[l], mq, q[l]);
      }
    };
    h->lazy_digits = sizeof(TQ) == 4 && h->relin_d <= MAXDIG && h->relin_w >= 1 && h->relin_w <= 29;
    if (h->lazy_digits) {
      const uint32_t wmask = (1u << h->relin_w) - 1u;
      for (int i = 0; i < L; ++i) {
        BigU x = M[i];
        for (int j = 0; j < h->relin_d; ++j) {
          const uint64_t lo = x.w.empty() ? 0 : x.w[0];
          h->dM[i][j] = (uint32_t)lo & wmask;
          for (int b = 0; b < h->relin_w; ++b) x.shr1();
        }
      }
    }
    crt(p2, P2, h->p2_hinv, h->p2_rcp, h->p2_hat_q, h->p2_v_q);
    if (h->ext_h) crt(aux, MA, h->a_hinv, h->a_rcp, h->a_hat_q, h->a_v_q);
  }
  auto* st = new TensorState();
  st->K = h->K; st->K2 = h->K2; st->L = L;
  st->q_lead = q_in && (int)aux.size() == L + (int)p2.size();
  for (int k = 0; st->q_lead && k < (int)p2.size(); ++k) st->q_lead = h->p2_idx[k] == L + k;
  st->host.assign(reinterpret_cast<const unsigned char*>(h), reinterpret_cast<const unsigned char*>(h) + sizeof(TensorConsts<TQ>));
  cudaError_t ce = cudaMalloc(&st->d_consts, sizeof(TensorConsts<TQ>));
  if (ce == cudaSuccess) ce = cudaMemcpy(st->d_consts, h, sizeof(TensorConsts<TQ>), cudaMemcpyHostToDevice);
  delete h;
  if (ce != cudaSuccess) { delete st; err = std::string("tensor constants: ") + cudaGetErrorString(ce); return -2; }
  c->tensor = st;
  return 0;
}

int build_tensor_consts(Ctx* c, std::string& err) {
  return c->base[BASE_Q].word == 4 ? build_tensor<uint32_t>(c, err) : build_tensor<uint64_t>(c, err);
}
void free_tensor_consts(TensorState* t) { delete t; }
int tensor_aux_count(const TensorState* t) { return t ? t->K : 0; }

}  // namespace ctb

using namespace ctb;


static int ensure_tensor(const ctb_ctx_t* ctx, const Ctx*& c) {
  c = reinterpret_cast<const Ctx*>(ctx);
  if (!c) { set_error("null context"); return ERR_ARG; }
  if (!c->tensor) {
    std::string err;
    const int rc = build_tensor_consts(const_cast<Ctx*>(c), err);
    if (rc) { set_error("tensoring setup: " + err); return rc == -2 ? ERR_CUDA : (rc == -3 ? ERR_UNSUPPORTED : ERR_ARG); }
  }
  return OK;
}

extern "C" int ctb_tensor_aux_size(const ctb_ctx_t* ctx) {
  const Ctx* c;
  const int rc = ensure_tensor(ctx, c);
  return rc ? rc : tensor_aux_count(c->tensor);
}

extern "C" int ctb_tensor_lift(const ctb_ctx_t* ctx, const void* ct, uint32_t* out, uint64_t batch, void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c;
  int rc = ensure_tensor(ctx, c);
  if (rc) return rc;
  if (!ct || !out) { set_error("ctb_tensor_lift: null buffer"); return ERR_ARG; }
  const uint64_t total = batch * 2 * c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int L = c->tensor->L, K = c->tensor->K;
  const unsigned grid = grid_stride(total, 4);
  if (c->base[BASE_Q].word == 4) {
    const auto& tc = *reinterpret_cast<const TensorConsts<uint32_t>*>(c->tensor->host.data());
    if (L == 7 && K == 17) k_tensor_lift<uint32_t, 7, 17><<<grid, 256, 0, s>>>((const uint32_t*)ct, out, tc, c->n, total);
    else k_tensor_lift<uint32_t, 0, 0><<<grid, 256, 0, s>>>((const uint32_t*)ct, out, tc, c->n, total);
  } else {
    const auto& tc = *reinterpret_cast<const TensorConsts<uint64_t>*>(c->tensor->host.data());
    if (L == 3 && K == 11) k_tensor_lift<uint64_t, 3, 11><<<grid, 256, 0, s>>>((const uint64_t*)ct, out, tc, c->n, total);
    else k_tensor_lift<uint64_t, 0, 0><<<grid, 256, 0, s>>>((const uint64_t*)ct, out, tc, c->n, total);
  }
  return cuda_status(cudaGetLastError(), "ctb_tensor_lift");
}

extern "C" int ctb_tensor_product(const ctb_ctx_t* ctx, const uint32_t* a_aux, const uint32_t* b_aux, uint32_t* h_aux,
                                  uint64_t batch, void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c;
  int rc = ensure_tensor(ctx, c);
  if (rc) return rc;
  if (!a_aux || !b_aux || !h_aux) { set_error("ctb_tensor_product: null buffer"); return ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  CTB_DISPATCH_LOGN(c->logn, e = (launch_tensor_product<LOGN>(c, a_aux, b_aux, h_aux, batch, s)));
  return cuda_status(e, "ctb_tensor_product");
}

extern "C" int ctb_tensor_round(const ctb_ctx_t* ctx, const uint32_t* h_aux, void* out, uint64_t batch, void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c;
  int rc = ensure_tensor(ctx, c);
  if (rc) return rc;
  if (!h_aux || !out) { set_error("ctb_tensor_round: null buffer"); return ERR_ARG; }
  const uint64_t total = batch * 3 * c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int L = c->tensor->L, K = c->tensor->K, K2 = c->tensor->K2;
  const unsigned grid = grid_stride(total, 4);
  // double-buffered aux residues: at most 2 x MAXA x 256 words = 40 KB, below the 48 KB default
  const size_t smem = 2 * (size_t)K * 256 * sizeof(uint32_t);
  if (c->base[BASE_Q].word == 4) {
    const auto& tc = *reinterpret_cast<const TensorConsts<uint32_t>*>(c->tensor->host.data());
    if (L == 7 && K == 17 && K2 == 10 && c->tensor->q_lead)
      k_tensor_round<uint32_t, 7, 17, 10><<<grid, 256, smem, s>>>(h_aux, (uint32_t*)out, tc, c->n, total);
    else
      k_tensor_round<uint32_t, 0, 0, 0><<<grid, 256, smem, s>>>(h_aux, (uint32_t*)out, tc, c->n, total);
  } else {
    const auto& tc = *reinterpret_cast<const TensorConsts<uint64_t>*>(c->tensor->host.data());
    bool p2_lead = true;  // P2 = aux primes 0..K2-1 (64-bit limbs: no cipher prime is an aux prime)
    for (int k = 0; k < K2; ++k) p2_lead = p2_lead && tc.p2_idx[k] == k;
    if (L == 3 && K == 11 && K2 == 7 && p2_lead)
      k_tensor_round<uint64_t, 3, 11, 7><<<grid, 256, smem, s>>>(h_aux, (uint64_t*)out, tc, c->n, total);
    else
      k_tensor_round<uint64_t, 0, 0, 0><<<grid, 256, smem, s>>>(h_aux, (uint64_t*)out, tc, c->n, total);
  }
  return cuda_status(cudaGetLastError(), "ctb_tensor_round");
}

extern "C" uint64_t ctb_ccmul_workspace_words(const ctb_ctx_t* ctx, uint64_t batch) {
  const Ctx* c;
  if (ensure_tensor(ctx, c)) return 0;
  return batch * 7ull * c->tensor->K * c->n;  // lifted a (2K) + lifted b (2K) + h (3K) polys, uint32
}

extern "C" int ctb_ccmul_raw(const ctb_ctx_t* ctx, const void* a, const void* b, void* out3, uint32_t* workspace,
                             uint64_t batch, void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c;
  int rc = ensure_tensor(ctx, c);
  if (rc) return rc;
  if (!a || !b || !out3 || !workspace) { set_error("ctb_ccmul_raw: null buffer"); return ERR_ARG; }
  const uint64_t poly = (uint64_t)c->tensor->K * c->n;
  uint32_t* la = workspace;
  uint32_t* lb = la + batch * 2 * poly;
  uint32_t* hh = lb + batch * 2 * poly;
  if ((rc = ctb_tensor_lift(ctx, a, la, batch, stream))) return rc;
  if ((rc = ctb_tensor_lift(ctx, b, lb, batch, stream))) return rc;
  if ((rc = ctb_tensor_product(ctx, la, lb, hh, batch, stream))) return rc;
  return ctb_tensor_round(ctx, hh, out3, batch, stream);
}

extern "C" int ctb_relin_digit_count(const ctb_ctx_t* ctx) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c) return ERR_ARG;
  BigU Q(1);
  for (uint64_t p : c->base[BASE_Q].primes) Q.mul_small(p);
  return (int)((Q.bit_length() + c->relin_base_bits - 1) / c->relin_base_bits);
}

extern "C" int ctb_relinearize(const ctb_ctx_t* ctx, const void* ct3, const void* keyprep, uint32_t* digits_ws,
                               void* out, uint64_t batch, void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c;
  int rc = ensure_tensor(ctx, c);
  if (rc) return rc;
  if (!ct3 || !keyprep || !digits_ws || !out) { set_error("ctb_relinearize: null buffer"); return ERR_ARG; }
  if (c->relin_base_bits < 1 || c->relin_base_bits > 29) { set_error("relinearisation base must be 1..29 bits"); return ERR_UNSUPPORTED; }
  const Base& B = c->base[BASE_Q];
  const int D = ctb_relin_digit_count(ctx);
  const uint64_t total = batch * c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  const auto& st = *c->tensor;
  if (B.word == 4) {
    using T = uint32_t;
    const auto& tc = *reinterpret_cast<const TensorConsts<T>*>(st.host.data());
    if (st.L == 7 && D == 14 && c->relin_base_bits == 16 && tc.lazy_digits)
      k_relin_digits<T, 7, 14, 16><<<grid_stride(total, 4), 256, 0, s>>>((const T*)ct3, digits_ws, tc, c->n, total);
    else
      k_relin_digits<T, 0, 0, 0><<<grid_stride(total, 4), 256, 0, s>>>((const T*)ct3, digits_ws, tc, c->n, total);
    e = cudaGetLastError();
    if (e == cudaSuccess)
      CTB_DISPATCH_LOGN(c->logn, e = (launch_relin_accum<T, LOGN>(c, ct3, 3, digits_ws, keyprep, out, batch, D, s)));
  } else {
    using T = uint64_t;
    const auto& tc = *reinterpret_cast<const TensorConsts<T>*>(st.host.data());
    if (st.L == 3 && D == 10 && c->relin_base_bits == 16)
      k_relin_digits<T, 3, 10, 16><<<grid_stride(total, 4), 256, 0, s>>>((const T*)ct3, digits_ws, tc, c->n, total);
    else
      k_relin_digits<T, 0, 0, 0><<<grid_stride(total, 4), 256, 0, s>>>((const T*)ct3, digits_ws, tc, c->n, total);
    e = cudaGetLastError();
    if (e == cudaSuccess)
      CTB_DISPATCH_LOGN(c->logn, e = (launch_relin_accum<T, LOGN>(c, ct3, 3, digits_ws, keyprep, out, batch, D, s)));
  }
  return cuda_status(e, "ctb_relinearize");
}

// ----------------------------------------------------------------------------- fused site sums (C ABI)
namespace {
constexpr uint64_t kSiteChunkBytes = 1ull << 30;  // H workspace budget per chunk

// Sites per chunk; CTB_SITE_CHUNK (sites) overrides the memory-derived value (tests use it to
// exercise the multi-chunk path on small jobs).
uint64_t site_chunk(uint64_t per_site_bytes) {
  static const uint64_t env = [] {
    const char* e = getenv("CTB_SITE_CHUNK");
    return e ? strtoull(e, nullptr, 10) : 0ull;
  }();
  return env ? env : std::max<uint64_t>(1, kSiteChunkBytes / per_site_bytes);
}

size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct SumLayout {
  size_t ax, aw, h, ct3, c01, ds, csr, total;
  uint64_t chunk;
};

SumLayout sum_layout(const Ctx* c, uint32_t n_x, uint32_t n_w, uint32_t n_out, uint32_t n_sites, uint32_t max_slot) {
  SumLayout l{};
  const size_t N = c->n, K = c->tensor->K, L = c->tensor->L, w = c->base[BASE_Q].word;
  const size_t D = (size_t)ctb_relin_digit_count(reinterpret_cast<const ctb_ctx_t*>(c));
  uint64_t chunk = site_chunk(3 * K * N * 4);
  chunk = std::max<uint64_t>(chunk, max_slot);
  chunk = std::min<uint64_t>(chunk, std::max<uint32_t>(n_sites, 1));
  l.chunk = chunk;
  l.ax = al256((size_t)n_x * 2 * K * N * 4);
  l.aw = al256((size_t)n_w * 2 * K * N * 4);
  l.h = al256(chunk * 3 * K * N * 4);
  l.ct3 = al256(chunk * 3 * L * N * w);
  l.c01 = al256(chunk * 2 * L * N * w);
  l.ds = al256(chunk * D * N * 4);
  l.csr = al256(((size_t)n_out + 1 + 2 * (size_t)n_sites) * 4);
  l.total = l.ax + l.aw + l.h + l.ct3 + l.c01 + l.ds + l.csr;
  return l;
}
}  // namespace

extern "C" uint64_t ctb_ccmul_sum_workspace_bytes(const ctb_ctx_t* ctx, uint32_t n_x, uint32_t n_w, uint32_t n_out,
                                                  uint32_t n_sites, uint32_t max_slot_sites) {
  const Ctx* c;
  if (ensure_tensor(ctx, c)) return 0;
  return sum_layout(c, n_x, n_w, n_out, n_sites, max_slot_sites).total;
}

extern "C" int ctb_ccmul_sum(const ctb_ctx_t* ctx, const void* ct_x, uint32_t n_x, const void* ct_w, uint32_t n_w,
                             const uint32_t* sites_host, uint32_t n_sites, uint32_t n_out, const void* keyprep,
                             void* out, void* workspace, uint64_t workspace_bytes, void* stream) {
  if (n_out == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c;
  int rc = ensure_tensor(ctx, c);
  if (rc) return rc;
  if (!ct_x || !ct_w || (n_sites && !sites_host) || !keyprep || !out || !workspace) {
    set_error("ctb_ccmul_sum: null buffer");
    return ERR_ARG;
  }
  if (c->relin_base_bits < 1 || c->relin_base_bits > 29) { set_error("relinearisation base must be 1..29 bits"); return ERR_UNSUPPORTED; }
  const Base& B = c->base[BASE_Q];
  const size_t N = c->n, L = B.size(), w = B.word, K = c->tensor->K;
  const int D = ctb_relin_digit_count(ctx);
  // CSR by output slot, reference site order kept within a slot
  std::vector<int32_t> ptr(n_out + 1, 0), sx(n_sites), sw(n_sites);
  for (uint32_t s = 0; s < n_sites; ++s) {
    const uint32_t xi = sites_host[3 * s], wi = sites_host[3 * s + 1], oi = sites_host[3 * s + 2];
    if (xi >= n_x || wi >= n_w || oi >= n_out) { set_error("ctb_ccmul_sum: site index out of range"); return ERR_ARG; }
    ptr[oi + 1]++;
  }
  uint32_t max_slot = 0;
  for (uint32_t o = 0; o < n_out; ++o) max_slot = std::max<uint32_t>(max_slot, ptr[o + 1]);
  if ((uint64_t)max_slot * ((1ull << c->relin_base_bits) - 1) >= (1ull << 32)) {
    set_error("ctb_ccmul_sum: too many sites in one output slot for 32-bit digit sums");
    return ERR_UNSUPPORTED;
  }
  for (uint32_t o = 0; o < n_out; ++o) ptr[o + 1] += ptr[o];
  {
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    for (uint32_t s = 0; s < n_sites; ++s) {
      const int32_t pos = fill[sites_host[3 * s + 2]]++;
      sx[pos] = (int32_t)sites_host[3 * s];
      sw[pos] = (int32_t)sites_host[3 * s + 1];
    }
  }
  const SumLayout lay = sum_layout(c, n_x, n_w, n_out, n_sites, max_slot);
  if (workspace_bytes < lay.total) { set_error("ctb_ccmul_sum: workspace too small"); return ERR_ARG; }
  char* ws = (char*)workspace;
  uint32_t* AX = (uint32_t*)ws; ws += lay.ax;
  uint32_t* AW = (uint32_t*)ws; ws += lay.aw;
  uint32_t* H = (uint32_t*)ws; ws += lay.h;
  void* CT3 = ws; ws += lay.ct3;
  void* C01 = ws; ws += lay.c01;
  uint32_t* DS = (uint32_t*)ws; ws += lay.ds;
  int32_t* csr = (int32_t*)ws;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int32_t> packed(n_out + 1 + 2 * (size_t)n_sites);
  std::copy(ptr.begin(), ptr.end(), packed.begin());
  std::copy(sx.begin(), sx.end(), packed.begin() + n_out + 1);
  std::copy(sw.begin(), sw.end(), packed.begin() + n_out + 1 + n_sites);
  cudaError_t e = stage_upload(csr, packed.data(), packed.size() * 4, s);  // no stream sync
  if (e != cudaSuccess) return cuda_status(e, "ctb_ccmul_sum csr");
  const int32_t* d_ptr = csr;
  const int32_t* d_sx = csr + n_out + 1;
  const int32_t* d_sw = d_sx + n_sites;
  // every distinct ciphertext: centred lift to the aux base, forward transform once
  if ((rc = ctb_tensor_lift(ctx, ct_x, AX, n_x, stream))) return rc;
  if ((rc = ctb_tensor_lift(ctx, ct_w, AW, n_w, stream))) return rc;
  // AX / AW are consumed only by k_site_product: thread-major chunk layout when it reads them so
  {
    bool strip = false;
    CTB_DISPATCH_LOGN(c->logn, strip = site_strip<LOGN>());
    if ((e = stream_forward(c, BASE_B, true, AX, AX, (uint64_t)n_x * 2, s, strip)) != cudaSuccess) return cuda_status(e, "ctb_ccmul_sum ntt");
    if ((e = stream_forward(c, BASE_B, false, AW, AW, (uint64_t)n_w * 2, s, strip)) != cudaSuccess) return cuda_status(e, "ctb_ccmul_sum ntt");
  }
  // chunks of whole slots
  uint32_t o0 = 0;
  while (o0 < n_out) {
    uint32_t o1 = o0 + 1;
    while (o1 < n_out && (uint64_t)(ptr[o1 + 1] - ptr[o0]) <= lay.chunk) ++o1;
    const int32_t s0 = ptr[o0], ns = ptr[o1] - ptr[o0];
    const uint32_t nslot = o1 - o0;
    if (ns > 0) {
      CTB_DISPATCH_LOGN(c->logn, e = (launch_site_product<LOGN>(c, AX, AW, d_sx + s0, d_sw + s0, H, (uint64_t)ns, s)));
      if (e != cudaSuccess) return cuda_status(e, "ctb_ccmul_sum product");
      if ((rc = ctb_tensor_round(ctx, H, CT3, (uint64_t)ns, stream))) return rc;
    }
    const uint64_t total = (uint64_t)nslot * N;
    if (w == 4) {
      const auto& tc = *reinterpret_cast<const TensorConsts<uint32_t>*>(c->tensor->host.data());
      if (L == 7 && D == 14 && c->relin_base_bits == 16 && tc.lazy_digits)
        k_slot_digits<uint32_t, 7, 14, 16><<<grid_stride(total, 4), 256, 0, s>>>((const uint32_t*)CT3, d_ptr + o0, s0,
                                                                        (uint32_t*)C01, DS, tc, (uint32_t)N, total);
      else
        k_slot_digits<uint32_t, 0, 0, 0><<<grid_stride(total, 4), 256, 0, s>>>((const uint32_t*)CT3, d_ptr + o0, s0,
                                                                       (uint32_t*)C01, DS, tc, (uint32_t)N, total);
    } else {
      const auto& tc = *reinterpret_cast<const TensorConsts<uint64_t>*>(c->tensor->host.data());
      if (L == 3 && D == 10 && c->relin_base_bits == 16)
        k_slot_digits<uint64_t, 3, 10, 16><<<grid_stride(total, 4), 256, 0, s>>>((const uint64_t*)CT3, d_ptr + o0, s0,
                                                                        (uint64_t*)C01, DS, tc, (uint32_t)N, total);
      else
        k_slot_digits<uint64_t, 0, 0, 0><<<grid_stride(total, 4), 256, 0, s>>>((const uint64_t*)CT3, d_ptr + o0, s0,
                                                                       (uint64_t*)C01, DS, tc, (uint32_t)N, total);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_status(e, "ctb_ccmul_sum digits");
    char* o_ptr = (char*)out + (size_t)o0 * 2 * L * N * w;
    if (w == 4) {
      CTB_DISPATCH_LOGN(c->logn, e = (launch_relin_accum<uint32_t, LOGN>(c, C01, 2, DS, keyprep, o_ptr, nslot, D, s)));
    } else {
      CTB_DISPATCH_LOGN(c->logn, e = (launch_relin_accum<uint64_t, LOGN>(c, C01, 2, DS, keyprep, o_ptr, nslot, D, s)));
    }
    if (e != cudaSuccess) return cuda_status(e, "ctb_ccmul_sum relin");
    o0 = o1;
  }
  (void)K;
  return OK;
}
