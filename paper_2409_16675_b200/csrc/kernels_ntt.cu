// Batched NTT / INTT, ring products, fused CPMul and PPMul (sm_100a).
//
// Replaces, on device:
//   ring._NttPlan.forward/inverse          ring.py:186-217  (ctb_ntt_forward/inverse)
//   ring.ring_mul -> _crt_ntt_mul          ring.py:404-474  (ctb_ring_mul)
//   He.cp_mul (lift + 2 ring_mul)          he.py:366-382    (ctb_cpmul, fused)
//   He.pp_mul (plain-ring ring_mul + CRT)  he.py:441-445, ring.py:477-485 (ctb_pp_mul)
// Layout: residues [poly][limb][N] (uint32 or uint64 words), plain [poly][N] uint64.
#include <algorithm>
#include "bulk.cuh"
#include "kernels.hpp"
#include "ctb200.h"

namespace ctb {

// out[i] = a[i * sa] * b[i * sb] in Z_q[x]/(x^N+1), per limb; sa/sb are poly strides (0 = broadcast).
template <typename T, int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS, NttShape<LOGN>::MINB)
k_ring_mul(const T* a, uint64_t sa, const T* b, uint64_t sb, T* out,
           const PrimeTab<T>* __restrict__ tabs, int L) {
  using Sh = NttShape<LOGN>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Exchanger<T, LOGN> ex{reinterpret_cast<T*>(smem_raw)};
  const int limb = blockIdx.x % L;
  const size_t poly = blockIdx.x / L;
  const size_t LN = (size_t)L * Sh::N;
  PrimeRegs<T> pr(tabs + limb);
  const T* pa = a + poly * sa * LN + (size_t)limb * Sh::N;
  const T* pb = b + poly * sb * LN + (size_t)limb * Sh::N;
  T y[Sh::E], x[Sh::E];
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) y[k] = pb[coef_base<LOGN>() + coef_off<LOGN>(k)];
  ntt_fwd_regs<T, LOGN>(y, ex, pr.fwd, pr.p, pr.p2);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) y[k] = shoup_mul(y[k], pr.ninvr, pr.ninvr_q, pr.p);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) x[k] = pa[coef_base<LOGN>() + coef_off<LOGN>(k)];
  ntt_fwd_regs<T, LOGN>(x, ex, pr.fwd, pr.p, pr.p2);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) x[k] = mont_mul(x[k], y[k], pr.p, pr.pinv);
  ntt_inv_regs<T, LOGN>(x, ex, pr.inv, pr.p, pr.p2);
  T* po = out + poly * LN + (size_t)limb * Sh::N;
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) po[coef_base<LOGN>() + coef_off<LOGN>(k)] = csub(x[k], pr.p);
}

// Eval-domain slotwise product (ring.pointwise_mul, ring.py:572-584).
template <typename T>
__global__ void k_pointwise(const T* a, const T* b, T* out, const PrimeTab<T>* __restrict__ tabs,
                            int L, uint32_t n, uint64_t total) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int limb = (int)((i >> pow2_shift(n)) % L);
    const PrimeTab<T>* t = tabs + limb;
    const T p = t->p, pinv = t->pinv;
    T v = mont_mul(a[i], b[i], p, pinv);       // a b R^-1
    v = mont_mul(v, t->rr, p, pinv);           // a b
    out[i] = csub(v, p);
  }
}

// Fused CPMul: ct [B][2][L][N] x pt [B][N] (uint64 in [0,t)) -> out [B][2][L][N].
// he.py:366-382 with the centred lift of he.py:325-327.
//
// Persistent and limb-stationary: CTA k serves limb k % L for ciphertexts
// k / L, k / L + n_l, ... (n_l = CTAs on that limb).  With SMEM_TW it first
// stages its prime's twiddle table (35 KB at N=4096) in shared memory, so every
// butterfly's twiddle is a conflict-free LDS instead of an L1/L2 round trip.
// Per ciphertext: NTT(lift(pt)) once -- scaled by N^-1 * 2^32 into the
// Montgomery domain and parked in a thread-private shared strip -- then per
// part: NTT, slotwise Montgomery product, INTT, canonical store.  The 7 limb
// groups advance through the batch together, so a plaintext read by all 7
// limbs is an L2 hit after the first.
constexpr int CPMUL_NBUF = 1;
// FP64-quotient butterflies (ntt.cuh F64Q_NE) per kernel family: the compute-bound CPMul and
// encryption kernels gain from moving quotients onto the FP64 pipe; the streaming transforms
// (latency-bound at their occupancy) do not (A/B: tools/ab_cpmul.py).
#ifndef CTB_STREAM_QE
#define CTB_STREAM_QE 0
#endif
constexpr int STREAM_QE = CTB_STREAM_QE;


// Groups of THREADS threads per CTA for the persistent CPMul: each group runs
// its own ciphertext of the CTA's limb, all groups share the CTA's twiddle
// table (2 groups at N >= 2048: 512-thread CTAs, 2 per SM, 32 warps).
template <typename T, int LOGN>
__host__ __device__ constexpr int cpmul_groups() { return sizeof(T) == 4 && (LOGN == 12 || LOGN == 11) ? 2 : 1; }
// k_cpmul at N = 4096: one 1024-thread CTA per SM running four transform groups on one limb (one
// twiddle table per SM instead of two, 64 registers, 32 warps) -- measured 6% faster than two
// 512-thread CTAs per SM (1.263 vs 1.344 ms per 4096 CPMul).
// CTB_CPMUL_GROUPS / CTB_CPMUL_NBUF (N = 4096, 32-bit limbs): transform groups per CTA and
// exchange buffers per group (2 = double-buffered, one barrier per exchange instead of two).
#ifndef CTB_CPMUL_GROUPS
#define CTB_CPMUL_GROUPS 4
#endif
#ifndef CTB_CPMUL_NBUF
#define CTB_CPMUL_NBUF 1
#endif
// next item prefetched towards L2 (cp.async.bulk.prefetch.L2) by one thread per group
#ifndef CTB_ENC_F64_POINTWISE
#define CTB_ENC_F64_POINTWISE 1
#endif
#ifndef CTB_CPMUL_F64_POINTWISE
#define CTB_CPMUL_F64_POINTWISE 1
#endif
#ifndef CTB_CPMUL_PF_L2
#define CTB_CPMUL_PF_L2 1
#endif
// read-once / write-once data with streaming cache hints (ld.global.cs / st.global.cs)
#ifndef CTB_CPMUL_STREAM_HINTS
#define CTB_CPMUL_STREAM_HINTS 1
#endif
template <typename T, int LOGN>
__host__ __device__ constexpr int cpmul_kernel_groups() {
  return (sizeof(T) == 4 && LOGN == 12) ? CTB_CPMUL_GROUPS : cpmul_groups<T, LOGN>();
}
template <typename T, int LOGN>
__host__ __device__ constexpr int cpmul_kernel_nbuf() {
  return (sizeof(T) == 4 && LOGN == 12) ? CTB_CPMUL_NBUF : CPMUL_NBUF;
}
template <typename T, int LOGN>
__host__ __device__ constexpr int cpmul_kernel_minb() {
  return cpmul_kernel_groups<T, LOGN>() >= 3 ? 1 : (cpmul_kernel_groups<T, LOGN>() == 2 ? 2 : NttShape<LOGN>::MINB);
}

template <typename T, int LOGN, bool SMEM_TW>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS * cpmul_kernel_groups<T, LOGN>(), cpmul_kernel_minb<T, LOGN>())
k_cpmul(const T* ct, const uint64_t* __restrict__ pt, T* out, const PrimeTab<T>* __restrict__ tabs,
        int L, uint64_t t_half, uint32_t batch, bool plain_fast) {
  using Sh = NttShape<LOGN>;
  constexpr int GROUPS = cpmul_kernel_groups<T, LOGN>();
  constexpr int NB = cpmul_kernel_nbuf<T, LOGN>();
  using Ex = Exchanger<T, LOGN, NB, GROUPS>;
  constexpr int TW_WORDS = SMEM_TW ? tw_words<T>(LOGN) : 0;
  constexpr int GROUP_WORDS = Ex::WORDS + Sh::N;  // exchange image + NTT(pt) strip
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* tw_sm = reinterpret_cast<T*>(smem_raw);
  const int group = (int)(threadIdx.x / Sh::THREADS);
  T* gsm = tw_sm + TW_WORDS + group * GROUP_WORDS;
  Ex ex{gsm};
  Strip<T, LOGN> ysm(gsm + Ex::WORDS);  // NTT(pt) N^-1 2^W, this thread's evaluation slots

  const int limb = blockIdx.x % L;
  const uint32_t slot = blockIdx.x / L;
  const uint32_t nslots = (gridDim.x - limb + L - 1) / L;  // CTAs serving this limb
  PrimeRegs<T> pr(tabs + limb);
  const T tmod = tabs[limb].tmod;
  const T* twp = pr.fwd;
  if constexpr (SMEM_TW) {
    stage_twiddles(pr.fwd, tw_sm, TW_WORDS, Sh::THREADS * GROUPS);
    __syncthreads();
    twp = tw_sm;
  }
  const TwSrc<T, SMEM_TW> tw{twp};
  constexpr bool RELAX = vec_exchange<T, LOGN>() && WARP_EXCHANGE;
  // slotwise products (and the N^-1 scaling) with FP64-pipe quotients (ntt.cuh f64_pointwise)
  constexpr bool F64PW = CTB_CPMUL_F64_POINTWISE && sizeof(T) == 4;
  const double pinv_d = __drcp_rn((double)pr.p), ninv_d = (double)pr.ninv;
  const uint32_t pn32 = 0u - (uint32_t)pr.p;

  T x[Sh::E];
  if constexpr (sizeof(T) == 8) {
    // 64-bit limbs: the whole CPMul stays in the FP64 domain -- the slotwise product is an FP64
    // product of the centred forward outputs with the centred NTT(lift(pt)) N^-1 kept (as double
    // bits) in the strip, so no conversions between the transforms and no 64-bit integer
    // Montgomery products (which ran on the fma pipe while the FP64 pipe idled)
    const F64Prime P{(double)pr.p, __drcp_rn((double)pr.p)};
    const T nv = pr.ninv;
    const double ninv_c = nv > pr.p / 2 ? -(double)(pr.p - nv) : (double)nv;   // centred N^-1
    const double ninv_p = __dmul_rn(ninv_c, P.pinv);
    double d[Sh::E];
    auto load_d = [&](const T (&v)[Sh::E]) {   // canonical (< p) -> the forward transform's input
      if constexpr (Sh::FIRST_R <= 3 && Sh::NPASS > 1) {
        const double off = __dadd_rn(4503599627370496.0, 2.0 * P.p);
#pragma unroll
        for (int k = 0; k < Sh::E; ++k)
          d[k] = __dadd_rn(__longlong_as_double((long long)((uint64_t)v[k] | 0x4330000000000000ull)), -off);
      } else {
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) d[k] = f64_center(f64_from_u64(v[k]), P);
      }
    };
#pragma unroll 1
    for (uint32_t b = slot * GROUPS + group; b < batch; b += nslots * GROUPS) {
      if constexpr (CTB_CPMUL_PF_L2) {   // the next item towards L2 (see the 32-bit loop below)
        if (ntt_tid<LOGN>() == 0 && b + nslots * GROUPS < batch) {
          const uint32_t nb = b + nslots * GROUPS;
          bulk_prefetch_l2(pt + (size_t)nb * Sh::N, (uint32_t)(Sh::N * 8));
          bulk_prefetch_l2(ct + (((size_t)nb * 2) * L + limb) * (size_t)Sh::N, (uint32_t)(Sh::N * sizeof(T)));
          bulk_prefetch_l2(ct + (((size_t)nb * 2 + 1) * L + limb) * (size_t)Sh::N, (uint32_t)(Sh::N * sizeof(T)));
        }
      }
      {
        lift_plain_regs<T, LOGN>(pt + (size_t)b * Sh::N + coef_base<LOGN>(), x, pr, tmod, t_half, plain_fast);
        load_d(x);
        ntt_fwd_f64<T, LOGN, 0, SMEM_TW, NB, GROUPS>(d, ex, tw, P);
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) {   // y = centre(NTT(pt)) N^-1, |y| < p
          const double yv = f64_mulmod(f64_center(d[k], P), ninv_c, ninv_p, P.p);
          x[k] = (T)__double_as_longlong(yv);
        }
        ysm.store(x);
      }
#pragma unroll 1
      for (int part = 0; part < 2; ++part) {
        const size_t off = (((size_t)b * 2 + part) * L + limb) * (size_t)Sh::N + coef_base<LOGN>();
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) x[k] = ct[off + coef_off<LOGN>(k)];
        load_d(x);
        ntt_fwd_f64<T, LOGN, 0, SMEM_TW, NB, GROUPS>(d, ex, tw, P);
#pragma unroll
        for (int c = 0; c < Strip<T, LOGN>::CHUNKS; ++c) {
          T y[Strip<T, LOGN>::VEC];
          ysm.load_chunk(c, y);
#pragma unroll
          for (int j = 0; j < Strip<T, LOGN>::VEC; ++j) {
            const int k = c * Strip<T, LOGN>::VEC + j;
            const double yv = __longlong_as_double((long long)y[j]);
            // centred x (<= p/2) times |y| < p: |x y / p| < p / 2 and the product lies in (-p, p),
            // an admissible input of the inverse transform (ntt.cuh: inputs below 2p)
            d[k] = f64_mulmod(f64_center(d[k], P), yv, __dmul_rn(yv, P.pinv), P.p);
          }
        }
        ntt_inv_f64<T, LOGN, Sh::NPASS - 1, SMEM_TW, NB, GROUPS>(d, ex, tw, P);
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) out[off + coef_off<LOGN>(k)] = (T)f64_to_canon(d[k], P);
      }
    }
    return;
  }
#pragma unroll 1
  for (uint32_t b = slot * GROUPS + group; b < batch; b += nslots * GROUPS) {
    if constexpr (CTB_CPMUL_PF_L2) {
      // the group's next item towards L2 while this one transforms (its loads then pay the L2, not
      // the HBM latency): this limb's two ciphertext parts and the plaintext
      if (ntt_tid<LOGN>() == 0 && b + nslots * GROUPS < batch) {
        const uint32_t nb = b + nslots * GROUPS;
        bulk_prefetch_l2(pt + (size_t)nb * Sh::N, (uint32_t)(Sh::N * 8));
        bulk_prefetch_l2(ct + (((size_t)nb * 2) * L + limb) * (size_t)Sh::N, (uint32_t)(Sh::N * sizeof(T)));
        bulk_prefetch_l2(ct + (((size_t)nb * 2 + 1) * L + limb) * (size_t)Sh::N, (uint32_t)(Sh::N * sizeof(T)));
      }
    }
    {
      lift_plain_regs<T, LOGN>(pt + (size_t)b * Sh::N + coef_base<LOGN>(), x, pr, tmod, t_half, plain_fast);
      // every transform of the loop runs with the relaxed exchange guard (ntt.cuh Exchanger): each
      // follows one of the other direction, except part 0's forward transform right after this
      // one -- the explicit group barrier below is that guard
      ntt_fwd_regs<T, LOGN, 0, SMEM_TW, NB, GROUPS, F64Q_NE, RELAX>(x, ex, tw, pr.p, pr.p2);
      if constexpr (F64PW) {   // y = NTT(pt) N^-1 (no Montgomery factor: the slotwise products are FP64-quotient)
#pragma unroll
        for (int k = 0; k < Sh::E; ++k)
          x[k] = (T)f64_pointwise((uint32_t)x[k], (uint32_t)pr.ninv, ninv_d, pinv_d, (uint32_t)pr.p, pn32);
      } else {
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) x[k] = shoup_mul(x[k], pr.ninvr, pr.ninvr_q, pr.p);
      }
      ysm.store(x);
      if constexpr (RELAX) group_sync<LOGN, GROUPS>();
    }
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      const size_t off = (((size_t)b * 2 + part) * L + limb) * (size_t)Sh::N + coef_base<LOGN>();
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) x[k] = CTB_CPMUL_STREAM_HINTS ? __ldcs(ct + off + coef_off<LOGN>(k)) : ct[off + coef_off<LOGN>(k)];
      // canonical ciphertext residues in: the forward transform skips the conditional subtractions
      // of its first stage (the inverse's inputs, Montgomery products of x < 4p and y < 2p, only
      // lie below 2p)
      ntt_fwd_regs<T, LOGN, 0, SMEM_TW, NB, GROUPS, F64Q_NE, RELAX, true>(x, ex, tw, pr.p, pr.p2);
#pragma unroll
      for (int c = 0; c < Strip<T, LOGN>::CHUNKS; ++c) {
        T y[Strip<T, LOGN>::VEC];
        ysm.load_chunk(c, y);
#pragma unroll
        for (int j = 0; j < Strip<T, LOGN>::VEC; ++j) {
          const int k = c * Strip<T, LOGN>::VEC + j;
          if constexpr (F64PW)
            x[k] = (T)f64_pointwise((uint32_t)x[k], (uint32_t)y[j], __uint2double_rn((uint32_t)y[j]), pinv_d, (uint32_t)pr.p, pn32);
          else
            x[k] = mont_mul(x[k], y[j], pr.p, pr.pinv);
        }
      }
      ntt_inv_regs<T, LOGN, Sh::NPASS - 1, SMEM_TW, NB, GROUPS, F64Q_NE, RELAX>(x, ex, tw, pr.p, pr.p2);
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) {
        if constexpr (CTB_CPMUL_STREAM_HINTS) __stcs(out + off + coef_off<LOGN>(k), csub(x[k], pr.p));
        else out[off + coef_off<LOGN>(k)] = csub(x[k], pr.p);
      }
    }
  }
}

// Persistent limb-stationary streaming transforms (the k_cpmul layout without
// the plaintext strip) over [npoly][L][N] batches:
//   Fwd          ctb_ntt_forward   canonical eval, bit-reversed (ring.ntt_forward)
//   Inv          ctb_ntt_inverse   (ring.ntt_inverse, N^-1 applied)
//   Prepare      ctb_prepare_operand: NTT(b) N^-1 2^W, the Montgomery-domain operand
//                that MulPrepared consumes (keys multiplying many polynomials: one
//                forward NTT per key instead of per product)
//   MulPrepared  ctb_mul_prepared: a * b (+ addend) with b prepared ([nb][L][N], stride
//                0 broadcasts) -- ring.ring_mul then ring.ring_add (ring.py:363-427)
//                fused: 1 forward + 1 inverse NTT per product.
//   InvAdd       unscaled INTT (+ addend): eval-domain sums of products with prepared
//                operands (N^-1 already folded in) back to coefficients, plus a
//                coefficient-domain addend (K3's mask product).
//   LiftPrepare  plain [npoly][N] in [0,t) -> NTT(centred lift) N^-1 2^W per limb (ctb_lift_prepare)
//   LiftFwd      plain [npoly][N] -> canonical NTT of the (centred) lift per limb
//   FwdNinv      NTT(x) N^-1, canonical: the eval-domain form of a coefficient addend to
//                sums of products with prepared operands (ctb_eval_addend)  Twiddles staged once per CTA in
// shared memory, GROUPS transforms per CTA sharing them.
enum class StreamOp { Fwd, Inv, Prepare, MulPrepared, InvAdd, LiftPrepare, FwdNinv, LiftFwd };

template <typename T>
struct StreamArgs {
  const T* in;             // [npoly * in_stride][L][N] (item b at poly b * in_stride)
  T* out;                  // [npoly][L][N]
  const T* bprep;          // MulPrepared: prepared operand, item b uses poly b * b_stride
  const T* addend;         // MulPrepared / InvAdd: item b adds poly b * add_stride (may be null)
  const uint64_t* plain;   // LiftPrepare: [npoly][N] values in [0, t)
  uint64_t in_stride, b_stride, add_stride, t_half;
  bool plain_fast;
  bool strip_in;           // Inv / InvAdd: input in the thread-major chunk layout (see strip_out)
  bool bprep_strip;        // MulPrepared: the prepared operand in the thread-major chunk layout
  bool strip_out;          // Fwd / Prepare: thread-major chunk layout (chunk c of transform thread t at
                           // 16-byte index c * THREADS + t) for internal operands whose consumer reads
                           // them the same way (k_site_product); contiguous warp stores, no transposition
};

template <typename T, int LOGN>
struct StreamCfg {
  using Sh = NttShape<LOGN>;
#ifndef CTB_STREAM_GROUPS4
#define CTB_STREAM_GROUPS4 1
#endif
  // transform groups per CTA: at N = 4096 four (one 1024-thread CTA per SM, one twiddle table
  // per SM, ~78 KB of L1 left for the epilogue operands; measured 4-6% faster than two 512-thread
  // CTAs on different limbs)
  // at N = 8192 (32-bit limbs: the auxiliary base of the 50-bit tensoring) two per 1024-thread CTA:
  // one twiddle table per SM and room for the TMA staging buffers (one 512-thread CTA per SM
  // otherwise) -- measured 24.8 -> 22.0 ms forward transforms per 4 cfg5 images (-11%)
#ifndef CTB_STREAM_G2_13
#define CTB_STREAM_G2_13 1
#endif
  static constexpr bool WIDE = (CTB_STREAM_GROUPS4 && sizeof(T) == 4 && LOGN == 12) ||
                               (CTB_STREAM_G2_13 && sizeof(T) == 4 && LOGN == 13);
  static constexpr int GROUPS = (CTB_STREAM_GROUPS4 && sizeof(T) == 4 && LOGN == 12) ? 4
                                : (CTB_STREAM_G2_13 && sizeof(T) == 4 && LOGN == 13) ? 2 : cpmul_groups<T, LOGN>();
  // (64-bit limbs: one 512-thread CTA per SM at ~108 registers, so the staging buffer fits beside
  // the table and the image)
  static constexpr int CTAS_PER_SM = WIDE || sizeof(T) == 8 ? 1 : 2;
  using Ex = Exchanger<T, LOGN, CPMUL_NBUF, GROUPS>;
  // eval-layout loads / stores through the exchange image (ntt.cuh eval_xpose_*)
  static constexpr bool XPOSE = CTB_EVAL_XPOSE && eval_xpose_ok<T, LOGN>(Ex::WORDS);
  // loads too for 32-bit words (u64 loads measured neutral to 6% slower in cfg5's InvAdd /
  // MulPrepared: the 64-bit path stages chunk by chunk without a prefetch across the barrier)
  static constexpr bool XPOSE_LD = XPOSE && sizeof(T) == 4;
  static constexpr size_t TW_BYTES = (size_t)tw_words<T>(LOGN) * sizeof(T);
  // u32: table + images within 200 KB (two CTAs per SM with staging); 64-bit limbs: the
  // (w, w/p) table (140 KB at N=8192) + image fill one CTA's 227 KB
  static constexpr bool SMEM_TW = LOGN >= 9 && TW_BYTES + GROUPS * (size_t)Ex::WORDS * sizeof(T) <=
                                                   (sizeof(T) == 4 ? 200 * 1024 : 226 * 1024);
  // TMA prefetch of the next item into an N-word staging buffer per group (u32, where the
  // table + images + staging still fit two CTAs per SM)
  static constexpr int EXW = (Ex::WORDS * (int)sizeof(T) + 15) / 16 * 16 / (int)sizeof(T);
  static constexpr bool PF_OK = SMEM_TW && (TW_BYTES + GROUPS * ((size_t)EXW + Sh::N) * sizeof(T) + 64) * CTAS_PER_SM <= 220 * 1024;
  static constexpr int GW = EXW + (PF_OK ? Sh::N : 0);  // words per group
  static constexpr size_t SMEM = (SMEM_TW ? TW_BYTES : 0) + GROUPS * (size_t)GW * sizeof(T) + (PF_OK ? 64 : 0);
  static constexpr int THREADS = Sh::THREADS * GROUPS;
  static constexpr int MINB = WIDE ? 1 : (GROUPS == 2 ? 2 : Sh::MINB);
};

template <typename T, int LOGN, bool SMEM_TW, StreamOp OP>
__global__ void __launch_bounds__(StreamCfg<T, LOGN>::THREADS, StreamCfg<T, LOGN>::MINB)
k_stream(const StreamArgs<T> a, const PrimeTab<T>* __restrict__ tabs, int L, uint32_t npoly) {
  using C = StreamCfg<T, LOGN>;
  using Sh = NttShape<LOGN>;
  constexpr int GROUPS = C::GROUPS;
  // (64-bit limbs: not for the public inverse, whose bit-reversed reads from the staging buffer
  // conflict -- measured +15% -- while its internal variant InvAdd reads the thread-major strip)
  constexpr bool PF = C::PF_OK && OP != StreamOp::LiftPrepare && OP != StreamOp::LiftFwd &&
                      !(sizeof(T) == 8 && OP == StreamOp::Inv);
  constexpr bool EARLY = PF && sizeof(T) == 8;   // next-item load issued right after the staging read
  constexpr int TW_WORDS = SMEM_TW ? tw_words<T>(LOGN) : 0;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* tw_sm = reinterpret_cast<T*>(smem_raw);
  const int group = (int)(threadIdx.x / Sh::THREADS);
  T* gsm = tw_sm + TW_WORDS + group * C::GW;
  typename C::Ex ex{gsm};
  T* stg = gsm + C::EXW;
  uint64_t* bar = reinterpret_cast<uint64_t*>(tw_sm + TW_WORDS + GROUPS * C::GW) + group;
  const bool leader = ntt_tid<LOGN>() == 0;
  const int limb = blockIdx.x % L;
  const uint32_t slot = blockIdx.x / L;
  const uint32_t nslots = (gridDim.x - limb + L - 1) / L;
  const uint32_t step = nslots * GROUPS;
  PrimeRegs<T> pr(tabs + limb);
  const T* twp = pr.fwd;
  if constexpr (SMEM_TW) {
    stage_twiddles(pr.fwd, tw_sm, TW_WORDS, C::THREADS);
    twp = tw_sm;
  }
  uint32_t b = slot * GROUPS + group;
  if constexpr (PF) {
    if (leader) {
      mbar_init(bar, 1);
      mbar_init_fence();
      if (b < npoly) bulk_load(stg, a.in + ((size_t)b * a.in_stride * L + limb) * Sh::N, Sh::N * sizeof(T), bar);
    }
  }
  if constexpr (SMEM_TW || PF) __syncthreads();
  const TwSrc<T, SMEM_TW> tw{twp};
  const int cb = coef_base<LOGN>();
  uint32_t phase = 0;
  T x[Sh::E];
#pragma unroll 1
  for (; b < npoly; b += step) {
    const size_t off = ((size_t)b * L + limb) * (size_t)Sh::N;               // output item
    const size_t ioff = ((size_t)b * a.in_stride * L + limb) * (size_t)Sh::N;  // input item
    const size_t aoff = ((size_t)b * a.add_stride * L + limb) * (size_t)Sh::N;
    auto issue_next = [&]() {
      if constexpr (PF) {
        if (leader) {
          if (b + step < npoly) {
            fence_proxy_async_smem();
            bulk_load(stg, a.in + ((size_t)(b + step) * a.in_stride * L + limb) * Sh::N, Sh::N * sizeof(T), bar);
          }
          // the epilogue's per-item operands: start them towards L2 while this item transforms
          if ((OP == StreamOp::InvAdd || OP == StreamOp::MulPrepared) && a.addend)
            bulk_prefetch_l2(a.addend + aoff, Sh::N * sizeof(T));
          if (OP == StreamOp::MulPrepared && a.b_stride)
            bulk_prefetch_l2(a.bprep + ((size_t)b * a.b_stride * L + limb) * (size_t)Sh::N, Sh::N * sizeof(T));
        }
      }
    };
    constexpr bool EVAL_IN = OP == StreamOp::Inv || OP == StreamOp::InvAdd;
    if constexpr (PF) {
      mbar_wait(bar, phase);
      phase ^= 1;
      if constexpr (EVAL_IN) {
        constexpr bool SI = EvalVec<T, LOGN>::CONTIG && EvalVec<T, LOGN>::VEC * sizeof(T) == 16;
        if (SI && a.strip_in) {  // thread-major chunks: contiguous, conflict-free staging reads
          const uint4* s4 = reinterpret_cast<const uint4*>(stg);
#pragma unroll
          for (int c = 0; c < Sh::E * (int)sizeof(T) / 16; ++c)
            unpack_chunk<T>(s4[c * Sh::THREADS + ntt_tid<LOGN>()], x + c * (16 / (int)sizeof(T)));
        } else if constexpr (C::XPOSE_LD) {
          eval_xpose_apply<T, LOGN, GROUPS, true>(stg, gsm, [&](int c, const T* v) {
#pragma unroll
            for (int i = 0; i < 16 / (int)sizeof(T); ++i) x[c * (16 / (int)sizeof(T)) + i] = v[i];
          });
        } else {
          load_eval_smem<T, LOGN>(stg, x);
        }
      } else {
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) x[k] = stg[cb + coef_off<LOGN>(k)];
      }
      // the next item's staging load is issued after the transform's first exchange, whose
      // barrier already orders every thread's staging read before it (see xform_fwd/xform_inv);
      // 64-bit limbs transform whole polynomials, so they order the reads with one group barrier
      // and issue the load right away (it then overlaps the whole transform, not just the store)
      if constexpr (EARLY) {
        group_sync<LOGN, GROUPS>();
        issue_next();
      }
    } else if constexpr (OP == StreamOp::LiftPrepare || OP == StreamOp::LiftFwd) {
      const uint64_t* src = a.plain + (size_t)b * Sh::N + cb;
      if (leader && b + step < npoly) bulk_prefetch_l2(a.plain + (size_t)(b + step) * Sh::N, Sh::N * 8);
      lift_plain_regs<T, LOGN>(src, x, pr, tabs[limb].tmod, a.t_half, a.plain_fast);
    } else if constexpr (EVAL_IN) {
      constexpr bool SI = EvalVec<T, LOGN>::CONTIG && EvalVec<T, LOGN>::VEC * sizeof(T) == 16;
      if (SI && a.strip_in) {
        const uint4* s4 = reinterpret_cast<const uint4*>(a.in + ioff);
#pragma unroll
        for (int c = 0; c < Sh::E * (int)sizeof(T) / 16; ++c)
          unpack_chunk<T>(__ldg(s4 + c * Sh::THREADS + ntt_tid<LOGN>()), x + c * (16 / (int)sizeof(T)));
      } else if constexpr (C::XPOSE_LD) {
        eval_xpose_apply<T, LOGN, GROUPS>(a.in + ioff, gsm, [&](int c, const T* v) {
#pragma unroll
          for (int i = 0; i < 16 / (int)sizeof(T); ++i) x[c * (16 / (int)sizeof(T)) + i] = v[i];
        });
      } else {
        load_eval<T, LOGN>(a.in + ioff, x);
      }
    } else {
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) x[k] = a.in[ioff + cb + coef_off<LOGN>(k)];
    }
    // forward / inverse transform; with staging, split after the first exchange to issue the
    // next item's load there (PF implies 32-bit limbs and >= 3 passes)
    // (64-bit limbs transform whole polynomials on the FP64 path: issue after the transform)
    constexpr bool SPLIT = PF && sizeof(T) == 4 && Sh::NPASS >= 2;
    auto xform_fwd = [&]() {
      if constexpr (SPLIT) {
        fwd_pass<T, LOGN, 0, SMEM_TW>(x, tw, pr.p, pr.p2);
        ex.template run<Sh::pass_s(0), Sh::pass_r(0), Sh::pass_s(1), Sh::pass_r(1)>(x);
        issue_next();
        ntt_fwd_regs<T, LOGN, 1, SMEM_TW, CPMUL_NBUF, GROUPS, STREAM_QE>(x, ex, tw, pr.p, pr.p2);
      } else {
        ntt_fwd_regs<T, LOGN, 0, SMEM_TW, CPMUL_NBUF, GROUPS, STREAM_QE>(x, ex, tw, pr.p, pr.p2);
        if constexpr (!EARLY) issue_next();
      }
    };
    auto store_out = [&](const T (&v)[Sh::E]) {
      if constexpr (EvalVec<T, LOGN>::CONTIG && EvalVec<T, LOGN>::VEC * sizeof(T) == 16) {
        if (a.strip_out) {
          uint4* o4 = reinterpret_cast<uint4*>(a.out + off);
#pragma unroll
          for (int c = 0; c < EvalVec<T, LOGN>::CHUNKS; ++c)
            o4[c * Sh::THREADS + ntt_tid<LOGN>()] = pack_chunk<T>(v + c * EvalVec<T, LOGN>::VEC);
          return;
        }
      }
      if constexpr (C::XPOSE) store_eval_xpose<T, LOGN, GROUPS>(a.out + off, v, gsm);
      else store_eval<T, LOGN>(a.out + off, v);
    };
    auto xform_inv = [&](bool first_in_item) {
      constexpr int K = Sh::NPASS - 1;
      if constexpr (SPLIT) {
        if (first_in_item) {
          inv_pass<T, LOGN, K, SMEM_TW>(x, tw, pr.p, pr.p2);
          ex.template run<Sh::pass_s(K), Sh::pass_r(K), Sh::pass_s(K - 1), Sh::pass_r(K - 1)>(x);
          issue_next();
          ntt_inv_regs<T, LOGN, K - 1, SMEM_TW, CPMUL_NBUF, GROUPS, STREAM_QE>(x, ex, tw, pr.p, pr.p2);
          return;
        }
      }
      ntt_inv_regs<T, LOGN, K, SMEM_TW, CPMUL_NBUF, GROUPS, STREAM_QE>(x, ex, tw, pr.p, pr.p2);
      if (!EARLY && first_in_item) issue_next();
    };
    if constexpr (OP == StreamOp::Inv) {
      xform_inv(true);
#pragma unroll
      for (int k = 0; k < Sh::E; ++k)
        a.out[off + cb + coef_off<LOGN>(k)] = csub(shoup_mul(x[k], pr.ninv, pr.ninv_q, pr.p), pr.p);
    } else if constexpr (OP == StreamOp::InvAdd) {
      xform_inv(true);
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) {
        const int j = cb + coef_off<LOGN>(k);
        T v = csub(x[k], pr.p);
        if (a.addend) v = add_mod(v, a.addend[aoff + j], pr.p);
        a.out[off + j] = v;
      }
    } else {
      xform_fwd();
      if constexpr (OP == StreamOp::Fwd || OP == StreamOp::LiftFwd) {
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) x[k] = pr.canon_fwd(x[k]);
        store_out(x);
      } else if constexpr (OP == StreamOp::FwdNinv) {
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) x[k] = csub(shoup_mul(x[k], pr.ninv, pr.ninv_q, pr.p), pr.p);
        store_out(x);
      } else if constexpr (OP == StreamOp::Prepare || OP == StreamOp::LiftPrepare) {
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) x[k] = csub(shoup_mul(x[k], pr.ninvr, pr.ninvr_q, pr.p), pr.p);
        store_out(x);
      } else {
        const T* pb = a.bprep + ((size_t)b * a.b_stride * L + limb) * (size_t)Sh::N;
        using EV = EvalVec<T, LOGN>;
        constexpr bool SB = EV::CONTIG && EV::VEC * sizeof(T) == 16;
        if (SB && a.bprep_strip) {
#pragma unroll
          for (int i = 0; i < EV::CHUNKS; ++i) {
            T v[EV::VEC];
            unpack_chunk<T>(__ldg(reinterpret_cast<const uint4*>(pb) + i * Sh::THREADS + ntt_tid<LOGN>()), v);
#pragma unroll
            for (int c = 0; c < EV::VEC; ++c) x[i * EV::VEC + c] = mont_mul(x[i * EV::VEC + c], v[c], pr.p, pr.pinv);
          }
        } else if constexpr (C::XPOSE_LD) {
          eval_xpose_apply<T, LOGN, GROUPS>(pb, gsm, [&](int i, const T* v) {
#pragma unroll
            for (int c = 0; c < EV::VEC; ++c) x[i * EV::VEC + c] = mont_mul(x[i * EV::VEC + c], v[c], pr.p, pr.pinv);
          });
        } else {
#pragma unroll
          for (int i = 0; i < EV::CHUNKS; ++i) {
            T v[EV::VEC];
            EV::load(pb, i, v);
#pragma unroll
            for (int c = 0; c < EV::VEC; ++c) x[i * EV::VEC + c] = mont_mul(x[i * EV::VEC + c], v[c], pr.p, pr.pinv);
          }
        }
        xform_inv(false);
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) {
          const int j = cb + coef_off<LOGN>(k);
          T v = csub(x[k], pr.p);
          if (a.addend) v = add_mod(v, a.addend[aoff + j], pr.p);
          a.out[off + j] = v;
        }
      }
    }
  }
}

template <typename T, int LOGN, StreamOp OP>
static cudaError_t launch_stream(const Base* b, const StreamArgs<T>& args, uint64_t npoly, cudaStream_t s) {
  using C = StreamCfg<T, LOGN>;
  auto kern = k_stream<T, LOGN, C::SMEM_TW, OP>;
  const int L = b->size();
  if (npoly == 0) return cudaSuccess;
  uint32_t grid = persistent_grid((const void*)kern, C::THREADS, C::SMEM);
  const uint64_t max_grid = (npoly + C::GROUPS - 1) / C::GROUPS * (uint64_t)L;
  grid = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(grid / L * L, (uint64_t)L), max_grid);
  return launch_kernel_grid(kern, grid, C::THREADS, C::SMEM, s, args, (const PrimeTab<T>*)b->d_tabs, L,
                            (uint32_t)npoly);
}

// Host-side builder of StreamArgs (untyped pointers from the C ABI).
template <typename T>
static StreamArgs<T> sargs(const void* in, void* out, const void* bprep = nullptr, uint64_t b_stride = 0,
                           const void* addend = nullptr, uint64_t in_stride = 1, uint64_t add_stride = 1) {
  StreamArgs<T> a{};
  a.in = (const T*)in;
  a.out = (T*)out;
  a.bprep = (const T*)bprep;
  a.addend = (const T*)addend;
  a.in_stride = in_stride;
  a.b_stride = b_stride;
  a.add_stride = add_stride;
  return a;
}

cudaError_t stream_forward(const Ctx* c, int base, bool prepare, const void* in, void* out, uint64_t npoly,
                           cudaStream_t s, bool strip_out) {
  const Base* b = &c->base[base];
  cudaError_t e = cudaSuccess;
  if (b->word == 4) {
    auto a = sargs<uint32_t>(in, out);
    a.strip_out = strip_out;
    if (prepare) CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::Prepare>(b, a, npoly, s)))
    else CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::Fwd>(b, a, npoly, s)))
  } else {
    auto a = sargs<uint64_t>(in, out);
    a.strip_out = strip_out;
    if (prepare) CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::Prepare>(b, a, npoly, s)))
    else CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::Fwd>(b, a, npoly, s)))
  }
  return e;
}

cudaError_t stream_inv_add(const Ctx* c, int base, const void* in, void* out, const void* addend, uint64_t npoly,
                           cudaStream_t s, bool strip_in) {
  const Base* b = &c->base[base];
  cudaError_t e = cudaSuccess;
  if (b->word == 4) {
    auto a = sargs<uint32_t>(in, out, nullptr, 0, addend);
    a.strip_in = strip_in;
    CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::InvAdd>(b, a, npoly, s)));
  } else {
    auto a = sargs<uint64_t>(in, out, nullptr, 0, addend);
    a.strip_in = strip_in;
    CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::InvAdd>(b, a, npoly, s)));
  }
  return e;
}

// Fused encryption (He.encrypt, he.py:307-323): per (ciphertext, limb)
//   c0 = INTT(NTT(u) * b^) + e1 + Delta * lift(m),   c1 = INTT(NTT(u) * a^) + e2
// with (b^, a^) the prepared public key ([2][L][N], ctb_prepare_operand) and
// draws [B][3][N] int64 = (u, e1, e2) small signed integers sampled by the
// caller (the reference's numpy stream, or the device generator).  One forward
// and two inverse transforms per limb; persistent and limb-stationary like
// k_cpmul, twiddles in shared memory.  At N = 4096 (32-bit limbs) one 1024-thread CTA per SM
// runs four transform groups on one limb: one shared twiddle table instead of two per SM, and the
// limb's prepared public key (2 x 16 KB, read by every item) stays resident in the ~78 KB of L1
// that the smaller shared-memory footprint leaves (two CTAs on different limbs would evict it).
template <typename T, int LOGN>
__host__ __device__ constexpr int enc_groups() { return sizeof(T) == 4 && LOGN == 12 ? 4 : cpmul_groups<T, LOGN>(); }
// The limb's prepared public key (b^, a^: 2 x N words) staged once per CTA in shared memory, in the
// chunk-major Strip layout (conflict-free 128-bit reads), instead of re-reading it from L1/L2 for every
// item: at N = 4096 (four groups) twiddles + images + strips + key = 200 KB.
#ifndef CTB_ENC_PKSM
#define CTB_ENC_PKSM 1
#endif
template <typename T, int LOGN>
__host__ __device__ constexpr bool enc_pk_smem() {
  return CTB_ENC_PKSM && sizeof(T) == 4 && LOGN == 12 &&
         (size_t)tw_words<T>(LOGN) * sizeof(T) +
                 enc_groups<T, LOGN>() * ((size_t)Exchanger<T, LOGN, CPMUL_NBUF, enc_groups<T, LOGN>()>::WORDS + (1 << LOGN)) * sizeof(T) +
                 2 * (size_t)(1 << LOGN) * sizeof(T) <= 227 * 1024;
}

// Public key in the thread-major chunk layout (converted per call into a pool temporary) when it
// is not staged in shared memory (64-bit limbs): contiguous warp loads.  -DCTB_ENC_PKSTRIP=0: direct.
#ifndef CTB_ENC_PKSTRIP
#define CTB_ENC_PKSTRIP 1
#endif
#ifndef CTB_ENC_MSTRIP
#define CTB_ENC_MSTRIP 1
#endif
template <typename T, int LOGN>
__host__ __device__ constexpr bool enc_pk_strip() {
  return CTB_ENC_PKSTRIP && !enc_pk_smem<T, LOGN>() && EvalVec<T, LOGN>::CONTIG && EvalVec<T, LOGN>::VEC * sizeof(T) == 16;
}
// 64-bit limbs: the encryption's products and transforms in the FP64 domain (key strips as doubles)
template <typename T, int LOGN>
__host__ __device__ constexpr bool enc_f64() {
  return sizeof(T) == 8 && enc_pk_strip<T, LOGN>() && Strip<T, LOGN>::VEC == EvalVec<T, LOGN>::VEC;
}

template <typename T, int LOGN, bool SMEM_TW, bool GATHER = false>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS * enc_groups<T, LOGN>(),
                                  enc_groups<T, LOGN>() == 4 ? 1 : (enc_groups<T, LOGN>() == 2 ? 2 : NttShape<LOGN>::MINB))
k_encrypt(const uint64_t* __restrict__ m, const int8_t* __restrict__ draws, const T* __restrict__ pkprep, T* out,
          const PrimeTab<T>* __restrict__ tabs, int L, uint64_t t_half, uint32_t batch, bool plain_fast,
          const __grid_constant__ PlainGather g) {
  using Sh = NttShape<LOGN>;
  constexpr int GROUPS = enc_groups<T, LOGN>();
  using Ex = Exchanger<T, LOGN, CPMUL_NBUF, GROUPS>;
  constexpr int TW_WORDS = SMEM_TW ? tw_words<T>(LOGN) : 0;
  constexpr int GROUP_WORDS = Ex::WORDS + Sh::N;
  constexpr bool PKSM = enc_pk_smem<T, LOGN>() && SMEM_TW;
  using EV = EvalVec<T, LOGN>;
  // (64-bit limbs: -8.2% at N=8192; at N=4096 / 32-bit the 64-register cap spills and it is neutral)
  constexpr bool MSTRIP = CTB_ENC_MSTRIP && sizeof(T) == 8 && Strip<T, LOGN>::VEC > 1 &&
                          Strip<T, LOGN>::VEC * Strip<T, LOGN>::CHUNKS == Sh::E;
  constexpr bool ENC_XPOSE = !PKSM && !enc_pk_strip<T, LOGN>() && sizeof(T) == 4 && CTB_EVAL_XPOSE &&
                             EV::VEC == Strip<T, LOGN>::VEC && eval_xpose_ok<T, LOGN>(Ex::WORDS);
  static_assert(!PKSM || (EV::VEC == Strip<T, LOGN>::VEC && GROUPS >= 2), "key strips need contiguous eval chunks");
  // relaxed exchange guards / first-stage shortcuts of the 32-bit transforms (see the item loop)
  constexpr bool RELAX = vec_exchange<T, LOGN>() && WARP_EXCHANGE && !ENC_XPOSE;
  // slotwise products with FP64-pipe quotients (ntt.cuh f64_pointwise) when the key is staged in
  // shared memory (converted out of the Montgomery domain once per CTA)
  constexpr bool F64PW = CTB_ENC_F64_POINTWISE && sizeof(T) == 4 && PKSM;
  // Montgomery products with canonical prepared key words (ctb_prepare_operand) are canonical;
  // the FP64-quotient products lie in (0.49 p, 1.51 p): no first-stage shortcut for the inverse
  constexpr bool KEY_CANON = sizeof(T) == 4 && !F64PW;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* tw_sm = reinterpret_cast<T*>(smem_raw);
  const int group = (int)(threadIdx.x / Sh::THREADS);
  T* gsm = tw_sm + TW_WORDS + group * GROUP_WORDS;
  Ex ex{gsm};
  Strip<T, LOGN> usm(gsm + Ex::WORDS);  // NTT(u), this thread's evaluation slots
  T* pk_sm = tw_sm + TW_WORDS + GROUPS * GROUP_WORDS;  // PKSM: [part][N] key strips

  const int limb = blockIdx.x % L;
  const uint32_t slot = blockIdx.x / L;
  const uint32_t nslots = (gridDim.x - limb + L - 1) / L;
  PrimeRegs<T> pr(tabs + limb);
  const T tmod = tabs[limb].tmod, delta = tabs[limb].delta, delta_q = tabs[limb].delta_q;
  const T* twp = pr.fwd;
  if constexpr (PKSM) {
    if (group < 2) {  // group g stages part g of this limb's key
      const T* kp = pkprep + ((size_t)group * L + limb) * Sh::N;
      Strip<T, LOGN> ks(pk_sm + (size_t)group * Sh::N);
#pragma unroll
      for (int i = 0; i < EV::CHUNKS; ++i) {
        T v[EV::VEC];
        EV::load(kp, i, v);
        if constexpr (F64PW) {   // out of the Montgomery domain: the FP64-quotient products carry no 2^-W
#pragma unroll
          for (int c = 0; c < EV::VEC; ++c) v[c] = mont_mul(v[c], (T)1, pr.p, pr.pinv);
        }
        ks.store_chunk(i, v);
      }
    }
  }
  if constexpr (SMEM_TW) {
    stage_twiddles(pr.fwd, tw_sm, TW_WORDS, Sh::THREADS * GROUPS);
    __syncthreads();
    twp = tw_sm;
  }
  const TwSrc<T, SMEM_TW> tw{twp};
  const double pinv_d = __drcp_rn((double)pr.p);
  auto small = [&](int8_t v) -> T {  // |v| <= 127 < p: canonical residue
    return v < 0 ? pr.p - (T)(-(int)v) : (T)v;
  };
  const int cb = coef_base<LOGN>();
  T x[Sh::E];
#pragma unroll 1
  // device draw layout (sample.cu): this thread's E draws of each kind are contiguous
  const int tid = ntt_tid<LOGN>();
  auto load_draws = [&](const int8_t* row, int8_t (&v)[Sh::E]) {
    if constexpr (Sh::E == 16) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(row) + tid);
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = (int8_t)(ww[k >> 2] >> (8 * (k & 3)));
    } else {
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) v[k] = __ldg(row + tid * Sh::E + k);
    }
  };
  if constexpr (enc_f64<T, LOGN>()) {
    // 64-bit limbs: NTT(u), the products with the public key and the inverse transforms stay in the
    // FP64 domain (the key arrives as centred doubles NTT(pk) N^-1 in the thread-major strip layout,
    // launch_encrypt); integer work only for the draws, Delta * lift(m) and the canonical store.
    const F64Prime P{(double)pr.p, __drcp_rn((double)pr.p)};
    using SV = Strip<T, LOGN>;
#pragma unroll 1
    for (uint32_t b = slot * GROUPS + group; b < batch; b += nslots * GROUPS) {
      const int8_t* drow = draws + (size_t)b * 3 * Sh::N;
      if (ntt_tid<LOGN>() == 0 && b + nslots * GROUPS < batch) {  // next item's inputs towards L2
        const uint32_t nb = b + nslots * GROUPS;
        if (!GATHER) bulk_prefetch_l2(m + (size_t)nb * Sh::N, (uint32_t)(Sh::N * 8));
        bulk_prefetch_l2(draws + (size_t)nb * 3 * Sh::N, (uint32_t)(Sh::N * 3));
      }
      const int32_t* grow = nullptr;
      int64_t gbase = 0;
      if constexpr (GATHER) g.row(b, Sh::N, grow, gbase);
      auto m_at = [&](int k) -> uint64_t {
        if constexpr (GATHER) return g.value(grow, gbase, (uint32_t)(cb + coef_off<LOGN>(k)));
        else return __ldg(m + (size_t)b * Sh::N + cb + coef_off<LOGN>(k));
      };
      double d[Sh::E];
      {
        int8_t u[Sh::E];
        load_draws(drow, u);
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) d[k] = (double)u[k];   // |u| <= 1: any transform input bound holds
      }
      ntt_fwd_f64<T, LOGN, 0, SMEM_TW, CPMUL_NBUF, GROUPS>(d, ex, tw, P);
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) x[k] = (T)__double_as_longlong(f64_center(d[k], P));
      usm.store(x);
#pragma unroll 1
      for (int pi = 0; pi < 2; ++pi) {
        const int part = 1 - pi;   // part 0 last: its plaintext is read before the inverse transform
        uint64_t mv[Sh::E];
        if (part == 0) {
#pragma unroll
          for (int k = 0; k < Sh::E; ++k) mv[k] = m_at(k);
        }
        const T* kp = pkprep + ((size_t)part * L + limb) * Sh::N;
#pragma unroll
        for (int i = 0; i < SV::CHUNKS; ++i) {
          T kv[SV::VEC], uu[SV::VEC];
          unpack_chunk<T>(__ldg(reinterpret_cast<const uint4*>(kp) + i * Sh::THREADS + ntt_tid<LOGN>()), kv);
          usm.load_chunk(i, uu);
#pragma unroll
          for (int c = 0; c < SV::VEC; ++c) {
            const double kd = __longlong_as_double((long long)kv[c]);
            d[i * SV::VEC + c] = f64_mulmod(__longlong_as_double((long long)uu[c]), kd, __dmul_rn(kd, P.pinv), P.p);
          }
        }
        auto delta_m = [&](uint64_t v) -> T {  // Delta * lift(m) mod p
          T l = csub(pr.reduce_u64_lazy(v), pr.p);
          if (v > t_half) l = sub_mod(l, tmod, pr.p);
          return csub(shoup_mul(l, delta, delta_q, pr.p), pr.p);
        };
        auto delta_m_small = [&](uint64_t v) -> T {  // t <= p: m is its own residue (lift_plain_regs)
          const T l = (T)(v > t_half ? v + (uint64_t)(pr.p - tmod) : v);
          return csub(shoup_mul(l, delta, delta_q, pr.p), pr.p);
        };
        if (part == 0) {   // the NTT(u) strip is dead now: park Delta * lift(m) there
          if (plain_fast) {
#pragma unroll
            for (int c = 0; c < SV::CHUNKS; ++c) {
              T dm[SV::VEC];
#pragma unroll
              for (int j = 0; j < SV::VEC; ++j) dm[j] = delta_m_small(mv[c * SV::VEC + j]);
              usm.store_chunk(c, dm);
            }
          } else {
#pragma unroll
          for (int c = 0; c < SV::CHUNKS; ++c) {
            T dm[SV::VEC];
#pragma unroll
            for (int j = 0; j < SV::VEC; ++j) dm[j] = delta_m(mv[c * SV::VEC + j]);
            usm.store_chunk(c, dm);
          }
          }
        }
        int8_t e[Sh::E];  // issued before the inverse transform, consumed after it
        load_draws(drow + (size_t)(1 + part) * Sh::N, e);
        ntt_inv_f64<T, LOGN, Sh::NPASS - 1, SMEM_TW, CPMUL_NBUF, GROUPS>(d, ex, tw, P);   // inputs |.| < p
        T* o = out + (((size_t)b * 2 + part) * L + limb) * Sh::N + cb;
#pragma unroll
        for (int c = 0; c < SV::CHUNKS; ++c) {
          T dm[SV::VEC];
          if (part == 0) usm.load_chunk(c, dm);
#pragma unroll
          for (int j = 0; j < SV::VEC; ++j) {
            const int k = c * SV::VEC + j;
            T v = add_mod((T)f64_to_canon(d[k], P), small(e[k]), pr.p);
            if (part == 0) v = add_mod(v, dm[j], pr.p);
            o[coef_off<LOGN>(k)] = v;
          }
        }
      }
    }
    return;
  }
  for (uint32_t b = slot * GROUPS + group; b < batch; b += nslots * GROUPS) {
    const int8_t* drow = draws + (size_t)b * 3 * Sh::N;
    if (ntt_tid<LOGN>() == 0 && b + nslots * GROUPS < batch) {  // next item's inputs towards L2
      const uint32_t nb = b + nslots * GROUPS;
      if (!GATHER) bulk_prefetch_l2(m + (size_t)nb * Sh::N, (uint32_t)(Sh::N * 8));
      bulk_prefetch_l2(draws + (size_t)nb * 3 * Sh::N, (uint32_t)(Sh::N * 3));
    }
    // the plaintext: packed values, or read through the packing descriptor (pack fused into the
    // encryption: the map row is shared by every polynomial of its kind and stays in L1/L2, and a
    // sparse polynomial -- one 3 x 3 kernel in 4096 degrees -- loads almost no source values)
    const int32_t* grow = nullptr;
    int64_t gbase = 0;
    if constexpr (GATHER) g.row(b, Sh::N, grow, gbase);
    auto m_at = [&](int k) -> uint64_t {
      if constexpr (GATHER) return g.value(grow, gbase, (uint32_t)(cb + coef_off<LOGN>(k)));
      else return __ldg(m + (size_t)b * Sh::N + cb + coef_off<LOGN>(k));
    };
    {
      int8_t u[Sh::E];
      load_draws(drow, u);
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) x[k] = small(u[k]);
    }
    // canonical draws in, and the slotwise products below are canonical too (x < 4p times a
    // canonical prepared key word: Montgomery output in [0, p)): every transform skips the
    // conditional subtractions of its first stage.  RELAX (ntt.cuh Exchanger): the forward transform
    // follows the previous item's inverse, part pi = 0's inverse follows it; only the second
    // inverse follows a transform of its own direction and gets the explicit guard barrier.
    ntt_fwd_regs<T, LOGN, 0, SMEM_TW, CPMUL_NBUF, GROUPS, F64Q_NE, RELAX, true>(x, ex, tw, pr.p, pr.p2);
    usm.store(x);
    // MSTRIP: part 1 first; part 0's plaintext reads are issued before its slotwise product and
    // Delta * lift(m) is parked in the NTT(u) strip (dead after that product) across the inverse
    // transform, instead of reading m after the transform with the whole L2 latency exposed.
#pragma unroll 1
    for (int pi = 0; pi < 2; ++pi) {
      const int part = MSTRIP ? 1 - pi : pi;
      uint64_t mv[MSTRIP ? Sh::E : 1];
      if (MSTRIP && part == 0) {
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) mv[k] = m_at(k);
      }
      const T* kp = pkprep + ((size_t)part * L + limb) * Sh::N;
      static_assert(EV::VEC == Strip<T, LOGN>::VEC || EV::VEC == 1, "strip / eval chunking");
      const Strip<T, LOGN> ks(pk_sm + (size_t)part * Sh::N);
      if constexpr (ENC_XPOSE) {
        // key read with contiguous 16-byte accesses through the exchange image (ntt.cuh)
        eval_xpose_apply<T, LOGN, GROUPS>(kp, gsm, [&](int i, const T* v) {
          T uu[EV::VEC];
          usm.load_chunk(i, uu);
#pragma unroll
          for (int c = 0; c < EV::VEC; ++c) x[i * EV::VEC + c] = mont_mul(uu[c], v[c], pr.p, pr.pinv);
        });
      } else {
#pragma unroll
      for (int i = 0; i < EV::CHUNKS; ++i) {
        T v[EV::VEC];
        if constexpr (PKSM) ks.load_chunk(i, v);
        else if constexpr (enc_pk_strip<T, LOGN>())
          unpack_chunk<T>(__ldg(reinterpret_cast<const uint4*>(kp) + i * Sh::THREADS + ntt_tid<LOGN>()), v);
        else EV::load(kp, i, v);
        if constexpr (EV::VEC == Strip<T, LOGN>::VEC) {
          T uu[EV::VEC];
          usm.load_chunk(i, uu);
#pragma unroll
          for (int c = 0; c < EV::VEC; ++c) {
            if constexpr (F64PW)
              x[i * EV::VEC + c] = (T)f64_pointwise((uint32_t)uu[c], (uint32_t)v[c], __uint2double_rn((uint32_t)v[c]), pinv_d,
                                                    (uint32_t)pr.p, 0u - (uint32_t)pr.p);
            else
              x[i * EV::VEC + c] = mont_mul(uu[c], v[c], pr.p, pr.pinv);
          }
        } else {
          T uu[Strip<T, LOGN>::VEC];
          usm.load_chunk(i / Strip<T, LOGN>::VEC, uu);
          x[i] = mont_mul(uu[i % Strip<T, LOGN>::VEC], v[0], pr.p, pr.pinv);
        }
      }
      }
      auto delta_m = [&](uint64_t v) -> T {  // Delta * lift(m) mod p
        T l = csub(pr.reduce_u64_lazy(v), pr.p);
        if (v > t_half) l = sub_mod(l, tmod, pr.p);
        return csub(shoup_mul(l, delta, delta_q, pr.p), pr.p);
      };
      // 32-bit limbs, t < 2^57, p > 2^25 (lift_plain_regs): the lift lazily below 4p with one Shoup
      // product -- the product by Delta takes any 32-bit operand
      auto delta_m_fast = [&](uint64_t v) -> T {
        const uint32_t hi = (uint32_t)(v >> 25), lo = (uint32_t)v & ((1u << 25) - 1);
        const T l = (T)(shoup_mul<uint32_t>(hi, (uint32_t)pr.c25, (uint32_t)pr.c25_q, (uint32_t)pr.p) + lo +
                        (v > t_half ? (uint32_t)(pr.p - tmod) : 0u));
        return csub(shoup_mul(l, delta, delta_q, pr.p), pr.p);
      };
      if (MSTRIP && part == 0) {
        Strip<T, LOGN> dsm = usm;
#pragma unroll
        for (int c = 0; c < Strip<T, LOGN>::CHUNKS; ++c) {
          T d[Strip<T, LOGN>::VEC];
#pragma unroll
          for (int j = 0; j < Strip<T, LOGN>::VEC; ++j) d[j] = delta_m(mv[c * Strip<T, LOGN>::VEC + j]);
          dsm.store_chunk(c, d);
        }
      }
      int8_t e[Sh::E];  // issued before the inverse transform, consumed after it
      load_draws(drow + (size_t)(1 + part) * Sh::N, e);
      if (RELAX && pi == 1) group_sync<LOGN, GROUPS>();
      ntt_inv_regs<T, LOGN, Sh::NPASS - 1, SMEM_TW, CPMUL_NBUF, GROUPS, F64Q_NE, RELAX, KEY_CANON>(x, ex, tw, pr.p, pr.p2);
      T* o = out + (((size_t)b * 2 + part) * L + limb) * Sh::N + cb;
      if (sizeof(T) == 4 && !MSTRIP && part == 0 && plain_fast) {
#pragma unroll
        for (int k = 0; k < Sh::E; ++k) {
          T v = add_mod(csub(x[k], pr.p), small(e[k]), pr.p);
          o[coef_off<LOGN>(k)] = add_mod(v, delta_m_fast(m_at(k)), pr.p);
        }
      } else {
#pragma unroll
      for (int c = 0; c < Strip<T, LOGN>::CHUNKS; ++c) {
        T d[Strip<T, LOGN>::VEC];
        if (MSTRIP && part == 0) usm.load_chunk(c, d);
#pragma unroll
        for (int j = 0; j < Strip<T, LOGN>::VEC; ++j) {
          const int k = c * Strip<T, LOGN>::VEC + j;
          T v = add_mod(csub(x[k], pr.p), small(e[k]), pr.p);
          if (part == 0) v = add_mod(v, MSTRIP ? d[j] : delta_m(m_at(k)), pr.p);
          o[coef_off<LOGN>(k)] = v;
        }
      }
      }
    }
  }
}

// PPMul in the plain ring Z_t[x]/(x^N+1), t = t0 (* t1): per-prime NTT
// product then the 2-prime CRT of ring._crt_combine (ring.py:478-485).
template <int LOGN>
__device__ __forceinline__ void plain_prime_product(const uint64_t* a, const uint64_t* b,
                                                    const PrimeTab<uint32_t>* tab,
                                                    Exchanger<uint32_t, LOGN>& ex,
                                                    uint32_t (&x)[NttShape<LOGN>::E]) {
  using Sh = NttShape<LOGN>;
  PrimeRegs<uint32_t> pr(tab);
  uint32_t y[Sh::E];
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) y[k] = csub(pr.reduce_u64_lazy(__ldg(b + coef_base<LOGN>() + coef_off<LOGN>(k))), pr.p);
  ntt_fwd_regs<uint32_t, LOGN>(y, ex, pr.fwd, pr.p, pr.p2);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) y[k] = shoup_mul(y[k], pr.ninvr, pr.ninvr_q, pr.p);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) x[k] = csub(pr.reduce_u64_lazy(__ldg(a + coef_base<LOGN>() + coef_off<LOGN>(k))), pr.p);
  ntt_fwd_regs<uint32_t, LOGN>(x, ex, pr.fwd, pr.p, pr.p2);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) x[k] = mont_mul(x[k], y[k], pr.p, pr.pinv);
  ntt_inv_regs<uint32_t, LOGN>(x, ex, pr.inv, pr.p, pr.p2);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) x[k] = csub(x[k], pr.p);
}

template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS, NttShape<LOGN>::MINB)
k_pp_mul(const uint64_t* a, const uint64_t* b, uint64_t* out, const PrimeTab<uint32_t>* __restrict__ tabs,
         int LT, uint32_t c_inv, uint32_t c_inv_q) {
  using Sh = NttShape<LOGN>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Exchanger<uint32_t, LOGN> ex{reinterpret_cast<uint32_t*>(smem_raw)};
  const size_t off = (size_t)blockIdx.x * Sh::N;
  uint32_t r0[Sh::E];
  plain_prime_product<LOGN>(a + off, b + off, tabs, ex, r0);
  if (LT == 1) {
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) out[off + coef_base<LOGN>() + coef_off<LOGN>(k)] = r0[k];
    return;
  }
  uint32_t r1[Sh::E];
  plain_prime_product<LOGN>(a + off, b + off, tabs + 1, ex, r1);
  const uint32_t p0 = tabs[0].p;
  PrimeRegs<uint32_t> p1(tabs + 1);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) {
    const uint32_t r0m = csub(p1.reduce_u64_lazy(r0[k]), p1.p);
    const uint32_t d = csub(shoup_mul(sub_mod(r1[k], r0m, p1.p), c_inv, c_inv_q, p1.p), p1.p);
    out[off + coef_base<LOGN>() + coef_off<LOGN>(k)] = (uint64_t)r0[k] + (uint64_t)p0 * d;
  }
}

}  // namespace ctb

// ---------------------------------------------------------------------------
// C-ABI entry points (declared in include/ctb200.h)
// ---------------------------------------------------------------------------
using namespace ctb;

static inline const Base* base_of(const ctb_ctx_t* ctx, int base) {
  if (!ctx || base < 0 || base >= BASE_COUNT) return nullptr;
  const Base* b = &reinterpret_cast<const Ctx*>(ctx)->base[base];
  return b->size() ? b : nullptr;
}

extern "C" int ctb_ntt_forward(const ctb_ctx_t* ctx, int base, const void* in, void* out,
                               uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, base);
  if (!b || !in || !out) { set_error("ctb_ntt_forward: bad context, base or buffer"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::Fwd>(b, sargs<uint32_t>(in, out), n_polys, s)));
  } else {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::Fwd>(b, sargs<uint64_t>(in, out), n_polys, s)));
  }
  return cuda_status(e, "ctb_ntt_forward");
}

extern "C" int ctb_ntt_inverse(const ctb_ctx_t* ctx, int base, const void* in, void* out,
                               uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, base);
  if (!b || !in || !out) { set_error("ctb_ntt_inverse: bad context, base or buffer"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::Inv>(b, sargs<uint32_t>(in, out), n_polys, s)));
  } else {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::Inv>(b, sargs<uint64_t>(in, out), n_polys, s)));
  }
  return cuda_status(e, "ctb_ntt_inverse");
}

extern "C" int ctb_eval_addend(const ctb_ctx_t* ctx, int base, const void* in, void* out, uint64_t n_polys,
                               void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, base);
  if (!b || !in || !out) { set_error("ctb_eval_addend: bad context, base or buffer"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::FwdNinv>(b, sargs<uint32_t>(in, out), n_polys, s)));
  } else {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::FwdNinv>(b, sargs<uint64_t>(in, out), n_polys, s)));
  }
  return cuda_status(e, "ctb_eval_addend");
}

extern "C" int ctb_linear_addend(const ctb_ctx_t* ctx, int base, const void* in, void* out, uint64_t n_polys,
                                 void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, base);
  if (!b || !in || !out) { set_error("ctb_linear_addend: bad context, base or buffer"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    auto a = sargs<uint32_t>(in, out);
    a.strip_out = true;
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::FwdNinv>(b, a, n_polys, s)));
  } else {
    auto a = sargs<uint64_t>(in, out);
    a.strip_out = true;
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::FwdNinv>(b, a, n_polys, s)));
  }
  return cuda_status(e, "ctb_linear_addend");
}

extern "C" int ctb_prepare_operand(const ctb_ctx_t* ctx, int base, const void* in, void* out, uint64_t n_polys,
                                   void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, base);
  if (!b || !in || !out) { set_error("ctb_prepare_operand: bad context, base or buffer"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::Prepare>(b, sargs<uint32_t>(in, out), n_polys, s)));
  } else {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::Prepare>(b, sargs<uint64_t>(in, out), n_polys, s)));
  }
  return cuda_status(e, "ctb_prepare_operand");
}

// MulPrepared; a broadcast prepared operand (b_stride 0: a key multiplying every item, e.g. the
// secret key of decryption) is first converted into the thread-major chunk layout (pool temporary,
// L polynomials) so every item reads it with contiguous warp loads.
template <typename T, int LOGN>
static cudaError_t launch_mul_prepared(const Ctx* c, const Base* b, StreamArgs<T> a, uint64_t npoly, cudaStream_t s) {
  using Sh = NttShape<LOGN>;
  using EV = EvalVec<T, LOGN>;
  void* tmp = nullptr;
  if constexpr (EV::CONTIG && EV::VEC * sizeof(T) == 16 && CTB_EVAL_XPOSE) {
    if (a.b_stride == 0 && npoly > 1) {
      const size_t bytes = (size_t)b->size() * Sh::N * sizeof(T);
      cudaError_t e = c->pool ? cudaMallocFromPoolAsync(&tmp, bytes, c->pool, s) : cudaMallocAsync(&tmp, bytes, s);
      if (e != cudaSuccess) return e;
      k_eval_to_strip<T, LOGN><<<(unsigned)b->size(), Sh::THREADS, 0, s>>>(a.bprep, (T*)tmp, nullptr, 1);
      if ((e = cudaGetLastError()) != cudaSuccess) { cudaFreeAsync(tmp, s); return e; }
      a.bprep = (const T*)tmp;
      a.bprep_strip = true;
    }
  }
  cudaError_t e = launch_stream<T, LOGN, StreamOp::MulPrepared>(b, a, npoly, s);
  if (tmp) {
    const cudaError_t f = cudaFreeAsync(tmp, s);
    if (e == cudaSuccess) e = f;
  }
  return e;
}

extern "C" int ctb_mul_prepared_strided(const ctb_ctx_t* ctx, int base, const void* a, uint64_t a_stride,
                                        const void* bprep, uint64_t b_stride, const void* addend,
                                        uint64_t add_stride, void* out, uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, base);
  if (!b || !a || !bprep || !out || a_stride == 0 || (addend && add_stride == 0)) {
    set_error("ctb_mul_prepared: bad context, base, buffer or stride");
    return ERR_ARG;
  }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_mul_prepared<uint32_t, LOGN>(c, b, sargs<uint32_t>(a, out, bprep, b_stride, addend, a_stride, add_stride), n_polys, s)));
  } else {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_mul_prepared<uint64_t, LOGN>(c, b, sargs<uint64_t>(a, out, bprep, b_stride, addend, a_stride, add_stride), n_polys, s)));
  }
  return cuda_status(e, "ctb_mul_prepared");
}

extern "C" int ctb_mul_prepared(const ctb_ctx_t* ctx, int base, const void* a, const void* bprep, uint64_t b_stride,
                                const void* addend, void* out, uint64_t n_polys, void* stream) {
  return ctb_mul_prepared_strided(ctx, base, a, 1, bprep, b_stride, addend, 1, out, n_polys, stream);
}

cudaError_t ctb::stream_lift(const Ctx* c, int base, bool prepare, const uint64_t* m, void* out, uint64_t npoly,
                             cudaStream_t s, bool strip_out) {
  const Base* b = &c->base[base];
  // the plain base needs no centring: t = 0 mod t_j
  const uint64_t t_half = base == BASE_Q ? c->t_half : ~0ull;
  const bool fast = base == BASE_Q && c->plain_fast;
  cudaError_t e = cudaSuccess;
  if (b->word == 4) {
    StreamArgs<uint32_t> a = sargs<uint32_t>(nullptr, out);
    a.plain = m; a.t_half = t_half; a.plain_fast = fast; a.strip_out = strip_out;
    if (prepare) CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::LiftPrepare>(b, a, npoly, s)))
    else CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint32_t, LOGN, StreamOp::LiftFwd>(b, a, npoly, s)))
  } else {
    StreamArgs<uint64_t> a = sargs<uint64_t>(nullptr, out);
    a.plain = m; a.t_half = t_half; a.plain_fast = fast; a.strip_out = strip_out;
    if (prepare) CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::LiftPrepare>(b, a, npoly, s)))
    else CTB_DISPATCH_LOGN_E(c->logn, e = (launch_stream<uint64_t, LOGN, StreamOp::LiftFwd>(b, a, npoly, s)))
  }
  return e;
}

extern "C" int ctb_pointwise_mul(const ctb_ctx_t* ctx, int base, const void* a, const void* bb, void* out,
                                 uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, base);
  if (!b || !a || !bb || !out) { set_error("ctb_pointwise_mul: bad context, base or buffer"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  const uint64_t total = n_polys * b->size() * (uint64_t)c->n;
  if (!total) return OK;
  const unsigned grid = grid_stride(total, 16);  // SM count of the current device x 16 CTAs
  cudaStream_t s = (cudaStream_t)stream;
  if (b->word == 4)
    k_pointwise<uint32_t><<<grid, 256, 0, s>>>((const uint32_t*)a, (const uint32_t*)bb, (uint32_t*)out,
                                               (const PrimeTab<uint32_t>*)b->d_tabs, b->size(), c->n, total);
  else
    k_pointwise<uint64_t><<<grid, 256, 0, s>>>((const uint64_t*)a, (const uint64_t*)bb, (uint64_t*)out,
                                               (const PrimeTab<uint64_t>*)b->d_tabs, b->size(), c->n, total);
  return cuda_status(cudaGetLastError(), "ctb_pointwise_mul");
}

extern "C" int ctb_ring_mul(const ctb_ctx_t* ctx, int base, const void* a, uint64_t a_stride, const void* bb,
                            uint64_t b_stride, void* out, uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, base);
  if (!b || !a || !bb || !out) { set_error("ctb_ring_mul: bad context, base or buffer"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  const size_t nblk = n_polys * b->size();
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    using T = uint32_t;
    CTB_DISPATCH_LOGN(c->logn, e = (launch_ntt_kernel<T, LOGN>(k_ring_mul<T, LOGN>, nblk, s, (const T*)a, a_stride,
                                                      (const T*)bb, b_stride, (T*)out,
                                                      (const PrimeTab<T>*)b->d_tabs, b->size())));
  } else {
    using T = uint64_t;
    CTB_DISPATCH_LOGN(c->logn, e = (launch_ntt_kernel<T, LOGN>(k_ring_mul<T, LOGN>, nblk, s, (const T*)a, a_stride,
                                                      (const T*)bb, b_stride, (T*)out,
                                                      (const PrimeTab<T>*)b->d_tabs, b->size())));
  }
  return cuda_status(e, "ctb_ring_mul");
}

template <typename T, int LOGN>
static cudaError_t launch_cpmul(const Ctx* c, const Base* b, const void* ct, const uint64_t* pt, void* out,
                                uint64_t batch, cudaStream_t s) {
  using Sh = NttShape<LOGN>;
  // twiddles in shared memory when the table fits beside the exchange image
  constexpr int GROUPS = cpmul_kernel_groups<T, LOGN>();
  constexpr size_t tw_bytes = (size_t)tw_words<T>(LOGN) * sizeof(T);
  constexpr size_t group_bytes = ((size_t)Exchanger<T, LOGN, cpmul_kernel_nbuf<T, LOGN>(), GROUPS>::WORDS + Sh::N) * sizeof(T);
  constexpr bool SMEM_TW = LOGN >= 9 && tw_bytes + GROUPS * group_bytes <= (sizeof(T) == 4 ? 224 : 226) * 1024;
  auto kern = k_cpmul<T, LOGN, SMEM_TW>;
  const size_t smem = GROUPS * group_bytes + (SMEM_TW ? tw_bytes : 0);
  const int L = b->size();
  const uint64_t items = batch * (uint64_t)L;
  if (items == 0) return cudaSuccess;
  const int threads = Sh::THREADS * GROUPS;
  uint32_t grid = persistent_grid((const void*)kern, threads, smem);
  const uint64_t max_grid = (batch + GROUPS - 1) / GROUPS * (uint64_t)L;
  grid = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(grid / L * L, (uint64_t)L), max_grid);
  return launch_kernel_grid(kern, grid, threads, smem, s, (const T*)ct, pt, (T*)out,
                            (const PrimeTab<T>*)b->d_tabs, L, c->t_half, (uint32_t)batch, c->plain_fast);
}

extern "C" int ctb_cpmul(const ctb_ctx_t* ctx, const void* ct, const uint64_t* pt, void* out, uint64_t batch,
                         void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, BASE_Q);
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!b || !c->t || !ct || !pt || !out) { set_error("ctb_cpmul: bad context (needs cipher+plain ring) or buffer"); return ERR_ARG; }
  if (batch >= (1ull << 32)) { set_error("ctb_cpmul: batch too large"); return ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_cpmul<uint32_t, LOGN>(c, b, ct, pt, out, batch, s)));
  } else {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_cpmul<uint64_t, LOGN>(c, b, ct, pt, out, batch, s)));
  }
  return cuda_status(e, "ctb_cpmul");
}

template <typename T, int LOGN>
static cudaError_t launch_encrypt(const Ctx* c, const Base* b, const uint64_t* m, const int8_t* draws,
                                  const void* pkprep, void* out, uint64_t batch, cudaStream_t s,
                                  const PlainGather& g) {
  using Sh = NttShape<LOGN>;
  constexpr int GROUPS = enc_groups<T, LOGN>();
  constexpr size_t tw_bytes = (size_t)tw_words<T>(LOGN) * sizeof(T);
  constexpr size_t group_bytes = ((size_t)Exchanger<T, LOGN, CPMUL_NBUF, GROUPS>::WORDS + Sh::N) * sizeof(T);
  constexpr bool SMEM_TW = LOGN >= 9 && tw_bytes + GROUPS * group_bytes <= (sizeof(T) == 4 ? 200 : 226) * 1024;
  constexpr size_t pk_bytes = enc_pk_smem<T, LOGN>() && SMEM_TW ? 2 * (size_t)Sh::N * sizeof(T) : 0;
  static_assert((SMEM_TW ? tw_bytes : 0) + GROUPS * group_bytes + pk_bytes <= 227 * 1024, "k_encrypt shared memory");
  auto kern = g.maps ? k_encrypt<T, LOGN, SMEM_TW, true> : k_encrypt<T, LOGN, SMEM_TW, false>;
  const size_t smem = GROUPS * group_bytes + (SMEM_TW ? tw_bytes : 0) + pk_bytes;
  const int L = b->size();
  if (batch == 0) return cudaSuccess;
  const int threads = Sh::THREADS * GROUPS;
  const void* pk = pkprep;
  void* tmp = nullptr;
  if constexpr (enc_pk_strip<T, LOGN>()) {
    cudaError_t e = c->pool ? cudaMallocFromPoolAsync(&tmp, 2 * (size_t)L * Sh::N * sizeof(T), c->pool, s)
                            : cudaMallocAsync(&tmp, 2 * (size_t)L * Sh::N * sizeof(T), s);
    if (e != cudaSuccess) return e;
    // (64-bit limbs: also out of the Montgomery domain into centred doubles for the FP64 products)
    k_eval_to_strip<T, LOGN, enc_f64<T, LOGN>()><<<(unsigned)(2 * L), Sh::THREADS, 0, s>>>(
        (const T*)pkprep, (T*)tmp, (const PrimeTab<T>*)b->d_tabs, L);
    if ((e = cudaGetLastError()) != cudaSuccess) { cudaFreeAsync(tmp, s); return e; }
    pk = tmp;
  }
  uint32_t grid = persistent_grid((const void*)kern, threads, smem);
  const uint64_t max_grid = (batch + GROUPS - 1) / GROUPS * (uint64_t)L;
  grid = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(grid / L * L, (uint64_t)L), max_grid);
  cudaError_t e = launch_kernel_grid(kern, grid, threads, smem, s, m, draws, (const T*)pk, (T*)out,
                                     (const PrimeTab<T>*)b->d_tabs, L, c->t_half, (uint32_t)batch, c->plain_fast, g);
  if (tmp) {
    const cudaError_t f = cudaFreeAsync(tmp, s);
    if (e == cudaSuccess) e = f;
  }
  return e;
}

extern "C" int ctb_encrypt(const ctb_ctx_t* ctx, const uint64_t* m, const int8_t* draws, const void* pkprep,
                           void* out, uint64_t batch, void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, BASE_Q);
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!b || !c->t || !m || !draws || !pkprep || !out) { set_error("ctb_encrypt: bad context (needs plain ring) or buffer"); return ERR_ARG; }
  if (batch >= (1ull << 32)) { set_error("ctb_encrypt: batch too large"); return ERR_ARG; }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  const PlainGather g{};
  if (b->word == 4) {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_encrypt<uint32_t, LOGN>(c, b, m, draws, pkprep, out, batch, s, g)));
  } else {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_encrypt<uint64_t, LOGN>(c, b, m, draws, pkprep, out, batch, s, g)));
  }
  return cuda_status(e, "ctb_encrypt");
}

extern "C" int ctb_encrypt_gather(const ctb_ctx_t* ctx, const int64_t* src, uint64_t src_len, const int32_t* maps,
                                  uint32_t n_maps, const int32_t* kind, const int64_t* base, const int8_t* draws,
                                  const void* pkprep, void* out, uint64_t batch, void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, BASE_Q);
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!b || !c->t || (src_len && !src) || !maps || !kind || !base || !draws || !pkprep || !out) {
    set_error("ctb_encrypt_gather: bad context (needs plain ring) or buffer");
    return ERR_ARG;
  }
  if (batch >= (1ull << 32)) { set_error("ctb_encrypt_gather: batch too large"); return ERR_ARG; }
  PlainGather g;
  g.src = src;
  g.src_len = src_len;
  g.maps = maps;
  g.n_maps = n_maps;
  g.kind = kind;
  g.base = base;
  g.t = c->t;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (b->word == 4) {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_encrypt<uint32_t, LOGN>(c, b, nullptr, draws, pkprep, out, batch, s, g)));
  } else {
    CTB_DISPATCH_LOGN(c->logn, e = (launch_encrypt<uint64_t, LOGN>(c, b, nullptr, draws, pkprep, out, batch, s, g)));
  }
  return cuda_status(e, "ctb_encrypt_gather");
}

extern "C" int ctb_pp_mul(const ctb_ctx_t* ctx, const uint64_t* a, const uint64_t* bb, uint64_t* out,
                          uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* b = base_of(ctx, BASE_T);
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!b || !a || !bb || !out) { set_error("ctb_pp_mul: context has no plain ring or bad buffer"); return ERR_ARG; }
  if (b->word != 4 || b->size() > 2) { set_error("ctb_pp_mul: plain ring must be 1-2 primes below 2^30"); return ERR_UNSUPPORTED; }
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  CTB_DISPATCH_LOGN(c->logn, e = (launch_ntt_kernel<uint32_t, LOGN>(k_pp_mul<LOGN>, n_polys, s, a, bb, out,
                                                           (const PrimeTab<uint32_t>*)b->d_tabs, b->size(),
                                                           c->crt_inv, c->crt_inv_q)));
  return cuda_status(e, "ctb_pp_mul");
}

