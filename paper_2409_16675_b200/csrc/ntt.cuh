// CTA-resident negacyclic NTT over one RNS limb of one polynomial.
//
// Mathematical contract (identical to the reference, ring.py:164-217):
//   forward: out[k] = a(psi^(2*bitrev_logN(k)+1)) mod p, i.e. the in-place
//            Cooley-Tukey pass over the twiddle table w[i] = psi^bitrev(i),
//            natural order in, bit-reversed order out, canonical [0, p);
//   inverse: the exact inverse map, canonical [0, p).
// psi is chosen exactly as ring._find_root_of_unity (ring.py:93-102), so the
// evaluation-domain layout is bit-identical to ring.ntt_forward.
//
// Execution model (B200, sm_100a): one CTA owns one (polynomial, limb).  Each
// of THREADS threads keeps E = N/THREADS residues in registers; the logN
// butterfly stages are grouped into passes of up to log2(E) stages that run
// entirely in registers (radix-2^r butterfly networks), and consecutive passes
// exchange data through an XOR-swizzled shared-memory image of the polynomial
// (bank-conflict-free for every pass layout: tools/swizzle_check.py).  The
// first pass reads coalesced from HBM (thread t owns t + j*THREADS) and the
// last forward pass leaves each thread 2^r contiguous evaluation slots, which
// is exactly the layout the first inverse pass needs, so a pointwise product
// between a forward and an inverse transform costs no data movement.
#pragma once
#include <cstdint>
#include "modarith.cuh"

namespace ctb {

// Per-prime constant block (device memory, read-only after ctx creation).
template <typename T>
struct PrimeTab {
  T p, p2, pinv;        // p, 2p, p^-1 mod 2^W
  T ninv, ninv_q;       // N^-1 mod p and its Shoup quotient
  T ninvr, ninvr_q;     // N^-1 * 2^W mod p (enters the Montgomery domain, 1/N folded)
  T one_q;              // floor(2^W / p): Shoup quotient of w = 1 (generic reduction)
  T r2, r2_q;           // 2^W mod p (u32: splitting 64-bit inputs) and Shoup quotient
  T rr;                 // 2^(2W) mod p (leaves the Montgomery domain)
  T tmod;               // plain modulus t mod p (cipher base only: centred lift)
  T delta, delta_q;     // floor(q/t) mod p and Shoup quotient (cipher base only)
  T c25, c25_q;         // 2^25 mod p and Shoup quotient (u32, p > 2^25): one-multiply plain reduction
  double dp, dpinv;     // p and 1/p as doubles (64-bit limbs: FP64 butterflies)
  const T* fwd;         // (w, w') pairs, pass-major / entry-major (see TwSrc); serves both directions
                        // (64-bit limbs: the bits of (double w, double w/p))
  const T* inv;         // == fwd (kept for layout stability)
};

// Pass schedule of the CTA transform, as runtime-capable constexpr functions
// so the host table builder (ctx.cu) and the device code agree exactly.
__host__ __device__ constexpr int shape_loge(int logn) { return logn >= 9 ? 4 : (logn >= 6 ? logn - 5 : 1); }
__host__ __device__ constexpr int shape_npass(int logn) { return (logn + shape_loge(logn) - 1) / shape_loge(logn); }
__host__ __device__ constexpr int shape_first_r(int logn) { return logn - (shape_npass(logn) - 1) * shape_loge(logn); }
__host__ __device__ constexpr int shape_pass_s(int logn, int k) { return k == 0 ? 0 : shape_first_r(logn) + (k - 1) * shape_loge(logn); }
__host__ __device__ constexpr int shape_pass_r(int logn, int k) { return k == 0 ? shape_first_r(logn) : shape_loge(logn); }
// Twiddles are stored pass-major: pass k, butterfly group B (2^s groups) owns
// 2^r consecutive (w, w') entries, entry (2^i - 1) + jb serving stage s+i,
// block jb -- one base pointer per pass and group, immediate offsets inside.
__host__ __device__ constexpr int shape_tw_off(int logn, int k) {
  int off = 0;
  for (int q = 0; q < k; ++q) off += 1 << (shape_pass_s(logn, q) + shape_pass_r(logn, q));
  return off;
}
__host__ __device__ constexpr int shape_tw_entries(int logn) { return shape_tw_off(logn, shape_npass(logn)); }
// 32-bit limbs: (w, w') pair index of entry e (= 2^i - 1 + jb) of group slot `slot` in pass k.
// Entries e and e + 1 with e odd (blocks jb, jb + 1 of one stage) are adjacent, so the passes read
// two entries per 128-bit load, conflict-free for consecutive slots; entry 0 is the second half of
// pair 0 (whose first half is unused).  64-bit limbs keep one word per entry at (e << s) + slot.
__host__ __device__ constexpr int shape_tw_pair(int logn, int k, int e, int slot) {
  return shape_tw_off(logn, k) + ((((e + 1) >> 1) << shape_pass_s(logn, k)) + slot) * 2 + ((e + 1) & 1);
}
// FP64-quotient butterflies (32-bit limbs).  The Shoup product a*w mod p costs IMAD.HI + 2 IMAD,
// all on the fma-heavy pipe (IMAD.HI at half rate), which is what bounds the transforms.  For the
// twiddle entries e < F64Q_NE of every pass (e = 2^i - 1 + jb: stage 0 and the first block of
// stage 1, 12 of the 32 butterflies of a radix-16 pass) the quotient comes from the otherwise idle
// FP64 pipe instead: one DFMA on the exponent-spliced double 2^52 + a gives rint(a * w'/p) with
// w'/p = round(w 2^52 / p) 2^-52 (|error| < 2^-21 for a < 2^32, so the quotient is floor or ceil of
// a*w/p), and a*w + p - q*p in (0, 2p) takes 2 IMAD -- the Shoup output range.  Measured register
// resident on this B200 (tools/probe/imad_probe.cu): Shoup 4.63 T/s, FP64-quotient 6.79 T/s.
// The quotients live in a second table after the (w, w') pairs: one double w'/p per entry,
// pass-major, [e][group slot] inside a pass.  -DCTB_F64Q_ENTRIES=0 restores pure Shoup.
#ifndef CTB_F64Q_ENTRIES
#define CTB_F64Q_ENTRIES 2
#endif
constexpr int F64Q_NE = CTB_F64Q_ENTRIES;
__host__ __device__ constexpr int shape_q_off(int logn, int k) {
  int off = 0;
  for (int q = 0; q < k; ++q) off += F64Q_NE << shape_pass_s(logn, q);
  return off;
}
// index of the FP64 quotient of entry e (< F64Q_NE): slot-major, a slot's entries adjacent
__host__ __device__ constexpr int shape_q_index(int logn, int k, int e, int slot) {
  return shape_q_off(logn, k) + slot * F64Q_NE + e;
}
// doubles in the quotient table, rounded up to a 16-byte multiple
__host__ __device__ constexpr int shape_q_entries(int logn) { return (shape_q_off(logn, shape_npass(logn)) + 1) & ~1; }
// Words per prime in the twiddle table: (w, w') pairs (+ the FP64 quotient table) for 32-bit
// limbs; one double w per entry for 64-bit limbs (the FP64 butterflies derive w/p as w * (1/p),
// see the f64 section below).
// (32-bit limbs: rounded up to 128 bytes, so the exchange images that follow a staged table keep
// the 128-byte alignment the warp-local exchange's XORed addresses need)
template <typename T>
__host__ __device__ constexpr int tw_words(int logn) {
  return sizeof(T) == 4 ? (2 * shape_tw_entries(logn) + 2 * shape_q_entries(logn) + 31) / 32 * 32 : shape_tw_entries(logn);
}

template <int LOGN>
struct NttShape {
  static constexpr int N = 1 << LOGN;
  static constexpr int LOGE = shape_loge(LOGN);
  static constexpr int E = 1 << LOGE;
  static constexpr int THREADS = N / E;
  // resident CTAs per SM the register allocation is capped for
  static constexpr int MINB = THREADS >= 512 ? 1 : (THREADS >= 256 ? 2 : 4);
  static constexpr int NPASS = shape_npass(LOGN);
  static constexpr int FIRST_R = shape_first_r(LOGN);
  __host__ __device__ static constexpr int pass_s(int k) { return shape_pass_s(LOGN, k); }
  __host__ __device__ static constexpr int pass_r(int k) { return shape_pass_r(LOGN, k); }
  __host__ __device__ static constexpr int tw_off(int k) { return shape_tw_off(LOGN, k); }
};

// Thread index inside the transform's thread group.  Kernels that run several
// independent transforms per CTA (one per group of THREADS threads) get the
// lane of the group; for one transform per CTA this is threadIdx.x.
template <int LOGN>
__device__ __forceinline__ int ntt_tid() {
  return (int)(threadIdx.x & (NttShape<LOGN>::THREADS - 1));
}

// Shared-memory image of a polynomial: element idx lives at word
// phys(idx) = sum over set bits b of idx of WEIGHT[b].  The weights are
// 2^b plus a little padding chosen so that, in every pass layout, the 32
// lanes of a warp (16 for 64-bit words) hit distinct banks
// (tools/swizzle_check.py proves it for every supported N >= 1024).  Because
// phys is additive over disjoint bit sets and the thread part and slot part of
// a pass index occupy disjoint bits, every access is [thread base + immediate].
template <typename T>
__host__ __device__ constexpr int smem_weight(int logn, int b) {
  constexpr int W32[14] = {1, 2, 4, 8, 16, 33, 66, 132, 272, 552, 1088, 2176, 4352, 8704};
  constexpr int W64[14] = {1, 2, 4, 8, 16, 33, 66, 132, 264, 528, 1056, 2112, 4224, 8448};
  return logn < 9 ? (1 << b) : (sizeof(T) == 4 ? W32[b] : W64[b]);
}

template <typename T, int LOGN>
__host__ __device__ constexpr int phys(int idx) {
  int r = 0;
  for (int b = 0; b < LOGN; ++b) r += ((idx >> b) & 1) * smem_weight<T>(LOGN, b);
  return r;
}

template <typename T, int LOGN>
struct SmemImage;

// Vectorised exchange maps (32-bit words, N = 4096: three radix-16 passes starting at stages 0,
// 4 and 8).  Each exchange gets its own additive map, chosen so that one side of it moves several
// consecutive slots per instruction and both sides stay bank-conflict-free
// (tools/swizzle_check.py --vector proves both):
//   map 1, passes 0 <-> 1: index bit 8 (pass 0's lowest slot bit) has weight 1, so pass 0 moves
//          slot pairs with 64-bit accesses; pass 1's lanes (index bits 0-3, 8) cover 32 banks;
//   map 2, passes 1 <-> 2: index bits 0-3 (pass 2's slots) have weights 1, 2, 4, 8, so pass 2
//          moves its 16 contiguous slots as four 128-bit accesses; the quarter-warp phases of
//          pass 2 (index bits 5-7) land on distinct 16-byte bank groups.
// One exchange then costs 24 (map 1) or 20 (map 2) shared-memory instructions per thread
// instead of 32.  Map 0 is the generic scalar layout (smem_weight).
template <typename T, int LOGN, int MAP>
__host__ __device__ constexpr int phys_map(int idx) {
  constexpr int M1[12] = {2, 4, 8, 16, 32, 64, 128, 256, 1, 512, 1024, 2048};
  constexpr int M2[12] = {1, 2, 4, 8, 16, 36, 72, 144, 304, 588, 1176, 2352};
  if constexpr (MAP == 0) {
    return phys<T, LOGN>(idx);
  } else {
    int r = 0;
    for (int b = 0; b < LOGN; ++b) r += ((idx >> b) & 1) * (MAP == 1 ? M1[b] : M2[b]);
    return r;
  }
}
template <typename T, int LOGN>
__host__ __device__ constexpr bool vec_exchange() { return sizeof(T) == 4 && LOGN == 12; }
// -DCTB_WARP_EXCHANGE=0 restores the group-wide map-2 exchange (A/B: tools/ab_variants.py)
#ifndef CTB_WARP_EXCHANGE
#define CTB_WARP_EXCHANGE 1
#endif
constexpr bool WARP_EXCHANGE = CTB_WARP_EXCHANGE;
// map of the exchange between the passes starting at stages SA and SB
template <typename T, int LOGN, int SA, int SB>
__host__ __device__ constexpr int exchange_map() {
  if constexpr (!vec_exchange<T, LOGN>()) return 0;
  else return (SA + SB == 4) ? 1 : (SA + SB == 12 ? 2 : 0);
}
// words per access on the side of pass S in map MAP
template <int MAP, int S>
__host__ __device__ constexpr int exchange_vec() { return MAP == 1 && S == 0 ? 2 : (MAP == 2 && S == 8 ? 4 : 1); }

template <typename T, int LOGN>
struct SmemImage {
  // vectorised exchanges: map 1 fills exactly N words and the warp-local exchange lives inside it
  static constexpr int RAW = vec_exchange<T, LOGN>() ? (WARP_EXCHANGE ? (1 << LOGN) : phys_map<T, LOGN, 2>((1 << LOGN) - 1) + 1)
                                                     : phys<T, LOGN>((1 << LOGN) - 1) + 1;
  // rounded to 16 bytes: whatever follows an image (strips, staging) is vector-accessed
  static constexpr int WORDS = (RAW + 16 / (int)sizeof(T) - 1) / (16 / (int)sizeof(T)) * (16 / (int)sizeof(T));
};

// Thread -> group permutation of a pass: the last pass of N >= 1024 rotates the
// low six thread bits so its lanes avoid the bank of the middle passes.
template <int LOGN, bool LAST>
__host__ __device__ constexpr int pass_thread(int t) {
  // N = 4096 rotates only the low five bits, so a warp's blocks in the last pass are the same 32
  // blocks (index bits 9-11 = warp) it owns in the middle pass: the exchange between those two
  // passes never leaves the warp (Exchanger::run_warp).  tools/swizzle_check.py covers both.
  if constexpr (LAST && LOGN == 12 && WARP_EXCHANGE) return ((t & 15) << 1) | ((t >> 4) & 1) | (t & ~31);
  if constexpr (LAST && LOGN >= 10) return ((t & 31) << 1) | ((t >> 5) & 1) | (t & ~63);
  return t;
}

// Index of register slot k of thread t in the layout of pass (S0, R).  The
// thread part (k = 0) and the slot part (t = 0) have disjoint bits, so
// pass_index(t, k) == pass_index(t, 0) | pass_index(0, k).
template <int LOGN, int S0, int R>
__host__ __device__ constexpr int pass_index(int t, int k) {
  using Sh = NttShape<LOGN>;
  constexpr int G = 1 << R;
  constexpr int S = Sh::N >> (S0 + R);
  constexpr bool LAST = (S0 + R == LOGN);
  const int gg = k / G, j = k % G;
  const int g = gg * Sh::THREADS + (t == 0 ? 0 : pass_thread<LOGN, LAST>(t));
  const int o = g & (S - 1);
  const int B = g >> (LOGN - S0 - R);
  return B * (Sh::N >> S0) + o + j * S;
}

// Twiddle table: ONE table per prime serves both directions.  Entry for
// forward stage s+i, butterfly block b = B*2^i + jb (pass k, group B) holds
// (w, w') with w = psi^bitrev(2^(s+i) + b).  Entries are stored entry-major
// inside a pass -- pair index tw_off(k) + e*2^s + B with e = 2^i - 1 + jb --
// so the lanes of a warp (distinct or equal B) read consecutive or identical
// pairs: coalesced from global, bank-conflict-free from shared memory.
// The inverse transform reads the same table mirrored (group 2^s-1-B, block
// 2^i-1-jb) because psi^-bitrev(m+b) = -psi^bitrev(2m-1-b); the sign is
// folded into the Gentleman-Sande butterfly as (Y - X) * w.
// Loads are volatile so the compiler cannot CSE table entries across the
// several transforms of one kernel (which pinned ~180 registers).
// Storage slot of the twiddle group served by (thread, gg) in pass (S0, R).
// Groups are stored in thread order: for the last pass, whose thread -> group
// map is permuted (pass_thread), slot = gg*THREADS + t rather than the group
// number, so consecutive lanes read consecutive pairs.  Complementing a group
// (the inverse's mirror) commutes with that bit permutation.
template <int LOGN, int S0, int R>
__device__ __forceinline__ int tw_slot(int gg) {
  using Sh = NttShape<LOGN>;
  if constexpr (S0 + R == LOGN) {
    return gg * Sh::THREADS + ntt_tid<LOGN>();
  } else {
    const int g = gg * Sh::THREADS + ntt_tid<LOGN>();
    return g >> (LOGN - S0 - R);
  }
}

// Host helper: storage slot of group B in pass (s, r) (inverse of the above).
__host__ __device__ constexpr int tw_group_slot(int logn, int s, int r, int B) {
  if (s + r == logn && logn == 12 && WARP_EXCHANGE) return ((B >> 1) & 15) | ((B & 1) << 4) | (B & ~31);
  if (s + r == logn && logn >= 10) return ((B >> 1) & 31) | ((B & 1) << 5) | (B & ~63);
  return B;
}

// Copy one prime's twiddle table (`words` words, 16-byte multiple) into shared memory with
// `nthreads` cooperating threads (callers synchronise before first use).
template <typename T>
__device__ __forceinline__ void stage_twiddles(const T* table, T* smem, int words, int nthreads) {
  const uint4* src = reinterpret_cast<const uint4*>(table);
  uint4* dst = reinterpret_cast<uint4*>(smem);
  for (int i = threadIdx.x; i < words * (int)sizeof(T) / 16; i += nthreads) dst[i] = __ldg(src + i);
}

template <typename T, bool SMEM>
struct TwSrc {
  const T* tab;  // generic pointer to pair 0 of this prime's table (global or shared)
  __device__ __forceinline__ double loadq(const double* at) const {
    double v;
    if constexpr (SMEM)
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((uint32_t)__cvta_generic_to_shared(at)));
    else
      asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(at));
    return v;
  }
  // two adjacent (w, w') entries with one 128-bit load (32-bit limbs); -DCTB_TW_LOAD2=0 reads them
  // with two 64-bit loads (A/B)
#ifndef CTB_TW_LOAD2
#define CTB_TW_LOAD2 1
#endif
  __device__ __forceinline__ void load2(const T* at, T& w0, T& wq0, T& w1, T& wq1) const {
    static_assert(sizeof(T) == 4, "paired twiddle entries: 32-bit limbs");
    if constexpr (!CTB_TW_LOAD2) {
      load(at, w0, wq0);
      load(at + 2, w1, wq1);
      return;
    }
    if constexpr (SMEM)
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(wq0), "=r"(w1), "=r"(wq1)
                   : "r"((uint32_t)__cvta_generic_to_shared(at)));
    else
      asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(w0), "=r"(wq0), "=r"(w1), "=r"(wq1) : "l"(at));
  }
  __device__ __forceinline__ void load(const T* at, T& w, T& wq) const {
    if constexpr (SMEM) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(at);
      if constexpr (sizeof(T) == 4)
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w), "=r"(wq) : "r"(sa));
      else
        asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(w), "=l"(wq) : "r"(sa));
    } else {
      if constexpr (sizeof(T) == 4)
        asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(w), "=r"(wq) : "l"(at));
      else
        asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(w), "=l"(wq) : "l"(at));
    }
  }
};

// ptxas turns two-input integer adds into IMAD.IADD (fma-heavy pipe, half rate on sm_100a -- the
// pipe that bounds the transforms) when it judges the ALU pipe busier.  -DCTB_ALU_ADD=1 writes the
// butterflies' two-input sums with a third operand the compiler cannot fold (a __constant__ zero),
// which keeps them IADD3 on the ALU pipe (tools/probe/bfly_probe.cu: +8% on pure Shoup passes).
#ifndef CTB_ALU_ADD
#define CTB_ALU_ADD 0
#endif
__device__ __constant__ uint32_t g_opaque_zero = 0;
template <typename T>
__device__ __forceinline__ T add2(T a, T b) {
  if constexpr (CTB_ALU_ADD && sizeof(T) == 4) return a + b + (T)g_opaque_zero;
  else return a + b;
}

// Harvey CT butterfly.
//  u32 (p < 2^30): X, Y in [0,4p) -> X+WY, X-WY in [0,4p).
//  u64 (p < 2^50 in practice, < 2^57 required): no conditional subtraction --
//    t = WY in [0,4p) (approximate Shoup), X+t and X-t+4p grow by < 4p per
//    stage, so canonical inputs stay below 53p after 13 stages (far below
//    2^64); consumers are Shoup / Montgomery products (valid for any such
//    input) or canon_fwd().
// NOCS (32-bit limbs): the caller knows the conditional subtraction is a no-op (forward: X < 2p;
// inverse: X + Y < 2p) -- the first stage of a transform whose inputs are canonical.
template <typename T, bool NOCS = false>
__device__ __forceinline__ void ct_bfly(T& X, T& Y, T w, T wq, T p, T p2) {
  if constexpr (sizeof(T) == 8) {
    const T t = shoup_mul_lazy4(Y, w, wq, p);
    const T x = X;
    X = x + t;
    Y = x + 2 * p2 - t;
  } else {
    T x = NOCS ? X : csub(X, p2);
    T t = shoup_mul(Y, w, wq, p);
    X = add2(x, t);
    Y = x - t + p2;
  }
}

// Harvey GS butterfly with the mirrored (negated) twiddle.
//  u32: X, Y in [0,2p) -> X+Y, (Y-X)W in [0,2p).
//  u64: X, Y in [0,4p) -> same, in [0,4p) (approximate Shoup); ntt_inv_regs
//       brings the outputs back below 2p after the last stage.
template <typename T, bool NOCS = false>
__device__ __forceinline__ void gs_bfly(T& X, T& Y, T w, T wq, T p, T p2) {
  if constexpr (sizeof(T) == 8) {
    const T p4 = 2 * p2;
    const T u = csub(X + Y, p4);
    const T v = Y - X + p4;
    Y = shoup_mul_lazy4(v, w, wq, p);
    X = u;
  } else {
    T u = NOCS ? X + Y : csub(add2(X, Y), p2);
    T v = Y - X + p2;
    Y = shoup_mul(v, w, wq, p);
    X = u;
  }
}

// FP64-quotient product (see F64Q_NE): a < 2^32, w < p < 2^30, wp = w'/p, kq = 1.5 2^52 - 2^52 wp
// (exact).  fma((2^52 + a), wp, kq) = 1.5 2^52 + a wp exactly before its one rounding, to the
// nearest integer (ulp 1 there): the low word is rint(a wp) in {floor, ceil}(a w / p).
// CONV converts a with I2F.F64.U32 (XU pipe, otherwise idle; no register pair to assemble, no kq)
// instead of the exponent splice: fma(a, wp, 1.5 2^52), same quotient.  Entries e in
// [CTB_F64Q_CONV_LO, CTB_F64Q_CONV_HI) convert, the others splice (A/B: tools/ab_variants.py;
// all-convert measured 1.197 vs all-splice 1.220 ms per 4096 CPMul).
#ifndef CTB_F64Q_CONV_LO
#define CTB_F64Q_CONV_LO 0
#endif
#ifndef CTB_F64Q_CONV_HI
#define CTB_F64Q_CONV_HI 16
#endif
template <bool CONV = true>
__device__ __forceinline__ uint32_t f64q_mul(uint32_t a, uint32_t w, double wp, double kq, uint32_t p, uint32_t pn) {
  const double qd = CONV ? __fma_rn(__uint2double_rn(a), wp, 6755399441055744.0)
                         : __fma_rn(__hiloint2double(0x43300000, (int)a), wp, kq);
  const uint32_t q = (uint32_t)__double2loint(qd);
  uint32_t t, r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(a), "r"(w), "r"(p));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(pn), "r"(t));
  return r;  // a*w + p - q*p in (0, 2p)
}
// Product of two DATA operands on the FP64 pipe (32-bit limbs): x < 2^32, y < 2^32, p < 2^30.
// q = rint(fl(x y) fl(1/p)) by the magic-constant FMA: |q - x y / p| <= 1/2 + 2^-19 (both roundings
// are relative 2^-53 on a quotient below 2^34), only its low word matters, and x y + p - q p in
// (0.49 p, 1.51 p) takes 2 IMAD -- 4 fma-heavy cycles instead of the Montgomery product's 12 (two
// IMAD.HI), the conversions on the XU pipe.  No Montgomery factor: the result is x y mod p.
__device__ __forceinline__ uint32_t f64_pointwise2(uint32_t x, uint32_t y, double xd, double yd, double pinv, uint32_t p,
                                                   uint32_t pn) {   // both operands already converted
  const double qd = __fma_rn(__dmul_rn(xd, yd), pinv, 6755399441055744.0);
  const uint32_t q = (uint32_t)__double2loint(qd);
  uint32_t t, r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(x), "r"(y), "r"(p));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(pn), "r"(t));
  return r;
}
__device__ __forceinline__ uint32_t f64_pointwise(uint32_t x, uint32_t y, double yd, double pinv, uint32_t p, uint32_t pn) {
  const double qd = __fma_rn(__dmul_rn(__uint2double_rn(x), yd), pinv, 6755399441055744.0);
  const uint32_t q = (uint32_t)__double2loint(qd);
  uint32_t t, r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(x), "r"(y), "r"(p));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(pn), "r"(t));
  return r;
}
__device__ __forceinline__ double f64q_k(double wp) { return __fma_rn(-4503599627370496.0, wp, 6755399441055744.0); }
// FP64 quotients of the group slot (pass K): entry e at [e] from it (ntt.cuh shape_q_index)
template <typename T, int LOGN, int K>
__device__ __forceinline__ const double* q_group(const T* tab, int slot) {
  return reinterpret_cast<const double*>(tab + 2 * shape_tw_entries(LOGN)) + shape_q_off(LOGN, K) + slot * F64Q_NE;
}

// CANON: the pass's inputs are below 2p (forward) / p (inverse), e.g. canonical residues from
// memory: the first stage skips its conditional subtractions.
// Twiddles are read two entries per 128-bit load (shape_tw_pair: the entries of blocks jb, jb + 1 of
// a stage are adjacent); entry 0 alone.
template <typename T, int LOGN, int K, bool SMEM, int QE = F64Q_NE, bool CANON = false>
__device__ __forceinline__ void fwd_pass(T (&x)[NttShape<LOGN>::E], TwSrc<T, SMEM> tw, T p, T p2) {
  static_assert(QE <= F64Q_NE, "FP64 quotient entries beyond the table");
  static_assert(sizeof(T) == 4, "integer butterflies: 32-bit limbs (64-bit limbs run the FP64 passes)");
  using Sh = NttShape<LOGN>;
  constexpr int S0 = Sh::pass_s(K), R = Sh::pass_r(K);
  constexpr int G = 1 << R;
  const T pn = (T)0 - p;
#pragma unroll
  for (int gg = 0; gg < Sh::E / G; ++gg) {
    const int slot = tw_slot<LOGN, S0, R>(gg);
    const T* tg = tw.tab + 2 * Sh::tw_off(K) + 4 * slot;   // entry pair q at + 4 (q << S0) words
    const double* qg = q_group<T, LOGN, K>(tw.tab, slot);
    auto block = [&](int i, int jb, T w, T wq) {
      const int h = 1 << (R - i - 1);
      const int e = (1 << i) - 1 + jb;
      if (e < QE) {
        const double wp = tw.loadq(qg + e);
        const double kq = f64q_k(wp);
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int a = gg * G + jb * 2 * h + jj;
          const T xx = (CANON && i == 0) ? x[a] : csub(x[a], p2);
          const T t = (e >= CTB_F64Q_CONV_LO && e < CTB_F64Q_CONV_HI)
                          ? (T)f64q_mul<true>((uint32_t)x[a + h], (uint32_t)w, wp, kq, (uint32_t)p, (uint32_t)pn)
                          : (T)f64q_mul<false>((uint32_t)x[a + h], (uint32_t)w, wp, kq, (uint32_t)p, (uint32_t)pn);
          x[a] = add2(xx, t);
          x[a + h] = xx - t + p2;
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int a = gg * G + jb * 2 * h + jj;
          if (CANON && i == 0) ct_bfly<T, true>(x[a], x[a + h], w, wq, p, p2);
          else ct_bfly(x[a], x[a + h], w, wq, p, p2);
        }
      }
    };
    {
      T w, wq;
      tw.load(tg + 2, w, wq);  // entry 0: second half of pair 0
      block(0, 0, w, wq);
    }
#pragma unroll
    for (int i = 1; i < R; ++i) {
#pragma unroll
      for (int jb = 0; jb < (1 << i); jb += 2) {
        T w0, wq0, w1, wq1;
        tw.load2(tg + 4 * ((((1 << i) + jb) >> 1) << S0), w0, wq0, w1, wq1);
        block(i, jb, w0, wq0);
        block(i, jb + 1, w1, wq1);
      }
    }
  }
}

template <typename T, int LOGN, int K, bool SMEM, int QE = F64Q_NE, bool CANON = false>
__device__ __forceinline__ void inv_pass(T (&x)[NttShape<LOGN>::E], TwSrc<T, SMEM> tw, T p, T p2) {
  static_assert(QE <= F64Q_NE, "FP64 quotient entries beyond the table");
  static_assert(sizeof(T) == 4, "integer butterflies: 32-bit limbs (64-bit limbs run the FP64 passes)");
  using Sh = NttShape<LOGN>;
  constexpr int S0 = Sh::pass_s(K), R = Sh::pass_r(K);
  constexpr int G = 1 << R;
  const T pn = (T)0 - p;
#pragma unroll
  for (int gg = 0; gg < Sh::E / G; ++gg) {
    const int slot = (1 << S0) - 1 - tw_slot<LOGN, S0, R>(gg);  // mirrored group
    const T* tg = tw.tab + 2 * Sh::tw_off(K) + 4 * slot;
    const double* qg = q_group<T, LOGN, K>(tw.tab, slot);
    // block jb of stage i with the mirrored entry e = 2^i - 1 + (2^i - 1 - jb)
    auto block = [&](int i, int jb, T w, T wq) {
      const int h = 1 << (R - i - 1);
      const int e = (1 << i) - 1 + ((1 << i) - 1 - jb);
      if (e < QE) {
        const double wp = tw.loadq(qg + e);
        const double kq = f64q_k(wp);
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int a = gg * G + jb * 2 * h + jj;
          const T X = x[a], Y = x[a + h];
          x[a] = (CANON && i == R - 1) ? X + Y : csub(add2(X, Y), p2);
          x[a + h] = (e >= CTB_F64Q_CONV_LO && e < CTB_F64Q_CONV_HI)
                         ? (T)f64q_mul<true>((uint32_t)(Y - X + p2), (uint32_t)w, wp, kq, (uint32_t)p, (uint32_t)pn)
                         : (T)f64q_mul<false>((uint32_t)(Y - X + p2), (uint32_t)w, wp, kq, (uint32_t)p, (uint32_t)pn);
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int a = gg * G + jb * 2 * h + jj;
          if (CANON && i == R - 1) gs_bfly<T, true>(x[a], x[a + h], w, wq, p, p2);
          else gs_bfly(x[a], x[a + h], w, wq, p, p2);
        }
      }
    };
#pragma unroll
    for (int i = R - 1; i >= 1; --i) {
#pragma unroll
      for (int jb = 0; jb < (1 << i); jb += 2) {
        // blocks jb, jb + 1 use entries e, e - 1 with e + 1 = 2^(i+1) - 1 - jb: halves 1 and 0 of one pair
        T w0, wq0, w1, wq1;
        tw.load2(tg + 4 * ((((1 << (i + 1)) - 1 - jb) >> 1) << S0), w0, wq0, w1, wq1);
        block(i, jb, w1, wq1);
        block(i, jb + 1, w0, wq0);
      }
    }
    {
      T w, wq;
      tw.load(tg + 2, w, wq);
      block(0, 0, w, wq);
    }
  }
}

// Barrier over the THREADS threads of one transform: the whole CTA (GROUPS = 1)
// or one named barrier per group (ids 1..GROUPS) when a CTA runs GROUPS
// independent transforms.
template <int LOGN, int GROUPS>
__device__ __forceinline__ void group_sync() {
  if constexpr (GROUPS == 1) {
    __syncthreads();
  } else {
    const int id = 1 + (int)(threadIdx.x / NttShape<LOGN>::THREADS);
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(NttShape<LOGN>::THREADS) : "memory");
  }
}

// Shared-memory exchange between two pass layouts.  NBUF = 2 double-buffers
// (one barrier per exchange); NBUF = 1 halves the footprint for one more
// resident CTA at the price of a second barrier (write-after-read guard).
//
// Vectorised case (32-bit words, N = 4096; one image whatever NBUF).  In the middle pass (stages
// 4-7) warp w of the transform owns the index bits 9-11 = w, and with the five-bit last-pass
// rotation (pass_thread) so it does in the last pass.  Map 1 keeps index bits 9-11 as address bits
// 9-11, so:
//   * the middle-pass side of the map-1 exchange touches only the warp's own 512-word block;
//   * the exchange between the middle and the last pass is a 16 x 16 transposition inside each
//     half-warp and runs INSIDE that block with __syncwarp only (run_warp): element (s = index bit
//     8, m = bits 4-7, j = bits 0-3) sits at block word
//         256 s + 32 (m & 7) + 16 (m3 ^ s) + 4 ((j >> 2) ^ ((m >> 1) & 3)) + (j & 3),
//     conflict-free for the middle pass's scalar accesses (lanes (s, j): bank bits m3 ^ s,
//     (j3 j2) ^ (m2 m1), j1 j0) and for the last pass's 128-bit accesses (a quarter warp varies
//     m3 m2 m1 at fixed s, m0: 16-byte bank group (m3 ^ s, c ^ (m2 m1))).  The XORed address bits
//     cost 7 LOP3 on the scalar side (8 bases, two stores each) and 3 on the vector side;
//   * the first-pass side of map 1 is thread-stationary: the inverse's last exchange reads exactly
//     the words the next forward transform's first exchange writes.
// Group-wide barriers per transform: one write-after-read guard before its first exchange and one
// read-after-write barrier in its map-1 exchange (instead of four).  RELAX drops the guard where
// the caller knows the image's previous use: a forward transform right after an inverse one
// (thread-stationary words: no synchronisation at all), an inverse right after a forward (the
// warp's own block: __syncwarp).  Not after a transform of the same direction, nor after any other
// use of the image (eval_xpose_*).
template <typename T, int LOGN, int NBUF = 2, int GROUPS = 1>
struct Exchanger {
  T* buf;      // NBUF * SmemImage::WORDS words
  int cur = 0;
  static constexpr bool WARPX = vec_exchange<T, LOGN>() && WARP_EXCHANGE;
  static constexpr int WORDS = (WARPX ? 1 : NBUF) * SmemImage<T, LOGN>::WORDS;

  // The warp-local exchange (see above).  FWD: middle pass -> last pass (scalar stores, 128-bit
  // loads); otherwise last -> middle (128-bit stores, scalar loads).
  template <bool FWD, bool RELAX, typename U>
  __device__ __forceinline__ void run_warp(U (&x)[NttShape<LOGN>::E]) {
    static_assert(vec_exchange<T, LOGN>() && NttShape<LOGN>::E == 16, "warp-local exchange: N = 4096, 32-bit words");
    const int t = ntt_tid<LOGN>();
    U* blk = reinterpret_cast<U*>(buf) + (t & ~31) * 16;                                   // 512 words per warp
    // middle-pass lane (s = t4, j = t3..t0): word 272 s + j, then ^ 4 (m >> 1), + 32 (m & 7) per element m
    const uint32_t mid = (uint32_t)__cvta_generic_to_shared(blk) + 4u * (272u * ((t >> 4) & 1) + (t & 15));
    // last-pass lane (m0 = t4, s = t3, m3 m2 m1 = t2 t1 t0): row 256 s + 32 (m & 7) + 16 (m3 ^ s), chunk c ^ (m2 m1)
    const int sl = (t >> 3) & 1;
    const uint32_t row = (uint32_t)__cvta_generic_to_shared(blk) +
                         4u * (256u * sl + 32u * (((t & 3) << 1) | ((t >> 4) & 1)) + 16u * (((t >> 2) & 1) ^ sl) + 4u * (t & 3));
    if constexpr (FWD || RELAX) __syncwarp();
    else group_sync<LOGN, GROUPS>();
    if constexpr (FWD) {
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const uint32_t a = mid ^ (16u * v);
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a + 128u * ((2 * v) & 7)), "r"((uint32_t)x[2 * v]) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a + 128u * ((2 * v + 1) & 7)), "r"((uint32_t)x[2 * v + 1]) : "memory");
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t a0, a1, a2, a3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(row ^ (16u * c)) : "memory");
        x[4 * c] = (U)a0; x[4 * c + 1] = (U)a1; x[4 * c + 2] = (U)a2; x[4 * c + 3] = (U)a3;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(row ^ (16u * c)), "r"((uint32_t)x[4 * c]),
                     "r"((uint32_t)x[4 * c + 1]), "r"((uint32_t)x[4 * c + 2]), "r"((uint32_t)x[4 * c + 3]) : "memory");
      __syncwarp();
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const uint32_t a = mid ^ (16u * v);
        uint32_t lo, hi;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(lo) : "r"(a + 128u * ((2 * v) & 7)) : "memory");
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hi) : "r"(a + 128u * ((2 * v + 1) & 7)) : "memory");
        x[2 * v] = (U)lo; x[2 * v + 1] = (U)hi;
      }
    }
  }

  template <int SA, int RA, int SB, int RB, bool RELAX = false, typename U>
  __device__ __forceinline__ void run(U (&x)[NttShape<LOGN>::E]) {
    static_assert(sizeof(U) == sizeof(T), "exchange element width");
    using Sh = NttShape<LOGN>;
    constexpr int MAP = exchange_map<T, LOGN, SA, SB>();
    if constexpr (MAP == 2 && WARPX) {
      run_warp<(SA < SB), RELAX>(x);
      return;
    }
    U* b = reinterpret_cast<U*>(buf + (WARPX ? 0 : cur) * SmemImage<T, LOGN>::WORDS);
    if constexpr (MAP == 1 && WARPX) {
      // write-after-read guard: forward (first exchange of its transform) a group barrier unless
      // RELAX; inverse (after the warp-local exchange, writing only the warp's own block) a warp one
      if constexpr (SA > SB) __syncwarp();
      else if constexpr (!RELAX) group_sync<LOGN, GROUPS>();
    } else {
      if constexpr (NBUF == 2) cur ^= 1;
      else group_sync<LOGN, GROUPS>();
    }
    constexpr int VA = exchange_vec<MAP, SA>(), VB = exchange_vec<MAP, SB>();
    U* wa = b + phys_map<T, LOGN, MAP>(pass_index<LOGN, SA, RA>(ntt_tid<LOGN>(), 0));
    U* wb = b + phys_map<T, LOGN, MAP>(pass_index<LOGN, SB, RB>(ntt_tid<LOGN>(), 0));
#pragma unroll
    for (int k = 0; k < Sh::E; k += VA) {
      U* at = wa + phys_map<T, LOGN, MAP>(pass_index<LOGN, SA, RA>(0, k));
      if constexpr (VA == 4)
        *reinterpret_cast<uint4*>(at) = make_uint4((uint32_t)x[k], (uint32_t)x[k + 1], (uint32_t)x[k + 2], (uint32_t)x[k + 3]);
      else if constexpr (VA == 2)
        *reinterpret_cast<uint2*>(at) = make_uint2((uint32_t)x[k], (uint32_t)x[k + 1]);
      else
        *at = x[k];
    }
    group_sync<LOGN, GROUPS>();
#pragma unroll
    for (int k = 0; k < Sh::E; k += VB) {
      const U* at = wb + phys_map<T, LOGN, MAP>(pass_index<LOGN, SB, RB>(0, k));
      if constexpr (VB == 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(at);
        x[k] = (U)v.x; x[k + 1] = (U)v.y; x[k + 2] = (U)v.z; x[k + 3] = (U)v.w;
      } else if constexpr (VB == 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(at);
        x[k] = (U)v.x; x[k + 1] = (U)v.y;
      } else {
        x[k] = *at;
      }
    }
  }
};

// Thread-private strip of E words per thread in shared memory (an operand kept in the
// evaluation layout between transforms: NTT(pt) in k_cpmul, NTT(u) in k_encrypt), stored
// chunk-major -- 16-byte chunk c of thread t at vector c * THREADS + t -- so it moves with
// conflict-free 128-bit accesses (E/4 instructions instead of E for 32-bit words).
// `region` (N words) must be 16-byte aligned.
template <typename T, int LOGN>
struct Strip {
  using Sh = NttShape<LOGN>;
  static constexpr int VEC = Sh::E * (int)sizeof(T) >= 16 ? 16 / (int)sizeof(T) : 1;  // scalar for tiny N
  static constexpr int CHUNKS = Sh::E / VEC;
  T* base;
  __device__ __forceinline__ explicit Strip(T* region) : base(region + VEC * ntt_tid<LOGN>()) {}
  __device__ __forceinline__ void store_chunk(int c, const T* v) {
    T* at = base + (size_t)c * VEC * Sh::THREADS;
    if constexpr (VEC == 1) {
      *at = v[0];
    } else if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<uint4*>(at) = make_uint4((uint32_t)v[0], (uint32_t)v[1], (uint32_t)v[2], (uint32_t)v[3]);
    } else {
      *reinterpret_cast<uint4*>(at) =
          make_uint4((uint32_t)v[0], (uint32_t)((uint64_t)v[0] >> 32), (uint32_t)v[1], (uint32_t)((uint64_t)v[1] >> 32));
    }
  }
  __device__ __forceinline__ void load_chunk(int c, T (&v)[VEC]) const {
    const T* at = base + (size_t)c * VEC * Sh::THREADS;
    if constexpr (VEC == 1) {
      v[0] = *at;
    } else {
      const uint4 w = *reinterpret_cast<const uint4*>(at);
      if constexpr (sizeof(T) == 4) {
        v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
      } else {
        v[0] = (T)((uint64_t)w.x | ((uint64_t)w.y << 32));
        v[1] = (T)((uint64_t)w.z | ((uint64_t)w.w << 32));
      }
    }
  }
  __device__ __forceinline__ void store(const T (&x)[Sh::E]) {
#pragma unroll
    for (int c = 0; c < CHUNKS; ++c) store_chunk(c, x + c * VEC);
  }
};

// ---- FP64 butterflies for 64-bit limbs (primes < 2^50) --------------------------------
// Residues are held as exact integers in doubles, signed and lazily reduced.  Twiddles are stored
// CENTRED, w in (-p/2, p/2] (ctx.cu), so |w/p| <= 1/2.  For |x w / p| < 2^51:
//   mulmod(x, w): hi = fl(x w), lo = x w - hi (exact, fma), q = rint(x * wp) with wp = fl(w fl(1/p))
//   (|wp - w/p| <= 2^-53 because |w/p| <= 1/2), so |q - x w / p| <= 1/2 + |x| 2^-53, and
//   r = (hi - q p) + lo is exact with |r| <= (1/2 + |x| 2^-53) p  (< 0.95 p for |x| <= 3.5 p);
//   center(x) = x - p rint(x / p) in [-p/2, p/2] (tiny slack), exact for |x| < 2^52.
// rint uses the 1.5 * 2^52 magic constant (exact for |y| < 2^51); sums stay exact below 2^53.
// Reduction schedule (bounds in units of p; p < 2^50, so 2^51 / p > 2):
//   forward CT  X' = X + t, Y' = X - t, t = mulmod(Y): a pass starts from centred values (0.5) and
//               runs its <= 4 stages WITHOUT reducing X: 0.5 -> 1.5 -> 2.5 -> 3.5 -> 4.5, the
//               multiplied operand never exceeds 3.5 (|Y wp| <= 1.75 p < 2^51); all 16 values are
//               centred once at the next pass boundary (3 ops per value per pass instead of 3 per
//               butterfly per stage).
//   inverse GS  X' = X + Y, Y' = mulmod(Y - X): X' is centred on every second global stage, starting
//               with the first, so the uncentred inputs may lie anywhere in [0, 2p) (every caller's
//               are: canonical values, Montgomery products, sums kept below 2p): the differences reach
//               at most 2p (first stage), then stay below 4p at the centring stages (|.| wp < 2p)
//               while products stay below p; no input centring.
// About 9.5 FP64 operations per butterfly instead of 11 with full reduction every stage.
struct F64Prime {
  double p, pinv;
};
__device__ __forceinline__ double f64_rint(double y) {
  constexpr double C = 6755399441055744.0;  // 1.5 * 2^52
  return __dadd_rn(__dadd_rn(y, C), -C);
}
// rint(a * b) for |a * b| < 2^51, the magic constant folded into the product's FMA
__device__ __forceinline__ double f64_rint_mul(double a, double b) {
  constexpr double C = 6755399441055744.0;  // 1.5 * 2^52
  return __dadd_rn(__fma_rn(a, b, C), -C);
}
__device__ __forceinline__ double f64_mulmod(double x, double w, double wp, double p) {
  const double hi = __dmul_rn(x, w);
  const double lo = __fma_rn(x, w, -hi);
  const double q = f64_rint_mul(x, wp);
  return __dadd_rn(__fma_rn(-q, p, hi), lo);
}
__device__ __forceinline__ double f64_center(double x, const F64Prime& P) {
  const double q = f64_rint_mul(x, P.pinv);
  return __fma_rn(-q, P.p, x);
}
// u64 residue (< 2^52) <-> double, exact, by exponent-bit splicing.
__device__ __forceinline__ double f64_from_u64(uint64_t x) {
  return __dadd_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), -4503599627370496.0);
}
__device__ __forceinline__ uint64_t f64_to_canon(double x, const F64Prime& P) {  // |x| < 2^52
  double y = f64_center(x, P);                   // [-p/2 - e, p/2 + e]
  y = y < 0.0 ? __dadd_rn(y, P.p) : y;           // [0, p)
  return (uint64_t)__double_as_longlong(__dadd_rn(y, 4503599627370496.0)) & 0x000FFFFFFFFFFFFFull;
}

// One table word per entry: w as a double; w/p = fl(w * fl(1/p)) (relative error < 2^-52, so
// |x fl(w/p) - x w / p| < 1/2 for |x| < 2^51 and the product bound |r| < p still holds).
template <typename T, bool SMEM>
__device__ __forceinline__ void tw_load_f64(const TwSrc<T, SMEM>& tw, const T* at, double pinv, double& w,
                                            double& wp) {
  uint64_t a;
  if constexpr (SMEM) {
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(a) : "r"((uint32_t)__cvta_generic_to_shared(at)));
  } else {
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(a) : "l"(at));
  }
  w = __longlong_as_double((long long)a);
  wp = __dmul_rn(w, pinv);
}

template <typename T, int LOGN, int K, bool SMEM>
__device__ __forceinline__ void fwd_pass_f64(double (&x)[NttShape<LOGN>::E], TwSrc<T, SMEM> tw, const F64Prime& P) {
  using Sh = NttShape<LOGN>;
  constexpr int S0 = Sh::pass_s(K), R = Sh::pass_r(K);
  constexpr int G = 1 << R;
  static_assert(R <= 4, "the lazy forward schedule assumes at most 4 stages per pass");
  if constexpr (K > 0) {
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) x[k] = f64_center(x[k], P);  // <= 4.5 p -> 0.5 p
  }
#pragma unroll
  for (int gg = 0; gg < Sh::E / G; ++gg) {
    const int slot = tw_slot<LOGN, S0, R>(gg);
    const T* tg = tw.tab + (Sh::tw_off(K) + slot);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int h = 1 << (R - i - 1);
#pragma unroll
      for (int jb = 0; jb < (1 << i); ++jb) {
        double w, wp;
        tw_load_f64(tw, tg + (((1 << i) - 1 + jb) << S0), P.pinv, w, wp);
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int a = gg * G + jb * 2 * h + jj;
          const double X = x[a];
          const double t = f64_mulmod(x[a + h], w, wp, P.p);
          x[a] = __dadd_rn(X, t);
          x[a + h] = __dadd_rn(X, -t);
        }
      }
    }
  }
}

template <typename T, int LOGN, int K, bool SMEM>
__device__ __forceinline__ void inv_pass_f64(double (&x)[NttShape<LOGN>::E], TwSrc<T, SMEM> tw, const F64Prime& P) {
  using Sh = NttShape<LOGN>;
  constexpr int S0 = Sh::pass_s(K), R = Sh::pass_r(K);
  constexpr int G = 1 << R;
  constexpr int DONE = LOGN - S0 - R;  // inverse stages run before this pass
#pragma unroll
  for (int gg = 0; gg < Sh::E / G; ++gg) {
    const int slot = (1 << S0) - 1 - tw_slot<LOGN, S0, R>(gg);
    const T* tg = tw.tab + (Sh::tw_off(K) + slot);
#pragma unroll
    for (int i = R - 1; i >= 0; --i) {
      const int h = 1 << (R - i - 1);
      const bool reduce = ((DONE + (R - 1 - i)) & 1) == 0;  // every second global stage, from the first
#pragma unroll
      for (int jb = 0; jb < (1 << i); ++jb) {
        double w, wp;
        tw_load_f64(tw, tg + (((1 << i) - 1 + ((1 << i) - 1 - jb)) << S0), P.pinv, w, wp);
#pragma unroll
        for (int jj = 0; jj < h; ++jj) {
          const int a = gg * G + jb * 2 * h + jj;
          const double X = x[a], Y = x[a + h];
          const double sum = __dadd_rn(X, Y);
          x[a] = reduce ? f64_center(sum, P) : sum;
          x[a + h] = f64_mulmod(__dadd_rn(Y, -X), w, wp, P.p);
        }
      }
    }
  }
}

template <typename T, int LOGN, int K, bool SMEM, int NBUF, int GROUPS>
__device__ __forceinline__ void ntt_fwd_f64(double (&x)[NttShape<LOGN>::E], Exchanger<T, LOGN, NBUF, GROUPS>& ex,
                                            TwSrc<T, SMEM> tw, const F64Prime& P) {
  using Sh = NttShape<LOGN>;
  fwd_pass_f64<T, LOGN, K, SMEM>(x, tw, P);
  if constexpr (K + 1 < Sh::NPASS) {
    ex.template run<Sh::pass_s(K), Sh::pass_r(K), Sh::pass_s(K + 1), Sh::pass_r(K + 1)>(x);
    ntt_fwd_f64<T, LOGN, K + 1, SMEM, NBUF, GROUPS>(x, ex, tw, P);
  }
}

template <typename T, int LOGN, int K, bool SMEM, int NBUF, int GROUPS>
__device__ __forceinline__ void ntt_inv_f64(double (&x)[NttShape<LOGN>::E], Exchanger<T, LOGN, NBUF, GROUPS>& ex,
                                            TwSrc<T, SMEM> tw, const F64Prime& P) {
  using Sh = NttShape<LOGN>;
  inv_pass_f64<T, LOGN, K, SMEM>(x, tw, P);
  if constexpr (K > 0) {
    ex.template run<Sh::pass_s(K), Sh::pass_r(K), Sh::pass_s(K - 1), Sh::pass_r(K - 1)>(x);
    ntt_inv_f64<T, LOGN, K - 1, SMEM, NBUF, GROUPS>(x, ex, tw, P);
  }
}

// RELAX (ntt_fwd_regs / ntt_inv_regs): the caller vouches for the image's previous use, see Exchanger.
// CANON: inputs below 2p (forward) / p (inverse), see fwd_pass; applies to the transform's first pass.
template <typename T, int LOGN, int K = 0, bool SMEM, int NBUF, int GROUPS, int QE = F64Q_NE, bool RELAX = false,
          bool CANON = false>
__device__ __forceinline__ void ntt_fwd_regs(T (&x)[NttShape<LOGN>::E], Exchanger<T, LOGN, NBUF, GROUPS>& ex,
                                             TwSrc<T, SMEM> tw, T p, T p2) {
  using Sh = NttShape<LOGN>;
  if constexpr (sizeof(T) == 8 && K != 0) {
    __trap();  // 64-bit limbs transform whole polynomials (never split)
  } else if constexpr (sizeof(T) == 8) {
    // 64-bit limbs: FP64 butterflies, inputs < 4p (< 2^52), outputs canonical [0, p) (the lazy
    // schedule leaves |d| <= 4.5 p, which f64_to_canon reduces exactly).  With at most 3 stages in
    // the first pass the inputs need no centring: x - 2p in [-2p, 2p) (one DADD fused into the
    // exponent splice) keeps the multiplied operand below 4p there (0.5 |Y| <= 2p < 2^51), and pass 1
    // centres everything.
    const F64Prime P{(double)p, __drcp_rn((double)p)};
    double d[Sh::E];
    if constexpr (Sh::FIRST_R <= 3 && Sh::NPASS > 1) {
      const double off = __dadd_rn(4503599627370496.0, 2.0 * (double)p);   // 2^52 + 2p, exact
#pragma unroll
      for (int k = 0; k < Sh::E; ++k)
        d[k] = __dadd_rn(__longlong_as_double((long long)((uint64_t)x[k] | 0x4330000000000000ull)), -off);
    } else {
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) d[k] = f64_center(f64_from_u64(x[k]), P);
    }
    ntt_fwd_f64<T, LOGN, 0, SMEM, NBUF, GROUPS>(d, ex, tw, P);
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) x[k] = f64_to_canon(d[k], P);
  } else {
    constexpr int S = Sh::pass_s(K), R = Sh::pass_r(K);
    fwd_pass<T, LOGN, K, SMEM, QE, CANON>(x, tw, p, p2);
    if constexpr (K + 1 < Sh::NPASS) {
      ex.template run<S, R, Sh::pass_s(K + 1), Sh::pass_r(K + 1), RELAX>(x);
      ntt_fwd_regs<T, LOGN, K + 1, SMEM, NBUF, GROUPS, QE, RELAX, false>(x, ex, tw, p, p2);
    }
  }
}

template <typename T, int LOGN, int K = NttShape<LOGN>::NPASS - 1, bool SMEM, int NBUF, int GROUPS, int QE = F64Q_NE,
          bool RELAX = false, bool CANON = false>
__device__ __forceinline__ void ntt_inv_regs(T (&x)[NttShape<LOGN>::E], Exchanger<T, LOGN, NBUF, GROUPS>& ex,
                                             TwSrc<T, SMEM> tw, T p, T p2) {
  using Sh = NttShape<LOGN>;
  if constexpr (sizeof(T) == 8 && K != Sh::NPASS - 1) {
    __trap();  // 64-bit limbs transform whole polynomials (never split)
  } else if constexpr (sizeof(T) == 8) {
    // 64-bit limbs: FP64 butterflies, inputs < 2p (taken as they are: the first stage centres),
    // outputs canonical [0, p)
    const F64Prime P{(double)p, __drcp_rn((double)p)};
    double d[Sh::E];
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) d[k] = f64_from_u64(x[k]);
    ntt_inv_f64<T, LOGN, Sh::NPASS - 1, SMEM, NBUF, GROUPS>(d, ex, tw, P);
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) x[k] = f64_to_canon(d[k], P);
  } else {
    constexpr int S = Sh::pass_s(K), R = Sh::pass_r(K);
    inv_pass<T, LOGN, K, SMEM, QE, CANON>(x, tw, p, p2);
    if constexpr (K > 0) {
      ex.template run<S, R, Sh::pass_s(K - 1), Sh::pass_r(K - 1), RELAX>(x);
      ntt_inv_regs<T, LOGN, K - 1, SMEM, NBUF, GROUPS, QE, RELAX, false>(x, ex, tw, p, p2);
    }
  }
}

// Convenience wrappers reading the twiddles through the global read-only path.
template <typename T, int LOGN>
__device__ __forceinline__ void ntt_fwd_regs(T (&x)[NttShape<LOGN>::E], Exchanger<T, LOGN>& ex,
                                             const T* tw, T p, T p2) {
  ntt_fwd_regs<T, LOGN, 0, false, 2, 1>(x, ex, TwSrc<T, false>{tw}, p, p2);
}
template <typename T, int LOGN>
__device__ __forceinline__ void ntt_inv_regs(T (&x)[NttShape<LOGN>::E], Exchanger<T, LOGN>& ex,
                                             const T* tw, T p, T p2) {
  ntt_inv_regs<T, LOGN, NttShape<LOGN>::NPASS - 1, false, 2, 1>(x, ex, TwSrc<T, false>{tw}, p, p2);
}

// Coefficient-domain layout (first pass, coalesced: thread t owns t + j*THREADS):
// element index = coef_base() + coef_off(k).
template <int LOGN>
__device__ __forceinline__ int coef_base() {
  return pass_index<LOGN, 0, NttShape<LOGN>::FIRST_R>(ntt_tid<LOGN>(), 0);
}
template <int LOGN>
__host__ __device__ constexpr int coef_off(int k) {
  return pass_index<LOGN, 0, NttShape<LOGN>::FIRST_R>(0, k);
}
// Evaluation-domain layout (last pass; bit-reversed storage order).
template <int LOGN>
__device__ __forceinline__ int eval_base() {
  using Sh = NttShape<LOGN>;
  return pass_index<LOGN, Sh::pass_s(Sh::NPASS - 1), Sh::pass_r(Sh::NPASS - 1)>(ntt_tid<LOGN>(), 0);
}
template <int LOGN>
__host__ __device__ constexpr int eval_off(int k) {
  using Sh = NttShape<LOGN>;
  return pass_index<LOGN, Sh::pass_s(Sh::NPASS - 1), Sh::pass_r(Sh::NPASS - 1)>(0, k);
}

// Vectorised global access in the evaluation layout.  In the last pass each
// thread owns E contiguous slots (when E/G == 1), so a thread's E words are one
// 16-byte-aligned run: 4 x 16-byte loads (u32) instead of 16 strided words that
// touch a separate sector per lane.  base must point at element 0 of the poly.
template <typename T, int LOGN>
__device__ __forceinline__ void load_eval(const T* __restrict__ base, T (&x)[NttShape<LOGN>::E]) {
  using Sh = NttShape<LOGN>;
  constexpr bool CONTIG = Sh::pass_r(Sh::NPASS - 1) == Sh::LOGE && Sh::E * sizeof(T) % 16 == 0;
  const T* p = base + eval_base<LOGN>();
  if constexpr (CONTIG) {
    const uint4* v = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int i = 0; i < Sh::E * (int)sizeof(T) / 16; ++i) {
      const uint4 w = __ldg(v + i);
      if constexpr (sizeof(T) == 4) {
        x[4 * i] = w.x; x[4 * i + 1] = w.y; x[4 * i + 2] = w.z; x[4 * i + 3] = w.w;
      } else {
        x[2 * i] = (uint64_t)w.x | ((uint64_t)w.y << 32);
        x[2 * i + 1] = (uint64_t)w.z | ((uint64_t)w.w << 32);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) x[k] = __ldg(p + eval_off<LOGN>(k));
  }
}

// Chunked form: chunk i holds slots [i*VEC, (i+1)*VEC) of the thread (VEC words = 16 B).
template <typename T, int LOGN>
struct EvalVec {
  using Sh = NttShape<LOGN>;
  static constexpr bool CONTIG = Sh::pass_r(Sh::NPASS - 1) == Sh::LOGE && Sh::E * sizeof(T) % 16 == 0;
  static constexpr int VEC = CONTIG ? 16 / (int)sizeof(T) : 1;
  static constexpr int CHUNKS = Sh::E / VEC;
  // base: element 0 of the polynomial
  __device__ __forceinline__ static void load(const T* __restrict__ base, int i, T (&v)[VEC]) {
    const T* p = base + eval_base<LOGN>();
    if constexpr (CONTIG) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(p) + i);
      if constexpr (sizeof(T) == 4) {
        v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
      } else {
        v[0] = (uint64_t)w.x | ((uint64_t)w.y << 32);
        v[1] = (uint64_t)w.z | ((uint64_t)w.w << 32);
      }
    } else {
      v[0] = __ldg(p + eval_off<LOGN>(i));
    }
  }
};

// load_eval from a shared-memory copy of the polynomial (natural word order).
template <typename T, int LOGN>
__device__ __forceinline__ void load_eval_smem(const T* base, T (&x)[NttShape<LOGN>::E]) {
  using Sh = NttShape<LOGN>;
  using EV = EvalVec<T, LOGN>;
  const T* p = base + eval_base<LOGN>();
  if constexpr (EV::CONTIG) {
#pragma unroll
    for (int i = 0; i < EV::CHUNKS; ++i) {
      const uint4 w = reinterpret_cast<const uint4*>(p)[i];
      if constexpr (sizeof(T) == 4) {
        x[4 * i] = w.x; x[4 * i + 1] = w.y; x[4 * i + 2] = w.z; x[4 * i + 3] = w.w;
      } else {
        x[2 * i] = (uint64_t)w.x | ((uint64_t)w.y << 32);
        x[2 * i + 1] = (uint64_t)w.z | ((uint64_t)w.w << 32);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) x[k] = p[eval_off<LOGN>(k)];
  }
}

template <typename T, int LOGN>
__device__ __forceinline__ void store_eval(T* base, const T (&x)[NttShape<LOGN>::E]) {
  using Sh = NttShape<LOGN>;
  constexpr bool CONTIG = Sh::pass_r(Sh::NPASS - 1) == Sh::LOGE && Sh::E * sizeof(T) % 16 == 0;
  T* p = base + eval_base<LOGN>();
  if constexpr (CONTIG) {
    uint4* v = reinterpret_cast<uint4*>(p);
#pragma unroll
    for (int i = 0; i < Sh::E * (int)sizeof(T) / 16; ++i) {
      uint4 w;
      if constexpr (sizeof(T) == 4) {
        w.x = x[4 * i]; w.y = x[4 * i + 1]; w.z = x[4 * i + 2]; w.w = x[4 * i + 3];
      } else {
        w.x = (uint32_t)x[2 * i]; w.y = (uint32_t)(x[2 * i] >> 32);
        w.z = (uint32_t)x[2 * i + 1]; w.w = (uint32_t)(x[2 * i + 1] >> 32);
      }
      v[i] = w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) p[eval_off<LOGN>(k)] = x[k];
  }
}

// Eval-layout global traffic through the group's (free) exchange image.  The last pass leaves
// thread t with the E-word block f(t) (pass_thread rotates the low thread bits, so a warp's blocks
// are 2 apart and each 16-byte access of store_eval / EvalVec lands in a different 128-byte line,
// and the natural-order TMA staging buffer read that way is an 8-way bank conflict).  Transposed
// through shared memory, each warp instruction moves 512 contiguous bytes instead.  16-byte chunk
// c of block B sits at slot
//   u32 (4 chunks per block): 8 (B/2) + 4 ((B ^ B/2) & 1) + (c ^ (B/4 mod 4))
//   u64 (8 chunks per block): 8 B + (c ^ (B/2 mod 8))
// so that both the block-wise side (a quarter warp holds blocks 2u + e for 8 consecutive u) and
// the contiguous side (a quarter warp holds 8 consecutive chunks) hit 8 distinct 16-byte bank
// groups, in exactly N words.  Barriers: the image may still be read by the last exchange (WAR),
// and the second side needs every write of the first (RAW); every later use of the image (an
// exchange, or the next transposition) starts with a group barrier.
// -DCTB_EVAL_XPOSE=0 restores the direct (line-per-lane) eval-layout accesses.
#ifndef CTB_EVAL_XPOSE
#define CTB_EVAL_XPOSE 1
#endif
template <typename T, int LOGN>
__host__ __device__ constexpr bool eval_xpose_ok(int image_words) {
  using Sh = NttShape<LOGN>;
  constexpr int CH = Sh::E * (int)sizeof(T) / 16;
  return Sh::pass_r(Sh::NPASS - 1) == Sh::LOGE && Sh::E * sizeof(T) % 16 == 0 && (CH == 4 || CH == 8) &&
         Sh::THREADS % 8 == 0 && image_words >= Sh::N;
}
template <int CH>
__device__ __forceinline__ int eval_xpose_slot(int B, int c) {
  if constexpr (CH == 4) return 8 * (B >> 1) + 4 * ((B ^ (B >> 1)) & 1) + (c ^ ((B >> 2) & 3));
  else return 8 * B + (c ^ ((B >> 1) & 7));
}
template <typename T>
__device__ __forceinline__ uint4 pack_chunk(const T* v) {
  if constexpr (sizeof(T) == 4) return make_uint4((uint32_t)v[0], (uint32_t)v[1], (uint32_t)v[2], (uint32_t)v[3]);
  else return make_uint4((uint32_t)v[0], (uint32_t)((uint64_t)v[0] >> 32), (uint32_t)v[1], (uint32_t)((uint64_t)v[1] >> 32));
}
template <typename T>
__device__ __forceinline__ void unpack_chunk(const uint4& w, T* v) {
  if constexpr (sizeof(T) == 4) {
    v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
  } else {
    v[0] = (T)((uint64_t)w.x | ((uint64_t)w.y << 32));
    v[1] = (T)((uint64_t)w.z | ((uint64_t)w.w << 32));
  }
}

template <typename T, int LOGN, int GROUPS>
__device__ __forceinline__ void store_eval_xpose(T* base, const T (&x)[NttShape<LOGN>::E], T* img) {
  using Sh = NttShape<LOGN>;
  constexpr int CH = Sh::E * (int)sizeof(T) / 16, VEC = 16 / (int)sizeof(T);
  uint4* img4 = reinterpret_cast<uint4*>(img);
  const int blk = eval_base<LOGN>() / Sh::E;
  group_sync<LOGN, GROUPS>();
#pragma unroll
  for (int c = 0; c < CH; ++c) img4[eval_xpose_slot<CH>(blk, c)] = pack_chunk<T>(x + c * VEC);
  group_sync<LOGN, GROUPS>();
  uint4* out4 = reinterpret_cast<uint4*>(base);
  const int t = ntt_tid<LOGN>();
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int G = j * Sh::THREADS + t;
    out4[G] = img4[eval_xpose_slot<CH>(G / CH, G % CH)];
  }
}

// The converse: an eval-layout polynomial at src (global, read-only; or shared memory in natural
// order) is staged into the image with contiguous 16-byte accesses (eval_xpose_stage), then each
// thread reads chunk c (VEC words) of its own block (eval_xpose_chunk) -- consumed chunk by chunk
// so only VEC extra registers are live.
template <typename T, int LOGN, int GROUPS, bool SRC_SMEM = false>
__device__ __forceinline__ void eval_xpose_stage(const T* src, T* img) {
  using Sh = NttShape<LOGN>;
  constexpr int CH = Sh::E * (int)sizeof(T) / 16;
  uint4* img4 = reinterpret_cast<uint4*>(img);
  const uint4* src4 = reinterpret_cast<const uint4*>(src);
  const int t = ntt_tid<LOGN>();
  if constexpr (CH == 4) {  // 16 registers: the loads fly across the WAR barrier
    uint4 w[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) w[j] = SRC_SMEM ? src4[j * Sh::THREADS + t] : __ldg(src4 + j * Sh::THREADS + t);
    group_sync<LOGN, GROUPS>();
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int G = j * Sh::THREADS + t;
      img4[eval_xpose_slot<CH>(G / CH, G % CH)] = w[j];
    }
  } else {  // 64-bit words (register-heavy kernels): load and place one chunk at a time
    group_sync<LOGN, GROUPS>();
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int G = j * Sh::THREADS + t;
      img4[eval_xpose_slot<CH>(G / CH, G % CH)] = SRC_SMEM ? src4[G] : __ldg(src4 + G);
    }
  }
  group_sync<LOGN, GROUPS>();
}
template <typename T, int LOGN>
__device__ __forceinline__ void eval_xpose_chunk(const T* img, int c, T* v) {
  using Sh = NttShape<LOGN>;
  constexpr int CH = Sh::E * (int)sizeof(T) / 16;
  unpack_chunk<T>(reinterpret_cast<const uint4*>(img)[eval_xpose_slot<CH>(eval_base<LOGN>() / Sh::E, c)], v);
}
template <typename T, int LOGN, int GROUPS, bool SRC_SMEM = false, typename F>
__device__ __forceinline__ void eval_xpose_apply(const T* src, T* img, F&& f) {
  using Sh = NttShape<LOGN>;
  constexpr int CH = Sh::E * (int)sizeof(T) / 16, VEC = 16 / (int)sizeof(T);
  eval_xpose_stage<T, LOGN, GROUPS, SRC_SMEM>(src, img);
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    T v[VEC];
    eval_xpose_chunk<T, LOGN>(img, c, v);
    f(c, v);
  }
}

// Eval layout ([npoly][N], e.g. prepared keys) -> thread-major chunk layout: chunk c of transform
// thread t at 16-byte index c * THREADS + t.  The eval layout gives thread t the block f(t)
// (ntt.cuh eval_xpose_*), so direct eval-layout key loads put every lane of a warp in its own
// 128-byte line; in this layout each warp load is 512 contiguous bytes.  One block per polynomial.
// TO_F64: the prepared operand (Montgomery domain, NTT * N^-1 * 2^W) leaves the Montgomery domain;
// 64-bit limbs store the bits of its centred double, the form the FP64 products take, 32-bit limbs
// the canonical word for the FP64-quotient products (`tabs` / `L`: the primes, block b being limb
// b % L).
template <typename T, int LOGN, bool TO_F64 = false>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS) k_eval_to_strip(const T* __restrict__ in, T* __restrict__ out,
                                                                          const PrimeTab<T>* __restrict__ tabs, int L) {
  using Sh = NttShape<LOGN>;
  using EV = EvalVec<T, LOGN>;
  const T* src = in + (size_t)blockIdx.x * Sh::N;
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)blockIdx.x * Sh::N);
  T p = 0, pinv = 0;
  if constexpr (TO_F64) {
    p = tabs[blockIdx.x % L].p;
    pinv = tabs[blockIdx.x % L].pinv;
  }
#pragma unroll
  for (int i = 0; i < EV::CHUNKS; ++i) {
    T v[EV::VEC];
    EV::load(src, i, v);
    if constexpr (TO_F64) {
#pragma unroll
      for (int c = 0; c < EV::VEC; ++c) {
        const T r = mont_mul(v[c], (T)1, p, pinv);   // x 2^-W: leaves the Montgomery domain, [0, p)
        if constexpr (sizeof(T) == 8) {
          const double dv = r > p / 2 ? -(double)(p - r) : (double)r;
          v[c] = (T)__double_as_longlong(dv);
        } else {
          v[c] = r;   // 32-bit limbs: the canonical word (FP64-quotient products convert it on use)
        }
      }
    }
    dst[i * Sh::THREADS + threadIdx.x] = pack_chunk<T>(v);
  }
}
// Load a PrimeTab into registers (uniform across the CTA).
template <typename T>
struct PrimeRegs {
  T p, p2, pinv, ninv, ninv_q, ninvr, ninvr_q, one_q, r2, r2_q, rr, c25, c25_q;
  const T* fwd;
  const T* inv;
  __device__ __forceinline__ explicit PrimeRegs(const PrimeTab<T>* tab) {
    p = tab->p; p2 = tab->p2; pinv = tab->pinv;
    ninv = tab->ninv; ninv_q = tab->ninv_q;
    ninvr = tab->ninvr; ninvr_q = tab->ninvr_q;
    one_q = tab->one_q; r2 = tab->r2; r2_q = tab->r2_q; rr = tab->rr;
    c25 = tab->c25; c25_q = tab->c25_q;
    fwd = tab->fwd; inv = tab->inv;
  }
  // Canonical [0, p) from a forward-transform output (u32: < 4p; u64: < 2^64).
  __device__ __forceinline__ T canon_fwd(T x) const {
    if constexpr (sizeof(T) == 4) return reduce4(x, p);
    else return csub(shoup_mul<uint64_t>(x, 1ull, one_q, p), p);
  }
  // Any 32-bit value into [0, p).
  __device__ __forceinline__ T reduce_digit(uint32_t v) const {
    return csub(shoup_mul<T>((T)v, (T)1, one_q, p), p);
  }
  // Reduce an arbitrary 64-bit value mod p into [0, 2p).
  __device__ __forceinline__ T reduce_u64_lazy(uint64_t v) const {
    if constexpr (sizeof(T) == 4) {
      uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
      uint32_t a = shoup_mul<uint32_t>(hi, r2, r2_q, p);   // hi * 2^32 mod p, [0,2p)
      uint32_t b = shoup_mul<uint32_t>(lo, 1u, one_q, p);  // lo mod p, [0,2p)
      return csub(a + b, p2);                               // [0,2p)
    } else {
      return shoup_mul<uint64_t>(v, 1ull, one_q, p);       // [0,2p)
    }
  }
};

// Centred lift of E plain values (he.py:325-327: v in [0, t) -> v - t when v > t/2, mod p) into
// the registers of a forward transform.  `src` points at coef_base().  32-bit limbs with `fast`
// (t < 2^57, p > 2^25): ONE Shoup product per value and no canonical reduction -- hi 2^25 + lo
// + (p - t mod p when v > t/2) < 2p + 2^25 + p < 4p, an admissible forward input (the butterflies
// take X in [0, 4p) and any 32-bit Y).  The branch on `fast` is hoisted out of the element loop:
// as a per-element select ptxas predicated both reductions and issued the unused one too (10 of
// 23 issue slots per value).  64-bit limbs with `fast` (t <= p): the value is its own residue.
// Otherwise canonical values in [0, p) through the general 64-bit reduction.
template <typename T, int LOGN>
__device__ __forceinline__ void lift_plain_regs(const uint64_t* __restrict__ src, T (&x)[NttShape<LOGN>::E],
                                                const PrimeRegs<T>& pr, T tmod, uint64_t t_half, bool fast) {
  using Sh = NttShape<LOGN>;
  if constexpr (sizeof(T) == 4) {
    if (fast) {
      const T ptm = pr.p - tmod;
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) {
        const uint64_t v = __ldg(src + coef_off<LOGN>(k));
        const uint32_t hi = (uint32_t)(v >> 25), lo = (uint32_t)v & ((1u << 25) - 1);
        x[k] = shoup_mul<uint32_t>(hi, pr.c25, pr.c25_q, pr.p) + lo + (v > t_half ? ptm : (T)0);
      }
      return;
    }
  } else {
    if (fast) {   // 64-bit limbs, t <= p: v is its own residue and t mod p = t -- no product
      const T ptm = pr.p - tmod;
#pragma unroll
      for (int k = 0; k < Sh::E; ++k) {
        const uint64_t v = __ldg(src + coef_off<LOGN>(k));
        x[k] = (T)(v > t_half ? v + ptm : v);              // canonical
      }
      return;
    }
  }
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) {
    const uint64_t v = __ldg(src + coef_off<LOGN>(k));
    T r = csub(pr.reduce_u64_lazy(v), pr.p);             // v mod p
    if (v > t_half) r = sub_mod(r, tmod, pr.p);           // centred lift: v - t
    x[k] = r;
  }
}

}  // namespace ctb
