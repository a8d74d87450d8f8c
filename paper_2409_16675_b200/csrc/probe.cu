// Roofline probe: register-resident throughput of the exact modular
// multiplication the butterflies use (Shoup, lazy [0,2p)), per word width.
// MEASURED_PEAKS.json carries no integer peak, so bench.py measures this one on
// the box and divides by it.
#include "ctb200.h"
#include "kernels.hpp"
#include <cmath>

using namespace ctb;

namespace {
constexpr int CHAINS = 8;

template <typename T>
__global__ void __launch_bounds__(256) k_probe_shoup(T* sink, uint64_t iters, T p, T w, T wq) {
  T a[CHAINS];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) a[j] = (T)(threadIdx.x * 131 + blockIdx.x * 7 + j) % p;
  for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) a[j] = shoup_mul(a[j], w, wq, p);
  }
  T acc = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) acc ^= a[j];
  if (acc == (T)0x5eed) sink[0] = acc;  // keep the chains alive
}

// The 32-bit butterfly mix of k_cpmul: NF of the 8 chains take their quotient from the FP64 pipe
// (ntt.cuh f64q_mul), the rest are Shoup products -- k_cpmul runs 12 of the 32 butterflies of a
// radix-16 pass (37.5% = 3/8) on the FP64 quotient.
// CONV: the quotient's operand converted with I2F.F64.U32 (as the kernels run it) or assembled by
// the exponent splice (the round-1 form).
template <int NF, bool CONV>
__global__ void __launch_bounds__(256) k_probe_mix(uint32_t* sink, uint64_t iters, uint32_t p, uint32_t w, uint32_t wq,
                                                   double wp) {
  uint32_t a[CHAINS];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) a[j] = (threadIdx.x * 131 + blockIdx.x * 7 + j) % p;
  const double kq = f64q_k(wp);
  const uint32_t pn = 0u - p;
  for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) a[j] = j < NF ? f64q_mul<CONV>(a[j], w, wp, kq, p, pn) : shoup_mul(a[j], w, wq, p);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) acc ^= a[j];
  if (acc == 0x5eedu) sink[0] = acc;
}
// The 50-bit product of the FP64 butterflies (ntt.cuh f64_mulmod): exact integers in doubles,
// centred twiddle, x w = hi + lo, q = rint(x w/p), r = (hi - q p) + lo -- 6 FP64 operations.
__global__ void __launch_bounds__(256) k_probe_f64(double* sink, uint64_t iters, double p, double w, double wp) {
  double a[CHAINS];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) a[j] = (double)((threadIdx.x * 131 + blockIdx.x * 7 + j) % 1000003);
  for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) a[j] = f64_mulmod(a[j], w, wp, p);
  }
  double acc = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) acc += a[j];
  if (acc == 12345.0) sink[0] = acc;
}
// The forward butterfly of the 64-bit-limb transforms as the kernels run it (ntt.cuh fwd_pass_f64):
// t = mulmod(Y, w), X' = X + t, Y' = X - t, every value centred once per 4 stages.  On the FP64
// pipe the butterfly's additions and its share of the lazy reduction cost as much as products, so
// this -- not the bare product -- is the ceiling of the transforms' own arithmetic; one modmul
// counted per butterfly.
__global__ void __launch_bounds__(256) k_probe_f64_bfly(double* sink, uint64_t iters, double p, double w,
                                                        double wp) {
  constexpr int PAIRS = CHAINS / 2;
  const F64Prime P{p, 1.0 / p};
  double x[CHAINS];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) x[j] = (double)((threadIdx.x * 131 + blockIdx.x * 7 + j) % 1000003);
  for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int st = 0; st < 4; ++st) {
#pragma unroll
      for (int j = 0; j < PAIRS; ++j) {
        const double X = x[2 * j];
        const double t = f64_mulmod(x[2 * j + 1], w, wp, p);
        x[2 * j] = __dadd_rn(X, t);
        x[2 * j + 1] = __dadd_rn(X, -t);
      }
    }
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) x[j] = f64_center(x[j], P);
  }
  double acc = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) acc += x[j];
  if (acc == 12345.0) sink[0] = acc;
}
}  // namespace

extern "C" int ctb_probe_bfly_f64(uint64_t iters, void* sink, uint64_t* modmuls, void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)sms * 8, block = 256;
  const uint64_t p = 1125899906826241ull;
  const double w = -(double)(p / 3);
  k_probe_f64_bfly<<<grid, block, 0, (cudaStream_t)stream>>>((double*)sink, iters, (double)p, w, w * (1.0 / (double)p));
  if (modmuls) *modmuls = (uint64_t)grid * block * (CHAINS / 2) * 4 * iters;
  return cuda_status(cudaGetLastError(), "ctb_probe_bfly_f64");
}

extern "C" int ctb_probe_modmul_f64(uint64_t iters, void* sink, uint64_t* modmuls, void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)sms * 8, block = 256;
  const uint64_t p = 1125899906826241ull;  // ntt_primes(8192, 50, 3)[0]
  const double w = -(double)(p / 3);        // a centred twiddle
  k_probe_f64<<<grid, block, 0, (cudaStream_t)stream>>>((double*)sink, iters, (double)p, w, w * (1.0 / (double)p));
  if (modmuls) *modmuls = (uint64_t)grid * block * CHAINS * iters;
  return cuda_status(cudaGetLastError(), "ctb_probe_modmul_f64");
}

// One radix-16 register pass of the 32-bit forward transform at N = 4096 exactly as k_cpmul runs it
// (ntt.cuh fwd_pass of the middle pass: 32 Harvey butterflies per thread -- conditional subtraction,
// product, sum, difference -- twiddles from the prime's table staged in shared memory, FP64 quotients
// on the first two entries), repeated register-resident: no exchanges, no global traffic, one
// 1024-thread CTA per SM like k_cpmul.  The ceiling of a transform's own arithmetic: the modmul
// probes above leave out the butterflies' ALU-pipe additions, which co-limit the kernels.
template <int LOGN>
__global__ void __launch_bounds__(1024, 1) k_probe_bfly_pass(uint32_t* sink, uint64_t iters,
                                                             const PrimeTab<uint32_t>* __restrict__ tabs) {
  using Sh = NttShape<LOGN>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* tw_sm = reinterpret_cast<uint32_t*>(smem_raw);
  PrimeRegs<uint32_t> pr(tabs);
  stage_twiddles(pr.fwd, tw_sm, tw_words<uint32_t>(LOGN), 1024);
  __syncthreads();
  const TwSrc<uint32_t, true> tw{tw_sm};
  uint32_t x[Sh::E];
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) x[k] = (threadIdx.x * 2654435761u + k * 40503u + blockIdx.x) % pr.p;
  for (uint64_t i = 0; i < iters; ++i) fwd_pass<uint32_t, LOGN, 1, true>(x, tw, pr.p, pr.p2);
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) acc ^= x[k];
  if (acc == 0x5eedu) sink[0] = acc;
}

extern "C" int ctb_probe_bfly_pass(const ctb_ctx_t* ctx, uint64_t iters, void* sink, uint64_t* bflys, void* stream) {
  if (!ctx) { set_error("ctb_probe_bfly_pass: null context"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  const Base& b = c->base[BASE_Q];
  if (c->logn != 12 || b.word != 4) { set_error("ctb_probe_bfly_pass: needs N = 4096 and 32-bit cipher limbs"); return ERR_ARG; }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = (size_t)tw_words<uint32_t>(12) * 4;
  auto kern = k_probe_bfly_pass<12>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_status(e, "ctb_probe_bfly_pass");
  kern<<<(unsigned)sms, 1024, smem, (cudaStream_t)stream>>>((uint32_t*)sink, iters, (const PrimeTab<uint32_t>*)b.d_tabs);
  if (bflys) *bflys = (uint64_t)sms * 1024 * 32 * iters;
  return cuda_status(cudaGetLastError(), "ctb_probe_bfly_pass");
}

static int probe_mix(int f64q_of_8, bool conv, uint64_t iters, void* sink, uint64_t* modmuls, void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)sms * 8, block = 256;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t p = 1073692673u, w = 510015274u;
  const uint32_t wq = (uint32_t)(((uint64_t)w << 32) / p);
  const double wp = std::ldexp((double)(uint64_t)((((unsigned __int128)w << 52) + p / 2) / p), -52);
  uint32_t* o = (uint32_t*)sink;
  switch (f64q_of_8 + (conv ? 16 : 0)) {
    case 0: case 16: k_probe_mix<0, false><<<grid, block, 0, s>>>(o, iters, p, w, wq, wp); break;
    case 3: k_probe_mix<3, false><<<grid, block, 0, s>>>(o, iters, p, w, wq, wp); break;
    case 8: k_probe_mix<8, false><<<grid, block, 0, s>>>(o, iters, p, w, wq, wp); break;
    case 19: k_probe_mix<3, true><<<grid, block, 0, s>>>(o, iters, p, w, wq, wp); break;
    case 24: k_probe_mix<8, true><<<grid, block, 0, s>>>(o, iters, p, w, wq, wp); break;
    default:
      set_error("ctb_probe_modmul_mix: f64q_of_8 must be 0, 3 or 8");
      return ERR_ARG;
  }
  if (modmuls) *modmuls = (uint64_t)grid * block * CHAINS * iters;
  return cuda_status(cudaGetLastError(), "ctb_probe_modmul_mix");
}
extern "C" int ctb_probe_modmul_mix(int f64q_of_8, uint64_t iters, void* sink, uint64_t* modmuls, void* stream) {
  return probe_mix(f64q_of_8, true, iters, sink, modmuls, stream);
}
extern "C" int ctb_probe_modmul_mix_splice(int f64q_of_8, uint64_t iters, void* sink, uint64_t* modmuls, void* stream) {
  return probe_mix(f64q_of_8, false, iters, sink, modmuls, stream);
}

extern "C" int ctb_probe_modmul(int word_bytes, uint64_t iters, void* sink, uint64_t* modmuls,
                                void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)sms * 8, block = 256;
  cudaStream_t s = (cudaStream_t)stream;
  if (word_bytes == 4) {
    const uint32_t p = 1073692673u, w = 510015274u;
    const uint32_t wq = (uint32_t)(((uint64_t)w << 32) / p);
    k_probe_shoup<uint32_t><<<grid, block, 0, s>>>((uint32_t*)sink, iters, p, w, wq);
  } else if (word_bytes == 8) {
    const uint64_t p = 1125899906826241ull, w = 123456789012345ull;
    const uint64_t wq = (uint64_t)(((unsigned __int128)w << 64) / p);
    k_probe_shoup<uint64_t><<<grid, block, 0, s>>>((uint64_t*)sink, iters, p, w, wq);
  } else {
    set_error("ctb_probe_modmul: word_bytes must be 4 or 8");
    return ERR_ARG;
  }
  if (modmuls) *modmuls = (uint64_t)grid * block * CHAINS * iters;
  return cuda_status(cudaGetLastError(), "ctb_probe_modmul");
}

// Device self-check of the FP64-quotient tables (ntt.cuh F64Q_NE) of one 32-bit base: for every
// prime and every quotient-table entry, f64q_mul(a, w, w'/p) must lie in [0, 2p) and equal a*w
// mod p, for the boundary inputs the butterflies can present (0, 1, p-1, p, 2p-1, 2p, 3p, 4p-1,
// 2^32-1) and `samples` pseudo-random a in [0, 2^32).  One CTA per (prime, entry).
namespace {
__global__ void k_check_f64q(const uint32_t* tw, int words, const uint64_t* primes, int logn, uint64_t samples,
                             uint64_t seed, unsigned long long* bad) {
  const int l = blockIdx.y;
  const uint32_t p = (uint32_t)primes[l];
  const uint32_t* f = tw + (size_t)l * words;
  const double* qt = reinterpret_cast<const double*>(f + 2 * shape_tw_entries(logn));
  // entry blockIdx.x -> (pass k, e, slot)
  int idx = blockIdx.x, k = 0;
  for (; k < shape_npass(logn); ++k) {
    const int n_k = F64Q_NE << shape_pass_s(logn, k);
    if (idx < n_k) break;
    idx -= n_k;
  }
  if (k == shape_npass(logn)) return;
  const int s = shape_pass_s(logn, k), r = shape_pass_r(logn, k);
  const int e = idx >> s, slot = idx & ((1 << s) - 1);
  if (e >= (1 << r) - 1) return;  // no such stage/block in a short pass: entry unused
  const uint32_t w = f[2 * shape_tw_pair(logn, k, e, slot)];
  const double wp = qt[shape_q_index(logn, k, e, slot)];
  const double kq = f64q_k(wp);
  const uint32_t pn = 0u - p;
  unsigned long long nbad = 0;
  const uint32_t edge[9] = {0u, 1u, p - 1, p, 2 * p - 1, 2 * p, 3 * p, 4 * p - 1, 0xFFFFFFFFu};
  for (uint64_t i = threadIdx.x; i < samples + 9; i += blockDim.x) {
    uint32_t a;
    if (i < 9) {
      a = edge[i];
    } else {  // splitmix64
      uint64_t z = seed + (uint64_t)l * 0x9E3779B97F4A7C15ull + (uint64_t)blockIdx.x * 0xBF58476D1CE4E5B9ull + i * 0x94D049BB133111EBull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      a = (uint32_t)(z ^ (z >> 31));
    }
    const uint32_t res = f64q_mul<true>(a, w, wp, kq, p, pn), res2 = f64q_mul<false>(a, w, wp, kq, p, pn);
    if (res2 != res) ++nbad;   // both quotient forms agree
    if (res >= 2 * p || res % p != (uint32_t)((uint64_t)a * w % p)) ++nbad;
  }
  if (nbad) atomicAdd(bad, nbad);
}
}  // namespace

extern "C" int ctb_check_f64q(const ctb_ctx_t* ctx, int base, uint64_t samples, uint64_t seed, uint64_t* bad,
                              void* stream) {
  if (!ctx || base < 0 || base >= BASE_COUNT || !bad) { set_error("ctb_check_f64q: bad arguments"); return ERR_ARG; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  const Base& b = c->base[base];
  if (!b.size()) { set_error("ctb_check_f64q: empty base"); return ERR_ARG; }
  *bad = 0;
  if (b.word != 4 || F64Q_NE == 0) return OK;  // 64-bit limbs run the FP64 butterflies; nothing to check
  cudaStream_t s = (cudaStream_t)stream;
  const int logn = (int)c->logn;
  unsigned long long* d_bad = nullptr;
  uint64_t* d_primes = nullptr;
  cudaError_t e = cudaMallocAsync(&d_bad, sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_primes, 8 * b.primes.size(), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_bad, 0, sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_primes, b.primes.data(), 8 * b.primes.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    const dim3 grid((unsigned)shape_q_off(logn, shape_npass(logn)), (unsigned)b.size());
    k_check_f64q<<<grid, 256, 0, s>>>((const uint32_t*)b.d_tw, tw_words<uint32_t>(logn), d_primes, logn, samples, seed,
                                      d_bad);
    e = cudaGetLastError();
  }
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d_bad, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (d_bad) cudaFreeAsync(d_bad, s);
  if (d_primes) cudaFreeAsync(d_primes, s);
  *bad = h;
  return cuda_status(e, "ctb_check_f64q");
}
