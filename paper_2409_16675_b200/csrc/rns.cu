// Exact conversions between the cipher base's residues and integers.
//
//   ctb_decrypt_round  he.py:347-349  out = floor((v t + floor(q/2)) / q) mod t
//   ctb_decrypt_round_extract  the same, fused with the client's c - p and job.extract (linprot.py:444-452)
//   ctb_rns_to_pos     ring.py:592-599 positional little-endian 64-bit words (wire format)
//   ctb_pos_to_rns     ring.py:602-615 the inverse (from_ints: value mod q)
//
// Decrypt rounding without big integers: with h = (q-1)/2 and
// R = (v t + h) mod q, the quotient is w = (v t + h - R) / q.  Modulo a plain
// prime t_j (which divides t), v t + h == h, so w == (h - R) q^-1 (mod t_j):
// one Garner conversion of R per coefficient, Horner-evaluated mod each t_j,
// then the plain CRT gives w mod t exactly (0 <= w <= t).
#include <algorithm>
#include <cstring>
#include <vector>
#include "bigint.hpp"
#include "ctb200.h"
#include "kernels.hpp"
#include "rns.cuh"

namespace ctb {

struct PlainEval {
  int LT = 0;
  uint32_t tp[2], oneq[2], r2[2], r2q[2];
  ShoupC<uint32_t> hc[2][MAX_MRC];  // q_k mod t_j, k < L-1
  uint32_t h_t[2];                  // h mod t_j
  ShoupC<uint32_t> qinv_t[2];       // q^-1 mod t_j
  ShoupC<uint32_t> crt;             // t0^-1 mod t1
};

template <typename T>
struct QConsts {
  MrcTab<T> mrc;
  ShoupC<T> t_q[MAX_MRC];   // t mod q_i
  T h_q[MAX_MRC];           // h mod q_i
  T r2[MAX_MRC];            // 2^W mod q_i  (u32: reducing 64-bit words)
  T r2q[MAX_MRC];
  int W;                    // 64-bit words per coefficient on the wire (ring.limb_count)
  ShoupC<T> pow64[MAX_MRC][8];  // 2^(64 k) mod q_i
  PlainEval pe;
};

// Decrypt rounding for u32 limbs by value (constant bank), lazy 64-bit accumulation:
// Garner digits a_j = (R_j - sum_{i<j} a_i M_i) M_j^-1 mod q_j, and R mod t_j as one dot
// product sum_i a_i (M_i mod t_j) (30-bit digits x 25-bit constants, one reduction).
constexpr int DEC_MAXQ = 8;
struct DecLazy {
  int L, LT;
  uint32_t q[DEC_MAXQ], one_q[DEC_MAXQ], r2[DEC_MAXQ], r2q[DEC_MAXQ], h_q[DEC_MAXQ];
  ShoupC<uint32_t> t_q[DEC_MAXQ];
  uint32_t gM[DEC_MAXQ][DEC_MAXQ];  // M_i mod q_j (i < j)
  ShoupC<uint32_t> gMinv[DEC_MAXQ];
  uint32_t tM[2][DEC_MAXQ];         // M_i mod t_j
  uint32_t tp[2], t_oneq[2], t_r2[2], t_r2q[2], h_t[2];
  ShoupC<uint32_t> qinv_t[2], crt;
};

// Optional epilogue of the decrypt rounding kernels (ctb_decrypt_round_extract): the client's
// unmasking c - p (linprot.py:444-450) and the job's extraction (packing.extract_output +
// to_signed_matrix, packing.py:476-522) as a scatter through per-kind degree maps.  With maps set,
// coefficients that are not outputs are skipped before any rounding work.
struct DecEpi {
  const uint64_t* sub = nullptr;   // [n][N] plain values subtracted mod t (may be null)
  const int32_t* maps = nullptr;   // [n_maps][N] destination offsets (-1: not an output); null: identity
  const int32_t* kind = nullptr;   // [n] map row per polynomial
  const int64_t* base = nullptr;   // [n] destination base per polynomial
  uint32_t n_maps = 0;
  int centered = 0;                // store (-t/2, t/2] signed values
  uint64_t dst_len = 0;
  uint64_t t = 0;
};

// destination of coefficient i of polynomial b, or -1 when the epilogue drops it
__device__ __forceinline__ int64_t epi_dst(const DecEpi& e, uint64_t b, uint64_t i, uint32_t n, uint64_t g) {
  if (!e.maps) return (int64_t)g;
  const uint32_t k = (uint32_t)e.kind[b];
  if (k >= e.n_maps) return -1;
  const int32_t m = e.maps[(uint64_t)k * n + i];
  if (m < 0) return -1;
  const uint64_t dst = (uint64_t)e.base[b] + (uint64_t)m;
  return dst < e.dst_len ? (int64_t)dst : -1;
}

__device__ __forceinline__ void epi_store(const DecEpi& e, uint64_t* out, int64_t dst, uint64_t g, uint64_t v) {
  if (e.sub) {
    const uint64_t b = e.sub[g];
    v = v >= b ? v - b : v + e.t - b;
  }
  if (e.centered && v > e.t / 2) v -= e.t;  // two's complement int64 view
  out[dst] = v;
}

struct RnsConsts {
  void* d_q = nullptr;  // QConsts<T> for the cipher base
  int word = 4;
  int W = 1;
  bool lazy = false;
  DecLazy dec{};
  ~RnsConsts() {
    if (d_q) cudaFree(d_q);
  }
};

// ----------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t red64_u32(uint64_t v, uint32_t m, uint32_t oneq, uint32_t r2, uint32_t r2q) {
  const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
  const uint32_t a = shoup_mul<uint32_t>(hi, r2, r2q, m);
  const uint32_t b = shoup_mul<uint32_t>(lo, 1u, oneq, m);
  return csub(csub(a + b, 2 * m), m);  // a,b < 2m < 2^31
}

template <typename T>
__device__ __forceinline__ T red64(uint64_t v, T m, T oneq, T r2, T r2q) {
  if constexpr (sizeof(T) == 4) return red64_u32(v, m, oneq, r2, r2q);
  else return csub(shoup_mul<uint64_t>(v, 1ull, oneq, m), m);
}

// Horner of mixed-radix digits (any word) mod a 32-bit prime.
template <typename T>
__device__ __forceinline__ uint32_t eval_mod_plain(int L, const T* a, const PlainEval& pe, int j) {
  const uint32_t m = pe.tp[j];
  uint32_t acc = red64_u32((uint64_t)a[L - 1], m, pe.oneq[j], pe.r2[j], pe.r2q[j]);
  for (int k = L - 2; k >= 0; --k) {
    acc = csub(shoup_mul<uint32_t>(acc, pe.hc[j][k].w, pe.hc[j][k].wq, m), m);
    acc = add_mod(acc, red64_u32((uint64_t)a[k], m, pe.oneq[j], pe.r2[j], pe.r2q[j]), m);
  }
  return acc;
}

template <typename T>
__global__ void k_decrypt_round(const T* v, uint64_t* out, const QConsts<T>* __restrict__ cq, uint32_t n,
                                uint64_t total, const DecEpi epi) {
  __shared__ QConsts<T> c;
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(cq);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&c);
    for (int i = threadIdx.x; i < (int)(sizeof(QConsts<T>) / 4); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int L = c.mrc.L;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = g >> pow2_shift(n), i = g & (n - 1);  // n = ring degree (power of two)
    const int64_t dst = epi_dst(epi, b, i, n, g);
    if (dst < 0) continue;
    T r[MAX_MRC], a[MAX_MRC];
    for (int l = 0; l < L; ++l) {
      const T q = c.mrc.q[l];
      const T x = v[(b * L + l) * n + i];
      r[l] = add_mod(csub(shoup_mul<T>(x, c.t_q[l].w, c.t_q[l].wq, q), q), c.h_q[l], q);  // (v t + h) mod q_l
    }
    mrc_digits(c.mrc, r, a);
    uint32_t w[2];
    for (int j = 0; j < c.pe.LT; ++j) {
      const uint32_t m = c.pe.tp[j];
      const uint32_t Rj = eval_mod_plain(L, a, c.pe, j);
      const uint32_t d = sub_mod(c.pe.h_t[j], Rj, m);
      w[j] = csub(shoup_mul<uint32_t>(d, c.pe.qinv_t[j].w, c.pe.qinv_t[j].wq, m), m);
    }
    uint64_t res = w[0];
    if (c.pe.LT == 2) {
      const uint32_t m1 = c.pe.tp[1];
      const uint32_t w0m = red64_u32(w[0], m1, c.pe.oneq[1], c.pe.r2[1], c.pe.r2q[1]);
      const uint32_t d = csub(shoup_mul<uint32_t>(sub_mod(w[1], w0m, m1), c.pe.crt.w, c.pe.crt.wq, m1), m1);
      res = (uint64_t)w[0] + (uint64_t)c.pe.tp[0] * d;
    }
    epi_store(epi, out, dst, g, res);
  }
}

template <int LC>
__global__ void __launch_bounds__(256) k_decrypt_round_lazy(const uint32_t* v, uint64_t* out,
                                                            const __grid_constant__ DecLazy c, uint32_t n,
                                                            uint64_t total, const __grid_constant__ DecEpi epi) {
  const int L = LC ? LC : c.L;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = g >> pow2_shift(n), i = g & (n - 1);  // n = ring degree (power of two)
    const int64_t dst = epi_dst(epi, b, i, n, g);
    if (dst < 0) continue;
    uint32_t a[DEC_MAXQ];
#pragma unroll
    for (int j = 0; j < (LC ? LC : DEC_MAXQ); ++j) {
      if (!LC && j >= L) break;
      const uint32_t q = c.q[j];
      const uint32_t x = v[(b * L + j) * n + i];
      const uint32_t r = add_mod(csub(shoup_mul<uint32_t>(x, c.t_q[j].w, c.t_q[j].wq, q), q), c.h_q[j], q);
      if (j == 0) {
        a[0] = r;
      } else {
        uint64_t sacc = 0;
#pragma unroll
        for (int k = 0; k < j; ++k) sacc += (uint64_t)a[k] * c.gM[j][k];
        const uint32_t sj = red64_u32(sacc, q, c.one_q[j], c.r2[j], c.r2q[j]);
        a[j] = csub(shoup_mul<uint32_t>(sub_mod(r, sj, q), c.gMinv[j].w, c.gMinv[j].wq, q), q);
      }
    }
    uint32_t w[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      if (t >= c.LT) break;
      uint64_t sacc = 0;
#pragma unroll
      for (int k = 0; k < (LC ? LC : DEC_MAXQ); ++k) {
        if (!LC && k >= L) break;
        sacc += (uint64_t)a[k] * c.tM[t][k];
      }
      const uint32_t m = c.tp[t];
      const uint32_t Rj = red64_u32(sacc, m, c.t_oneq[t], c.t_r2[t], c.t_r2q[t]);
      const uint32_t d = sub_mod(c.h_t[t], Rj, m);
      w[t] = csub(shoup_mul<uint32_t>(d, c.qinv_t[t].w, c.qinv_t[t].wq, m), m);
    }
    uint64_t res = w[0];
    if (c.LT == 2) {
      const uint32_t m1 = c.tp[1];
      const uint32_t w0m = red64_u32(w[0], m1, c.t_oneq[1], c.t_r2[1], c.t_r2q[1]);
      const uint32_t d = csub(shoup_mul<uint32_t>(sub_mod(w[1], w0m, m1), c.crt.w, c.crt.wq, m1), m1);
      res = (uint64_t)w[0] + (uint64_t)c.tp[0] * d;
    }
    epi_store(epi, out, dst, g, res);
  }
}

template <typename T>
__global__ void k_rns_to_pos(const T* x, uint64_t* out, const QConsts<T>* __restrict__ cq, uint32_t n,
                             uint64_t total) {
  __shared__ MrcTab<T> m;
  __shared__ int W;
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&cq->mrc);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&m);
    for (int i = threadIdx.x; i < (int)(sizeof(MrcTab<T>) / 4); i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0) W = cq->W;
  }
  __syncthreads();
  const int L = m.L;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = g >> pow2_shift(n), i = g & (n - 1);  // n = ring degree (power of two)
    T r[MAX_MRC], a[MAX_MRC];
    for (int l = 0; l < L; ++l) r[l] = x[(b * L + l) * n + i];
    mrc_digits(m, r, a);
    uint32_t X[2 * 8 + 2];
    mrc_positional(m, a, X, 2 * W + 2);
    for (int w = 0; w < W; ++w) out[g * W + w] = (uint64_t)X[2 * w] | ((uint64_t)X[2 * w + 1] << 32);
  }
}

template <typename T>
__global__ void k_pos_to_rns(const uint64_t* in, T* x, const QConsts<T>* __restrict__ cq, uint32_t n,
                             uint64_t total) {
  __shared__ QConsts<T> c;
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(cq);
    uint32_t* dst = reinterpret_cast<uint32_t*>(&c);
    for (int i = threadIdx.x; i < (int)(sizeof(QConsts<T>) / 4); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int L = c.mrc.L, W = c.W;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = g >> pow2_shift(n), i = g & (n - 1);  // n = ring degree (power of two)
    uint64_t words[8];
    for (int w = 0; w < W; ++w) words[w] = in[g * W + w];
    for (int l = 0; l < L; ++l) {
      const T q = c.mrc.q[l];
      T acc = 0;
      for (int w = 0; w < W; ++w) {
        const T d = red64<T>(words[w], q, c.mrc.one_q[l], c.r2[l], c.r2q[l]);
        acc = add_mod(acc, csub(shoup_mul<T>(d, c.pow64[l][w].w, c.pow64[l][w].wq, q), q), q);
      }
      x[(b * L + l) * n + i] = acc;
    }
  }
}

// ----------------------------------------------------------------- host constants
template <typename T>
static ShoupC<T> shoup_pair(uint64_t w, uint64_t p) {
  constexpr int W = 8 * sizeof(T);
  return ShoupC<T>{(T)w, (T)(((unsigned __int128)w << W) / p)};
}

template <typename T>
static void fill_mrc(MrcTab<T>& m, const std::vector<uint64_t>& q) {
  constexpr int W = 8 * sizeof(T);
  m.L = (int)q.size();
  for (int j = 0; j < m.L; ++j) {
    m.q[j] = (T)q[j];
    m.q2[j] = (T)(2 * q[j]);
    m.one_q[j] = (T)(((unsigned __int128)1 << W) / q[j]);
    for (int i = 0; i < j; ++i) m.inv[j * (j - 1) / 2 + i] = shoup_pair<T>(invmod(q[i] % q[j], q[j]), q[j]);
  }
}

template <typename T>
static int build_q_consts(Ctx* c, RnsConsts* rc, std::string& err) {
  const std::vector<uint64_t>& q = c->base[BASE_Q].primes;
  const std::vector<uint64_t>& tp = c->base[BASE_T].primes;
  constexpr int W = 8 * sizeof(T);
  if ((int)q.size() > MAX_MRC) { err = "too many cipher primes for the exact conversions"; return -3; }
  auto* h = new QConsts<T>();
  std::memset((void*)h, 0, sizeof(QConsts<T>));
  fill_mrc(h->mrc, q);
  BigU Q(1);
  for (uint64_t p : q) Q.mul_small(p);
  BigU hq = BigU::sub(Q, BigU(1));  // h = (q - 1) / 2  (q odd)
  hq.shr1();
  h->W = std::max<int>(1, (int)((Q.bit_length() + 63) / 64));
  if (h->W > 8) { delete h; err = "cipher modulus above 512 bits"; return -3; }
  for (size_t i = 0; i < q.size(); ++i) {
    h->t_q[i] = shoup_pair<T>(c->t % q[i], q[i]);
    h->h_q[i] = (T)hq.mod_small(q[i]);
    const uint64_t r2 = (uint64_t)(((unsigned __int128)1 << W) % q[i]);
    h->r2[i] = (T)(sizeof(T) == 4 ? r2 : 0);
    h->r2q[i] = (T)(sizeof(T) == 4 ? (uint64_t)(((unsigned __int128)r2 << W) / q[i]) : 0);
    uint64_t pw = 1;  // 2^(64 k) mod q_i
    const uint64_t two64 = (uint64_t)(((unsigned __int128)1 << 64) % q[i]);
    for (int k = 0; k < h->W; ++k) {
      h->pow64[i][k] = shoup_pair<T>(pw, q[i]);
      pw = mulmod(pw, two64, q[i]);
    }
  }
  PlainEval& pe = h->pe;
  pe.LT = (int)tp.size();
  if (pe.LT > 2) { delete h; err = "plain modulus must have at most 2 primes"; return -3; }
  for (int j = 0; j < pe.LT; ++j) {
    const uint64_t m = tp[j];
    pe.tp[j] = (uint32_t)m;
    pe.oneq[j] = (uint32_t)(((uint64_t)1 << 32) / m);
    const uint64_t r2 = ((uint64_t)1 << 32) % m;
    pe.r2[j] = (uint32_t)r2;
    pe.r2q[j] = (uint32_t)((r2 << 32) / m);
    for (size_t k = 0; k + 1 < q.size(); ++k) pe.hc[j][k] = shoup_pair<uint32_t>(q[k] % m, m);
    pe.h_t[j] = (uint32_t)hq.mod_small(m);
    pe.qinv_t[j] = shoup_pair<uint32_t>(invmod(Q.mod_small(m), m), m);
  }
  if (pe.LT == 2) pe.crt = shoup_pair<uint32_t>(invmod(tp[0] % tp[1], tp[1]), tp[1]);
  if (sizeof(T) == 4 && (int)q.size() <= DEC_MAXQ && pe.LT >= 1) {
    DecLazy& d = rc->dec;
    d.L = (int)q.size();
    d.LT = pe.LT;
    std::vector<BigU> M(q.size() + 1, BigU(1));
    for (size_t i = 1; i <= q.size(); ++i) { M[i] = M[i - 1]; M[i].mul_small(q[i - 1]); }
    for (size_t j = 0; j < q.size(); ++j) {
      d.q[j] = (uint32_t)q[j];
      d.one_q[j] = (uint32_t)h->mrc.one_q[j];
      d.r2[j] = (uint32_t)h->r2[j];
      d.r2q[j] = (uint32_t)h->r2q[j];
      d.h_q[j] = (uint32_t)h->h_q[j];
      d.t_q[j] = ShoupC<uint32_t>{(uint32_t)h->t_q[j].w, (uint32_t)h->t_q[j].wq};
      for (size_t i = 0; i < j; ++i) d.gM[j][i] = (uint32_t)M[i].mod_small(q[j]);
      d.gMinv[j] = shoup_pair<uint32_t>(invmod(M[j].mod_small(q[j]), q[j]), q[j]);
    }
    for (int j = 0; j < pe.LT; ++j) {
      d.tp[j] = pe.tp[j]; d.t_oneq[j] = pe.oneq[j]; d.t_r2[j] = pe.r2[j]; d.t_r2q[j] = pe.r2q[j];
      d.h_t[j] = pe.h_t[j]; d.qinv_t[j] = pe.qinv_t[j];
      for (size_t i = 0; i < q.size(); ++i) d.tM[j][i] = (uint32_t)M[i].mod_small(tp[j]);
    }
    d.crt = pe.crt;
    rc->lazy = true;
  }
  cudaError_t e = cudaMalloc(&rc->d_q, sizeof(QConsts<T>));
  if (e == cudaSuccess) e = cudaMemcpy(rc->d_q, h, sizeof(QConsts<T>), cudaMemcpyHostToDevice);
  rc->W = h->W;
  delete h;
  if (e != cudaSuccess) { err = std::string("rns constants: ") + cudaGetErrorString(e); return -2; }
  return 0;
}

int build_rns_consts(Ctx* c, std::string& err) {
  auto* rc = new RnsConsts();
  rc->word = c->base[BASE_Q].word;
  const int rcode = rc->word == 4 ? build_q_consts<uint32_t>(c, rc, err) : build_q_consts<uint64_t>(c, rc, err);
  if (rcode) { delete rc; return rcode; }
  c->rns = rc;
  return 0;
}

void free_rns_consts(RnsConsts* rc) { delete rc; }
int rns_words(const RnsConsts* rc) { return rc ? rc->W : 0; }

}  // namespace ctb

using namespace ctb;


namespace {
int launch_decrypt_round(const Ctx* c, const void* v, uint64_t* out, uint64_t n_polys, const DecEpi& epi,
                         cudaStream_t s) {
  const uint64_t total = n_polys * c->n;
  if (!total) return OK;
  if (c->rns->lazy) {
    if (c->rns->dec.L == 7)
      k_decrypt_round_lazy<7><<<grid_stride(total, 8), 256, 0, s>>>((const uint32_t*)v, out, c->rns->dec, c->n, total,
                                                                    epi);
    else
      k_decrypt_round_lazy<0><<<grid_stride(total, 8), 256, 0, s>>>((const uint32_t*)v, out, c->rns->dec, c->n, total,
                                                                    epi);
  } else if (c->rns->word == 4)
    k_decrypt_round<uint32_t><<<grid_stride(total, 8), 256, 0, s>>>((const uint32_t*)v, out,
                                                              (const QConsts<uint32_t>*)c->rns->d_q, c->n, total, epi);
  else
    k_decrypt_round<uint64_t><<<grid_stride(total, 8), 256, 0, s>>>((const uint64_t*)v, out,
                                                              (const QConsts<uint64_t>*)c->rns->d_q, c->n, total, epi);
  return cuda_status(cudaGetLastError(), "ctb_decrypt_round");
}
}  // namespace

extern "C" int ctb_decrypt_round(const ctb_ctx_t* ctx, const void* v, uint64_t* out, uint64_t n_polys,
                                 void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !c->rns || !c->t || !v || !out) { set_error("ctb_decrypt_round: context lacks plain ring or bad buffer"); return ERR_ARG; }
  return launch_decrypt_round(c, v, out, n_polys, DecEpi{}, (cudaStream_t)stream);
}

extern "C" int ctb_decrypt_round_extract(const ctb_ctx_t* ctx, const void* v, const uint64_t* sub,
                                         const int32_t* maps, uint32_t n_maps, const int32_t* kind,
                                         const int64_t* base, uint64_t dst_len, int centered, int64_t* out,
                                         uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !c->rns || !c->t || !v || !maps || !kind || !base || (dst_len && !out)) {
    set_error("ctb_decrypt_round_extract: context lacks plain ring or bad buffer");
    return ERR_ARG;
  }
  DecEpi e;
  e.sub = sub;
  e.maps = maps;
  e.kind = kind;
  e.base = base;
  e.n_maps = n_maps;
  e.centered = centered;
  e.dst_len = dst_len;
  e.t = c->t;
  return launch_decrypt_round(c, v, reinterpret_cast<uint64_t*>(out), n_polys, e, (cudaStream_t)stream);
}

extern "C" int ctb_rns_to_pos(const ctb_ctx_t* ctx, const void* x, uint64_t* out, uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !c->rns || !x || !out) { set_error("ctb_rns_to_pos: bad context or buffer"); return ERR_ARG; }
  const uint64_t total = n_polys * c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (c->rns->word == 4)
    k_rns_to_pos<uint32_t><<<grid_stride(total, 8), 256, 0, s>>>((const uint32_t*)x, out,
                                                           (const QConsts<uint32_t>*)c->rns->d_q, c->n, total);
  else
    k_rns_to_pos<uint64_t><<<grid_stride(total, 8), 256, 0, s>>>((const uint64_t*)x, out,
                                                           (const QConsts<uint64_t>*)c->rns->d_q, c->n, total);
  return cuda_status(cudaGetLastError(), "ctb_rns_to_pos");
}

extern "C" int ctb_pos_to_rns(const ctb_ctx_t* ctx, const uint64_t* in, void* x, uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !c->rns || !in || !x) { set_error("ctb_pos_to_rns: bad context or buffer"); return ERR_ARG; }
  const uint64_t total = n_polys * c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (c->rns->word == 4)
    k_pos_to_rns<uint32_t><<<grid_stride(total, 8), 256, 0, s>>>(in, (uint32_t*)x, (const QConsts<uint32_t>*)c->rns->d_q,
                                                           c->n, total);
  else
    k_pos_to_rns<uint64_t><<<grid_stride(total, 8), 256, 0, s>>>(in, (uint64_t*)x, (const QConsts<uint64_t>*)c->rns->d_q,
                                                           c->n, total);
  return cuda_status(cudaGetLastError(), "ctb_pos_to_rns");
}

extern "C" int ctb_ctx_pos_words(const ctb_ctx_t* ctx) {
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  return c ? rns_words(c->rns) : ERR_ARG;
}
