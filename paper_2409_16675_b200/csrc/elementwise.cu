// Coefficient-wise ring operations (ring.py:363-401) and lifts (he.py:292-327).
//
//   ctb_rns_elementwise   ring_add / ring_sub / ring_neg on residues        ring.py:363-389
//   ctb_rns_scalar_mul    ring_scalar_mul (per-limb constant)              ring.py:392-401
//   ctb_rns_from_small    RingElem.from_ints of small signed ints (s, u, e) ring.py:267-279
//   ctb_lift_plain        scale * centred lift of plain values into Z_q    he.py:318, 325-327
//   ctb_plain_elementwise the same ops mod t on uint64 plain values
#include <algorithm>
#include "ctb200.h"
#include "kernels.hpp"

using namespace ctb;

namespace {

constexpr int MAXL = 24;

template <typename T>
struct LimbConsts {
  T p[MAXL];
  T s[MAXL], sq[MAXL];  // Shoup pair per limb (scalar) or t mod p (lift)
  T oneq[MAXL], r2[MAXL], r2q[MAXL];
  T tm[MAXL];           // plain modulus t mod p (centred lift)
};


template <typename T>
__device__ __forceinline__ T reduce_word(uint64_t v, const LimbConsts<T>& c, int l) {
  if constexpr (sizeof(T) == 4) {
    const uint32_t p = c.p[l];
    const uint32_t a = shoup_mul<uint32_t>((uint32_t)(v >> 32), c.r2[l], c.r2q[l], p);
    const uint32_t b = shoup_mul<uint32_t>((uint32_t)v, 1u, c.oneq[l], p);
    return csub(csub(a + b, 2 * p), p);
  } else {
    return csub(shoup_mul<uint64_t>(v, 1ull, c.oneq[l], c.p[l]), c.p[l]);
  }
}

template <typename T>
__global__ void k_rns_elementwise(int op, const T* a, const T* b, T* out, LimbConsts<T> c, int L, uint32_t n,
                                  uint64_t total) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const int l = (int)((i >> pow2_shift(n)) % L);
    const T p = c.p[l];
    T r;
    if (op == 0) r = add_mod(a[i], b[i], p);
    else if (op == 1) r = sub_mod(a[i], b[i], p);
    else if (op == 2) r = sub_mod((T)0, a[i], p);
    else r = csub(shoup_mul<T>(a[i], c.s[l], c.sq[l], p), p);  // op 3: scalar
    out[i] = r;
  }
}

template <typename T>
__global__ void k_rns_from_small(const int64_t* in, T* out, LimbConsts<T> c, int L, uint32_t n, uint64_t total) {
  // total = n_polys * L * N; output [poly][L][N]
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t poly = i / ((uint64_t)L * n);
    const int l = (int)((i >> pow2_shift(n)) % L);
    const int64_t v = in[poly * n + (i & (n - 1))];
    const uint64_t mag = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
    T r = reduce_word<T>(mag, c, l);
    if (v < 0) r = sub_mod((T)0, r, c.p[l]);
    out[i] = r;
  }
}

template <typename T>
__global__ void k_lift_plain(const uint64_t* m, T* out, LimbConsts<T> c, int L, uint32_t n, uint64_t t_half,
                             uint64_t total) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t poly = i / ((uint64_t)L * n);
    const int l = (int)((i >> pow2_shift(n)) % L);
    const T p = c.p[l];
    const uint64_t v = m[poly * n + (i & (n - 1))];
    T r = reduce_word<T>(v, c, l);
    if (v > t_half) r = sub_mod(r, c.tm[l], p);
    out[i] = csub(shoup_mul<T>(r, c.s[l], c.sq[l], p), p);
  }
}

__global__ void k_plain_elementwise(int op, const uint64_t* a, const uint64_t* b, uint64_t scalar, uint64_t* out,
                                    uint64_t t, uint64_t total) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = a[i];
    uint64_t r;
    if (op == 0) r = x + b[i], r = r >= t ? r - t : r;
    else if (op == 1) r = x >= b[i] ? x - b[i] : x + t - b[i];
    else if (op == 2) r = x ? t - x : 0;
    else r = (uint64_t)((unsigned __int128)x * scalar % t);
    out[i] = r;
  }
}

template <typename T>
LimbConsts<T> limb_consts(const Base& b, const uint64_t* scal, const uint64_t* aux) {
  constexpr int W = 8 * sizeof(T);
  LimbConsts<T> c{};
  for (int l = 0; l < b.size(); ++l) {
    const uint64_t p = b.primes[l];
    c.p[l] = (T)p;
    c.oneq[l] = (T)(((unsigned __int128)1 << W) / p);
    const uint64_t r2 = sizeof(T) == 4 ? ((1ull << 32) % p) : 0;
    c.r2[l] = (T)r2;
    c.r2q[l] = sizeof(T) == 4 ? (T)((r2 << 32) / p) : 0;
    if (scal) {
      const uint64_t s = scal[l] % p;
      c.s[l] = (T)s;
      c.sq[l] = (T)(((unsigned __int128)s << W) / p);
    }
  }
  if (aux)
    for (int l = 0; l < b.size(); ++l) c.tm[l] = (T)(aux[l] % b.primes[l]);
  return c;
}

const Base* base_ptr(const ctb_ctx_t* ctx, int base) {
  if (!ctx || base < 0 || base >= BASE_COUNT) return nullptr;
  const Base* b = &reinterpret_cast<const Ctx*>(ctx)->base[base];
  return b->size() ? b : nullptr;
}

}  // namespace

extern "C" int ctb_rns_elementwise(const ctb_ctx_t* ctx, int base, int op, const void* a, const void* b, void* out,
                                   uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* B = base_ptr(ctx, base);
  if (!B || op < 0 || op > 2 || !a || !out || (op < 2 && !b)) { set_error("ctb_rns_elementwise: bad arguments"); return ERR_ARG; }
  if (B->size() > MAXL) { set_error("ctb_rns_elementwise: too many limbs"); return ERR_UNSUPPORTED; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  const uint64_t total = n_polys * B->size() * (uint64_t)c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (B->word == 4)
    k_rns_elementwise<uint32_t><<<grid_stride(total, 16), 256, 0, s>>>(op, (const uint32_t*)a, (const uint32_t*)b,
                                                                (uint32_t*)out, limb_consts<uint32_t>(*B, nullptr, nullptr),
                                                                B->size(), c->n, total);
  else
    k_rns_elementwise<uint64_t><<<grid_stride(total, 16), 256, 0, s>>>(op, (const uint64_t*)a, (const uint64_t*)b,
                                                                (uint64_t*)out, limb_consts<uint64_t>(*B, nullptr, nullptr),
                                                                B->size(), c->n, total);
  return cuda_status(cudaGetLastError(), "ctb_rns_elementwise");
}

extern "C" int ctb_rns_scalar_mul(const ctb_ctx_t* ctx, int base, const void* a, const uint64_t* scalars, void* out,
                                  uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* B = base_ptr(ctx, base);
  if (!B || !a || !scalars || !out) { set_error("ctb_rns_scalar_mul: bad arguments"); return ERR_ARG; }
  if (B->size() > MAXL) { set_error("ctb_rns_scalar_mul: too many limbs"); return ERR_UNSUPPORTED; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  const uint64_t total = n_polys * B->size() * (uint64_t)c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (B->word == 4)
    k_rns_elementwise<uint32_t><<<grid_stride(total, 16), 256, 0, s>>>(3, (const uint32_t*)a, nullptr, (uint32_t*)out,
                                                                limb_consts<uint32_t>(*B, scalars, nullptr),
                                                                B->size(), c->n, total);
  else
    k_rns_elementwise<uint64_t><<<grid_stride(total, 16), 256, 0, s>>>(3, (const uint64_t*)a, nullptr, (uint64_t*)out,
                                                                limb_consts<uint64_t>(*B, scalars, nullptr),
                                                                B->size(), c->n, total);
  return cuda_status(cudaGetLastError(), "ctb_rns_scalar_mul");
}

extern "C" int ctb_rns_from_small(const ctb_ctx_t* ctx, int base, const int64_t* in, void* out, uint64_t n_polys,
                                  void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* B = base_ptr(ctx, base);
  if (!B || !in || !out) { set_error("ctb_rns_from_small: bad arguments"); return ERR_ARG; }
  if (B->size() > MAXL) { set_error("ctb_rns_from_small: too many limbs"); return ERR_UNSUPPORTED; }
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  const uint64_t total = n_polys * B->size() * (uint64_t)c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (B->word == 4)
    k_rns_from_small<uint32_t><<<grid_stride(total, 16), 256, 0, s>>>(in, (uint32_t*)out, limb_consts<uint32_t>(*B, nullptr, nullptr),
                                                               B->size(), c->n, total);
  else
    k_rns_from_small<uint64_t><<<grid_stride(total, 16), 256, 0, s>>>(in, (uint64_t*)out, limb_consts<uint64_t>(*B, nullptr, nullptr),
                                                               B->size(), c->n, total);
  return cuda_status(cudaGetLastError(), "ctb_rns_from_small");
}

extern "C" int ctb_lift_plain(const ctb_ctx_t* ctx, const uint64_t* m, const uint64_t* scale, void* out,
                              uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Base* B = base_ptr(ctx, CTB_BASE_Q);
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!B || !c->t || !m || !scale || !out) { set_error("ctb_lift_plain: bad arguments (needs plain ring)"); return ERR_ARG; }
  if (B->size() > MAXL) { set_error("ctb_lift_plain: too many limbs"); return ERR_UNSUPPORTED; }
  const uint64_t total = n_polys * B->size() * (uint64_t)c->n;
  if (!total) return OK;
  std::vector<uint64_t> tm(B->size());
  for (int l = 0; l < B->size(); ++l) tm[l] = c->t % B->primes[l];
  cudaStream_t s = (cudaStream_t)stream;
  if (B->word == 4)
    k_lift_plain<uint32_t><<<grid_stride(total, 16), 256, 0, s>>>(m, (uint32_t*)out, limb_consts<uint32_t>(*B, scale, tm.data()),
                                                           B->size(), c->n, c->t_half, total);
  else
    k_lift_plain<uint64_t><<<grid_stride(total, 16), 256, 0, s>>>(m, (uint64_t*)out, limb_consts<uint64_t>(*B, scale, tm.data()),
                                                           B->size(), c->n, c->t_half, total);
  return cuda_status(cudaGetLastError(), "ctb_lift_plain");
}

extern "C" int ctb_plain_elementwise(const ctb_ctx_t* ctx, int op, const uint64_t* a, const uint64_t* b,
                                     uint64_t scalar, uint64_t* out, uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !c->t || op < 0 || op > 3 || !a || !out || (op < 2 && !b)) { set_error("ctb_plain_elementwise: bad arguments"); return ERR_ARG; }
  const uint64_t total = n_polys * (uint64_t)c->n;
  if (!total) return OK;
  k_plain_elementwise<<<grid_stride(total, 16), 256, 0, (cudaStream_t)stream>>>(op, a, b, scalar % c->t, out, c->t, total);
  return cuda_status(cudaGetLastError(), "ctb_plain_elementwise");
}
