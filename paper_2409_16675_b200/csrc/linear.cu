// K3: the precompute-protocol online server step of one linear job, batched.
//
// Reference loop (linprot.precompute_online_server, linprot.py:473-482):
//   for (xi, wi, oi) in sites:
//       c_slot[oi] += cp_mul([x_xi], w_wi - r_w) + cp_mul([w_wi], x_xi - r_x)
//       p_slot[oi] += (x_xi - r_x) * (w_wi - r_w)                 (plain ring)
//   c_slot[oi] += [r_x r_w]_oi                                    (mask product)
// Everything above is linear mod q (mod t for p), so it is computed exactly in
// the evaluation domain: every x/w ciphertext part and every lifted masked
// plaintext is transformed ONCE, each slot accumulates its sites' slotwise
// products in registers, and each slot part is inverse-transformed ONCE --
// instead of 2 x (3 forward + 2 inverse) NTTs per site in the reference.
//
//   k_lift_prepare  plain [P][N] -> NTT(lift(m)) N^-1 2^W per limb (prepared operand)
//   k_lin_cipher    CTA per (slot, limb): 2 parts x sum over the slot's sites, INTT, + mask product
//   k_lin_plain     CTA per (slot, plain prime): sum of prepared products, INTT
//   k_plain_crt     plain residues -> uint64 mod t (ring._crt_combine, ring.py:478-485)
//   k_slot_sum      segmented sum of ciphertexts per slot (offline CCAdd accumulation)
#include <algorithm>
#include <cstring>
#include <vector>
#include "ctb200.h"
#include "kernels.hpp"

namespace ctb {

template <typename T, int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS, NttShape<LOGN>::MINB)
k_lift_prepare(const uint64_t* __restrict__ m, T* out, const PrimeTab<T>* __restrict__ tabs, int L, uint64_t t_half) {
  using Sh = NttShape<LOGN>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Exchanger<T, LOGN> ex{reinterpret_cast<T*>(smem_raw)};
  const int limb = blockIdx.x % L;
  const size_t poly = blockIdx.x / L;
  PrimeRegs<T> pr(tabs + limb);
  const T tmod = tabs[limb].tmod;
  const uint64_t* src = m + poly * Sh::N + coef_base<LOGN>();
  T x[Sh::E];
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) {
    const uint64_t v = __ldg(src + coef_off<LOGN>(k));
    T r = csub(pr.reduce_u64_lazy(v), pr.p);
    if (v > t_half) r = sub_mod(r, tmod, pr.p);
    x[k] = r;
  }
  ntt_fwd_regs<T, LOGN>(x, ex, pr.fwd, pr.p, pr.p2);
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) x[k] = csub(shoup_mul(x[k], pr.ninvr, pr.ninvr_q, pr.p), pr.p);
  store_eval<T, LOGN>(out + (size_t)blockIdx.x * Sh::N, x);
}

// X [n_x][2][L][N], W [n_w][2][L][N]: canonical eval; MXp [n_x][L][N], MWp [n_w][L][N]: prepared.
template <typename T, int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS, NttShape<LOGN>::MINB)
k_lin_cipher(const T* X, const T* W, const T* MXp, const T* MWp, const int32_t* __restrict__ slot_ptr,
             const int32_t* __restrict__ site_x, const int32_t* __restrict__ site_w, const T* maskprod, T* out,
             const PrimeTab<T>* __restrict__ tabs, int L) {
  using Sh = NttShape<LOGN>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Exchanger<T, LOGN> ex{reinterpret_cast<T*>(smem_raw)};
  const int limb = blockIdx.x % L;
  const int slot = blockIdx.x / L;
  PrimeRegs<T> pr(tabs + limb);
  const size_t N = Sh::N, LN = (size_t)L * N;
  using EV = EvalVec<T, LOGN>;
  T a0[Sh::E], a1[Sh::E];
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) a0[k] = a1[k] = 0;
  const int s0 = slot_ptr[slot], s1 = slot_ptr[slot + 1];
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const size_t xi = (size_t)site_x[s], wi = (size_t)site_w[s];
    const T* x0 = X + (xi * 2 + 0) * LN + limb * N;
    const T* x1 = X + (xi * 2 + 1) * LN + limb * N;
    const T* w0 = W + (wi * 2 + 0) * LN + limb * N;
    const T* w1 = W + (wi * 2 + 1) * LN + limb * N;
    const T* mx = MXp + xi * LN + limb * N;
    const T* mw = MWp + wi * LN + limb * N;
#pragma unroll
    for (int i = 0; i < EV::CHUNKS; ++i) {
      T vx0[EV::VEC], vx1[EV::VEC], vw0[EV::VEC], vw1[EV::VEC], vmx[EV::VEC], vmw[EV::VEC];
      EV::load(x0, i, vx0); EV::load(x1, i, vx1); EV::load(w0, i, vw0);
      EV::load(w1, i, vw1); EV::load(mx, i, vmx); EV::load(mw, i, vmw);
#pragma unroll
      for (int c = 0; c < EV::VEC; ++c) {
        const int k = i * EV::VEC + c;
        a0[k] = csub(a0[k] + mont_mul(vx0[c], vmw[c], pr.p, pr.pinv), pr.p2);
        a0[k] = csub(a0[k] + mont_mul(vw0[c], vmx[c], pr.p, pr.pinv), pr.p2);
        a1[k] = csub(a1[k] + mont_mul(vx1[c], vmw[c], pr.p, pr.pinv), pr.p2);
        a1[k] = csub(a1[k] + mont_mul(vw1[c], vmx[c], pr.p, pr.pinv), pr.p2);
      }
    }
  }
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    T acc[Sh::E];
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) acc[k] = part == 0 ? a0[k] : a1[k];
    ntt_inv_regs<T, LOGN>(acc, ex, pr.inv, pr.p, pr.p2);
    const size_t off = ((size_t)slot * 2 + part) * LN + limb * N + coef_base<LOGN>();
#pragma unroll
    for (int k = 0; k < Sh::E; ++k) {
      T v = csub(acc[k], pr.p);
      if (maskprod) v = add_mod(v, maskprod[off + coef_off<LOGN>(k)], pr.p);
      out[off + coef_off<LOGN>(k)] = v;
    }
  }
}

// Plain side over the plain primes (u32): MXt canonical eval [n_x][LT][N], MWtp prepared.
template <int LOGN>
__global__ void __launch_bounds__(NttShape<LOGN>::THREADS, NttShape<LOGN>::MINB)
k_lin_plain(const uint32_t* MXt, const uint32_t* MWtp, const int32_t* __restrict__ slot_ptr,
            const int32_t* __restrict__ site_x, const int32_t* __restrict__ site_w, uint32_t* out,
            const PrimeTab<uint32_t>* __restrict__ tabs, int LT) {
  using Sh = NttShape<LOGN>;
  using T = uint32_t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Exchanger<T, LOGN> ex{reinterpret_cast<T*>(smem_raw)};
  const int j = blockIdx.x % LT;
  const int slot = blockIdx.x / LT;
  PrimeRegs<T> pr(tabs + j);
  const size_t N = Sh::N, LN = (size_t)LT * N;
  using EV = EvalVec<T, LOGN>;
  T acc[Sh::E];
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) acc[k] = 0;
  const int s0 = slot_ptr[slot], s1 = slot_ptr[slot + 1];
#pragma unroll 1
  for (int s = s0; s < s1; ++s) {
    const T* mx = MXt + (size_t)site_x[s] * LN + j * N;
    const T* mw = MWtp + (size_t)site_w[s] * LN + j * N;
#pragma unroll
    for (int i = 0; i < EV::CHUNKS; ++i) {
      T vx[EV::VEC], vw[EV::VEC];
      EV::load(mx, i, vx);
      EV::load(mw, i, vw);
#pragma unroll
      for (int c = 0; c < EV::VEC; ++c)
        acc[i * EV::VEC + c] = csub(acc[i * EV::VEC + c] + mont_mul(vx[c], vw[c], pr.p, pr.pinv), pr.p2);
    }
  }
  ntt_inv_regs<T, LOGN>(acc, ex, pr.inv, pr.p, pr.p2);
  T* dst = out + ((size_t)slot * LT + j) * N + coef_base<LOGN>();
#pragma unroll
  for (int k = 0; k < Sh::E; ++k) dst[coef_off<LOGN>(k)] = csub(acc[k], pr.p);
}

__global__ void k_plain_crt(const uint32_t* res, uint64_t* out, int LT, uint32_t n, uint32_t p0, uint32_t p1,
                            uint32_t cinv, uint32_t cinv_q, uint32_t p1_oneq, uint64_t total) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t poly = g / n, i = g % n;
    const uint32_t r0 = res[(poly * LT) * n + i];
    if (LT == 1) { out[g] = r0; continue; }
    const uint32_t r1 = res[(poly * LT + 1) * n + i];
    const uint32_t r0m = csub(shoup_mul<uint32_t>(r0, 1u, p1_oneq, p1), p1);
    const uint32_t d = csub(shoup_mul<uint32_t>(sub_mod(r1, r0m, p1), cinv, cinv_q, p1), p1);
    out[g] = (uint64_t)r0 + (uint64_t)p0 * d;
  }
}

// out[o] = sum over members s of slot o of in[idx[s]] (mod p), [*][parts][L][N] layouts.
template <typename T>
__global__ void k_slot_sum(const T* in, const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ idx,
                           T* out, const PrimeTab<T>* __restrict__ tabs, int L, int parts, uint32_t n, uint64_t total) {
  // total = n_out * parts * L * n
  const uint64_t per = (uint64_t)parts * L * n;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t o = g / per, r = g % per;
    const int limb = (int)((r / n) % L);
    const T p = tabs[limb].p;
    T acc = 0;
    for (int s = slot_ptr[o]; s < slot_ptr[o + 1]; ++s) acc = add_mod(acc, in[(uint64_t)idx[s] * per + r], p);
    out[g] = acc;
  }
}

}  // namespace ctb

using namespace ctb;

namespace {
const Ctx* cctx(const ctb_ctx_t* ctx) { return reinterpret_cast<const Ctx*>(ctx); }
unsigned grid_lin(uint64_t total) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((total + 255) / 256, 148ull * 16));
}
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
}  // namespace

extern "C" int ctb_lift_prepare(const ctb_ctx_t* ctx, const uint64_t* m, void* out, uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = cctx(ctx);
  if (!c || !c->t || !m || !out) { set_error("ctb_lift_prepare: needs plain ring and buffers"); return ERR_ARG; }
  const Base& B = c->base[BASE_Q];
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (B.word == 4) {
    using T = uint32_t;
    CTB_DISPATCH_LOGN(c->logn, e = (launch_ntt_kernel<T, LOGN>(k_lift_prepare<T, LOGN>, n_polys * B.size(), s, m, (T*)out,
                                                      (const PrimeTab<T>*)B.d_tabs, B.size(), c->t_half)));
  } else {
    using T = uint64_t;
    CTB_DISPATCH_LOGN(c->logn, e = (launch_ntt_kernel<T, LOGN>(k_lift_prepare<T, LOGN>, n_polys * B.size(), s, m, (T*)out,
                                                      (const PrimeTab<T>*)B.d_tabs, B.size(), c->t_half)));
  }
  return cuda_status(e, "ctb_lift_prepare");
}

extern "C" uint64_t ctb_linear_online_workspace_bytes(const ctb_ctx_t* ctx, uint32_t n_x, uint32_t n_w, uint32_t n_out,
                                                      uint32_t n_sites) {
  const Ctx* c = cctx(ctx);
  if (!c) return 0;
  const size_t N = c->n, L = c->base[BASE_Q].size(), LT = c->base[BASE_T].size();
  const size_t w = c->base[BASE_Q].word;
  size_t b = 0;
  b += align256((size_t)n_x * 2 * L * N * w);   // X eval
  b += align256((size_t)n_w * 2 * L * N * w);   // W eval
  b += align256((size_t)n_x * L * N * w);       // MX prepared
  b += align256((size_t)n_w * L * N * w);       // MW prepared
  b += align256((size_t)n_x * LT * N * 4);      // mx mod t_j (eval)
  b += align256((size_t)n_w * LT * N * 4);      // mw mod t_j (prepared)
  b += align256((size_t)n_out * LT * N * 4);    // p slot residues
  b += align256((size_t)(n_out + 1 + 2 * (size_t)n_sites) * 4);  // CSR
  return b;
}

extern "C" int ctb_linear_online(const ctb_ctx_t* ctx, const void* ct_x, uint32_t n_x, const void* ct_w, uint32_t n_w,
                                 const uint64_t* mx, const uint64_t* mw, const uint32_t* sites_host, uint32_t n_sites,
                                 uint32_t n_out, const void* maskprod, void* out_ct, uint64_t* out_p, void* workspace,
                                 void* stream) {
  if (n_out == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = cctx(ctx);
  if (!c || !c->t || !ct_x || !ct_w || !mx || !mw || !sites_host || !out_ct || !out_p || !workspace) {
    set_error("ctb_linear_online: bad context (needs plain ring) or buffer");
    return ERR_ARG;
  }
  const Base& B = c->base[BASE_Q];
  const Base& BT = c->base[BASE_T];
  if (BT.word != 4 || BT.size() > 2) { set_error("ctb_linear_online: plain ring must be 1-2 primes < 2^30"); return ERR_UNSUPPORTED; }
  const size_t N = c->n, L = B.size(), LT = BT.size(), w = B.word;
  // CSR of the sites by output slot (stable: keeps the reference's site order per slot)
  std::vector<int32_t> ptr(n_out + 1, 0), sx(n_sites), sw(n_sites);
  for (uint32_t s = 0; s < n_sites; ++s) {
    const uint32_t xi = sites_host[3 * s], wi = sites_host[3 * s + 1], oi = sites_host[3 * s + 2];
    if (xi >= n_x || wi >= n_w || oi >= n_out) { set_error("ctb_linear_online: site index out of range"); return ERR_ARG; }
    ptr[oi + 1]++;
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
  char* ws = (char*)workspace;
  auto take = [&](size_t bytes) { char* p = ws; ws += align256(bytes); return (void*)p; };
  void* X = take((size_t)n_x * 2 * L * N * w);
  void* W = take((size_t)n_w * 2 * L * N * w);
  void* MX = take((size_t)n_x * L * N * w);
  void* MW = take((size_t)n_w * L * N * w);
  uint32_t* MXt = (uint32_t*)take((size_t)n_x * LT * N * 4);
  uint32_t* MWt = (uint32_t*)take((size_t)n_w * LT * N * 4);
  uint32_t* PR = (uint32_t*)take((size_t)n_out * LT * N * 4);
  int32_t* csr = (int32_t*)take((size_t)(n_out + 1 + 2 * (size_t)n_sites) * 4);
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<int32_t> packed(n_out + 1 + 2 * (size_t)n_sites);
  std::copy(ptr.begin(), ptr.end(), packed.begin());
  std::copy(sx.begin(), sx.end(), packed.begin() + n_out + 1);
  std::copy(sw.begin(), sw.end(), packed.begin() + n_out + 1 + n_sites);
  cudaError_t e = cudaMemcpyAsync(csr, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_status(e, "ctb_linear_online csr");
  e = cudaStreamSynchronize(s);  // the host vector dies at return
  if (e != cudaSuccess) return cuda_status(e, "ctb_linear_online csr");
  const int32_t* d_ptr = csr;
  const int32_t* d_sx = csr + n_out + 1;
  const int32_t* d_sw = d_sx + n_sites;
  int rc;
  // forward transforms of every ciphertext part, lifted+prepared masked plaintexts
  if ((rc = ctb_ntt_forward(ctx, CTB_BASE_Q, ct_x, X, (uint64_t)n_x * 2, stream))) return rc;
  if ((rc = ctb_ntt_forward(ctx, CTB_BASE_Q, ct_w, W, (uint64_t)n_w * 2, stream))) return rc;
  if ((rc = ctb_lift_prepare(ctx, mx, MX, n_x, stream))) return rc;
  if ((rc = ctb_lift_prepare(ctx, mw, MW, n_w, stream))) return rc;
  // plain side: residues mod t_j of mx (eval) and mw (prepared)
  if ((rc = ctb_rns_from_small(ctx, CTB_BASE_T, (const int64_t*)mx, MXt, n_x, stream))) return rc;
  if ((rc = ctb_ntt_forward(ctx, CTB_BASE_T, MXt, MXt, n_x, stream))) return rc;
  if ((rc = ctb_rns_from_small(ctx, CTB_BASE_T, (const int64_t*)mw, MWt, n_w, stream))) return rc;
  if ((rc = ctb_prepare_operand(ctx, CTB_BASE_T, MWt, MWt, n_w, stream))) return rc;
  if (B.word == 4) {
    using T = uint32_t;
    CTB_DISPATCH_LOGN(c->logn, e = (launch_ntt_kernel<T, LOGN>(k_lin_cipher<T, LOGN>, (size_t)n_out * L, s,
                                                      (const T*)X, (const T*)W, (const T*)MX, (const T*)MW, d_ptr,
                                                      d_sx, d_sw, (const T*)maskprod, (T*)out_ct,
                                                      (const PrimeTab<T>*)B.d_tabs, (int)L)));
  } else {
    using T = uint64_t;
    CTB_DISPATCH_LOGN(c->logn, e = (launch_ntt_kernel<T, LOGN>(k_lin_cipher<T, LOGN>, (size_t)n_out * L, s,
                                                      (const T*)X, (const T*)W, (const T*)MX, (const T*)MW, d_ptr,
                                                      d_sx, d_sw, (const T*)maskprod, (T*)out_ct,
                                                      (const PrimeTab<T>*)B.d_tabs, (int)L)));
  }
  if (e != cudaSuccess) return cuda_status(e, "ctb_linear_online cipher");
  CTB_DISPATCH_LOGN(c->logn, e = (launch_ntt_kernel<uint32_t, LOGN>(k_lin_plain<LOGN>, (size_t)n_out * LT, s,
                                                           (const uint32_t*)MXt, (const uint32_t*)MWt, d_ptr, d_sx,
                                                           d_sw, PR, (const PrimeTab<uint32_t>*)BT.d_tabs, (int)LT)));
  if (e != cudaSuccess) return cuda_status(e, "ctb_linear_online plain");
  const uint64_t total = (uint64_t)n_out * N;
  const uint32_t p0 = (uint32_t)BT.primes[0], p1 = LT > 1 ? (uint32_t)BT.primes[1] : 1u;
  const uint32_t p1_oneq = (uint32_t)((1ull << 32) / p1);
  if (total)
    k_plain_crt<<<grid_lin(total), 256, 0, s>>>(PR, out_p, (int)LT, (uint32_t)N, p0, p1, c->crt_inv, c->crt_inv_q,
                                                p1_oneq, total);
  return cuda_status(cudaGetLastError(), "ctb_linear_online crt");
}

extern "C" int ctb_slot_sum(const ctb_ctx_t* ctx, int base, const void* in, uint32_t parts, const int32_t* slot_ptr,
                            const int32_t* members, uint32_t n_out, void* out, void* stream) {
  if (n_out == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = cctx(ctx);
  if (!c || base < 0 || base >= BASE_COUNT || !in || !slot_ptr || !members || !out) {
    set_error("ctb_slot_sum: bad arguments");
    return ERR_ARG;
  }
  const Base& B = c->base[base];
  const uint64_t total = (uint64_t)n_out * parts * B.size() * c->n;
  if (!total) return OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (B.word == 4)
    k_slot_sum<uint32_t><<<grid_lin(total), 256, 0, s>>>((const uint32_t*)in, slot_ptr, members, (uint32_t*)out,
                                                         (const PrimeTab<uint32_t>*)B.d_tabs, B.size(), (int)parts,
                                                         c->n, total);
  else
    k_slot_sum<uint64_t><<<grid_lin(total), 256, 0, s>>>((const uint64_t*)in, slot_ptr, members, (uint64_t*)out,
                                                         (const PrimeTab<uint64_t>*)B.d_tabs, B.size(), (int)parts,
                                                         c->n, total);
  return cuda_status(cudaGetLastError(), "ctb_slot_sum");
}
