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
//   LiftPrepare     plain [P][N] -> NTT(lift(m)) N^-1 2^W per limb (k_stream, kernels_ntt.cu)
//   k_lin_accum     per (slot, limb, 16-byte vector): 2 parts x sum over the slot's sites (eval)
//   k_stream InvAdd persistent INTT of the slot sums, + mask product (kernels_ntt.cu)
//   k_lin_accum_plain + k_stream InvAdd: the plain side, same structure over the plain primes
//   k_plain_crt     plain residues -> uint64 mod t (ring._crt_combine, ring.py:478-485)
//   k_slot_sum      segmented sum of ciphertexts per slot (offline CCAdd accumulation)
#include <algorithm>
#include <cstring>
#include <vector>
#include "ctb200.h"
#include "kernels.hpp"

namespace ctb {

// X [n_x][2][L][N], W [n_w][2][L][N]: canonical eval; MXp [n_x][L][N], MWp [n_w][L][N]: prepared.
// ACC [n_out][2][L][N] (eval, [0,2p), N^-1 folded) = per slot the sum over its sites of
// X (x) MW + W (x) MX.  Elementwise in the eval domain, so the thread mapping is free:
// one thread per 16-byte vector of one (slot, limb), sites two at a time so a thread
// has 12 independent 16-byte loads in flight -- this phase is a gather over HBM/L2 and
// lives on memory-level parallelism, while the transforms run in k_stream (InvAdd).
// resident k_lin_accum blocks per SM of the grid-stride launch
#ifndef CTB_LIN_BLOCKS_PER_SM
#define CTB_LIN_BLOCKS_PER_SM 4
#endif
// resident blocks the registers are capped for (the gather lives on memory-level parallelism: 32-bit
// limbs 4 blocks of 64 registers instead of 3 of 70, 636 -> 605 us per cfg4 job; 5 blocks spill)
#ifndef CTB_LIN_MINB
#define CTB_LIN_MINB 4
#endif
template <typename T>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? CTB_LIN_MINB : 1)
k_lin_accum(const T* __restrict__ X, const T* __restrict__ W, const T* __restrict__ MXp, const T* __restrict__ MWp,
            const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ site_x,
            const int32_t* __restrict__ site_w, const T* __restrict__ init, T* __restrict__ acc,
            const PrimeTab<T>* __restrict__ tabs, int L, uint32_t n, uint32_t chunks, uint64_t units) {
  constexpr int VEC = 16 / sizeof(T);
  union V { uint4 u; T t[VEC]; };
  // grid-stride over (slot, limb, chunk) units: a few resident blocks per SM instead of one short
  // block per unit (the gather is latency-bound; block turnover costs issue slots)
#pragma unroll 1
  for (uint64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
  uint32_t bid = (uint32_t)unit;
  const uint32_t chunk = bid % chunks;
  bid /= chunks;
  const int limb = (int)(bid % L);
  const uint32_t slot = bid / L;
  const uint32_t nv = n / VEC;
  const uint32_t v = chunk * blockDim.x + threadIdx.x;
  if (v >= nv) continue;
  const T p = tabs[limb].p, p2 = 2 * p, pinv = tabs[limb].pinv;
  const size_t LN = (size_t)L * n;
  const uint4* X4 = reinterpret_cast<const uint4*>(X + (size_t)limb * n) + v;
  const uint4* W4 = reinterpret_cast<const uint4*>(W + (size_t)limb * n) + v;
  const uint4* MX4 = reinterpret_cast<const uint4*>(MXp + (size_t)limb * n) + v;
  const uint4* MW4 = reinterpret_cast<const uint4*>(MWp + (size_t)limb * n) + v;
  const size_t part4 = LN / VEC, poly4 = 2 * part4;  // uint4 strides
  T a0[VEC], a1[VEC];
  uint4* A4 = reinterpret_cast<uint4*>(acc + (size_t)limb * n) + v + (size_t)slot * poly4;
  if (init) {  // eval-domain mask product (ctb_eval_addend form), same layout as acc
    V i0, i1;
    const uint4* I4 = reinterpret_cast<const uint4*>(init + (size_t)limb * n) + v + (size_t)slot * poly4;
    i0.u = __ldg(I4);
    i1.u = __ldg(I4 + part4);
#pragma unroll
    for (int c = 0; c < VEC; ++c) { a0[c] = i0.t[c]; a1[c] = i1.t[c]; }
  } else {
#pragma unroll
    for (int c = 0; c < VEC; ++c) a0[c] = a1[c] = 0;
  }
  auto site = [&](const V& x0, const V& x1, const V& w0, const V& w1, const V& mx, const V& mw) {
#pragma unroll
    for (int c = 0; c < VEC; ++c) {
      a0[c] = csub(a0[c] + mont_mul(x0.t[c], mw.t[c], p, pinv), p2);
      a0[c] = csub(a0[c] + mont_mul(w0.t[c], mx.t[c], p, pinv), p2);
      a1[c] = csub(a1[c] + mont_mul(x1.t[c], mw.t[c], p, pinv), p2);
      a1[c] = csub(a1[c] + mont_mul(w1.t[c], mx.t[c], p, pinv), p2);
    }
  };
  int s = slot_ptr[slot];
  const int s1 = slot_ptr[slot + 1];
#pragma unroll 1
  for (; s + 1 < s1; s += 2) {
    const size_t xa = site_x[s], wa = site_w[s], xb = site_x[s + 1], wb = site_w[s + 1];
    V x0a, x1a, w0a, w1a, mxa, mwa, x0b, x1b, w0b, w1b, mxb, mwb;
    x0a.u = __ldg(X4 + xa * poly4); x1a.u = __ldg(X4 + xa * poly4 + part4);
    w0a.u = __ldg(W4 + wa * poly4); w1a.u = __ldg(W4 + wa * poly4 + part4);
    mxa.u = __ldg(MX4 + xa * part4); mwa.u = __ldg(MW4 + wa * part4);
    x0b.u = __ldg(X4 + xb * poly4); x1b.u = __ldg(X4 + xb * poly4 + part4);
    w0b.u = __ldg(W4 + wb * poly4); w1b.u = __ldg(W4 + wb * poly4 + part4);
    mxb.u = __ldg(MX4 + xb * part4); mwb.u = __ldg(MW4 + wb * part4);
    site(x0a, x1a, w0a, w1a, mxa, mwa);
    site(x0b, x1b, w0b, w1b, mxb, mwb);
  }
  if (s < s1) {
    const size_t xa = site_x[s], wa = site_w[s];
    V x0a, x1a, w0a, w1a, mxa, mwa;
    x0a.u = __ldg(X4 + xa * poly4); x1a.u = __ldg(X4 + xa * poly4 + part4);
    w0a.u = __ldg(W4 + wa * poly4); w1a.u = __ldg(W4 + wa * poly4 + part4);
    mxa.u = __ldg(MX4 + xa * part4); mwa.u = __ldg(MW4 + wa * part4);
    site(x0a, x1a, w0a, w1a, mxa, mwa);
  }
  V o0, o1;
#pragma unroll
  for (int c = 0; c < VEC; ++c) { o0.t[c] = a0[c]; o1.t[c] = a1[c]; }
  A4[0] = o0.u;
  A4[part4] = o1.u;
  }
}

// Plain side over the plain primes (u32): MXt canonical eval [n_x][LT][N], MWtp prepared;
// PR [n_out][LT][N] (eval, N^-1 folded) = per slot the sum over its sites of MXt (x) MWtp -- the
// same memory-level-parallel gather as k_lin_accum, one product per site; k_stream InvAdd
// (no addend) then transforms the slot sums back in place.
__global__ void __launch_bounds__(256)
k_lin_accum_plain(const uint32_t* __restrict__ MXt, const uint32_t* __restrict__ MWtp,
                  const int32_t* __restrict__ slot_ptr, const int32_t* __restrict__ site_x,
                  const int32_t* __restrict__ site_w, uint32_t* __restrict__ acc,
                  const PrimeTab<uint32_t>* __restrict__ tabs, int LT, uint32_t n, uint32_t chunks) {
  union V { uint4 u; uint32_t t[4]; };
  uint32_t bid = blockIdx.x;
  const uint32_t chunk = bid % chunks;
  bid /= chunks;
  const int j = (int)(bid % LT);
  const uint32_t slot = bid / LT;
  const uint32_t nv = n / 4;
  const uint32_t v = chunk * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const uint32_t p = tabs[j].p, p2 = 2 * p, pinv = tabs[j].pinv;
  const size_t LN4 = (size_t)LT * n / 4;
  const uint4* X4 = reinterpret_cast<const uint4*>(MXt + (size_t)j * n) + v;
  const uint4* W4 = reinterpret_cast<const uint4*>(MWtp + (size_t)j * n) + v;
  uint32_t a[4] = {0, 0, 0, 0};
  int s = slot_ptr[slot];
  const int s1 = slot_ptr[slot + 1];
#pragma unroll 1
  for (; s + 1 < s1; s += 2) {
    V xa, wa, xb, wb;
    xa.u = __ldg(X4 + (size_t)site_x[s] * LN4);
    wa.u = __ldg(W4 + (size_t)site_w[s] * LN4);
    xb.u = __ldg(X4 + (size_t)site_x[s + 1] * LN4);
    wb.u = __ldg(W4 + (size_t)site_w[s + 1] * LN4);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      a[c] = csub(a[c] + mont_mul(xa.t[c], wa.t[c], p, pinv), p2);
      a[c] = csub(a[c] + mont_mul(xb.t[c], wb.t[c], p, pinv), p2);
    }
  }
  if (s < s1) {
    V xa, wa;
    xa.u = __ldg(X4 + (size_t)site_x[s] * LN4);
    wa.u = __ldg(W4 + (size_t)site_w[s] * LN4);
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = csub(a[c] + mont_mul(xa.t[c], wa.t[c], p, pinv), p2);
  }
  V o;
#pragma unroll
  for (int c = 0; c < 4; ++c) o.t[c] = a[c];
  reinterpret_cast<uint4*>(acc + ((size_t)slot * LT + j) * n)[v] = o.u;
}

__global__ void k_plain_crt(const uint32_t* res, uint64_t* out, int LT, uint32_t n, uint32_t p0, uint32_t p1,
                            uint32_t cinv, uint32_t cinv_q, uint32_t p1_oneq, uint64_t total) {
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t poly = g >> pow2_shift(n), i = g & (n - 1);
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
    const int limb = (int)((r >> pow2_shift(n)) % L);
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
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
}  // namespace

extern "C" int ctb_lift_prepare(const ctb_ctx_t* ctx, const uint64_t* m, void* out, uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = cctx(ctx);
  if (!c || !c->t || !m || !out) { set_error("ctb_lift_prepare: needs plain ring and buffers"); return ERR_ARG; }
  return cuda_status(stream_lift(c, BASE_Q, true, m, out, n_polys, (cudaStream_t)stream), "ctb_lift_prepare");
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
                                 uint32_t n_out, const void* maskprod, int maskprod_eval, void* out_ct, uint64_t* out_p,
                                 void* workspace, void* stream) {
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
  cudaError_t e = stage_upload(csr, packed.data(), packed.size() * 4, s);  // no stream sync
  if (e != cudaSuccess) return cuda_status(e, "ctb_linear_online csr");
  const int32_t* d_ptr = csr;
  const int32_t* d_sx = csr + n_out + 1;
  const int32_t* d_sw = d_sx + n_sites;
  int rc;
  // Every eval-domain operand of this call is internal (and the eval-form mask product comes from
  // ctb_linear_addend), so they all use the thread-major chunk layout (k_stream strip_out /
  // strip_in): contiguous warp stores in the forward transforms and conflict-free staging reads in
  // the inverse ones, no transposition; the slot sums below are elementwise, layout-agnostic.
  // forward transforms of every ciphertext part, lifted+prepared masked plaintexts
  if ((e = stream_forward(c, BASE_Q, false, ct_x, X, (uint64_t)n_x * 2, s, true)) != cudaSuccess) return cuda_status(e, "ctb_linear_online ntt");
  if ((e = stream_forward(c, BASE_Q, false, ct_w, W, (uint64_t)n_w * 2, s, true)) != cudaSuccess) return cuda_status(e, "ctb_linear_online ntt");
  if ((e = stream_lift(c, BASE_Q, true, mx, MX, n_x, s, true)) != cudaSuccess) return cuda_status(e, "ctb_linear_online lift");
  if ((e = stream_lift(c, BASE_Q, true, mw, MW, n_w, s, true)) != cudaSuccess) return cuda_status(e, "ctb_linear_online lift");
  // plain side: residues mod t_j of mx (eval) and mw (prepared)
  if ((e = stream_lift(c, BASE_T, false, mx, MXt, n_x, s, true)) != cudaSuccess) return cuda_status(e, "ctb_linear_online lift");
  if ((e = stream_lift(c, BASE_T, true, mw, MWt, n_w, s, true)) != cudaSuccess) return cuda_status(e, "ctb_linear_online lift");
  {
    // cipher side: gather-accumulate into out_ct (eval domain), then INTT in place + mask product
    const uint32_t nv = (uint32_t)(N * w / 16);
    const uint32_t chunks = (nv + 255) / 256;
    const uint64_t blocks = (uint64_t)n_out * L * chunks;
    if (blocks >= (1ull << 31)) { set_error("ctb_linear_online: job too large"); return ERR_ARG; }
    const unsigned grid = (unsigned)std::min<uint64_t>(blocks, (uint64_t)grid_stride(blocks * 256, CTB_LIN_BLOCKS_PER_SM));
    if (B.word == 4)
      k_lin_accum<uint32_t><<<grid, 256, 0, s>>>((const uint32_t*)X, (const uint32_t*)W,
          (const uint32_t*)MX, (const uint32_t*)MW, d_ptr, d_sx, d_sw,
          maskprod_eval ? (const uint32_t*)maskprod : nullptr, (uint32_t*)out_ct,
          (const PrimeTab<uint32_t>*)B.d_tabs, (int)L, (uint32_t)N, chunks, blocks);
    else
      k_lin_accum<uint64_t><<<grid, 256, 0, s>>>((const uint64_t*)X, (const uint64_t*)W,
          (const uint64_t*)MX, (const uint64_t*)MW, d_ptr, d_sx, d_sw,
          maskprod_eval ? (const uint64_t*)maskprod : nullptr, (uint64_t*)out_ct,
          (const PrimeTab<uint64_t>*)B.d_tabs, (int)L, (uint32_t)N, chunks, blocks);
    e = cudaGetLastError();
    if (e == cudaSuccess)
      e = stream_inv_add(c, BASE_Q, out_ct, out_ct, maskprod_eval ? nullptr : maskprod, (uint64_t)n_out * 2, s, true);
  }
  if (e != cudaSuccess) return cuda_status(e, "ctb_linear_online cipher");
  {
    const uint32_t nv = (uint32_t)(N / 4);
    const uint32_t chunks = (nv + 255) / 256;
    const uint64_t blocks = (uint64_t)n_out * LT * chunks;
    k_lin_accum_plain<<<(unsigned)blocks, 256, 0, s>>>(MXt, MWt, d_ptr, d_sx, d_sw, PR,
                                                        (const PrimeTab<uint32_t>*)BT.d_tabs, (int)LT, (uint32_t)N,
                                                        chunks);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = stream_inv_add(c, BASE_T, PR, PR, nullptr, (uint64_t)n_out, s, true);
  }
  if (e != cudaSuccess) return cuda_status(e, "ctb_linear_online plain");
  const uint64_t total = (uint64_t)n_out * N;
  const uint32_t p0 = (uint32_t)BT.primes[0], p1 = LT > 1 ? (uint32_t)BT.primes[1] : 1u;
  const uint32_t p1_oneq = (uint32_t)((1ull << 32) / p1);
  if (total)
    k_plain_crt<<<grid_stride(total, 16), 256, 0, s>>>(PR, out_p, (int)LT, (uint32_t)N, p0, p1, c->crt_inv, c->crt_inv_q,
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
    k_slot_sum<uint32_t><<<grid_stride(total, 16), 256, 0, s>>>((const uint32_t*)in, slot_ptr, members, (uint32_t*)out,
                                                         (const PrimeTab<uint32_t>*)B.d_tabs, B.size(), (int)parts,
                                                         c->n, total);
  else
    k_slot_sum<uint64_t><<<grid_stride(total, 16), 256, 0, s>>>((const uint64_t*)in, slot_ptr, members, (uint64_t*)out,
                                                         (const PrimeTab<uint64_t>*)B.d_tabs, B.size(), (int)parts,
                                                         c->n, total);
  return cuda_status(cudaGetLastError(), "ctb_slot_sum");
}
