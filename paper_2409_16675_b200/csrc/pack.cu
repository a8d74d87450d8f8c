// Client-side encode / decode of the correlated linear layer (K3's client side), as gather / scatter
// kernels driven by per-plan degree maps.
//
//   ctb_pack_gather        packing.pack_input_correlated / pack_kernel_correlated   packing.py:407-445
//                          pack_fc_input / pack_fc_matrix / pack_outer_left         packing.py:545-597
//                          (+ the masking x - r_x, w - r_w of linprot.py:438-441, fused)
//   ctb_plain_scatter      packing.extract_output (+ to_signed_matrix)              packing.py:476-522
//                          extract_fc_output / extract_outer                        packing.py:577-605
//   (ctb_decrypt_round_extract, rns.cu: the same scatter as the decrypt epilogue)
//
// A packing plan is value-independent (packing.plan_correlated), so the host turns it once into
// maps[kind][d] = the source element feeding degree d of a polynomial of that kind (-1: zero degree)
// -- one kind per tile for inputs, one for kernels -- and into the inverse maps for extraction
// (maps[kind][d] = destination of product coefficient d, -1: not an output).  A job (or a whole
// batch of jobs) is then one launch: polynomial p reads src[base[p] + maps[kind[p]][d]].  Every warp
// writes 256 contiguous bytes per row; the map row is shared by all polynomials of a kind (L1/L2
// resident) and the source tensor (a few KB per image) is gathered from L1/L2.
#include <algorithm>
#include "ctb200.h"
#include "kernels.hpp"

using namespace ctb;

namespace {

// Four consecutive degrees per thread: one 16-byte map load, four independent source loads and
// 16-byte mask loads / stores, so each thread keeps several memory requests in flight (the kernel is
// latency-bound on the dependent map -> source loads with one degree per thread).
__global__ void __launch_bounds__(256) k_pack_gather(const int64_t* __restrict__ src, uint64_t src_len,
                                                     const int32_t* __restrict__ maps, uint32_t n_maps,
                                                     const int32_t* __restrict__ kind,
                                                     const int64_t* __restrict__ base,
                                                     const uint64_t* __restrict__ r, uint64_t* out_plain,
                                                     uint64_t* out_masked, uint64_t t, uint32_t logn,
                                                     uint64_t total4) {
  const uint32_t n = 1u << logn;
  for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < total4;
       q += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = q * 4;
    const uint64_t p = g >> logn;
    const uint32_t d = (uint32_t)g & (n - 1);
    const uint32_t k = (uint32_t)__ldg(kind + p);
    uint64_t v[4] = {0, 0, 0, 0};
    if (k < n_maps) {
      const int4 m = __ldg(reinterpret_cast<const int4*>(maps + (uint64_t)k * n + d));
      const uint64_t b = (uint64_t)__ldg(base + p);
      const int mm[4] = {m.x, m.y, m.z, m.w};
      int64_t sv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t at = b + (uint64_t)mm[j];
        sv[j] = (mm[j] >= 0 && at < src_len) ? __ldg(src + at) : 0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = mod_signed(sv[j], t);
    }
    if (out_plain) {
      reinterpret_cast<ulonglong2*>(out_plain + g)[0] = make_ulonglong2(v[0], v[1]);
      reinterpret_cast<ulonglong2*>(out_plain + g)[1] = make_ulonglong2(v[2], v[3]);
    }
    if (out_masked) {
      const ulonglong2 r01 = __ldg(reinterpret_cast<const ulonglong2*>(r + g));
      const ulonglong2 r23 = __ldg(reinterpret_cast<const ulonglong2*>(r + g) + 1);
      const uint64_t rv[4] = {r01.x, r01.y, r23.x, r23.y};
      uint64_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = v[j] >= rv[j] ? v[j] - rv[j] : v[j] + t - rv[j];
      reinterpret_cast<ulonglong2*>(out_masked + g)[0] = make_ulonglong2(o[0], o[1]);
      reinterpret_cast<ulonglong2*>(out_masked + g)[1] = make_ulonglong2(o[2], o[3]);
    }
  }
}

__global__ void __launch_bounds__(256) k_plain_scatter(const uint64_t* __restrict__ in,
                                                       const uint64_t* __restrict__ sub,
                                                       const int32_t* __restrict__ maps, uint32_t n_maps,
                                                       const int32_t* __restrict__ kind,
                                                       const int64_t* __restrict__ base, uint64_t dst_len,
                                                       int centered, int64_t* out, uint64_t t, uint32_t logn,
                                                       uint64_t total) {
  const uint32_t n = 1u << logn;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = g >> logn;
    const uint32_t d = (uint32_t)g & (n - 1);
    const uint32_t k = (uint32_t)kind[s];
    if (k >= n_maps) continue;
    const int32_t m = maps[(uint64_t)k * n + d];
    if (m < 0) continue;
    const uint64_t dst = (uint64_t)base[s] + (uint64_t)m;
    if (dst >= dst_len) continue;
    uint64_t v = in[g];
    if (sub) {
      const uint64_t b = sub[g];
      v = v >= b ? v - b : v + t - b;
    }
    out[dst] = centered && v > t / 2 ? (int64_t)v - (int64_t)t : (int64_t)v;
  }
}

}  // namespace

extern "C" int ctb_pack_gather(const ctb_ctx_t* ctx, const int64_t* src, uint64_t src_len, const int32_t* maps,
                               uint32_t n_maps, const int32_t* kind, const int64_t* base, const uint64_t* r,
                               uint64_t* out_plain, uint64_t* out_masked, uint64_t n_polys, void* stream) {
  if (n_polys == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !c->t || !maps || !kind || !base || (src_len && !src) || (!out_plain && !out_masked) ||
      (out_masked && !r)) {
    set_error("ctb_pack_gather: context lacks a plain ring or bad buffer");
    return ERR_ARG;
  }
  const uint64_t total4 = n_polys * (uint64_t)c->n / 4;   // ring degree >= 4, a multiple of 4
  k_pack_gather<<<grid_stride(total4, 8), 256, 0, (cudaStream_t)stream>>>(src, src_len, maps, n_maps, kind, base, r,
                                                                          out_plain, out_masked, c->t, c->logn, total4);
  return cuda_status(cudaGetLastError(), "ctb_pack_gather");
}

extern "C" int ctb_plain_scatter(const ctb_ctx_t* ctx, const uint64_t* in, const uint64_t* sub, const int32_t* maps,
                                 uint32_t n_maps, const int32_t* kind, const int64_t* base, uint64_t dst_len,
                                 int centered, int64_t* out, uint64_t n_slots, void* stream) {
  if (n_slots == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !c->t || !in || !maps || !kind || !base || (dst_len && !out)) {
    set_error("ctb_plain_scatter: context lacks a plain ring or bad buffer");
    return ERR_ARG;
  }
  const uint64_t total = n_slots * (uint64_t)c->n;
  k_plain_scatter<<<grid_stride(total, 8), 256, 0, (cudaStream_t)stream>>>(in, sub, maps, n_maps, kind, base, dst_len,
                                                                           centered, out, c->t, c->logn, total);
  return cuda_status(cudaGetLastError(), "ctb_plain_scatter");
}
