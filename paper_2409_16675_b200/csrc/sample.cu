// Device sampling of encryption randomness (He._ternary / He._error, he.py:292-303).
//
// Counter-based Philox4x32-10 keyed by a 64-bit seed; the counter is
// (global polynomial index, coefficient), so every limb of an encryption sees
// the same draws and the stream is independent of the launch shape.  One
// Philox block per coefficient gives u (ternary, uniform over {-1, 0, 1}) and,
// through Box-Muller, the two Gaussian errors e1, e2 ~ N(0, sigma^2), rounded
// to the nearest integer and clipped to +-bound like the reference.  Output:
// int8 draws [batch][3][N] = (u, e1, e2) in the device draw layout ctb_encrypt consumes:
// thread-major, position t*E + k holds the draw of the coefficient that register k of
// NTT thread t owns (coef_base/coef_off of the first pass), so a thread loads its 16
// draws of each kind with one 16-byte load.  ctb_draws_from_natural converts.
#include <algorithm>
#include <cstdint>
#include "ctb200.h"
#include "kernels.hpp"

namespace ctb {

struct Philox4x32 {
  static __device__ __forceinline__ uint4 run(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
      c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

template <int LOGN>
__host__ __device__ constexpr int draw_coef(int pos) {  // device position -> coefficient
  using Sh = NttShape<LOGN>;
  return pass_index<LOGN, 0, Sh::FIRST_R>(pos / Sh::E, pos % Sh::E);
}

template <int LOGN>
__global__ void k_sample_draws(int8_t* out, uint64_t seed, uint64_t first_poly, uint64_t total, float sigma, int bound) {
  constexpr uint32_t n = 1u << LOGN;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t poly = g >> pow2_shift(n);
    const uint32_t pos = (uint32_t)(g & (n - 1));
    const uint32_t i = (uint32_t)draw_coef<LOGN>((int)pos);
    const uint64_t gp = first_poly + poly;
    const uint4 r = Philox4x32::run(make_uint4(i, (uint32_t)gp, (uint32_t)(gp >> 32), 0x43544232u), key);
    const int u = (int)(((uint64_t)r.x * 3u) >> 32) - 1;
    const float u1 = ((float)r.y + 1.0f) * 2.3283064365386963e-10f;   // (0, 1]
    const float th = (float)r.z * 1.4629180792671596e-09f;             // 2 pi / 2^32
    // fast SFU intrinsics: absolute errors ~1e-6 on z, irrelevant after rint(sigma z)
    const float rad = sqrtf(-2.0f * __logf(u1));
    float sn, cs;
    __sincosf(th, &sn, &cs);
    const int e1 = max(-bound, min(bound, __float2int_rn(sigma * rad * cs)));
    const int e2 = max(-bound, min(bound, __float2int_rn(sigma * rad * sn)));
    int8_t* o = out + poly * 3 * n + pos;
    o[0] = (int8_t)u;
    o[n] = (int8_t)e1;
    o[2 * n] = (int8_t)e2;
  }
}

template <int LOGN>
__global__ void k_draws_layout(const int8_t* in, int8_t* out, uint64_t total) {
  constexpr uint32_t n = 1u << LOGN;
  for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < total; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t row = g >> pow2_shift(n);   // poly * 3 + kind
    const uint32_t pos = (uint32_t)(g & (n - 1));
    out[g] = in[row * n + (uint32_t)draw_coef<LOGN>((int)pos)];
  }
}

}  // namespace ctb

using namespace ctb;


extern "C" int ctb_sample_draws(const ctb_ctx_t* ctx, uint64_t seed, uint64_t first_poly, double sigma, int bound,
                                int8_t* out, uint64_t batch, void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !out) { set_error("ctb_sample_draws: bad context or buffer"); return ERR_ARG; }
  if (bound < 0 || bound > 127 || !(sigma >= 0.0)) { set_error("ctb_sample_draws: bound must be in [0, 127], sigma >= 0"); return ERR_ARG; }
  const uint64_t total = batch * c->n;
  cudaStream_t s = (cudaStream_t)stream;
  CTB_DISPATCH_LOGN(c->logn, (k_sample_draws<LOGN><<<grid_stride(total, 16), 256, 0, s>>>(out, seed, first_poly, total,
                                                                                (float)sigma, bound)));
  return cuda_status(cudaGetLastError(), "ctb_sample_draws");
}

extern "C" int ctb_draws_from_natural(const ctb_ctx_t* ctx, const int8_t* in, int8_t* out, uint64_t batch,
                                      void* stream) {
  if (batch == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  const Ctx* c = reinterpret_cast<const Ctx*>(ctx);
  if (!c || !in || !out || in == out) { set_error("ctb_draws_from_natural: bad context or buffer (no in-place)"); return ERR_ARG; }
  const uint64_t total = batch * 3 * c->n;
  cudaStream_t s = (cudaStream_t)stream;
  CTB_DISPATCH_LOGN(c->logn, (k_draws_layout<LOGN><<<grid_stride(total, 16), 256, 0, s>>>(in, out, total)));
  return cuda_status(cudaGetLastError(), "ctb_draws_from_natural");
}
