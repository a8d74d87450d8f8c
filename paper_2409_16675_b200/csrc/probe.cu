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
template <int NF>
__global__ void __launch_bounds__(256) k_probe_mix(uint32_t* sink, uint64_t iters, uint32_t p, uint32_t w, uint32_t wq,
                                                   double wp) {
  uint32_t a[CHAINS];
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) a[j] = (threadIdx.x * 131 + blockIdx.x * 7 + j) % p;
  const double kq = f64q_k(wp);
  const uint32_t pn = 0u - p;
  for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) a[j] = j < NF ? f64q_mul(a[j], w, wp, kq, p, pn) : shoup_mul(a[j], w, wq, p);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; ++j) acc ^= a[j];
  if (acc == 0x5eedu) sink[0] = acc;
}
}  // namespace

extern "C" int ctb_probe_modmul_mix(int f64q_of_8, uint64_t iters, void* sink, uint64_t* modmuls, void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)sms * 8, block = 256;
  cudaStream_t s = (cudaStream_t)stream;
  const uint32_t p = 1073692673u, w = 510015274u;
  const uint32_t wq = (uint32_t)(((uint64_t)w << 32) / p);
  const double wp = std::ldexp((double)(uint64_t)((((unsigned __int128)w << 52) + p / 2) / p), -52);
  uint32_t* o = (uint32_t*)sink;
  switch (f64q_of_8) {
    case 0: k_probe_mix<0><<<grid, block, 0, s>>>(o, iters, p, w, wq, wp); break;
    case 3: k_probe_mix<3><<<grid, block, 0, s>>>(o, iters, p, w, wq, wp); break;
    case 8: k_probe_mix<8><<<grid, block, 0, s>>>(o, iters, p, w, wq, wp); break;
    default:
      set_error("ctb_probe_modmul_mix: f64q_of_8 must be 0, 3 or 8");
      return ERR_ARG;
  }
  if (modmuls) *modmuls = (uint64_t)grid * block * CHAINS * iters;
  return cuda_status(cudaGetLastError(), "ctb_probe_modmul_mix");
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
