// Roofline probe: register-resident throughput of the exact modular
// multiplication the butterflies use (Shoup, lazy [0,2p)), per word width.
// MEASURED_PEAKS.json carries no integer peak, so bench.py measures this one on
// the box and divides by it.
#include "ctb200.h"
#include "kernels.hpp"

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
}  // namespace

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
