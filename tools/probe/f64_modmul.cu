// Throughput probe: 50-bit modular multiply by a constant, u64 Shoup (IMAD) vs FP64 (DFMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe f64_modmul.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mulhi64_approx(uint64_t a, uint64_t b) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  const uint64_t m1 = (uint64_t)a1 * b0, m2 = (uint64_t)a0 * b1, hh = (uint64_t)a1 * b1;
  return hh + (m1 >> 32) + (m2 >> 32);
}

__global__ void k_u64(uint64_t* out, uint64_t p, uint64_t w, uint64_t wq, int iters) {
  uint64_t x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint64_t r = x[k] * w - mulhi64_approx(x[k], wq) * p;
      x[k] = r;
    }
  }
  uint64_t s = 0;
  for (int k = 0; k < 8; ++k) s ^= x[k];
  if (s == 12345) out[0] = s;
}

// FP64: x, w exact integers < 2^52; r = x*w mod p in (-p, 2p) then folded to [0, 2p) lazily.
__global__ void k_f64(double* out, double p, double w, double wp, int iters) {
  const double C = 6755399441055744.0;  // 1.5 * 2^52: round-to-nearest integer magic
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double hi = x[k] * w;
      const double lo = fma(x[k], w, -hi);
      const double q = fma(x[k], wp, C) - C;
      double r = fma(-q, p, hi) + lo;      // exact, in (-p, 2p)
      r = r < 0.0 ? r + p : r;
      x[k] = r;
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.0) out[0] = s;
}

int main() {
  const uint64_t p = 1125899906826241ull;  // ntt_primes(8192, 50, 3)[0]
  const uint64_t w = 987654321012345ull % p;
  const uint64_t wq = (uint64_t)(((unsigned __int128)w << 64) / p);
  uint64_t* du; double* dd;
  cudaMalloc(&du, 8); cudaMalloc(&dd, 8);
  int blocks = 148 * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_u64<<<blocks, threads>>>(du, p, w, wq, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double n = (double)blocks * threads * iters * 8;
    printf("u64 shoup : %.1f G modmul/s\n", n / ms / 1e6);
    cudaEventRecord(a);
    k_f64<<<blocks, threads>>>(dd, (double)p, (double)w, (double)w / (double)p, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("f64       : %.1f G modmul/s\n", n / ms / 1e6);
  }
  return 0;
}
