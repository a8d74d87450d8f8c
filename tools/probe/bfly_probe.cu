// Register-resident radix-16 forward pass (4 Harvey CT stages on 16 residues per thread, 30-bit
// prime, twiddles from shared memory like k_cpmul) with a choice of quotient per twiddle entry:
//   Shoup          IMAD.HI + 2 IMAD                      (fma-heavy pipe only)
//   splice         MOV + DFMA + 2 IMAD                   (2^52 + a exponent splice, ntt.cuh f64q_mul)
//   convert        I2F.F64.U32 + DFMA + 2 IMAD           (conversion on the XU pipe, no register pair)
// Entries e < QS use the splice, QS <= e < QS + QC the conversion, the rest Shoup (e = 2^i - 1 + jb:
// stage i, block jb; entry 0 serves 8 butterflies, 1-2 four each, 3-6 two each, 7-14 one each).
// Prints G butterflies/s per variant: the ceiling of a transform's own arithmetic per pipe mix.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/bfly_probe tools/probe/bfly_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t csub(uint32_t x, uint32_t y) { return min(x - y, x); }
__device__ __forceinline__ uint32_t shoup(uint32_t a, uint32_t w, uint32_t wq, uint32_t p) {
  return a * w - __umulhi(a, wq) * p;
}
__device__ __forceinline__ uint32_t fin(uint32_t a, uint32_t w, double qd, uint32_t p, uint32_t pn) {
  const uint32_t q = (uint32_t)__double2loint(qd);
  uint32_t t, r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(a), "r"(w), "r"(p));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(pn), "r"(t));
  return r;
}
__device__ __forceinline__ uint32_t f64_splice(uint32_t a, uint32_t w, double wp, double kq, uint32_t p, uint32_t pn) {
  return fin(a, w, __fma_rn(__hiloint2double(0x43300000, (int)a), wp, kq), p, pn);
}
__device__ __forceinline__ uint32_t f64_conv(uint32_t a, uint32_t w, double wp, uint32_t p, uint32_t pn) {
  return fin(a, w, __fma_rn(__uint2double_rn(a), wp, 6755399441055744.0), p, pn);
}

struct Tw { uint32_t w, wq; };

// AM: how the two-input add X' = xx + t is written.  ptxas turns plain two-input adds into IMAD.IADD
// (fma-heavy pipe, half rate on sm_100) when it thinks the ALU is the busier pipe; a third, opaque
// operand (a kernel parameter that is 0 / 0xffffffff at run time) keeps them on the ALU pipe:
//   0 plain,  1 IADD3 xx + t + zero,  2 VIADDMNMX min(xx + t, big)
template <int AM>
__device__ __forceinline__ uint32_t add2(uint32_t a, uint32_t b, uint32_t zero, uint32_t big) {
  if constexpr (AM == 1) return a + b + zero;
  else if constexpr (AM == 2) return __viaddmin_u32(a, b, big);
  else return a + b;
}
template <int QS, int QC, int AM = 0>
__global__ void __launch_bounds__(1024, 1) k_pass(uint32_t* out, const Tw* gtw, const double* gwp, uint32_t p, int iters,
                                                  uint32_t zero, uint32_t big) {
  __shared__ Tw tw[16 * 64];
  __shared__ double wps[16 * 64];
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) { tw[i] = gtw[i]; wps[i] = gwp[i]; }
  __syncthreads();
  const uint32_t p2 = 2 * p, pn = 0u - p;
  uint32_t x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = (threadIdx.x * 77 + k * 1315423911u) % p;
  const int slot = threadIdx.x & 63;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int h = 1 << (3 - i);
#pragma unroll
      for (int jb = 0; jb < (1 << i); ++jb) {
        const int e = (1 << i) - 1 + jb;
        const volatile Tw* t = &tw[e * 64 + slot];
        uint32_t w, wq;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w), "=r"(wq) : "r"((uint32_t)__cvta_generic_to_shared((const void*)t)));
        if (e < QS + QC) {
          double wp;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(wp) : "r"((uint32_t)__cvta_generic_to_shared(&wps[e * 64 + slot])));
          const double kq = __fma_rn(-4503599627370496.0, wp, 6755399441055744.0);
#pragma unroll
          for (int jj = 0; jj < h; ++jj) {
            const int a = jb * 2 * h + jj;
            const uint32_t xx = csub(x[a], p2);
            const uint32_t tt = e < QS ? f64_splice(x[a + h], w, wp, kq, p, pn) : f64_conv(x[a + h], w, wp, p, pn);
            x[a] = add2<AM>(xx, tt, zero, big);
            x[a + h] = xx - tt + p2;
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < h; ++jj) {
            const int a = jb * 2 * h + jj;
            const uint32_t xx = csub(x[a], p2);
            const uint32_t tt = shoup(x[a + h], w, wq, p);
            x[a] = add2<AM>(xx, tt, zero, big);
            x[a + h] = xx - tt + p2;
          }
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s ^= x[k];
  if (s == 12345) out[0] = s;
}

template <int QS, int QC, int AM = 0>
static void run(const char* name, uint32_t* out, const Tw* tw, const double* wp, uint32_t p, int threads) {
  const int iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = 148 * (1024 / threads);
  k_pass<QS, QC, AM><<<blocks, threads>>>(out, tw, wp, p, 50, 0u, 0xffffffffu);
  cudaEventRecord(a);
  k_pass<QS, QC, AM><<<blocks, threads>>>(out, tw, wp, p, iters, 0u, 0xffffffffu);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bf = (double)blocks * threads * iters * 32.0;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_pass<QS, QC, AM>);
  printf("%-22s add%d splice<%2d conv<%2d  %8.1f G bfly/s  (%.3f ms, %d regs, %s)\n", name, AM, QS, QS + QC, bf / ms / 1e6, ms,
         fa.numRegs, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint32_t p = 1073692673u;
  Tw htw[16 * 64]; double hwp[16 * 64];
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < 16 * 64; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const uint32_t w = (uint32_t)(s % p);
    htw[i] = {w, (uint32_t)(((uint64_t)w << 32) / p)};
    hwp[i] = std::ldexp((double)(uint64_t)((((unsigned __int128)w << 52) + p / 2) / p), -52);
  }
  Tw* dtw; double* dwp; uint32_t* out;
  cudaMalloc(&dtw, sizeof htw); cudaMalloc(&dwp, sizeof hwp); cudaMalloc(&out, 64);
  cudaMemcpy(dtw, htw, sizeof htw, cudaMemcpyHostToDevice);
  cudaMemcpy(dwp, hwp, sizeof hwp, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    run<0, 0>("shoup", out, dtw, dwp, p, 1024);
    run<0, 0, 1>("shoup", out, dtw, dwp, p, 1024);
    run<0, 0, 2>("shoup", out, dtw, dwp, p, 1024);
    run<2, 0, 1>("splice e<2", out, dtw, dwp, p, 1024);
    run<2, 0, 2>("splice e<2", out, dtw, dwp, p, 1024);
    run<3, 0, 1>("splice e<3", out, dtw, dwp, p, 1024);
    run<7, 0, 1>("splice e<7", out, dtw, dwp, p, 1024);
    run<7, 0, 2>("splice e<7", out, dtw, dwp, p, 1024);
    run<15, 0, 1>("splice all", out, dtw, dwp, p, 1024);
    run<0, 3, 1>("conv e<3", out, dtw, dwp, p, 1024);
    run<0, 7, 1>("conv e<7", out, dtw, dwp, p, 1024);
    run<0, 15, 1>("conv all", out, dtw, dwp, p, 1024);
    run<3, 4, 1>("splice 3 conv 4", out, dtw, dwp, p, 1024);
    run<3, 12, 1>("splice 3 conv 12", out, dtw, dwp, p, 1024);
    run<2, 0>("splice e<2 (today)", out, dtw, dwp, p, 1024);
    run<3, 0>("splice e<3", out, dtw, dwp, p, 1024);
    run<7, 0>("splice e<7", out, dtw, dwp, p, 1024);
    run<15, 0>("splice all", out, dtw, dwp, p, 1024);
    run<0, 2>("conv e<2", out, dtw, dwp, p, 1024);
    run<0, 3>("conv e<3", out, dtw, dwp, p, 1024);
    run<0, 7>("conv e<7", out, dtw, dwp, p, 1024);
    run<0, 15>("conv all", out, dtw, dwp, p, 1024);
    run<1, 1>("splice 1 conv 1", out, dtw, dwp, p, 1024);
    run<1, 2>("splice 1 conv 2", out, dtw, dwp, p, 1024);
    run<2, 1>("splice 2 conv 1", out, dtw, dwp, p, 1024);
    run<1, 6>("splice 1 conv 6", out, dtw, dwp, p, 1024);
    run<2, 5>("splice 2 conv 5", out, dtw, dwp, p, 1024);
    run<3, 4>("splice 3 conv 4", out, dtw, dwp, p, 1024);
    run<1, 14>("splice 1 conv 14", out, dtw, dwp, p, 1024);
    run<3, 12>("splice 3 conv 12", out, dtw, dwp, p, 1024);
  }
  return 0;
}
