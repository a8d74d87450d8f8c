// Pipe-throughput probe for the 30-bit modular multiply by a known constant (the NTT butterfly's
// twiddle product), register resident:
//   imad     a = a*w + c                         (IMAD, fma-heavy pipe)
//   imadhi   a = hi(a*wq) + a                    (IMAD.HI)
//   dfma     d = d*x + y                         (DFMA, FP64 pipe)
//   shoup    a*w - hi(a*wq)*p                    (IMAD.HI + 2 IMAD)   <- the butterfly today
//   f64q     quotient rint(a*w/p) from ONE DFMA on the exponent-spliced double of a, then
//            a*w + p - q*p in (0, 2p) with 2 IMAD  (MOV + DFMA + 2 IMAD)
//   mix      half the chains shoup, half f64q
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe/imad_probe tools/probe/imad_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int CH = 8;

__device__ __forceinline__ uint32_t shoup(uint32_t a, uint32_t w, uint32_t wq, uint32_t p) {
  return a * w - __umulhi(a, wq) * p;
}
// wpk = the double 1.5*2^52 - 2^52 * wp' with wp' = round(w/p * 2^52) / 2^52 (an exact integer)
__device__ __forceinline__ uint32_t f64q(uint32_t a, uint32_t w, double wp, double kw, uint32_t p) {
  const double ad = __hiloint2double(0x43300000, (int)a);  // 2^52 + a, exact
  const double qd = __fma_rn(ad, wp, kw);                   // 1.5*2^52 + rint(a*wp'), exact sum rounded once
  const uint32_t q = (uint32_t)__double2loint(qd);
  uint32_t t, r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(a), "r"(w), "r"(p));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(0u - p), "r"(t));
  return r;                                                 // a*w + p - q*p in (0, 2p)
}

__device__ __forceinline__ uint32_t f64qc(uint32_t a, uint32_t w, double wp, uint32_t p) {
  const double qd = __fma_rn(__uint2double_rn(a), wp, 6755399441055744.0);  // I2F.F64.U32 + DFMA
  const uint32_t q = (uint32_t)__double2loint(qd);
  uint32_t t, r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(a), "r"(w), "r"(p));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(q), "r"(0u - p), "r"(t));
  return r;
}
__global__ void k_f64qc(uint32_t* out, uint32_t p, uint32_t w, double wp, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = (threadIdx.x * 77 + k) % p;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = f64qc(a[k], w, wp, p);
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
template <int NF>
__global__ void k_mixc(uint32_t* out, uint32_t p, uint32_t w, uint32_t wq, double wp, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = (threadIdx.x * 77 + k) % p;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = k < NF ? f64qc(a[k], w, wp, p) : shoup(a[k], w, wq, p);
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
__global__ void k_i2f(double* out, int iters) {
  uint32_t a[CH];
  double acc[CH];
  for (int k = 0; k < CH; ++k) { a[k] = threadIdx.x * 77 + k; acc[k] = 0; }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) { acc[k] = __uint2double_rn(a[k] + i); }
  double s = 0;
  for (int k = 0; k < CH; ++k) s += acc[k];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_imad(uint32_t* out, uint32_t w, uint32_t c, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = a[k] * w + c;
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
// ALU-pipe instructions of the butterfly: IADD3, VIADDMNMX (the fused conditional subtraction
// min(x - 2p, x)), VIMNMX
__global__ void k_iadd3(uint32_t* out, uint32_t b, uint32_t c, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(a[k]) : "r"(b), "r"(c));
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
__global__ void k_csub(uint32_t* out, uint32_t b, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = __viaddmin_u32(a[k], b, a[k]) ^ (uint32_t)i;
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
__global__ void k_min(uint32_t* out, uint32_t b, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = min(a[k], b) ^ (uint32_t)i;
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
__global__ void k_xor(uint32_t* out, uint32_t b, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = (a[k] & b) ^ (uint32_t)i;
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
__global__ void k_imadhi(uint32_t* out, uint32_t wq, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = __umulhi(a[k], wq) + a[k];
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
__global__ void k_dfma(double* out, double x, double y, int iters) {
  double a[CH];
  for (int k = 0; k < CH; ++k) a[k] = threadIdx.x * 77 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = __fma_rn(a[k], x, y);
  double s = 0;
  for (int k = 0; k < CH; ++k) s += a[k];
  if (s == 12345.0) out[0] = s;
}
__global__ void k_shoup(uint32_t* out, uint32_t p, uint32_t w, uint32_t wq, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = (threadIdx.x * 77 + k) % p;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = shoup(a[k], w, wq, p);
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
__global__ void k_f64q(uint32_t* out, uint32_t p, uint32_t w, double wp, double kw, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = (threadIdx.x * 77 + k) % p;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = f64q(a[k], w, wp, kw, p);
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
template <int NF>
__global__ void k_mix(uint32_t* out, uint32_t p, uint32_t w, uint32_t wq, double wp, double kw, int iters) {
  uint32_t a[CH];
  for (int k = 0; k < CH; ++k) a[k] = (threadIdx.x * 77 + k) % p;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) a[k] = k < NF ? f64q(a[k], w, wp, kw, p) : shoup(a[k], w, wq, p);
  uint32_t s = 0;
  for (int k = 0; k < CH; ++k) s ^= a[k];
  if (s == 12345) out[0] = s;
}
// correctness of f64q over many (a, w): r == a*w mod p (mod p) and 0 < r < 2p
__global__ void k_check(uint32_t* bad, uint32_t p, const uint32_t* ws, const double* wps, const double* kws, int nw) {
  const uint32_t a0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (int j = 0; j < nw; ++j) {
    for (uint32_t a = a0; a < 4u * p; a += gridDim.x * blockDim.x * 97u) {
      const uint32_t r = f64q(a, ws[j], wps[j], kws[j], p);
      const uint64_t want = (uint64_t)a * ws[j] % p;
      if (r >= 2 * p || (r % p) != want) atomicAdd(bad, 1u);
    }
  }
}

static void time_it(const char* name, double ops, void (*launch)(void*), void* arg) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch(arg);
  cudaEventRecord(a);
  launch(arg);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-10s %8.1f G op/s  (%.3f ms)\n", name, ops / ms / 1e6, ms);
}

struct Args { uint32_t* u; double* d; uint32_t p, w, wq; double wp, kw; int iters; };
static const int BLOCKS = 148 * 8, THREADS = 256;

int main() {
  const uint32_t p = 1073692673u;  // ntt_primes(4096, 30, 7)[0]
  const uint32_t w = 510015274u;
  const uint32_t wq = (uint32_t)(((uint64_t)w << 32) / p);
  const double wpr = (double)w / (double)p;
  const double wp = nearbyint(wpr * 4503599627370496.0) / 4503599627370496.0;
  const double kw = 6755399441055744.0 - 4503599627370496.0 * wp;
  Args A{nullptr, nullptr, p, w, wq, wp, kw, 4096};
  cudaMalloc(&A.u, 64); cudaMalloc(&A.d, 64);
  const double n = (double)BLOCKS * THREADS * A.iters * CH;
  for (int rep = 0; rep < 2; ++rep) {
    time_it("imad", n, [](void* v) { Args* a = (Args*)v; k_imad<<<BLOCKS, THREADS>>>(a->u, a->w, a->p, a->iters); }, &A);
    time_it("imadhi", n, [](void* v) { Args* a = (Args*)v; k_imadhi<<<BLOCKS, THREADS>>>(a->u, a->wq, a->iters); }, &A);
    time_it("iadd3", n, [](void* v) { Args* a = (Args*)v; k_iadd3<<<BLOCKS, THREADS>>>(a->u, a->w, a->p, a->iters); }, &A);
    time_it("csub+xor", n, [](void* v) { Args* a = (Args*)v; k_csub<<<BLOCKS, THREADS>>>(a->u, 0u - 2 * a->p, a->iters); }, &A);
    time_it("min+xor", n, [](void* v) { Args* a = (Args*)v; k_min<<<BLOCKS, THREADS>>>(a->u, a->p, a->iters); }, &A);
    time_it("lop3", n, [](void* v) { Args* a = (Args*)v; k_xor<<<BLOCKS, THREADS>>>(a->u, a->p, a->iters); }, &A);
    time_it("dfma", n, [](void* v) { Args* a = (Args*)v; k_dfma<<<BLOCKS, THREADS>>>(a->d, 0.999, 1.0, a->iters); }, &A);
    time_it("shoup", n, [](void* v) { Args* a = (Args*)v; k_shoup<<<BLOCKS, THREADS>>>(a->u, a->p, a->w, a->wq, a->iters); }, &A);
    time_it("f64q", n, [](void* v) { Args* a = (Args*)v; k_f64q<<<BLOCKS, THREADS>>>(a->u, a->p, a->w, a->wp, a->kw, a->iters); }, &A);
    time_it("mix2/8", n, [](void* v) { Args* a = (Args*)v; k_mix<2><<<BLOCKS, THREADS>>>(a->u, a->p, a->w, a->wq, a->wp, a->kw, a->iters); }, &A);
    time_it("mix3/8", n, [](void* v) { Args* a = (Args*)v; k_mix<3><<<BLOCKS, THREADS>>>(a->u, a->p, a->w, a->wq, a->wp, a->kw, a->iters); }, &A);
    time_it("f64qc", n, [](void* v) { Args* a = (Args*)v; k_f64qc<<<BLOCKS, THREADS>>>(a->u, a->p, a->w, a->wp, a->iters); }, &A);
    time_it("mixc2/8", n, [](void* v) { Args* a = (Args*)v; k_mixc<2><<<BLOCKS, THREADS>>>(a->u, a->p, a->w, a->wq, a->wp, a->iters); }, &A);
    time_it("mixc3/8", n, [](void* v) { Args* a = (Args*)v; k_mixc<3><<<BLOCKS, THREADS>>>(a->u, a->p, a->w, a->wq, a->wp, a->iters); }, &A);
    time_it("i2f", n, [](void* v) { Args* a = (Args*)v; k_i2f<<<BLOCKS, THREADS>>>(a->d, a->iters); }, &A);
    time_it("mix4/8", n, [](void* v) { Args* a = (Args*)v; k_mix<4><<<BLOCKS, THREADS>>>(a->u, a->p, a->w, a->wq, a->wp, a->kw, a->iters); }, &A);
  }
  // correctness sweep: random twiddles incl. extremes
  const int NW = 64;
  uint32_t hw[NW]; double hwp[NW], hkw[NW];
  srand(7);
  for (int j = 0; j < NW; ++j) {
    uint32_t ww = j == 0 ? 1u : j == 1 ? p - 1 : j == 2 ? p / 2 : (uint32_t)(((uint64_t)rand() << 16 ^ rand()) % p);
    hw[j] = ww;
    hwp[j] = nearbyint((double)ww / (double)p * 4503599627370496.0) / 4503599627370496.0;
    hkw[j] = 6755399441055744.0 - 4503599627370496.0 * hwp[j];
  }
  uint32_t *dw, *dbad; double *dwp, *dkw;
  cudaMalloc(&dw, sizeof hw); cudaMalloc(&dwp, sizeof hwp); cudaMalloc(&dkw, sizeof hkw); cudaMalloc(&dbad, 4);
  cudaMemcpy(dw, hw, sizeof hw, cudaMemcpyHostToDevice);
  cudaMemcpy(dwp, hwp, sizeof hwp, cudaMemcpyHostToDevice);
  cudaMemcpy(dkw, hkw, sizeof hkw, cudaMemcpyHostToDevice);
  cudaMemset(dbad, 0, 4);
  k_check<<<148 * 4, 256>>>(dbad, p, dw, dwp, dkw, NW);
  uint32_t bad = 0;
  cudaMemcpy(&bad, dbad, 4, cudaMemcpyDeviceToHost);
  printf("f64q check: %u bad of %.0f (err=%s)\n", bad, (double)NW * 4.0 * p / 97.0, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
