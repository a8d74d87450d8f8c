// Shared launch plumbing for the ring kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "ctx.hpp"
#include "ntt.cuh"

namespace ctb {

constexpr int OK = 0;
constexpr int ERR_ARG = -1;
constexpr int ERR_CUDA = -2;
constexpr int ERR_UNSUPPORTED = -3;

inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return ERR_CUDA;
}

// Launch a CTA-per-polynomial-limb kernel with the double-buffered exchange image.
// Per-kernel record of the dynamic shared-memory opt-in (cudaFuncSetAttribute
// is per function, so it is keyed by the kernel pointer).
bool smem_attr_done(const void* kern);
void smem_attr_mark(const void* kern);

// EXTRA_POLYS: additional N-word thread-private strips after the image.
template <typename T, int LOGN, int EXTRA_POLYS = 0, typename... KArgs, typename... Args>
inline cudaError_t launch_ntt_kernel(void (*kern)(KArgs...), size_t nblocks, cudaStream_t s,
                                     Args... args) {
  using Sh = NttShape<LOGN>;
  const size_t smem = ((size_t)Exchanger<T, LOGN>::WORDS + (size_t)EXTRA_POLYS * Sh::N) * sizeof(T);   // default NBUF = 2
  if (!smem_attr_done((const void*)kern)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_attr_mark((const void*)kern);
  }
  if (nblocks == 0) return cudaSuccess;
  kern<<<(unsigned)nblocks, Sh::THREADS, smem, s>>>(args...);
  return cudaGetLastError();
}

// Resident CTAs per SM x SM count for a persistent kernel (cached per kernel).
uint32_t persistent_grid(const void* kern, int threads, size_t smem);

// x mod t for a signed 64-bit value (RingElem.from_ints semantics), t < 2^63.
__device__ __forceinline__ uint64_t mod_signed(int64_t v, uint64_t t) {
  if (v >= 0) return (uint64_t)v < t ? (uint64_t)v : (uint64_t)v % t;
  const uint64_t a = (uint64_t)(-(v + 1)) + 1;  // |v| without overflow at INT64_MIN
  const uint64_t r = a < t ? a : a % t;
  return r ? t - r : 0;
}

// A packed plaintext given by its packing descriptor instead of its values (ctb_pack_gather's
// arguments): coefficient i of polynomial p is src[base[p] + maps[kind[p]][i]] mod t, 0 where the
// map is -1.  Kernels that consume plaintexts (encryption) read them through this directly, so the
// packed polynomial is never written out; `maps == nullptr` means "not used".
struct PlainGather {
  const int64_t* src = nullptr;
  uint64_t src_len = 0;
  const int32_t* maps = nullptr;
  uint32_t n_maps = 0;
  const int32_t* kind = nullptr;
  const int64_t* base = nullptr;
  uint64_t t = 0;
  // (kind, base) of one polynomial, loaded once per item
  __device__ __forceinline__ void row(uint64_t poly, uint32_t n, const int32_t*& mrow, int64_t& b) const {
    const uint32_t k = (uint32_t)__ldg(kind + poly);
    mrow = k < n_maps ? maps + (size_t)k * n : nullptr;
    b = __ldg(base + poly);
  }
  __device__ __forceinline__ uint64_t value(const int32_t* mrow, int64_t b, uint32_t i) const {
    if (!mrow) return 0;
    const int32_t m = __ldg(mrow + i);
    if (m < 0) return 0;
    const uint64_t at = (uint64_t)b + (uint64_t)m;
    return at < src_len ? mod_signed(__ldg(src + at), t) : 0;
  }
};

// Streaming multiprocessors of the current device (cached).
uint32_t sm_count();

// Grid for a 256-thread grid-stride elementwise kernel over `total` items: enough CTAs for
// `per_sm` resident per SM, never more than the items need.
inline unsigned grid_stride(uint64_t total, unsigned per_sm) {
  const uint64_t cap = (uint64_t)sm_count() * per_sm;
  const uint64_t need = (total + 255) / 256;
  return (unsigned)(need < 1 ? 1 : (need < cap ? need : cap));
}

// Launch with an explicit grid and dynamic shared memory (opt-in handled).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kernel_grid(void (*kern)(KArgs...), uint32_t grid, int threads, size_t smem,
                                      cudaStream_t s, Args... args) {
  if (!smem_attr_done((const void*)kern)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_attr_mark((const void*)kern);
  }
  if (grid == 0) return cudaSuccess;
  kern<<<grid, threads, smem, s>>>(args...);
  return cudaGetLastError();
}

#define CTB_CASE_LOGN(L_, ...) \
  case L_: {                   \
    constexpr int LOGN = L_;   \
    __VA_ARGS__;               \
  } break;

// Dispatch a body over the supported ring degrees N = 2^2 .. 2^13.
#define CTB_DISPATCH_LOGN(logn, ...)                                  \
  switch (logn) {                                                     \
    CTB_CASE_LOGN(2, __VA_ARGS__)                                     \
    CTB_CASE_LOGN(3, __VA_ARGS__)                                     \
    CTB_CASE_LOGN(4, __VA_ARGS__)                                     \
    CTB_CASE_LOGN(5, __VA_ARGS__)                                     \
    CTB_CASE_LOGN(6, __VA_ARGS__)                                     \
    CTB_CASE_LOGN(7, __VA_ARGS__)                                     \
    CTB_CASE_LOGN(8, __VA_ARGS__)                                     \
    CTB_CASE_LOGN(9, __VA_ARGS__)                                     \
    CTB_CASE_LOGN(10, __VA_ARGS__)                                    \
    CTB_CASE_LOGN(11, __VA_ARGS__)                                    \
    CTB_CASE_LOGN(12, __VA_ARGS__)                                    \
    CTB_CASE_LOGN(13, __VA_ARGS__)                                    \
    default:                                                          \
      set_error("ring degree 2^" + std::to_string(logn) + " unsupported"); \
      return ERR_UNSUPPORTED;                                         \
  }

// Same dispatch for helpers returning cudaError_t (unsupported degree -> cudaErrorInvalidValue).
#define CTB_DISPATCH_LOGN_E(logn, ...)        \
  switch (logn) {                             \
    CTB_CASE_LOGN(2, __VA_ARGS__)             \
    CTB_CASE_LOGN(3, __VA_ARGS__)             \
    CTB_CASE_LOGN(4, __VA_ARGS__)             \
    CTB_CASE_LOGN(5, __VA_ARGS__)             \
    CTB_CASE_LOGN(6, __VA_ARGS__)             \
    CTB_CASE_LOGN(7, __VA_ARGS__)             \
    CTB_CASE_LOGN(8, __VA_ARGS__)             \
    CTB_CASE_LOGN(9, __VA_ARGS__)             \
    CTB_CASE_LOGN(10, __VA_ARGS__)            \
    CTB_CASE_LOGN(11, __VA_ARGS__)            \
    CTB_CASE_LOGN(12, __VA_ARGS__)            \
    CTB_CASE_LOGN(13, __VA_ARGS__)            \
    default:                                  \
      return cudaErrorInvalidValue;           \
  }

// Unscaled inverse NTT of eval-domain [npoly][L][N] (+ coefficient addend), persistent
// (kernels_ntt.cu k_stream InvAdd).  In place allowed.
// strip_in: input in the thread-major chunk layout (stream_forward strip_out).
cudaError_t stream_inv_add(const Ctx* c, int base, const void* in, void* out, const void* addend, uint64_t npoly,
                           cudaStream_t s, bool strip_in = false);

// Persistent forward NTT of [npoly][L][N] over base `base`: canonical eval, or prepared
// (N^-1 2^W Montgomery operand) when `prepare` (k_stream Fwd / Prepare).  In place allowed.
// strip_out: thread-major chunk layout instead of the eval layout (internal operands only).
cudaError_t stream_forward(const Ctx* c, int base, bool prepare, const void* in, void* out, uint64_t npoly,
                           cudaStream_t s, bool strip_out = false);

// NTT of the lift of plain [npoly][N] (centred for the cipher base) per limb of `base`:
// prepared (N^-1 2^W, k_stream LiftPrepare) or canonical eval (LiftFwd).
cudaError_t stream_lift(const Ctx* c, int base, bool prepare, const uint64_t* m, void* out, uint64_t npoly,
                        cudaStream_t s, bool strip_out = false);

}  // namespace ctb
