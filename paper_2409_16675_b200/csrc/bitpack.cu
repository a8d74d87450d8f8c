// Dense bit-packed host format for the PCIe leg of the end-to-end path.
//
// A residue of a 30-bit prime needs 30 bits, a plaintext value of t < 2^50 needs 50, but the device
// layouts hold them in 32- and 64-bit words.  Across PCIe (the end-to-end CPMul path is bound by it)
// the batch travels as one little-endian bitstream instead -- value j at bits [j b, (j+1) b) -- and
// is expanded / compacted on the device by these kernels (HBM is ~100x faster than the link).
//
//   ctb_bits_unpack  packed words -> uint32 / uint64 values   (one thread per value)
//   ctb_bits_pack    uint32 / uint64 values -> packed words   (one thread per output word, so the
//                                                              stores need no atomics)
#include "ctb200.h"
#include "kernels.hpp"

using namespace ctb;

namespace {

template <typename T>
__global__ void __launch_bounds__(256) k_bits_unpack(const uint32_t* __restrict__ in, T* __restrict__ out, uint32_t bits,
                                                     uint64_t count) {
  const uint64_t mask = bits == 64 ? ~0ull : ((1ull << bits) - 1);
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t bit = j * bits;
    const uint64_t w = bit >> 5;
    const uint32_t s = (uint32_t)(bit & 31);
    uint64_t v = (uint64_t)__ldg(in + w) >> s;
    if (s + bits > 32) v |= (uint64_t)__ldg(in + w + 1) << (32 - s);
    if (s + bits > 64) v |= (uint64_t)__ldg(in + w + 2) << (64 - s);
    out[j] = (T)(v & mask);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_bits_pack(const T* __restrict__ in, uint32_t* __restrict__ out, uint32_t bits,
                                                   uint64_t count, uint64_t words) {
  const uint64_t mask = bits == 64 ? ~0ull : ((1ull << bits) - 1);
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t lo = w * 32, hi = lo + 32;  // this word's bit range
    uint32_t acc = 0;
    for (uint64_t j = lo / bits; j * bits < hi && j < count; ++j) {
      const uint64_t v = (uint64_t)__ldg(in + j) & mask;
      const int64_t sh = (int64_t)(j * bits) - (int64_t)lo;  // value's first bit relative to the word
      if (sh >= 0) acc |= (uint32_t)(v << sh);
      else acc |= (uint32_t)(v >> (-sh));
    }
    out[w] = acc;
  }
}

}  // namespace

extern "C" uint64_t ctb_bits_words(uint32_t bits, uint64_t count) { return (count * bits + 31) / 32; }

extern "C" int ctb_bits_unpack(const ctb_ctx_t* ctx, int word_bytes, const uint32_t* in, uint32_t bits, void* out,
                               uint64_t count, void* stream) {
  if (count == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  if (!ctx || !in || !out || (word_bytes != 4 && word_bytes != 8) || bits < 1 || bits > 8u * (uint32_t)word_bytes) {
    set_error("ctb_bits_unpack: bad arguments (word 4 or 8 bytes, 1 <= bits <= word bits)");
    return ERR_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (word_bytes == 4)
    k_bits_unpack<uint32_t><<<grid_stride(count, 8), 256, 0, s>>>(in, (uint32_t*)out, bits, count);
  else
    k_bits_unpack<uint64_t><<<grid_stride(count, 8), 256, 0, s>>>(in, (uint64_t*)out, bits, count);
  return cuda_status(cudaGetLastError(), "ctb_bits_unpack");
}

extern "C" int ctb_bits_pack(const ctb_ctx_t* ctx, int word_bytes, const void* in, uint32_t bits, uint32_t* out,
                             uint64_t count, void* stream) {
  if (count == 0 && ctx) return OK;  // empty batch: no-op, buffers may be null
  if (!ctx || !in || !out || (word_bytes != 4 && word_bytes != 8) || bits < 1 || bits > 8u * (uint32_t)word_bytes) {
    set_error("ctb_bits_pack: bad arguments (word 4 or 8 bytes, 1 <= bits <= word bits)");
    return ERR_ARG;
  }
  const uint64_t words = ctb_bits_words(bits, count);
  cudaStream_t s = (cudaStream_t)stream;
  if (word_bytes == 4)
    k_bits_pack<uint32_t><<<grid_stride(words, 8), 256, 0, s>>>((const uint32_t*)in, out, bits, count, words);
  else
    k_bits_pack<uint64_t><<<grid_stride(words, 8), 256, 0, s>>>((const uint64_t*)in, out, bits, count, words);
  return cuda_status(cudaGetLastError(), "ctb_bits_pack");
}
