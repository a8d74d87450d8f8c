// Host-side context: per-base prime tables resident in device memory.
//
// Replaces the reference's per-(n, modulus) plan cache `_plan` / `_NttPlan`
// (ring.py:164-229) and the derived constants of `HeParams` (he.py:61-132).
// Read-only after creation, so concurrent calls from two party threads on
// different streams are safe (threading).
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "ntt.cuh"

namespace ctb {

enum BaseId { BASE_Q = 0, BASE_T = 1, BASE_B = 2, BASE_COUNT = 3 };

struct Base {
  std::vector<uint64_t> primes;
  int word = 4;            // 4 -> uint32 residues, 8 -> uint64 residues
  void* d_tabs = nullptr;  // PrimeTab<T>[L]
  void* d_tw = nullptr;    // twiddle pairs, L * 2 * 2N words
  int size() const { return (int)primes.size(); }
};

// Constants for exact RNS <-> integer work (mixed-radix / Garner), filled by
// rns.cu.  All device arrays are uint64 words regardless of the base word.
struct RnsConsts;
struct TensorState;

struct Ctx {
  uint32_t n = 0, logn = 0;
  Base base[BASE_COUNT];
  uint64_t t = 0, t_half = 0;   // plain modulus (0 when the context has no plain ring)
  uint32_t crt_inv = 0, crt_inv_q = 0;  // (t0^-1 mod t1) and Shoup quotient, 2-prime plain CRT
  bool plain_fast = false;      // cheap plaintext lift (lift_plain_regs, ntt.cuh): u32 limbs t < 2^57 and every
                                // cipher prime > 2^25; u64 limbs t <= every cipher prime
  uint32_t relin_base_bits = 16;
  uint32_t wave_chunk = 296;    // items per limb-major chunk (= 2 x SM count, set at creation)
  RnsConsts* rns = nullptr;
  TensorState* tensor = nullptr;  // built lazily on first CCMul (tensor.cu)
  // stream-ordered scratch (per-call temporaries, e.g. relinearisation keys in the thread-major
  // layout); its own pool keeps freed memory mapped across synchronisations (release threshold
  // max) and is safe for concurrent calls from the party threads sharing the context
  cudaMemPool_t pool = nullptr;
  ~Ctx();
};

// thread-local error text for ctb_last_error()
void set_error(const std::string& msg);
const char* get_error();

// stream-ordered copy of a small host table through a thread-local pinned ring buffer (ctx.cu):
// returns without synchronising the stream; the host source may be freed right after the call
cudaError_t stage_upload(void* dst, const void* src, size_t bytes, cudaStream_t s);

// exact host arithmetic
inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
  return (uint64_t)((unsigned __int128)a * b % m);
}
inline uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod(r, b, m);
    b = mulmod(b, b, m);
    e >>= 1;
  }
  return r;
}
inline uint64_t invmod(uint64_t a, uint64_t m) { return powmod(a, m - 2, m); }  // m prime

// extra per-prime constants of the cipher base (may be null): t mod p, floor(q/t) mod p
int build_base(Base& b, const uint64_t* primes, int count, uint32_t logn, std::string& err,
               const uint64_t* tmod = nullptr, const uint64_t* delta = nullptr);
void free_base(Base& b);
// rns.cu: exact conversion constants of the cipher base (needs BASE_Q and BASE_T built)
int build_rns_consts(Ctx* c, std::string& err);
void free_rns_consts(RnsConsts* rc);
// tensor.cu: auxiliary base + constants for exact tensoring / relinearisation
int build_tensor_consts(Ctx* c, std::string& err);
void free_tensor_consts(TensorState* t);

}  // namespace ctb
