// Context lifetime and introspection entry points of the C ABI.
#include <cstdlib>
#include <string>
#include "bigint.hpp"
#include "ctb200.h"
#include "kernels.hpp"

using namespace ctb;

namespace ctb {
Ctx::~Ctx() {
  if (pool) cudaMemPoolDestroy(pool);
  free_tensor_consts(tensor);
  free_rns_consts(rns);
  for (auto& b : base) free_base(b);
}
}  // namespace ctb

extern "C" const char* ctb_last_error(void) { return get_error(); }
extern "C" int ctb_version(void) { return 1; }

extern "C" int ctb_ctx_create(ctb_ctx_t** out, uint32_t n, const uint64_t* q_primes, uint32_t n_q,
                              const uint64_t* t_primes, uint32_t n_t, uint32_t relin_base_bits) {
  if (!out) { set_error("ctb_ctx_create: null output"); return ERR_ARG; }
  *out = nullptr;
  if (n < 4 || (n & (n - 1))) { set_error("ring degree must be a power of two >= 4"); return ERR_ARG; }
  if (!q_primes || n_q == 0) { set_error("ctb_ctx_create: no cipher primes"); return ERR_ARG; }
  uint32_t logn = 0;
  while ((1u << logn) < n) ++logn;
  if (logn > 13) { set_error("ring degree above 8192 unsupported"); return ERR_UNSUPPORTED; }
  Ctx* c = new Ctx();
  c->n = n; c->logn = logn; c->relin_base_bits = relin_base_bits;
  {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    c->wave_chunk = 2u * (uint32_t)(sms > 0 ? sms : 148);
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&c->pool, &props) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep);
    } else {
      c->pool = nullptr;
      cudaGetLastError();
    }
    if (const char* env = std::getenv("CTB_WAVE_CHUNK")) {  // tuning knob
      const long v = std::strtol(env, nullptr, 10);
      if (v > 0) c->wave_chunk = (uint32_t)v;
    }
  }
  std::string err;
  // plain modulus t = prod t_j (< 2^63, as the reference's uint64 plain ring, ring.py:151-152)
  std::vector<uint64_t> tmod, delta;
  if (n_t) {
    BigU tb(1);
    for (uint32_t j = 0; j < n_t; ++j) tb.mul_small(t_primes[j]);
    if (tb.bit_length() > 63) { delete c; set_error("plain modulus must be below 2^63"); return ERR_UNSUPPORTED; }
    c->t = tb.word64(0);
    c->t_half = c->t / 2;
    BigU q(1);
    for (uint32_t i = 0; i < n_q; ++i) q.mul_small(q_primes[i]);
    BigU dq = q;
    dq.divmod_small(c->t);  // Delta = floor(q / t)  (he.py:88-90)
    for (uint32_t i = 0; i < n_q; ++i) {
      tmod.push_back(c->t % q_primes[i]);
      delta.push_back(dq.mod_small(q_primes[i]));
    }
    int rc = build_base(c->base[BASE_T], t_primes, (int)n_t, logn, err);
    if (rc) { delete c; set_error("plain base: " + err); return rc == -2 ? ERR_CUDA : ERR_ARG; }
    if (n_t == 2) {
      const uint64_t inv = invmod(t_primes[0] % t_primes[1], t_primes[1]);
      c->crt_inv = (uint32_t)inv;
      c->crt_inv_q = (uint32_t)(((unsigned __int128)inv << 32) / t_primes[1]);
    }
  }
  int rc = build_base(c->base[BASE_Q], q_primes, (int)n_q, logn, err, n_t ? tmod.data() : nullptr,
                      n_t ? delta.data() : nullptr);
  if (rc) { delete c; set_error("cipher base: " + err); return rc == -2 ? ERR_CUDA : ERR_ARG; }
  {
    // 32-bit limbs: t < 2^57 and every cipher prime > 2^25 (one Shoup product per lifted value);
    // 64-bit limbs: t <= every cipher prime (a plain value is its own residue: no product at all)
    bool fast = c->t != 0;
    if (c->base[BASE_Q].word == 4) {
      fast = fast && c->t < (1ull << 57);
      for (uint32_t i = 0; i < n_q; ++i) fast = fast && q_primes[i] > (1ull << 25);
    } else {
      for (uint32_t i = 0; i < n_q; ++i) fast = fast && c->t <= q_primes[i];
    }
    c->plain_fast = fast;
  }
  rc = build_rns_consts(c, err);
  if (rc) { delete c; set_error("conversion constants: " + err); return rc == -2 ? ERR_CUDA : (rc == -3 ? ERR_UNSUPPORTED : ERR_ARG); }
  *out = reinterpret_cast<ctb_ctx_t*>(c);
  return OK;
}

extern "C" int ctb_ctx_destroy(ctb_ctx_t* ctx) {
  delete reinterpret_cast<Ctx*>(ctx);
  return OK;
}

extern "C" int ctb_ctx_word_bytes(const ctb_ctx_t* ctx, int base) {
  if (!ctx || base < 0 || base >= BASE_COUNT) return ERR_ARG;
  const Base& b = reinterpret_cast<const Ctx*>(ctx)->base[base];
  return b.size() ? b.word : ERR_ARG;
}

extern "C" int ctb_ctx_base_size(const ctb_ctx_t* ctx, int base) {
  if (!ctx || base < 0 || base >= BASE_COUNT) return ERR_ARG;
  return reinterpret_cast<const Ctx*>(ctx)->base[base].size();
}

extern "C" int ctb_ctx_base_primes(const ctb_ctx_t* ctx, int base, uint64_t* out, uint32_t cap) {
  if (!ctx || base < 0 || base >= BASE_COUNT || !out) return ERR_ARG;
  const Base& b = reinterpret_cast<const Ctx*>(ctx)->base[base];
  uint32_t k = 0;
  for (; k < cap && k < (uint32_t)b.size(); ++k) out[k] = b.primes[k];
  return (int)k;
}
