/*
 * ctb200.h -- C ABI of the B200-native HE linear-layer hot path of CryptoTrain
 * (arXiv 2409.16675).  Library: paper_2409_16675_b200/lib/libctb200.so.
 *
 * The reference (pkg/src/privtrain, pure Python + numpy) has no FFI: its
 * boundary is the Python object API of he.He / ring / packing / linprot.
 * Each entry point below names the reference function whose arithmetic it
 * replaces; the Python mirror in paper_2409_16675_b200/ (he.py, ring.py,
 * linprot.py) is the binding a reference maintainer would call, see
 * INTEGRATION.md.
 *
 * Conventions
 *   - Every buffer argument is a DEVICE pointer owned by the caller; the
 *     library never frees or retains it.  Inputs are never written unless the
 *     same pointer is passed as the output (in-place is allowed where noted).
 *   - Residue layout is [poly][limb][N]; a limb's word is uint32 when every
 *     prime of its base is < 2^30 and uint64 otherwise (ctb_ctx_word_bytes).
 *     Plain-ring polynomials are [poly][N] uint64 in [0, t).
 *   - Ciphertexts are [batch][parts][L][N] residues of the cipher base.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *     asynchronous on that stream; a context is read-only after creation, so
 *     two threads may use one context on different streams concurrently.
 *   - Return value: CTB_OK (0) or a negative CTB_ERR_*; ctb_last_error()
 *     returns the thread-local message of the last failure.
 */
#ifndef CTB200_H
#define CTB200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ctb_ctx ctb_ctx_t;

enum { CTB_OK = 0, CTB_ERR_ARG = -1, CTB_ERR_CUDA = -2, CTB_ERR_UNSUPPORTED = -3 };

/* RNS bases held by a context. */
enum {
  CTB_BASE_Q = 0, /* cipher modulus q = prod q_i  (he.HeParams.cipher_ring, he.py:61-99) */
  CTB_BASE_T = 1, /* plain modulus  t = prod t_j  (he.HeParams.plain_ring)               */
  CTB_BASE_B = 2  /* auxiliary 30-bit NTT primes for exact tensoring (ring.py:498-541)   */
};

const char* ctb_last_error(void);
int ctb_version(void);

/* Context: replaces ring._plan/_NttPlan (ring.py:164-229) and the derived
 * constants of he.HeParams (he.py:61-132).  q_primes: the declared factorisation
 * of the cipher (or single) ring modulus, each = 1 mod 2N, < 2^62.  t_primes:
 * factorisation of the plain modulus (n_t = 0 for a ring-only context).
 * relin_base_bits: he.HeParams.relin_base_bits (he.py:68). */
int ctb_ctx_create(ctb_ctx_t** out, uint32_t n, const uint64_t* q_primes, uint32_t n_q,
                   const uint64_t* t_primes, uint32_t n_t, uint32_t relin_base_bits);
int ctb_ctx_destroy(ctb_ctx_t* ctx);
int ctb_ctx_word_bytes(const ctb_ctx_t* ctx, int base);  /* 4 or 8; <0 if absent */
int ctb_ctx_base_size(const ctb_ctx_t* ctx, int base);   /* number of primes     */
int ctb_ctx_base_primes(const ctb_ctx_t* ctx, int base, uint64_t* out, uint32_t cap);

/* Negacyclic NTT of n_polys polynomials over every limb of `base`
 * (ring.ntt_forward / ring.ntt_inverse, ring.py:549-569; the per-prime
 * transform of ring._NttPlan.forward/inverse, ring.py:186-217).  Output is
 * canonical; forward output is in the reference's bit-reversed order.
 * In-place allowed. */
int ctb_ntt_forward(const ctb_ctx_t* ctx, int base, const void* in, void* out, uint64_t n_polys,
                    void* stream);
int ctb_ntt_inverse(const ctb_ctx_t* ctx, int base, const void* in, void* out, uint64_t n_polys,
                    void* stream);
/* Slotwise product of evaluation-domain polys (ring.pointwise_mul, ring.py:572-584). */
int ctb_pointwise_mul(const ctb_ctx_t* ctx, int base, const void* a, const void* b, void* out,
                      uint64_t n_polys, void* stream);

/* out[i] = a[i*a_stride] * b[i*b_stride] mod (x^N+1, base modulus); strides in
 * polynomials (0 broadcasts one operand).  ring.ring_mul -> _crt_ntt_mul
 * (ring.py:404-474), exact per limb. */
int ctb_ring_mul(const ctb_ctx_t* ctx, int base, const void* a, uint64_t a_stride, const void* b,
                 uint64_t b_stride, void* out, uint64_t n_polys, void* stream);

/* CPMul: out[k] = (c0*lift(pt[k]), c1*lift(pt[k])) for `batch` 2-part
 * ciphertexts ct[k] ([batch][2][L][N]) and plain polys pt[k] ([batch][N]
 * uint64 in [0,t)).  He.cp_mul (he.py:366-382) with He._lift (he.py:325-327).
 * In-place (out == ct) allowed. */
int ctb_cpmul(const ctb_ctx_t* ctx, const void* ct, const uint64_t* pt, void* out, uint64_t batch,
              void* stream);

/* PPMul in the plain ring: He.pp_mul (he.py:441-445) = ring.ring_mul over the
 * plain primes + 2-prime CRT (ring.py:477-485). */
int ctb_pp_mul(const ctb_ctx_t* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out,
               uint64_t n_polys, void* stream);

/* Instrumentation (not a reference interface): launch a register-resident
 * Shoup modmul throughput probe on `stream` (grid = 8 x SM count, 256 threads,
 * 8 chains) for word width 4 or 8; *modmuls receives the number of modular
 * multiplications it performs.  Time it with events on the same stream to
 * obtain the integer roofline denominator used by bench.py.  `sink` is a
 * device word that is written only in a never-taken branch. */
int ctb_probe_modmul(int word_bytes, uint64_t iters, void* sink, uint64_t* modmuls, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CTB200_H */
