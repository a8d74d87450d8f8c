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
 *   - A call whose item count (n_polys / batch / n_out) is zero is a no-op
 *     returning CTB_OK; its buffers may then be NULL.
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
 * of the cipher (or single) ring modulus, each = 1 mod 2N, < 2^50.  t_primes:
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
 * Inputs must be reduced residues (< p; 64-bit limbs accept up to 2p for the inverse and 4p for
 * the forward transform).  In-place allowed. */
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

/* out = NTT(in) * N^-1 (canonical eval): the evaluation-domain form of a coefficient
 * addend to sums of products with prepared operands, e.g. K3's mask products
 * (ctb_linear_online maskprod_eval = 1).  In place allowed. */
int ctb_eval_addend(const ctb_ctx_t* ctx, int base, const void* in, void* out, uint64_t n_polys, void* stream);

/* The same values (NTT(in) * N^-1, canonical) in ctb_linear_online's internal evaluation layout
 * (16-byte chunk c of transform thread t at chunk index c * (N/16) + t): the form its
 * maskprod_eval = 1 argument takes.  Replaces the server's per-slot mask-product addition of
 * precompute_online_server (linprot.py:482-484), moved offline.  In place allowed. */
int ctb_linear_addend(const ctb_ctx_t* ctx, int base, const void* in, void* out, uint64_t n_polys, void* stream);

/* Prepared operand for repeated products: out = NTT(in) scaled into the
 * Montgomery domain with N^-1 folded (layout [poly][L][N], evaluation order).
 * Keys (public, secret, relinearisation) are prepared once per session. */
int ctb_prepare_operand(const ctb_ctx_t* ctx, int base, const void* in, void* out, uint64_t n_polys,
                        void* stream);
/* out[i] = a[i] * b[i*b_stride] (+ addend[i] if non-NULL) with b prepared by
 * ctb_prepare_operand: ring.ring_mul followed by ring.ring_add (ring.py:363-427). */
int ctb_mul_prepared(const ctb_ctx_t* ctx, int base, const void* a, const void* bprep, uint64_t b_stride,
                     const void* addend, void* out, uint64_t n_polys, void* stream);

/* ctb_mul_prepared over strided operands: item k reads a at poly k * a_stride and the
 * addend at poly k * add_stride (strides in [L][N] polys), e.g. c0 + c1 * s straight from
 * [B][2][L][N] ciphertexts (a = &ct[0][1], addend = &ct[0][0], strides 2). */
int ctb_mul_prepared_strided(const ctb_ctx_t* ctx, int base, const void* a, uint64_t a_stride, const void* bprep,
                             uint64_t b_stride, const void* addend, uint64_t add_stride, void* out,
                             uint64_t n_polys, void* stream);

/* CPMul: out[k] = (c0*lift(pt[k]), c1*lift(pt[k])) for `batch` 2-part
 * ciphertexts ct[k] ([batch][2][L][N]) and plain polys pt[k] ([batch][N]
 * uint64 in [0,t)).  He.cp_mul (he.py:366-382) with He._lift (he.py:325-327).
 * In-place (out == ct) allowed. */
int ctb_cpmul(const ctb_ctx_t* ctx, const void* ct, const uint64_t* pt, void* out, uint64_t batch,
              void* stream);

/* Encryption (He.encrypt, he.py:307-323), fused: out[k] = (b u + e1 + Delta lift(m), a u + e2)
 * for m [batch][N] uint64 in [0,t), draws [batch][3][N] int8 = (u, e1, e2) small signed
 * integers (ternary u, rounded-Gaussian e clipped to the error bound, |e| <= 127) in the
 * DEVICE DRAW LAYOUT (thread-major: see ctb_sample_draws; convert natural-order draws,
 * e.g. the reference's numpy draws, with ctb_draws_from_natural), pkprep =
 * ctb_prepare_operand of the public key (b, a) as [2][L][N]; out [batch][2][L][N]. */
int ctb_encrypt(const ctb_ctx_t* ctx, const uint64_t* m, const int8_t* draws, const void* pkprep, void* out,
                uint64_t batch, void* stream);

/* ctb_encrypt with the plaintexts given by their packing descriptor (the arguments of
 * ctb_pack_gather) instead of packed values: the correlated / FC packing fused into the encryption
 * (packing.py:407-445, 545-597 then he.py:307-323), so packed plaintexts are never written out.
 * Identical ciphertexts to ctb_pack_gather followed by ctb_encrypt. */
int ctb_encrypt_gather(const ctb_ctx_t* ctx, const int64_t* src, uint64_t src_len, const int32_t* maps, uint32_t n_maps,
                       const int32_t* kind, const int64_t* base, const int8_t* draws, const void* pkprep, void* out,
                       uint64_t batch, void* stream);

/* Device sampler for ctb_encrypt's draws (He._ternary / He._error, he.py:292-303):
 * Philox4x32-10 keyed by `seed`, counter = (first_poly + k, coefficient), so the
 * stream is launch-shape independent; u uniform over {-1,0,1}, e1/e2 = clip(rint(
 * sigma * z), -bound, bound) for z ~ N(0,1) by Box-Muller.  out [batch][3][N] int8 in
 * the device draw layout: position t*E + k of each row holds the draw of the coefficient
 * owned by register k of transform thread t (E = 16 residues per thread for N >= 512).
 * The distribution is the reference's; the stream is not numpy's. */
int ctb_sample_draws(const ctb_ctx_t* ctx, uint64_t seed, uint64_t first_poly, double sigma, int bound,
                     int8_t* out, uint64_t batch, void* stream);

/* Natural-order draws [batch][3][N] (coefficient i at index i) -> device draw layout
 * (not in place). */
int ctb_draws_from_natural(const ctb_ctx_t* ctx, const int8_t* in, int8_t* out, uint64_t batch, void* stream);

/* PPMul in the plain ring: He.pp_mul (he.py:441-445) = ring.ring_mul over the
 * plain primes + 2-prime CRT (ring.py:477-485). */
int ctb_pp_mul(const ctb_ctx_t* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out,
               uint64_t n_polys, void* stream);

/* Coefficient-wise ring operations (ring.py:363-401) on residues [n][L][N]:
 * op 0 = add, 1 = sub (a - b), 2 = neg (b unused).  In-place allowed. */
int ctb_rns_elementwise(const ctb_ctx_t* ctx, int base, int op, const void* a, const void* b, void* out,
                        uint64_t n_polys, void* stream);
/* out = a * c mod q with c given per limb (host array of L words, c_i < q_i). */
int ctb_rns_scalar_mul(const ctb_ctx_t* ctx, int base, const void* a, const uint64_t* scalars, void* out,
                       uint64_t n_polys, void* stream);
/* Small signed integers [n][N] (int64; ternary s/u, Gaussian e) -> residues [n][L][N]. */
int ctb_rns_from_small(const ctb_ctx_t* ctx, int base, const int64_t* in, void* out, uint64_t n_polys,
                       void* stream);
/* out = scale * lift(m) mod q: m [n][N] uint64 in [0,t), centred lift of he.py:325-327,
 * scale per limb (host array; Delta mod q_i for encryption, 1 for a plain lift). */
int ctb_lift_plain(const ctb_ctx_t* ctx, const uint64_t* m, const uint64_t* scale, void* out, uint64_t n_polys,
                   void* stream);
/* Plain ring (mod t) coefficient ops on uint64 [n][N]: op 0 add, 1 sub, 2 neg, 3 scalar multiply. */
int ctb_plain_elementwise(const ctb_ctx_t* ctx, int op, const uint64_t* a, const uint64_t* b, uint64_t scalar,
                          uint64_t* out, uint64_t n_polys, void* stream);

/* Decrypt's exact scale-and-round: v [n][L][N] residues of c0 + c1 s (+ c2 s^2)
 * -> out [n][N] = floor((v t + floor(q/2)) / q) mod t   (He.decrypt, he.py:347-349). */
int ctb_decrypt_round(const ctb_ctx_t* ctx, const void* v, uint64_t* out, uint64_t n_polys, void* stream);
/* ctb_decrypt_round fused with the client's unmasking and extraction (precompute_online_client,
 * linprot.py:444-452: decrypt(c) - p, then job.extract = packing.extract_output / to_signed_matrix,
 * packing.py:476-522, or the FC / outer extractions :577-605): for polynomial b and coefficient d
 * with m = maps[kind[b]][d] >= 0 and base[b] + m < dst_len,
 *   out[base[b] + m] = (round(v[b])[d] - sub[b][d]) mod t   (sub may be NULL),
 * centred into (-t/2, t/2] when `centered` (to_signed_matrix).  maps [n_maps][N] int32, kind [n]
 * int32, base [n] int64, out int64 -- all device.  Coefficients without a destination are not
 * rounded at all. */
int ctb_decrypt_round_extract(const ctb_ctx_t* ctx, const void* v, const uint64_t* sub, const int32_t* maps,
                              uint32_t n_maps, const int32_t* kind, const int64_t* base, uint64_t dst_len,
                              int centered, int64_t* out, uint64_t n_polys, void* stream);

/* Encode side of the correlated linear layer as one gather (packing.pack_input_correlated /
 * pack_kernel_correlated, packing.py:407-445; pack_fc_input / pack_fc_matrix / pack_outer_left,
 * packing.py:545-597; affine_job's packing, linprot.py:243-257):
 *   out_plain[p][d] = m >= 0 && base[p] + m < src_len ? src[base[p] + m] mod t : 0,
 *   m = maps[kind[p]][d]
 * src int64 signed values (reduced like RingElem.from_ints); maps [n_maps][N] int32 (-1 = empty
 * degree), kind [n_polys] int32, base [n_polys] int64 -- all device.  When r != NULL also
 * out_masked[p][d] = (out_plain[p][d] - r[p][d]) mod t, the client's masking x - r_x / w - r_w of
 * precompute_online_client (linprot.py:438-441), fused; out_plain may then be NULL. */
int ctb_pack_gather(const ctb_ctx_t* ctx, const int64_t* src, uint64_t src_len, const int32_t* maps, uint32_t n_maps,
                    const int32_t* kind, const int64_t* base, const uint64_t* r, uint64_t* out_plain,
                    uint64_t* out_masked, uint64_t n_polys, void* stream);

/* Decode side as one scatter (packing.extract_output packing.py:476-509 + to_signed_matrix :512-522,
 * extract_fc_output / extract_outer :577-605) from plain values in [n_slots][N] uint64:
 *   out[base[s] + m] = (in[s][d] - sub[s][d]) mod t (sub may be NULL), centred if `centered`,
 * for m = maps[kind[s]][d] >= 0 and base[s] + m < dst_len. */
int ctb_plain_scatter(const ctb_ctx_t* ctx, const uint64_t* in, const uint64_t* sub, const int32_t* maps,
                      uint32_t n_maps, const int32_t* kind, const int64_t* base, uint64_t dst_len, int centered,
                      int64_t* out, uint64_t n_slots, void* stream);

/* Dense bit-packed transfer format (not a reference format: the end-to-end path's PCIe leg).
 * `count` values of `bits` bits (uint32 values for word_bytes 4, uint64 for 8; values must be
 * < 2^bits) form one little-endian bitstream, value j at bits [j*bits, (j+1)*bits), in
 * ctb_bits_words(bits, count) uint32 words -- e.g. 30-bit residues at 3.75 B instead of 4 B and
 * 50-bit plaintexts at 6.25 B instead of 8 B.  Device buffers, stream-ordered. */
uint64_t ctb_bits_words(uint32_t bits, uint64_t count);
int ctb_bits_pack(const ctb_ctx_t* ctx, int word_bytes, const void* in, uint32_t bits, uint32_t* out, uint64_t count,
                  void* stream);
int ctb_bits_unpack(const ctb_ctx_t* ctx, int word_bytes, const uint32_t* in, uint32_t bits, void* out, uint64_t count,
                    void* stream);

/* Wire format: residues [n][L][N] <-> positional little-endian 64-bit words
 * [n][N][W], W = ctb_ctx_pos_words = ring.RingParams.limb_count (ring.py:147,
 * ring_to_bytes / ring_from_bytes ring.py:592-615; input words reduced mod q). */
int ctb_ctx_pos_words(const ctb_ctx_t* ctx);
int ctb_rns_to_pos(const ctb_ctx_t* ctx, const void* x, uint64_t* out, uint64_t n_polys, void* stream);
int ctb_pos_to_rns(const ctb_ctx_t* ctx, const uint64_t* in, void* x, uint64_t n_polys, void* stream);

/* CCMul tensoring (He.cc_mul_raw, he.py:384-407; ring.int_negacyclic_mul,
 * ring.py:516-541), exact: a, b [batch][2][L][N] -> out3 [batch][3][L][N] =
 * round(h_k t / q) mod q.  `workspace` holds ctb_ccmul_workspace_words(batch)
 * uint32 words.  The auxiliary 30-bit NTT base is built on first use. */
uint64_t ctb_ccmul_workspace_words(const ctb_ctx_t* ctx, uint64_t batch);
int ctb_ccmul_raw(const ctb_ctx_t* ctx, const void* a, const void* b, void* out3, uint32_t* workspace,
                  uint64_t batch, void* stream);
/* The three stages of ctb_ccmul_raw, exposed for pipelining: centred lift onto the
 * auxiliary base ([batch][2][K][N] uint32), tensor products ([batch][3][K][N]),
 * and the exact scale-and-round back to the cipher base. */
int ctb_tensor_aux_size(const ctb_ctx_t* ctx);
int ctb_tensor_lift(const ctb_ctx_t* ctx, const void* ct, uint32_t* out, uint64_t batch, void* stream);
int ctb_tensor_product(const ctb_ctx_t* ctx, const uint32_t* a_aux, const uint32_t* b_aux, uint32_t* h_aux,
                       uint64_t batch, void* stream);
int ctb_tensor_round(const ctb_ctx_t* ctx, const uint32_t* h_aux, void* out, uint64_t batch, void* stream);
/* Relinearisation (He.relinearize, he.py:409-432): ct3 [batch][3][L][N] and the
 * relinearisation keys prepared by ctb_prepare_operand as [D][2][L][N]
 * ((b_i, a_i), D = ctb_relin_digit_count) -> out [batch][2][L][N].
 * digits_ws: batch * D * N uint32 words of scratch. */
int ctb_relin_digit_count(const ctb_ctx_t* ctx);
int ctb_relinearize(const ctb_ctx_t* ctx, const void* ct3, const void* keyprep, uint32_t* digits_ws, void* out,
                    uint64_t batch, void* stream);

/* Fused per-slot CCMul sums -- the server side of the precompute protocol's offline
 * phase (precompute_offline_server, linprot.py:407-427: per site cc_mul(r_x, r_w),
 * relinearised, CCAdd into its slot) and of protocol b (linear_b_server, linprot.py:
 * 371-379).  ct_x [n_x][2][L][N], ct_w [n_w][2][L][N]; sites_host [n_sites][3] = (x, w,
 * slot) in HOST memory; keyprep as ctb_relinearize; out [n_out][2][L][N] with
 * out[o] = sum over the sites of slot o of relinearize(cc_mul_raw(x, w)), identical to
 * the per-site computation.  Each distinct ciphertext is lifted and transformed once and
 * relinearisation runs once per slot (digit sums; a slot may hold at most
 * (2^32 - 1) / (2^w - 1) sites).  workspace: ctb_ccmul_sum_workspace_bytes(..., largest
 * slot's site count).  The host site table is copied stream-ordered through a pinned staging
 * buffer: the call does not synchronise `stream` and sites_host may be freed on return. */
uint64_t ctb_ccmul_sum_workspace_bytes(const ctb_ctx_t* ctx, uint32_t n_x, uint32_t n_w, uint32_t n_out,
                                       uint32_t n_sites, uint32_t max_slot_sites);
int ctb_ccmul_sum(const ctb_ctx_t* ctx, const void* ct_x, uint32_t n_x, const void* ct_w, uint32_t n_w,
                  const uint32_t* sites_host, uint32_t n_sites, uint32_t n_out, const void* keyprep, void* out,
                  void* workspace, uint64_t workspace_bytes, void* stream);

/* Prepared lifted plaintext: NTT(lift(m)) in the Montgomery domain, N^-1
 * folded (m [n][N] uint64 in [0,t)) -> [n][L][N]. */
int ctb_lift_prepare(const ctb_ctx_t* ctx, const uint64_t* m, void* out, uint64_t n_polys, void* stream);

/* K3 -- server step of the precompute protocol for one linear job
 * (linprot.precompute_online_server, linprot.py:455-485), exact:
 *   out_ct[o] = sum_{(x,w,o) in sites} ( ct_x[x] * lift(mw[w]) + ct_w[w] * lift(mx[x]) ) + maskprod[o]
 *   out_p[o]  = sum_{(x,w,o) in sites} mx[x] * mw[w]       (plain ring)
 * ct_x [n_x][2][L][N], ct_w [n_w][2][L][N] ciphertexts; mx [n_x][N], mw [n_w][N]
 * masked plaintexts (x - r_x, w - r_w); sites_host: HOST array of n_sites
 * (x index, w index, out slot) triples (linprot.JobShape.sites); maskprod
 * [n_out][2][L][N] or NULL, as ciphertexts (maskprod_eval = 0) or in the
 * ctb_linear_addend form (maskprod_eval = 1: the server transformed its mask products
 * offline, so the online step adds them in the evaluation domain);
 * out_ct [n_out][2][L][N]; out_p [n_out][N].
 * workspace: ctb_linear_online_workspace_bytes() bytes of device memory.
 * Every ciphertext part and masked plaintext is NTT'd once; each slot is
 * accumulated in the evaluation domain and inverse-transformed once.  Like ctb_ccmul_sum the
 * call returns without synchronising `stream` (sites_host may be freed on return). */
uint64_t ctb_linear_online_workspace_bytes(const ctb_ctx_t* ctx, uint32_t n_x, uint32_t n_w, uint32_t n_out,
                                           uint32_t n_sites);
int ctb_linear_online(const ctb_ctx_t* ctx, const void* ct_x, uint32_t n_x, const void* ct_w, uint32_t n_w,
                      const uint64_t* mx, const uint64_t* mw, const uint32_t* sites_host, uint32_t n_sites,
                      uint32_t n_out, const void* maskprod, int maskprod_eval, void* out_ct, uint64_t* out_p,
                      void* workspace, void* stream);
/* Segmented sum (the CCAdd accumulation of linprot._accumulate, linprot.py:343-344):
 * out[o] = sum_{s in [slot_ptr[o], slot_ptr[o+1])} in[members[s]] over [*][parts][L][N]
 * (slot_ptr / members are DEVICE int32 arrays). */
int ctb_slot_sum(const ctb_ctx_t* ctx, int base, const void* in, uint32_t parts, const int32_t* slot_ptr,
                 const int32_t* members, uint32_t n_out, void* out, void* stream);

/* Instrumentation (not a reference interface): launch a register-resident
 * Shoup modmul throughput probe on `stream` (grid = 8 x SM count, 256 threads,
 * 8 chains) for word width 4 or 8; *modmuls receives the number of modular
 * multiplications it performs.  Time it with events on the same stream to
 * obtain the integer roofline denominator used by bench.py.  `sink` is a
 * device word that is written only in a never-taken branch. */
int ctb_probe_modmul(int word_bytes, uint64_t iters, void* sink, uint64_t* modmuls, void* stream);

/* Instrumentation: the 30-bit butterfly product mix of ctb_cpmul -- f64q_of_8 (0, 3 or 8) of
 * the 8 chains take the FP64-pipe quotient (3 = the share k_cpmul uses), the rest are Shoup
 * products.  Same launch shape and contract as ctb_probe_modmul; bench.py divides by it. */
int ctb_probe_modmul_mix(int f64q_of_8, uint64_t iters, void* sink, uint64_t* modmuls, void* stream);
/* The same mix with the quotient's operand assembled by the exponent splice (the round-1 form;
 * ctb_probe_modmul_mix converts it with I2F.F64.U32 like the kernels do now). */
int ctb_probe_modmul_mix_splice(int f64q_of_8, uint64_t iters, void* sink, uint64_t* modmuls, void* stream);

/* Instrumentation: one radix-16 register pass of the 32-bit forward transform at N = 4096 exactly as
 * ctb_cpmul runs it (32 complete Harvey butterflies per thread: conditional subtraction, product,
 * sum, difference; twiddles from shared memory), repeated register-resident with no exchanges and no
 * global traffic, one 1024-thread CTA per SM; *bflys receives the butterflies performed.  The
 * ceiling of a transform's own arithmetic (the modmul probes leave out the ALU-pipe additions).
 * Needs a context with N = 4096 and 32-bit cipher limbs. */
int ctb_probe_bfly_pass(const ctb_ctx_t* ctx, uint64_t iters, void* sink, uint64_t* bflys, void* stream);

/* Instrumentation: the 50-bit product of the FP64 butterflies (64-bit limbs: exact integers in
 * doubles, 6 FP64 operations per product, ntt.cuh f64_mulmod).  Same launch shape and contract as
 * ctb_probe_modmul; bench.py divides the 50-bit configurations by it. */
int ctb_probe_modmul_f64(uint64_t iters, void* sink, uint64_t* modmuls, void* stream);

/* Instrumentation: the forward butterfly of the 64-bit-limb transforms (product + add + sub + its share
 * of the once-per-pass reduction, ntt.cuh fwd_pass_f64), one modmul counted per butterfly: the FP64
 * pipe's ceiling for the transforms' own arithmetic. */
int ctb_probe_bfly_f64(uint64_t iters, void* sink, uint64_t* modmuls, void* stream);

/* Self-check (not a reference interface): for every prime of 32-bit base `base` and every entry of
 * its FP64-quotient twiddle table, the butterfly product a*w mod p with the FP64-pipe quotient must
 * lie in [0, 2p) and be congruent to a*w for boundary inputs and `samples` pseudo-random 32-bit a
 * (seeded by `seed`).  Blocking; *bad receives the number of failures (0 expected).  A no-op for
 * 64-bit bases. */
int ctb_check_f64q(const ctb_ctx_t* ctx, int base, uint64_t samples, uint64_t seed, uint64_t* bad, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CTB200_H */
