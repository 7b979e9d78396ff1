/* pcb200.h — C ABI of the B200-native Paillier / 3P-ADMM-PC2 hot path.
 *
 * This is the drop-in boundary.  The reference has no FFI: its seam is the C++ class
 * pcadmm::Paillier (/root/reference/proj/include/pcadmm/paillier.hpp:104-181) and the quantizer
 * free functions (quantize.hpp:32-71).  Each entry point below names the reference member it
 * replaces.  The C++ drop-in (paper_2601_14980_b200/cpp/pcb200_pcadmm.hpp, pcadmm::Paillier) and the Python package
 * re-expose the reference signatures on top of these calls; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *   - Big integers are fixed-width little-endian uint32 limb arrays.  For a context with an
 *     L-limb modulus n (L = pcb_ctx_n_limbs):  plaintexts and r use L limbs (or a narrower
 *     m_limbs for quantized plaintexts), ciphertexts use 2L limbs.  Batches are AoS:
 *     element i occupies [i*width, (i+1)*width).
 *   - Pointers may be device pointers (stream-ordered, no hidden copies) or host pointers
 *     (staged through device scratch; the call synchronises the stream before returning).
 *   - Exceptions of the reference become pcb_status values; batched calls also write one int32
 *     status per element (nullable) so a single bad element does not hide the others.
 *   - There is no CPU fallback: without a CUDA device every compute call returns PCB_E_CUDA.
 *   - Thread-safety: one context may be used from several host threads on distinct streams.
 */
#ifndef PCB200_H
#define PCB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pcb_ctx pcb_ctx;
typedef struct CUstream_st* pcb_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  PCB_OK = 0,
  PCB_E_PLAINTEXT_RANGE = 1,  /* m >= n            invalid_argument  paillier.cpp:242        */
  PCB_E_RANDOMNESS_RANGE = 2, /* r == 0 or r >= n  invalid_argument  paillier.cpp:322-323    */
  PCB_E_CIPHER_RANGE = 3,     /* c >= n^2          invalid_argument  paillier.cpp:348,356    */
  PCB_E_NOT_UNIT = 4,         /* gcd(c,n) != 1     runtime_error     paillier.cpp:34-41      */
  PCB_E_OVERFLOW = 5,         /* plain_bits guard  overflow_error    paillier.cpp:245-251    */
  PCB_E_NO_PRIVATE = 6,       /* private op on a public-only context   logic_error             */
  PCB_E_SHAPE = 7,            /* bad sizes/window/key size              invalid_argument        */
  PCB_E_UNSUPPORTED = 8,      /* valid request this build does not implement (e.g. random g)    */
  PCB_E_CUDA = 9,             /* CUDA runtime error or no device                                  */
  PCB_E_ALLOC = 10,           /* device/host allocation failed                                    */
  PCB_E_RANGE_UPDATE = 11     /* decrypted ADMM update out of range: ProtocolError protocol.cpp:20-27 */
} pcb_status;

/* ---- keys (host; one-time work) ------------------------------------------ */

/* pcadmm::keygen(Rng&, key_bits, GMode::binomial) — paillier.cpp:106-123, bit-exact including
 * the splitmix64 stream consumption.  *rng_state is the Rng::state before/after.  key_bits must
 * be 64, 1024, 2048 or 4096 (the reference's accepted set).  n gets key_bits/32 limbs (64-bit:
 * 2), p and q get half of that. */
pcb_status pcb_keygen(uint64_t* rng_state, uint32_t key_bits, uint32_t* n, uint32_t* p, uint32_t* q);

/* pcadmm::random_prime(Rng&, bits, 40) — bignat.cpp:497-515 (used for 3072-bit keys via
 * keypair_from_primes).  out gets ceil(bits/32) limbs. */
pcb_status pcb_random_prime(uint64_t* rng_state, uint32_t bits, uint32_t* out);

/* The same two calls with the Miller-Rabin rounds batched (csrc/prime.cu, host/hbn.cpp
 * random_prime_batched): the rounds of many candidates run at once, speculating that every
 * trial-division survivor fails its first round, then committing / rewinding the stream exactly
 * as the reference consumes it -- identical primes, keys and *rng_state.  device >= 0 evaluates
 * the batches on that CUDA device (bits <= 2048 per prime); device < 0 evaluates them with the
 * host pow_mod (the checker the CPU tests pin the speculation with). */
pcb_status pcb_keygen_speculative(uint64_t* rng_state, uint32_t key_bits, int device, uint32_t* n, uint32_t* p,
                                  uint32_t* q);
pcb_status pcb_random_prime_speculative(uint64_t* rng_state, uint32_t bits, int device, uint32_t* out);

/* ---- context ------------------------------------------------------------------------------ */

/* Builds the per-key device constants (Montgomery contexts for p^2, q^2, p, q, n^2, exponent
 * window schedules, CRT factors).  Replaces Paillier(KeyPair) / Paillier(PublicKey)
 * (paillier.cpp:193-212).  p and q (pq_limbs each) may be NULL for a public-key-only context
 * (the edge role).  binomial g = n+1 only (the reference default, GMode::binomial). */
pcb_status pcb_ctx_create(pcb_ctx** out, int device, const uint32_t* n, uint32_t n_limbs,
                          const uint32_t* p, const uint32_t* q, uint32_t pq_limbs);
void pcb_ctx_destroy(pcb_ctx* ctx);
/* GMode::random_g (paillier.cpp:80-100): sets the generator g (g_limbs words, 1 < g < n^2,
 * gcd(g, n) = 1, L(g^eps mod n^2) invertible mod n) of a context made by pcb_ctx_create.  The
 * decryption constants are rebuilt from g (h_p = L_p(g^(p-1) mod p^2)^-1, mu = L(g^eps)^-1), and
 * pcb_encrypt / pcb_encrypt_rn / pcb_finish_split_encrypt compute g^m mod n^2 on the device from
 * the 64-bit digit powers g^(2^(64 j)) mod n^2.  g = n + 1 restores the binomial form.  The fused
 * pcb_quantize_encrypt (the g = n + 1 hot path) returns PCB_E_UNSUPPORTED on a random-g context. */
pcb_status pcb_ctx_set_generator(pcb_ctx* ctx, const uint32_t* g, uint32_t g_limbs);
uint32_t pcb_ctx_n_limbs(const pcb_ctx* ctx);   /* L: limb width of plaintexts and r       */
uint32_t pcb_ctx_n_bits(const pcb_ctx* ctx);    /* bit length of n (plain_bits guard bound) */
int pcb_ctx_has_private(const pcb_ctx* ctx);
/* Core that runs the CRT halves of Enc/Dec: 0 = 32-bit carry-chain Montgomery (side_kernel),
 * 1 = RNS Montgomery with tensor-core base extensions (rns_pow_kernel; 2048-bit keys, default;
 * PCB_RNS=0 in the environment at context creation selects 0), 2 = radix-2^28 (3072-bit). */
/* Stream priority of the context's internal CRT-half side streams (used for batches below one
 * full wave): high != 0 -> the device's greatest priority, 0 -> least (e.g. offline precompute). */
pcb_status pcb_ctx_set_priority(pcb_ctx* ctx, int high);
int pcb_ctx_engine(const pcb_ctx* ctx);
/* Copies n (L limbs) / n^2 (2L limbs) out of the context. */
pcb_status pcb_ctx_get_n(const pcb_ctx* ctx, uint32_t* n, uint32_t* n2);
/* Exponentiation ledger, pcadmm::OpCount (paillier.hpp:84-87): same counting rules as the
 * reference (pow_half per p^2/q^2 exponentiation, pow_full per n^2 exponentiation/matvec row). */
void pcb_ctx_counters(const pcb_ctx* ctx, uint64_t* pow_full, uint64_t* pow_half);
void pcb_ctx_reset_counters(pcb_ctx* ctx);

/* ---- randomness ---------------------------------------------------------------------------- */

/* count x Paillier::sample_r(rng) — paillier.cpp:233-239 with bignat.cpp:388-445: splitmix64
 * words, rejection until 0 < r < n, gcd(r, n) == 1.  Generated on the GPU from the counter form
 * of splitmix64 and stream-compacted, so r_out and the final *rng_state are identical to the
 * reference's serial draw loop (paillier.cpp:499-500). */
pcb_status pcb_sample_r(pcb_ctx* ctx, uint64_t* rng_state, size_t count, uint32_t* r_out,
                        pcb_stream stream);

/* ---- encryption / decryption -------------------------------------------------------------- */

/* c_i = (1 + m_i n) r_i^n mod n^2.
 *   use_crt = 1: Paillier::crt_encrypt_with_r (paillier.cpp:334-344), needs p, q;
 *   use_crt = 0: Paillier::encrypt_with_r     (paillier.cpp:320-328), public key only.
 * m: count x m_limbs (m_limbs <= L), r: count x L, c: count x 2L. */
pcb_status pcb_encrypt(pcb_ctx* ctx, const uint32_t* m, uint32_t m_limbs, const uint32_t* r,
                       size_t count, uint32_t* c, int use_crt, int32_t* status, pcb_stream stream);

/* Offline/online split of encryption.  Offline: rn_i = r_i^n mod n^2, which is pcb_encrypt with
 * m = 0 (the randomness stream does not depend on the data, so it can run ahead, e.g. during
 * the previous ADMM iteration's edge step).  Online: c_i = (1 + m_i n) rn_i mod n^2 — bit-equal
 * to crt_encrypt_with_r / encrypt_with_r (paillier.cpp:320-344) with the same r.  Per element:
 * PCB_E_PLAINTEXT_RANGE if m >= n, PCB_E_RANDOMNESS_RANGE if rn is 0 or >= n^2 (c = 0).  Works on
 * public-key contexts.  m: count x m_limbs u32, rn / c: count x 2L. */
pcb_status pcb_encrypt_rn(pcb_ctx* ctx, const uint32_t* m, uint32_t m_limbs, const uint32_t* rn,
                          size_t count, uint32_t* c, int32_t* status, pcb_stream stream);

/* m_i = L(c_i^eps mod n^2) mu mod n.
 *   use_crt = 1: Paillier::crt_decrypt (paillier.cpp:354-361);  use_crt = 0: decrypt (346-352).
 * Both compute the same residue (c^(p-1) mod p^2 / L_p / h_p form + CRT on the device).
 * c: count x 2L, m: count x L. */
pcb_status pcb_decrypt(pcb_ctx* ctx, const uint32_t* c, size_t count, uint32_t* m, int use_crt,
                       int32_t* status, pcb_stream stream);

/* ---- collaborative variant (paper Alg. 3): the p^2 side delegated to an edge ------------------- */

/* m_i = L(x_i) mu mod n, x_i = CRT(p2_power_i mod p^2, c_i^(eps mod phi(q^2)) mod q^2) —
 * Paillier::decrypt_with_half (paillier.cpp:363-369).  p2_power: count x pw_limbs (pw_limbs <= 2L),
 * e.g. an edge's delegated_power (protocol.cpp:15-18).  Statuses as pcb_decrypt.  Every key size (keys
 * up to 1024 bits run it on the K = 40 RNS core, 2048/3072-bit keys on the Enc/Dec core). */
pcb_status pcb_decrypt_with_half(pcb_ctx* ctx, const uint32_t* c, const uint32_t* p2_power, uint32_t pw_limbs,
                                 size_t count, uint32_t* m, int32_t* status, pcb_stream stream);

/* An edge's CrtShare {p^2, phi(p^2)} (paillier.hpp:64-66) on the device: no other key material. */
typedef struct pcb_share pcb_share;
pcb_status pcb_share_create(pcb_share** share, int device, const uint32_t* p2, uint32_t p2_limbs,
                            const uint32_t* phi_p2, uint32_t phi_limbs);
void pcb_share_destroy(pcb_share* share);
/* out_i = (base_i mod p^2)^(obf_i mod phi(p^2)) mod p^2 — delegated_power (protocol.cpp:15-18), with
 * per-element exponents (e.g. obfuscate_exponent(value, n eps, mask), protocol.cpp:11-13).
 * base: count x base_limbs (<= 2 x p^2 words), obf: count x obf_limbs, out: count x (p^2 words). */
pcb_status pcb_delegated_power(pcb_share* share, const uint32_t* base, uint32_t base_limbs, const uint32_t* obf,
                               uint32_t obf_limbs, size_t count, uint32_t* out, pcb_stream stream);
/* The same for the binomial generator g = n + 1 shared by the batch (n: n_limbs words): the
 * collapse (1 + n)^e = 1 + e n (mod p^2) (n^2 = 0 mod p^2, as g_power_half, paillier.cpp:259-263);
 * bit-identical to pcb_delegated_power(base = n + 1, obf) without the exponentiation. */
pcb_status pcb_delegated_power_binomial(pcb_share* share, const uint32_t* n, uint32_t n_limbs, const uint32_t* obf,
                                        uint32_t obf_limbs, size_t count, uint32_t* out, pcb_stream stream);
/* The same for exponents that are multiples of p - 1, e_i = u_i (p - 1) with 0 < u_i < p (half_pow
 * with w = 0, paillier.cpp:275-305): out_i = 1 + p (L_p(base_i^(p-1) mod p^2) u_i mod p), or 0 when
 * p | base_i -- one |p|-bit chain instead of a |p^2|-bit one; bit-identical to pcb_delegated_power
 * with obf_i = e_i.  The collaborative session's obf_dec = eps (1 + mask n) reduces to this form.
 * u_mont: count x (p^2 words / 2), u_i R mod p with R = 2^(16 x p^2 words).  2048/3072/4096-bit keys. */
pcb_status pcb_delegated_power_fermat(pcb_share* share, const uint32_t* base, uint32_t base_limbs,
                                      const uint32_t* u_mont, size_t count, uint32_t* out, pcb_stream stream);

/* out_i = value_i + mask_i * n_eps — obfuscate_exponent (protocol.cpp:11-13), the master's masked
 * exponents for the edges' delegated powers.  value: count x value_limbs, mask: count u64 (draw_mask,
 * protocol.cpp:86-93), n_eps: ne_limbs (n * eps), out: count x out_limbs (>= ne_limbs + 3). */
pcb_status pcb_obfuscate_exponent(const uint32_t* value, uint32_t value_limbs, const uint64_t* mask,
                                  const uint32_t* n_eps, uint32_t ne_limbs, size_t count, uint32_t* out,
                                  uint32_t out_limbs, pcb_stream stream);

/* c_i = CRT((p2_g_power_i mod p^2) r_i^(n mod phi(p^2)) mod p^2, (1 + m_i n) r_i^(n mod phi(q^2)) mod q^2)
 * — Paillier::finish_split_encrypt (paillier.cpp:402-414).  Statuses as pcb_encrypt. */
pcb_status pcb_finish_split_encrypt(pcb_ctx* ctx, const uint32_t* m, uint32_t m_limbs, const uint32_t* p2_g_power,
                                    uint32_t pg_limbs, const uint32_t* r, size_t count, uint32_t* c,
                                    int32_t* status, pcb_stream stream);

/* The pooled form — Paillier::finish_split_encrypt_with_factor (paillier.cpp:416-426): rn = the
 * factor's r^n mod n^2 (RnFactor.full, whose residues mod p^2 / q^2 are half_p2 / half_q2), count x 2L
 * limbs; c_i = CRT(p2_g_power_i mod p^2, (1 + m_i n) mod q^2) rn_i mod n^2, no exponentiation with r.
 * rn_i = 0 or >= n^2 fails that element with PCB_E_RANDOMNESS_RANGE.  Statuses as pcb_encrypt. */
pcb_status pcb_finish_split_encrypt_rn(pcb_ctx* ctx, const uint32_t* m, uint32_t m_limbs, const uint32_t* p2_g_power,
                                       uint32_t pg_limbs, const uint32_t* rn, size_t count, uint32_t* c,
                                       int32_t* status, pcb_stream stream);

/* ---- edge setup: node factors ---------------------------------------- */

/* pcadmm::node_factor (admm.cpp:63-75) for every block of a column split at once:
 * normal_k = A_k^T A_k + rho I,  b_bar_k = rho normal_k^-1,  alpha_k = normal_k^-1 A_k^T y_s,
 * y_s = y / k_total when over_k (YScaling::over_k) else y.  a: rows x cols FP64 row-major with row
 * stride lda; block k = the sizes[k] consecutive columns after blocks 0..k-1 (sum sizes = cols).
 * b_bar: the blocks' sizes[k]^2 row-major matrices back to back; alpha: cols.  FP64 blocked
 * Cholesky + triangular inverse on DMMA (csrc/factor.cu); equal to the reference's LDLT solve to
 * rounding.  Errors (check_inputs, admm.cpp:8-16): empty shapes, rho <= 0, k_total < 1, sizes not
 * summing to cols -> PCB_E_SHAPE; a non-finite input (normal not positive definite) -> PCB_E_SHAPE. */
pcb_status pcb_node_factors(const double* a, size_t rows, size_t cols, size_t lda, const double* y, size_t nblocks,
                            const uint32_t* sizes, double rho, uint32_t k_total, int over_k, double* b_bar,
                            double* alpha, pcb_stream stream);

/* ---- homomorphic operations (public key suffices) ----------------------------------------- */

/* out_i = a_i * b_i mod n^2 — Paillier::hom_add (paillier.cpp:428-432).  plain_bits tracking
 * stays on the host (facade), exactly as the reference formula. */
pcb_status pcb_hom_add(pcb_ctx* ctx, const uint32_t* a, const uint32_t* b, size_t count,
                       uint32_t* out, pcb_stream stream);

/* out_i = c_i^k_i mod n^2 — Paillier::hom_scalar_mul (paillier.cpp:434-439), k_i < 2^64. */
pcb_status pcb_hom_scalar_mul(pcb_ctx* ctx, const uint64_t* k, const uint32_t* c, size_t count,
                              uint32_t* out, pcb_stream stream);

/* out_i = alpha_i * prod_j zv_j^expo[i][j] mod n^2 — Paillier::hom_matvec
 * (paillier.cpp:441-493).  expo is rows x cols row-major u64; window in [1, 8] selects the
 * reference's table width (the result does not depend on it). */
pcb_status pcb_hom_matvec(pcb_ctx* ctx, const uint32_t* alpha, const uint64_t* expo,
                          const uint32_t* zv, size_t rows, size_t cols, uint32_t window,
                          uint32_t* out, pcb_stream stream);

/* Edge step (protocol.cpp:264-271): zv_j = z_j * v_j mod n^2 (hom_add), then hom_matvec.
 * Also range-checks z_j, v_j < n^2 (ProtocolError "ciphertext outside the group"). */
pcb_status pcb_edge_step(pcb_ctx* ctx, const uint32_t* alpha, const uint64_t* expo,
                         const uint32_t* zc, const uint32_t* vc, size_t cols, uint32_t window,
                         uint32_t* out, pcb_stream stream);

/* The edge steps of nblocks independent edges in one batch (the per-edge loop of one ADMM
 * iteration, protocol.cpp:486-511 -> 264-271 for each k): block k is square of side sizes[k];
 * alpha / zc / vc / out hold sum(sizes) ciphertexts block after block, expo the row-major
 * sizes[k] x sizes[k] exponent matrices back to back.  Result of block k == pcb_edge_step on
 * block k alone.  PCB_E_CIPHER_RANGE if any z_j or v_j is not below n^2. */
pcb_status pcb_edge_step_blocks(pcb_ctx* ctx, size_t nblocks, const uint32_t* sizes,
                                const uint32_t* alpha, const uint64_t* expo, const uint32_t* zc,
                                const uint32_t* vc, uint32_t window, uint32_t* out,
                                pcb_stream stream);

/* out = prod_i c_i mod n^2 (balanced reduction tree; order-independent value, SURVEY.md §0
 * fact 9).  count >= 1. */
pcb_status pcb_aggregate(pcb_ctx* ctx, const uint32_t* c, size_t count, uint32_t* out,
                         pcb_stream stream);

/* ---- fused quantize / dequantize (quantize.cpp, FP64 without contraction) ------------------ */

/* Gamma2 (fine = 0, quantize.cpp:31-35) or Gamma1 (fine = 1, 37-41) of count doubles, then
 * encryption with r (as pcb_encrypt; use_crt = 0 is the public-key form the edge uses for
 * alpha, protocol.cpp:207-212).  q_out (nullable) receives the quantized integers
 * (u64, or u128 as lo/hi pairs when fine); clamps (nullable, host) receives {low, high}. */
pcb_status pcb_quantize_encrypt(pcb_ctx* ctx, const double* v, size_t count, double z_min,
                                double z_max, double delta, int fine, const uint32_t* r,
                                int use_crt, uint32_t* c, uint64_t* q_out, uint64_t* clamps,
                                pcb_stream stream);

/* gamma2_vec / gamma1_vec (quantize.cpp:52-64) on the GPU: q_out gets u64 (fine = 0) or u128 as
 * (lo, hi) pairs (fine = 1); clamps (nullable, host) receives {low, high}.  A non-finite value
 * returns PCB_E_SHAPE (clamp_in throws invalid_argument, quantize.cpp:18-19). */
pcb_status pcb_quantize(const double* v, size_t count, double z_min, double z_max, double delta, int fine,
                        uint64_t* q_out, uint64_t* clamps, pcb_stream stream);

/* Master block update (protocol.cpp:494-511): decrypt count updates, range-gate them
 * (check_update_range, protocol.cpp:20-27), inverse_quantize_x (quantize.cpp:84-112) with the
 * block's Gamma2(B) row sums, then z = S_{lambda/rho}(x + v), v = x + v - z in place.
 * q_z, q_nv: the Gamma2 integers the block was encrypted from (count each). */
pcb_status pcb_decrypt_update(pcb_ctx* ctx, const uint32_t* c, size_t count,
                              const uint64_t* rowsum, const uint64_t* q_z, const uint64_t* q_nv,
                              double z_min, double z_max, double delta, double kappa, double* x,
                              double* z, double* v, int32_t* status, pcb_stream stream);

/* pcb_decrypt_update over nblocks blocks laid out back to back (sizes[k] rows each); sum_zv and
 * the range cap use each block's own columns (quantize.cpp:96-99, protocol.cpp:23-24), so the
 * result equals nblocks separate pcb_decrypt_update calls. */
pcb_status pcb_decrypt_update_blocks(pcb_ctx* ctx, size_t nblocks, const uint32_t* sizes,
                                     const uint32_t* c, const uint64_t* rowsum,
                                     const uint64_t* q_z, const uint64_t* q_nv, double z_min,
                                     double z_max, double delta, double kappa, double* x, double* z,
                                     double* v, int32_t* status, pcb_stream stream);

/* pcb_decrypt_update_blocks of the collaborative variant: the p^2 side of every Dec comes from the
 * edge (p2_power: count x 2L words, delegated_power of c with the obfuscated eps) and the master
 * finishes with decrypt_with_half (protocol.cpp:490-492).  2048/3072-bit keys. */
pcb_status pcb_decrypt_update_blocks_half(pcb_ctx* ctx, size_t nblocks, const uint32_t* sizes, const uint32_t* c,
                                          const uint32_t* p2_power, const uint64_t* rowsum, const uint64_t* q_z,
                                          const uint64_t* q_nv, double z_min, double z_max, double delta,
                                          double kappa, double* x, double* z, double* v, int32_t* status,
                                          pcb_stream stream);

/* combined_quantized_update (quantize.cpp:66-82) on the device: out_i = q_alpha_i +
 * sum_j q_b[i][j] (q_z_j + q_nv_j) in u128 (wrapping as the reference).  q_alpha / out: rows (lo, hi)
 * u64 pairs, q_b: rows x cols row-major.  The plaintext oracle of the encrypted edge step. */
pcb_status pcb_combined_update(const uint64_t* q_alpha, const uint64_t* q_b, const uint64_t* q_z,
                               const uint64_t* q_nv, size_t rows, size_t cols, uint64_t* out, pcb_stream stream);

/* inverse_quantize_x (quantize.cpp:84-112) on the device, FP64 in the reference's operation order
 * (no contraction; the sequential sum over columns in one thread).  q: rows (lo, hi) u64 pairs. */
pcb_status pcb_inverse_quantize_x(const uint64_t* q, const uint64_t* rowsum, const uint64_t* q_z,
                                  const uint64_t* q_nv, size_t rows, size_t cols, double z_min, double z_max,
                                  double delta, double* x, pcb_stream stream);

/* ---- asynchronous forms for a resident iteration loop --------------------------------------
 * Same results as the calls above, for DEVICE pointers only and without any host synchronisation
 * (the round-1 forms synchronised the stream up to three times per call).  Instead of returning
 * per-element failures they record the first failing element's code in *err_dev (a device int32
 * the caller zeroes; atomicCAS from 0, so the earliest-arriving failure wins) and the caller checks
 * it once per iteration.  The call's own return value reports argument / launch errors only. */

/* pcb_quantize without the host round trip: clamps_dev (nullable, device u64[2]) is ACCUMULATED
 * {low, high}; a non-finite value sets *err_dev = PCB_E_SHAPE. */
pcb_status pcb_quantize_async(const double* v, size_t count, double z_min, double z_max, double delta,
                              int fine, uint64_t* q_out, uint64_t* clamps_dev, int32_t* err_dev,
                              pcb_stream stream);

/* pcb_edge_step_blocks without host synchronisation.  expo_bits: an upper bound of the bit length
 * of every exponent (the largest Gamma2(B) entry, constant over a session; 0 = compute it, which
 * synchronises once).  z_j or v_j >= n^2 sets *err_dev = PCB_E_CIPHER_RANGE. */
pcb_status pcb_edge_step_blocks_async(pcb_ctx* ctx, size_t nblocks, const uint32_t* sizes,
                                      const uint32_t* alpha, const uint64_t* expo, uint32_t expo_bits,
                                      const uint32_t* zc, const uint32_t* vc, uint32_t window,
                                      uint32_t* out, int32_t* err_dev, pcb_stream stream);

/* pcb_decrypt_update_blocks without host synchronisation: rows whose decryption or range gate
 * fails keep x / z / v and set *err_dev (PCB_E_NOT_UNIT, PCB_E_CIPHER_RANGE, PCB_E_RANGE_UPDATE). */
pcb_status pcb_decrypt_update_blocks_async(pcb_ctx* ctx, size_t nblocks, const uint32_t* sizes,
                                           const uint32_t* c, const uint64_t* rowsum,
                                           const uint64_t* q_z, const uint64_t* q_nv, double z_min,
                                           double z_max, double delta, double kappa, double* x,
                                           double* z, double* v, int32_t* err_dev, pcb_stream stream);

/* The master's own CRT half of Paillier::decrypt_with_half (paillier.cpp:366) on its own: the q^2
 * chain, q2_half (count x S words, S = the CRT half width).  eps mod phi(q^2) = u (q - 1), so for
 * u != 0 (every key but toy ones) the chain is c^(q-1) mod q^2 and the factor u is applied in the
 * finish (half_pow, paillier.cpp:275-305); else (c mod q^2)^(eps mod phi(q^2)) mod q^2.  An
 * intermediate for pcb_decrypt_update_blocks_half_async on the same context.  It needs only c, so
 * the master can run it while the edge computes the p^2 side (delegated_power); device pointers,
 * no host synchronisation. */
pcb_status pcb_decrypt_half_q(pcb_ctx* ctx, const uint32_t* c, size_t count, uint32_t* q2_half, pcb_stream stream);

/* pcb_decrypt_update_blocks_half without host synchronisation (errors into *err_dev as above).
 * q2_half: nullable; the pcb_decrypt_half_q output for the same c, else it is computed here. */
pcb_status pcb_decrypt_update_blocks_half_async(pcb_ctx* ctx, size_t nblocks, const uint32_t* sizes,
                                                const uint32_t* c, const uint32_t* p2_power,
                                                const uint32_t* q2_half, const uint64_t* rowsum,
                                                const uint64_t* q_z, const uint64_t* q_nv, double z_min,
                                                double z_max, double delta, double kappa, double* x,
                                                double* z, double* v, int32_t* err_dev, pcb_stream stream);

/* ---- wire format (interop with the reference's SimCarrier / TcpCarrier sessions) ---------- */

/* put_cipher_vec (wire.cpp:125-132) on the device: u32 BE count, then per element u32 BE byte
 * length, the minimal big-endian magnitude of c_i (bignat.cpp:414-418) and u32 BE plain_bits_i.
 * c: count x W LE u32 limbs, plain_bits: count u32 (nullable -> 0).  *out_len gets the byte count;
 * out = NULL only queries it.  PCB_E_SHAPE if out_cap is too small. */
pcb_status pcb_wire_put_cipher_vec(const uint32_t* c, uint32_t W, const uint32_t* plain_bits, size_t count,
                                   uint8_t* out, size_t out_cap, size_t* out_len, pcb_stream stream);
/* get_cipher_vec (wire.cpp:134-146): parses the vector at byte *off of in (in_len bytes) into c
 * (count x W limbs, zero-extended) and plain_bits (nullable); *count_out = count, *off advances.
 * PCB_E_SHAPE on truncation (runtime_error), more than max_count elements or a magnitude wider
 * than W limbs. */
pcb_status pcb_wire_get_cipher_vec(const uint8_t* in, size_t in_len, size_t* off, uint32_t W, size_t max_count,
                                   size_t* count_out, uint32_t* c, uint32_t* plain_bits, pcb_stream stream);
/* encode_envelope (wire.cpp:148-159): u32 BE (7 + payload_len), type (1..7, wire.hpp:16-24), u16 BE
 * session, u32 BE iteration, payload.  PCB_E_SHAPE past kFrameCap (length_error).  out = NULL
 * queries *out_len. */
pcb_status pcb_encode_envelope(uint8_t type, uint16_t session, uint32_t iteration, const uint8_t* payload,
                               size_t payload_len, uint8_t* out, size_t out_cap, size_t* out_len, pcb_stream stream);

/* ---- generic primitive + measurement ------------------------------------------------------ */

/* y_i = x_i^e mod m for an odd modulus m (m_limbs <= 96) and a batch-uniform exponent e —
 * the batched ModArith::pow (paillier.cpp:26-30).  Inputs/outputs m_limbs wide. */
pcb_status pcb_modexp_batch(const uint32_t* m, uint32_t m_limbs, const uint32_t* e, uint32_t e_limbs,
                            const uint32_t* x, size_t count, uint32_t* y, pcb_stream stream);

/* IMAD roofline microbenchmark on the current device: kind 0 = IMAD.WIDE.U32 chains,
 * kind 1 = IMAD.LO + IMAD.HI pairs.  Returns MAC32/s (< 0 on error). */
double pcb_imad_peak(int kind, int iters, float* ms_out);

/* Number of kernels this library has launched (process-wide), for bench.py's gpu_launches. */
uint64_t pcb_launch_count(void);

/* Hot-kernel timing for the roofline (bench.py): while enabled, every launch of the modexp
 * "side" kernel is bracketed by CUDA events on the stream it runs on, and its algorithmic
 * MAC32 count (canonical formula) is accumulated.  pcb_profile_end
 * synchronises, sums the per-launch event durations and disables recording. */
void pcb_profile_begin(void);
pcb_status pcb_profile_end(double* side_ms_total, uint64_t* side_launches, double* side_alg_mac32);
/* int8 tensor-core MACs issued by the RNS kernels (base extensions) in the last profile window. */
double pcb_profile_int8_macs(void);

const char* pcb_status_str(pcb_status s);

#ifdef __cplusplus
}
#endif
#endif /* PCB200_H */
