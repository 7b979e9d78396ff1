// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never on the product path).
//
// A thin C ABI over the UNMODIFIED reference objects compiled from
// /root/reference/proj/src/{bignat,coeffrep,fft,modexp,paillier,quantize}.cpp by
// oracle/Makefile into oracle/_ref/libpcref.so.  It lets the Python tests, the golden-vector
// generator (oracle/gen_golden.py) and bench.py's cpu_baseline / --impl reference leg drive the
// reference's own pcadmm::Paillier / quantize code with plain pointers.
//
// Every value crosses the boundary as fixed-width little-endian u32 limbs.  Exceptions thrown by
// the reference are mapped to per-element status codes with the same numbering as
// include/pcb200.h (pcb_status), so the GPU path's error behaviour is compared 1:1.
#include <omp.h>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "pcadmm/bignat.hpp"
#include "pcadmm/paillier.hpp"
#include "pcadmm/quantize.hpp"

using namespace pcadmm;

namespace {

enum : int {
  ST_OK = 0,
  ST_PLAINTEXT_RANGE = 1,   // std::invalid_argument("plaintext not below n")
  ST_RANDOMNESS_RANGE = 2,  // std::invalid_argument("randomness not in [1, n)")
  ST_CIPHER_RANGE = 3,      // std::invalid_argument("ciphertext not below n^2")
  ST_NOT_UNIT = 4,          // std::runtime_error("ciphertext outside the multiplicative group")
  ST_OVERFLOW = 5,          // std::overflow_error (plain_bits guard)
  ST_NO_PRIVATE = 6,        // std::logic_error
  ST_SHAPE = 7,             // std::invalid_argument (shape / window)
  ST_OTHER = 99,
};

BigNat from_limbs32(const uint32_t* p, size_t n) {
  std::vector<u64> l((n + 1) / 2, 0);
  for (size_t i = 0; i < n; i++) l[i / 2] |= (u64)p[i] << (32 * (i % 2));
  return BigNat::from_limbs(std::move(l));
}

int to_limbs32(const BigNat& v, uint32_t* out, size_t n) {
  std::memset(out, 0, n * 4);
  const auto& l = v.limbs();
  if (v.bit_length() > 32 * n) return -1;
  for (size_t i = 0; i < l.size(); i++) {
    if (2 * i < n) out[2 * i] = (uint32_t)l[i];
    if (2 * i + 1 < n) out[2 * i + 1] = (uint32_t)(l[i] >> 32);
  }
  return 0;
}

int classify(const std::exception& e) {
  std::string w = e.what();
  if (dynamic_cast<const std::overflow_error*>(&e)) return ST_OVERFLOW;
  if (dynamic_cast<const std::logic_error*>(&e) && !dynamic_cast<const std::invalid_argument*>(&e) &&
      !dynamic_cast<const std::domain_error*>(&e))
    return ST_NO_PRIVATE;
  if (w.find("plaintext") != std::string::npos) return ST_PLAINTEXT_RANGE;
  if (w.find("randomness") != std::string::npos) return ST_RANDOMNESS_RANGE;
  if (w.find("ciphertext not below") != std::string::npos) return ST_CIPHER_RANGE;
  if (w.find("multiplicative group") != std::string::npos) return ST_NOT_UNIT;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return ST_SHAPE;
  return ST_OTHER;
}

struct RefKey {
  KeyPair kp;
  Paillier* ph = nullptr;
  Paillier* pub = nullptr;
};

}  // namespace

extern "C" {

// ---- keys -------------------------------------------------------------------------------
// keygen(Rng(seed), bits, binomial) — paillier.cpp:106-123.  Writes n, p, q (LE u32 limbs,
// widths nl, nl/2+1, nl/2+1) and returns an opaque handle holding the KeyPair + a Paillier.
void* pcref_keygen(uint64_t seed, uint32_t bits, int binomial, uint64_t* rng_state_inout) {
  try {
    Rng rng(rng_state_inout ? *rng_state_inout : seed);
    auto* k = new RefKey;
    k->kp = keygen(rng, bits, binomial ? GMode::binomial : GMode::random_g);
    if (rng_state_inout) *rng_state_inout = rng.state;
    k->ph = new Paillier(k->kp);
    k->pub = new Paillier(k->kp.pub);
    return k;
  } catch (...) {
    return nullptr;
  }
}

// keypair_from_primes — paillier.cpp:125-130.
void* pcref_from_primes(const uint32_t* p, const uint32_t* q, uint32_t limbs, int binomial,
                        uint64_t g_seed) {
  try {
    auto* k = new RefKey;
    k->kp = keypair_from_primes(from_limbs32(p, limbs), from_limbs32(q, limbs),
                                binomial ? GMode::binomial : GMode::random_g, g_seed);
    k->ph = new Paillier(k->kp);
    k->pub = new Paillier(k->kp.pub);
    return k;
  } catch (...) {
    return nullptr;
  }
}

void pcref_free(void* h) {
  auto* k = (RefKey*)h;
  if (!k) return;
  delete k->ph;
  delete k->pub;
  delete k;
}

uint32_t pcref_n_bits(void* h) { return (uint32_t)((RefKey*)h)->kp.pub.n.bit_length(); }

// which: 0 n, 1 p, 2 q, 3 epsilon, 4 mu, 5 n2, 6 g, 7 p2_inv_q2, 8 n_mod_phi_p2, 9 n_mod_phi_q2,
//        10 eps_mod_phi_p2, 11 eps_mod_phi_q2, 12 p2, 13 q2
int pcref_get(void* h, int which, uint32_t* out, uint32_t limbs) {
  const KeyPair& kp = ((RefKey*)h)->kp;
  const BigNat* v = nullptr;
  switch (which) {
    case 0: v = &kp.pub.n; break;
    case 1: v = &kp.prv.p; break;
    case 2: v = &kp.prv.q; break;
    case 3: v = &kp.prv.epsilon; break;
    case 4: v = &kp.prv.mu; break;
    case 5: v = &kp.pub.n2; break;
    case 6: v = &kp.pub.g; break;
    case 7: v = &kp.crt.p2_inv_q2; break;
    case 8: v = &kp.crt.n_mod_phi_p2; break;
    case 9: v = &kp.crt.n_mod_phi_q2; break;
    case 10: v = &kp.crt.eps_mod_phi_p2; break;
    case 11: v = &kp.crt.eps_mod_phi_q2; break;
    case 12: v = &kp.crt.p2; break;
    case 13: v = &kp.crt.q2; break;
    default: return -2;
  }
  return to_limbs32(*v, out, limbs);
}

// serialize_keypair — paillier.cpp:152-166.  Returns the byte count (call with out=NULL first).
size_t pcref_serialize(void* h, uint8_t* out, size_t cap) {
  std::vector<uint8_t> b = serialize_keypair(((RefKey*)h)->kp);
  if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  return b.size();
}

void* pcref_parse(const uint8_t* bytes, size_t len) {
  try {
    auto* k = new RefKey;
    k->kp = parse_keypair(std::vector<uint8_t>(bytes, bytes + len));
    k->ph = new Paillier(k->kp);
    k->pub = new Paillier(k->kp.pub);
    return k;
  } catch (...) {
    return nullptr;
  }
}

// ---- randomness ----------------------------------------------------------------------------
// Paillier::sample_r x count — paillier.cpp:233-239 on Rng(state).  r is written with width
// limbs; *state is advanced exactly as the reference's serial draw loop (paillier.cpp:499-500).
void pcref_sample_r(void* h, uint64_t* state, size_t count, uint32_t* r_out, uint32_t limbs) {
  RefKey* k = (RefKey*)h;
  Rng rng(*state);
  for (size_t i = 0; i < count; i++) to_limbs32(k->pub->sample_r(rng), r_out + i * limbs, limbs);
  *state = rng.state;
}

uint64_t pcref_rng_next(uint64_t* state) {
  Rng r(*state);
  uint64_t v = r.next();
  *state = r.state;
  return v;
}

// ---- encryption / decryption ---------------------------------------------------------------
// mode: 0 encrypt_with_r (public key, paillier.cpp:320-328), 1 crt_encrypt_with_r (334-344).
// Element i uses m[i*m_limbs..], r[i*r_limbs..]; c written with width c_limbs; st[i] status.
// OpenMP over elements (the reference's own vector form parallelises the same way,
// paillier.cpp:502-505); threads <= 0 keeps the OpenMP default.
void pcref_encrypt(void* h, int mode, const uint32_t* m, uint32_t m_limbs, const uint32_t* r,
                   uint32_t r_limbs, size_t count, uint32_t* c, uint32_t c_limbs, int32_t* st,
                   int threads) {
  RefKey* k = (RefKey*)h;
  Paillier* ph = mode == 1 ? k->ph : k->pub;
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1) if (threads != 1)
  for (ptrdiff_t i = 0; i < (ptrdiff_t)count; i++) {
    try {
      BigNat mi = from_limbs32(m + i * m_limbs, m_limbs);
      BigNat ri = from_limbs32(r + i * r_limbs, r_limbs);
      Ciphertext ct = mode == 1 ? ph->crt_encrypt_with_r(mi, ri) : ph->encrypt_with_r(mi, ri);
      to_limbs32(ct.value, c + i * c_limbs, c_limbs);
      if (st) st[i] = ST_OK;
    } catch (const std::exception& e) {
      std::memset(c + i * c_limbs, 0, c_limbs * 4);
      if (st) st[i] = classify(e);
    }
  }
}

// mode: 0 decrypt (paillier.cpp:346-352), 1 crt_decrypt (354-361).
void pcref_decrypt(void* h, int mode, const uint32_t* c, uint32_t c_limbs, size_t count,
                   uint32_t* m, uint32_t m_limbs, int32_t* st, int threads) {
  RefKey* k = (RefKey*)h;
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1) if (threads != 1)
  for (ptrdiff_t i = 0; i < (ptrdiff_t)count; i++) {
    try {
      Ciphertext ct{from_limbs32(c + i * c_limbs, c_limbs), 0};
      BigNat mi = mode == 1 ? k->ph->crt_decrypt(ct) : k->ph->decrypt(ct);
      to_limbs32(mi, m + i * m_limbs, m_limbs);
      if (st) st[i] = ST_OK;
    } catch (const std::exception& e) {
      std::memset(m + i * m_limbs, 0, m_limbs * 4);
      if (st) st[i] = classify(e);
    }
  }
}

// ---- collaborative variant: decrypt_with_half (paillier.cpp:363-369), finish_split_encrypt
// (paillier.cpp:402-414).  Element i: c / p2 values of c_limbs / p_limbs words.
void pcref_decrypt_with_half(void* h, const uint32_t* c, uint32_t c_limbs, const uint32_t* p2, uint32_t p_limbs,
                             size_t count, uint32_t* m, uint32_t m_limbs, int32_t* st) {
  RefKey* k = (RefKey*)h;
  for (size_t i = 0; i < count; i++) {
    try {
      Ciphertext ct{from_limbs32(c + i * c_limbs, c_limbs), 0};
      BigNat mi = k->ph->decrypt_with_half(ct, from_limbs32(p2 + i * p_limbs, p_limbs));
      to_limbs32(mi, m + i * m_limbs, m_limbs);
      if (st) st[i] = ST_OK;
    } catch (const std::exception& e) {
      std::memset(m + i * m_limbs, 0, m_limbs * 4);
      if (st) st[i] = classify(e);
    }
  }
}

void pcref_finish_split_encrypt(void* h, const uint32_t* m, uint32_t m_limbs, const uint32_t* g, uint32_t g_limbs,
                                const uint32_t* r, uint32_t r_limbs, size_t count, uint32_t* c, uint32_t c_limbs,
                                int32_t* st) {
  RefKey* k = (RefKey*)h;
  for (size_t i = 0; i < count; i++) {
    try {
      Ciphertext ct = k->ph->finish_split_encrypt(from_limbs32(m + i * m_limbs, m_limbs),
                                                  from_limbs32(g + i * g_limbs, g_limbs),
                                                  from_limbs32(r + i * r_limbs, r_limbs));
      to_limbs32(ct.value, c + i * c_limbs, c_limbs);
      if (st) st[i] = ST_OK;
    } catch (const std::exception& e) {
      std::memset(c + i * c_limbs, 0, c_limbs * 4);
      if (st) st[i] = classify(e);
    }
  }
}

// ---- homomorphic operations ------------------------------------------------------------------
// hom_add (paillier.cpp:428-432) with plain_bits in/out; status ST_OVERFLOW when the guard trips.
void pcref_hom_add(void* h, const uint32_t* a, const uint32_t* b, const uint32_t* a_bits,
                   const uint32_t* b_bits, size_t count, uint32_t c_limbs, uint32_t* out,
                   uint32_t* out_bits, int32_t* st) {
  RefKey* k = (RefKey*)h;
  for (size_t i = 0; i < count; i++) {
    try {
      Ciphertext x{from_limbs32(a + i * c_limbs, c_limbs), a_bits ? a_bits[i] : 0};
      Ciphertext y{from_limbs32(b + i * c_limbs, c_limbs), b_bits ? b_bits[i] : 0};
      Ciphertext z = k->pub->hom_add(x, y);
      to_limbs32(z.value, out + i * c_limbs, c_limbs);
      if (out_bits) out_bits[i] = z.plain_bits;
      if (st) st[i] = ST_OK;
    } catch (const std::exception& e) {
      if (st) st[i] = classify(e);
    }
  }
}

// hom_scalar_mul (paillier.cpp:434-439), scalar k as u64.
void pcref_hom_scalar_mul(void* h, const uint64_t* ks, const uint32_t* c, const uint32_t* c_bits,
                          size_t count, uint32_t c_limbs, uint32_t* out, uint32_t* out_bits,
                          int32_t* st) {
  RefKey* k = (RefKey*)h;
  for (size_t i = 0; i < count; i++) {
    try {
      Ciphertext x{from_limbs32(c + i * c_limbs, c_limbs), c_bits ? c_bits[i] : 0};
      Ciphertext z = k->pub->hom_scalar_mul(BigNat(ks[i]), x);
      to_limbs32(z.value, out + i * c_limbs, c_limbs);
      if (out_bits) out_bits[i] = z.plain_bits;
      if (st) st[i] = ST_OK;
    } catch (const std::exception& e) {
      if (st) st[i] = classify(e);
    }
  }
}

// hom_matvec (paillier.cpp:441-493): expo is rows x cols row-major u64.
int pcref_hom_matvec(void* h, const uint32_t* alpha, const uint32_t* alpha_bits,
                     const uint64_t* expo, const uint32_t* zv, const uint32_t* zv_bits,
                     size_t rows, size_t cols, uint32_t window, uint32_t c_limbs, uint32_t* out,
                     uint32_t* out_bits, int threads) {
  RefKey* k = (RefKey*)h;
  // the reference parallelises the row loop with OpenMP (paillier.cpp:477); pin the team size
  if (threads > 0) omp_set_num_threads(threads);
  try {
    std::vector<Ciphertext> a(rows), z(cols);
    std::vector<std::vector<u64>> e(rows, std::vector<u64>(cols));
    for (size_t i = 0; i < rows; i++) {
      a[i] = Ciphertext{from_limbs32(alpha + i * c_limbs, c_limbs), alpha_bits ? alpha_bits[i] : 0};
      for (size_t j = 0; j < cols; j++) e[i][j] = expo[i * cols + j];
    }
    for (size_t j = 0; j < cols; j++)
      z[j] = Ciphertext{from_limbs32(zv + j * c_limbs, c_limbs), zv_bits ? zv_bits[j] : 0};
    std::vector<Ciphertext> o = k->pub->hom_matvec(a, e, z, window);
    for (size_t i = 0; i < rows; i++) {
      to_limbs32(o[i].value, out + i * c_limbs, c_limbs);
      if (out_bits) out_bits[i] = o[i].plain_bits;
    }
    return ST_OK;
  } catch (const std::exception& ex) {
    return classify(ex);
  }
}

// Counters (paillier.hpp:84-87) of the private-key instance.
void pcref_counters(void* h, uint64_t* pow_full, uint64_t* pow_half) {
  OpCount c = ((RefKey*)h)->ph->counters();
  *pow_full = c.pow_full;
  *pow_half = c.pow_half;
}

// ---- quantization (quantize.cpp) -------------------------------------------------------------
// gamma2 / gamma1 over a vector; clamps[0]=low, clamps[1]=high.  q1 is u128 as 2 x u64 (lo, hi).
int pcref_gamma2(const double* v, size_t n, double zmin, double zmax, double delta, uint64_t* out,
                 uint64_t* clamps) {
  try {
    ClampStats cs;
    QuantSpec s{zmin, zmax, delta};
    for (size_t i = 0; i < n; i++) out[i] = gamma2(v[i], s, &cs);
    if (clamps) { clamps[0] = cs.low; clamps[1] = cs.high; }
    return 0;
  } catch (...) {
    return ST_SHAPE;
  }
}

int pcref_gamma1(const double* v, size_t n, double zmin, double zmax, double delta, uint64_t* out,
                 uint64_t* clamps) {
  try {
    ClampStats cs;
    QuantSpec s{zmin, zmax, delta};
    for (size_t i = 0; i < n; i++) {
      u128 q = gamma1(v[i], s, &cs);
      out[2 * i] = (uint64_t)q;
      out[2 * i + 1] = (uint64_t)(q >> 64);
    }
    if (clamps) { clamps[0] = cs.low; clamps[1] = cs.high; }
    return 0;
  } catch (...) {
    return ST_SHAPE;
  }
}

double pcref_degamma2(uint64_t q, double zmin, double zmax, double delta) {
  return degamma2(q, QuantSpec{zmin, zmax, delta});
}

// combined_quantized_update (quantize.cpp:66-82): q_alpha u128 pairs, q_b rows x cols.
void pcref_combined_update(const uint64_t* q_alpha, const uint64_t* q_b, const uint64_t* q_z,
                           const uint64_t* q_nv, size_t rows, size_t cols, uint64_t* out) {
  std::vector<u128> qa(rows);
  std::vector<std::vector<u64>> qb(rows, std::vector<u64>(cols));
  for (size_t i = 0; i < rows; i++) {
    qa[i] = ((u128)q_alpha[2 * i + 1] << 64) | q_alpha[2 * i];
    for (size_t j = 0; j < cols; j++) qb[i][j] = q_b[i * cols + j];
  }
  std::vector<u64> z(q_z, q_z + cols), nv(q_nv, q_nv + cols);
  std::vector<u128> o = combined_quantized_update(qa, qb, z, nv);
  for (size_t i = 0; i < rows; i++) {
    out[2 * i] = (uint64_t)o[i];
    out[2 * i + 1] = (uint64_t)(o[i] >> 64);
  }
}

// inverse_quantize_x (quantize.cpp:84-112).
void pcref_inverse_quantize_x(const uint64_t* q, const uint64_t* rowsum, const uint64_t* q_z,
                              const uint64_t* q_nv, size_t rows, size_t cols, double zmin,
                              double zmax, double delta, double* out) {
  std::vector<u128> qq(rows);
  for (size_t i = 0; i < rows; i++) qq[i] = ((u128)q[2 * i + 1] << 64) | q[2 * i];
  std::vector<u64> rs(rowsum, rowsum + rows), z(q_z, q_z + cols), nv(q_nv, q_nv + cols);
  std::vector<double> o = inverse_quantize_x(qq, rs, z, nv, QuantSpec{zmin, zmax, delta});
  for (size_t i = 0; i < rows; i++) out[i] = o[i];
}

// widen_bounds (quantize.cpp:114-129).
int pcref_widen_bounds(double lo, double hi, double margin, double delta, double* zmin,
                       double* zmax) {
  try {
    QuantSpec s = widen_bounds(lo, hi, margin, delta);
    *zmin = s.z_min;
    *zmax = s.z_max;
    return 0;
  } catch (...) {
    return ST_SHAPE;
  }
}

}  // extern "C"
