// pcb200_pcadmm.hpp — the C++ drop-in for the reference's hot-path API, over the C ABI of
// include/pcb200.h (libpcb200.so).  A program written against pcadmm::Paillier and the key types
// (/root/reference/proj/include/pcadmm/paillier.hpp:30-181, bignat.hpp:19-125) compiles against
// this header unchanged (cpp/include/pcadmm/{paillier,bignat}.hpp forward here) and every
// per-element operation -- encryption, decryption, r sampling, hom_add, hom_scalar_mul,
// hom_matvec, the vector forms, the pooled / split / delegated forms -- runs as one batched CUDA
// call on the B200.  Host code here is bookkeeping only: key material and CRT constants (one-time,
// as in the reference), plain_bits tracking, exception mapping, operation counters.
//
// Notes:
//   * GMode::random_g keys work: the generator search is the reference's (host key work), and the
//     device computes g^m from 64-bit digit powers (pcb_ctx_set_generator).  The fused ADMM hot
//     path (pcb_quantize_encrypt) is the g = n + 1 form, as north_star fixes it.
//   * Engine::coeff_fft is accepted and runs the same CUDA path (the reference pins the two lanes
//     to identical results, test_paillier.cpp:242-257); there is no second lane to dispatch to.
//   * Keys up to 4096 bits (the reference keygen's largest size); larger moduli are refused by the
//     device context.
// Errors map 1:1 to the reference's exception types (paillier.cpp; pcb_status in pcb200.h).
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace pcadmm {

using u32 = uint32_t;
using u64 = uint64_t;
using u128 = unsigned __int128;

// Natural number, canonical little-endian 64-bit limbs (bignat.hpp:19-61 semantics).  Host-side
// value type for keys, plaintexts and ciphertexts crossing the API; the arithmetic behind it is
// the library's host big-integer code (csrc/host/hbn.cpp), used for key setup and bookkeeping.
class BigNat {
 public:
  BigNat() = default;
  explicit BigNat(u64 v) {
    if (v) limbs_.push_back(v);
  }
  static BigNat from_u128(u128 v);
  static BigNat from_limbs(std::vector<u64> limbs);
  static BigNat from_decimal(const std::string& s);
  static BigNat from_bytes_be(const uint8_t* data, size_t len);

  const std::vector<u64>& limbs() const { return limbs_; }
  bool is_zero() const { return limbs_.empty(); }
  bool is_odd() const { return !limbs_.empty() && (limbs_[0] & 1u); }
  size_t bit_length() const;
  bool bit(size_t i) const;
  u64 to_u64() const;
  u128 to_u128() const;
  double to_double() const;
  std::string to_decimal() const;
  std::vector<uint8_t> to_bytes_be() const;

  // 32-bit limb views for the C ABI (fixed width, zero padded)
  std::vector<uint32_t> to_u32(size_t width) const;
  static BigNat from_u32(const uint32_t* w, size_t n);

  friend int cmp(const BigNat& a, const BigNat& b);
  bool operator==(const BigNat& o) const { return limbs_ == o.limbs_; }
  bool operator!=(const BigNat& o) const { return limbs_ != o.limbs_; }
  bool operator<(const BigNat& o) const { return cmp(*this, o) < 0; }
  bool operator<=(const BigNat& o) const { return cmp(*this, o) <= 0; }
  bool operator>(const BigNat& o) const { return cmp(*this, o) > 0; }
  bool operator>=(const BigNat& o) const { return cmp(*this, o) >= 0; }
  friend BigNat operator+(const BigNat& a, const BigNat& b);
  friend BigNat operator-(const BigNat& a, const BigNat& b);
  friend BigNat operator*(const BigNat& a, const BigNat& b);
  friend BigNat operator<<(const BigNat& a, size_t bits);
  friend BigNat operator>>(const BigNat& a, size_t bits);
  BigNat& operator+=(const BigNat& o) { return *this = *this + o; }
  BigNat& operator-=(const BigNat& o) { return *this = *this - o; }

 private:
  void trim() {
    while (!limbs_.empty() && !limbs_.back()) limbs_.pop_back();
  }
  std::vector<u64> limbs_;
};

struct DivModResult {
  BigNat quot, rem;
};
DivModResult divmod(const BigNat& a, const BigNat& b);
BigNat mod(const BigNat& a, const BigNat& m);
BigNat gcd(BigNat a, BigNat b);
BigNat lcm(const BigNat& a, const BigNat& b);
std::optional<BigNat> mod_inverse(const BigNat& a, const BigNat& m);
BigNat pow_mod(const BigNat& base, const BigNat& exp, const BigNat& m);  // host; key setup only

// splitmix64, the reference's stream (bignat.cpp:388-412)
struct Rng {
  u64 state;
  explicit Rng(u64 seed) : state(seed) {}
  u64 next();
  u64 below(u64 bound);
  double unit();
  double gaussian();
};
BigNat random_bits(Rng& rng, size_t bits);
BigNat random_below(Rng& rng, const BigNat& bound);
bool is_probable_prime(const BigNat& n, Rng& rng, int rounds = 40);
BigNat random_prime(Rng& rng, size_t bits, int mr_rounds = 40);

enum class Engine { packed, coeff_fft };
enum class GMode { binomial, random_g };

struct PublicKey {
  BigNat n, n2, g;
  size_t key_bits = 0;
  bool binomial_g = true;
};
struct PrivateKey {
  BigNat p, q, epsilon, mu;
};
struct CrtContext {
  BigNat p2, q2, g_p2, g_q2, phi_p2, phi_q2, p2_inv_q2;
  BigNat n_mod_phi_p2, n_mod_phi_q2, eps_mod_phi_p2, eps_mod_phi_q2;
};
struct KeyPair {
  PublicKey pub;
  PrivateKey prv;
  CrtContext crt;
};
struct CrtShare {
  BigNat p2, phi_p2;
};
struct Ciphertext {
  BigNat value;
  u32 plain_bits = 0;
};
struct RnFactor {
  BigNat r, full, half_p2, half_q2;
};
struct OpCount {
  u64 pow_full = 0, pow_half = 0;
};

KeyPair keygen(Rng& rng, size_t key_bits, GMode gmode = GMode::binomial);
KeyPair keypair_from_primes(const BigNat& p, const BigNat& q, GMode gmode = GMode::binomial, u64 g_seed = 1);
CrtShare crt_share(const KeyPair& keys);
std::vector<uint8_t> serialize_keypair(const KeyPair& keys);
KeyPair parse_keypair(const std::vector<uint8_t>& bytes);

// One key, its device context (pcb_ctx on the CUDA device PCB_DEVICE, default 0) and the
// operation counters of one protocol role.
class Paillier {
 public:
  Paillier(PublicKey pub, Engine engine = Engine::packed);
  Paillier(const KeyPair& keys, Engine engine = Engine::packed);
  ~Paillier();
  Paillier(const Paillier&) = delete;
  Paillier& operator=(const Paillier&) = delete;

  const PublicKey& pub() const { return pub_; }
  bool has_private() const { return has_prv_; }
  const PrivateKey& prv() const;
  const CrtContext& crt() const;
  Engine engine() const { return engine_; }
  OpCount counters() const { return OpCount{pow_full_.load(), pow_half_.load()}; }
  void reset_counters() {
    pow_full_ = 0;
    pow_half_ = 0;
  }

  BigNat sample_r(Rng& rng) const;
  Ciphertext encrypt(const BigNat& m, Rng& rng);
  Ciphertext encrypt_with_r(const BigNat& m, const BigNat& r);
  Ciphertext crt_encrypt(const BigNat& m, Rng& rng);
  Ciphertext crt_encrypt_with_r(const BigNat& m, const BigNat& r);
  BigNat decrypt(const Ciphertext& c);
  BigNat crt_decrypt(const Ciphertext& c);

  RnFactor make_rn_factor(const BigNat& r);
  Ciphertext encrypt_with_factor(const BigNat& m, const RnFactor& f);
  Ciphertext crt_encrypt_with_factor(const BigNat& m, const RnFactor& f);
  Ciphertext finish_split_encrypt(const BigNat& m, const BigNat& p2_g_power, const BigNat& r);
  Ciphertext finish_split_encrypt_with_factor(const BigNat& m, const BigNat& p2_g_power, const RnFactor& f);
  BigNat decrypt_with_half(const Ciphertext& c, const BigNat& p2_power);

  Ciphertext hom_add(const Ciphertext& a, const Ciphertext& b);
  Ciphertext hom_scalar_mul(const BigNat& k, const Ciphertext& c);
  std::vector<Ciphertext> hom_matvec(const std::vector<Ciphertext>& alpha, const std::vector<std::vector<u64>>& expo,
                                     const std::vector<Ciphertext>& zv, unsigned window = 6);
  std::vector<Ciphertext> encrypt_vec(const std::vector<BigNat>& ms, Rng& rng, bool use_crt);
  std::vector<BigNat> decrypt_vec(const std::vector<Ciphertext>& cs, bool use_crt);

 private:
  void need_private(const char* what) const;
  void bump_bits_or_throw(u32 bits) const;
  std::vector<BigNat> enc_batch(const std::vector<BigNat>& ms, const std::vector<BigNat>& rs, bool use_crt,
                                bool count_g = true);
  void set_generator();
  std::vector<BigNat> dec_batch(const std::vector<Ciphertext>& cs, bool use_crt);

  PublicKey pub_;
  bool has_prv_ = false;
  PrivateKey prv_;
  CrtContext crt_;
  Engine engine_;
  void* ctx_ = nullptr;  // pcb_ctx*
  size_t L_ = 0;         // u32 limbs of n
  std::atomic<u64> pow_full_{0}, pow_half_{0};
};

}  // namespace pcadmm
