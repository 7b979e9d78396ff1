// pcb200_pcadmm.cpp — pcadmm::Paillier and the key types over the C ABI (include/pcb200.h).
// Per-element work is one batched call of libpcb200.so on the device; this file keeps the
// reference's host bookkeeping: key constants (paillier.cpp:43-130 semantics), plain_bits
// (paillier.cpp:245-251, 327, 429-437, 457-489), counters (paillier.hpp:84-87) and exceptions.
#include "pcb200_pcadmm.hpp"

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "host/hbn.hpp"
#include "pcb200.h"

namespace pcadmm {
namespace {

using pcb::HBN;

HBN to_h(const BigNat& a) {
  std::vector<uint64_t> l = a.limbs();
  return HBN::from_u64_limbs(l);
}
BigNat from_h(const HBN& h) {
  std::vector<u64> l((h.w.size() + 1) / 2, 0);
  for (size_t i = 0; i < h.w.size(); i++) l[i / 2] |= (u64)h.w[i] << (32 * (i % 2));
  return BigNat::from_limbs(std::move(l));
}

// pcb_status -> the reference's exception type (pcb200.h enum comments)
[[noreturn]] void throw_status(int st, const char* what) {
  std::string msg = std::string(what) + ": " + pcb_status_str((pcb_status)st);
  switch (st) {
    case PCB_E_NOT_UNIT: throw std::runtime_error(msg);
    case PCB_E_OVERFLOW: throw std::overflow_error(msg);
    case PCB_E_NO_PRIVATE: throw std::logic_error(msg);
    case PCB_E_CUDA:
    case PCB_E_ALLOC:
    case PCB_E_RANGE_UPDATE: throw std::runtime_error(msg);
    default: throw std::invalid_argument(msg);
  }
}
void check(int st, const char* what) {
  if (st != PCB_OK) throw_status(st, what);
}
// first failing element of a batch, as the reference's element loop would throw it
void check_elems(const std::vector<int32_t>& st, const char* what) {
  for (int32_t s : st)
    if (s != PCB_OK) throw_status(s, what);
}

int device_index() {
  const char* d = std::getenv("PCB_DEVICE");
  return d ? std::atoi(d) : 0;
}

KeyPair finish_binomial(const BigNat& p, const BigNat& q, size_t key_bits) {
  // paillier.cpp:63-104, binomial generator: g = n + 1, mu = (eps mod n)^-1 mod n
  KeyPair k;
  const HBN hp = to_h(p), hq = to_h(q), n = hp * hq;
  const HBN eps = pcb::lcm(hp - HBN(1), hq - HBN(1));
  HBN mu;
  if (!pcb::mod_inverse(pcb::mod(eps, n), n, mu)) throw std::invalid_argument("lcm(p-1, q-1) shares a factor with n");
  k.pub.n = from_h(n);
  k.pub.n2 = from_h(n * n);
  k.pub.g = from_h(n + HBN(1));
  k.pub.key_bits = key_bits;
  k.pub.binomial_g = true;
  k.prv.p = p;
  k.prv.q = q;
  k.prv.epsilon = from_h(eps);
  k.prv.mu = from_h(mu);
  // make_crt (paillier.cpp:43-60)
  const HBN p2 = hp * hp, q2 = hq * hq, phip = p2 - hp, phiq = q2 - hq;
  HBN inv;
  if (!pcb::mod_inverse(pcb::mod(p2, q2), q2, inv)) throw std::invalid_argument("p and q share a factor");
  k.crt.p2 = from_h(p2);
  k.crt.q2 = from_h(q2);
  k.crt.g_p2 = from_h(pcb::mod(n + HBN(1), p2));
  k.crt.g_q2 = from_h(pcb::mod(n + HBN(1), q2));
  k.crt.phi_p2 = from_h(phip);
  k.crt.phi_q2 = from_h(phiq);
  k.crt.p2_inv_q2 = from_h(inv);
  k.crt.n_mod_phi_p2 = from_h(pcb::mod(n, phip));
  k.crt.n_mod_phi_q2 = from_h(pcb::mod(n, phiq));
  k.crt.eps_mod_phi_p2 = from_h(pcb::mod(eps, phip));
  k.crt.eps_mod_phi_q2 = from_h(pcb::mod(eps, phiq));
  return k;
}

// Random generator (paillier.cpp:80-100): g = random_below(Rng(g_seed), n^2) until g is a unit
// with L(g^eps mod n^2) invertible mod n; mu = that inverse.  One-time key work on the host, as in
// the reference; every per-element g power then runs on the device (pcb_ctx_set_generator).
void finish_random_g(KeyPair& k, u64 g_seed) {
  const HBN n = to_h(k.pub.n), n2 = to_h(k.pub.n2), eps = to_h(k.prv.epsilon);
  pcb::HRng gr(g_seed);
  for (int budget = 256;; budget--) {
    if (budget == 0) throw std::runtime_error("generator search exhausted");
    const HBN g = pcb::random_below(gr, n2);
    if (g.bit_length() < 2 || pcb::gcd(g, n) != HBN(1)) continue;
    HBN l, r, mu;
    pcb::divmod(pcb::pow_mod(g, eps, n2) - HBN(1), n, l, r);
    if (!pcb::mod_inverse(l, n, mu)) continue;
    k.pub.g = from_h(g);
    k.pub.binomial_g = false;
    k.prv.mu = from_h(mu);
    const HBN p2 = to_h(k.crt.p2), q2 = to_h(k.crt.q2);
    k.crt.g_p2 = from_h(pcb::mod(g, p2));
    k.crt.g_q2 = from_h(pcb::mod(g, q2));
    return;
  }
}

}  // namespace

// ---- BigNat ---------------------------------------------------------------------------------
BigNat BigNat::from_u128(u128 v) {
  return from_limbs({(u64)v, (u64)(v >> 64)});
}
BigNat BigNat::from_limbs(std::vector<u64> l) {
  BigNat b;
  b.limbs_ = std::move(l);
  b.trim();
  return b;
}
BigNat BigNat::from_decimal(const std::string& s) {
  if (s.empty()) throw std::invalid_argument("empty decimal string");
  BigNat r;
  for (char c : s) {
    if (c < '0' || c > '9') throw std::invalid_argument("non-digit in decimal string");
    r = r * BigNat(10) + BigNat((u64)(c - '0'));
  }
  return r;
}
BigNat BigNat::from_bytes_be(const uint8_t* d, size_t len) {
  std::vector<u64> l((len + 7) / 8, 0);
  for (size_t i = 0; i < len; i++) l[i / 8] |= (u64)d[len - 1 - i] << (8 * (i % 8));
  return from_limbs(std::move(l));
}
size_t BigNat::bit_length() const {
  if (limbs_.empty()) return 0;
  return 64 * (limbs_.size() - 1) + (64 - (size_t)__builtin_clzll(limbs_.back()));
}
bool BigNat::bit(size_t i) const {
  return i / 64 < limbs_.size() && ((limbs_[i / 64] >> (i % 64)) & 1u);
}
u64 BigNat::to_u64() const {
  if (limbs_.size() > 1) throw std::overflow_error("BigNat wider than 64 bits");
  return limbs_.empty() ? 0 : limbs_[0];
}
u128 BigNat::to_u128() const {
  if (limbs_.size() > 2) throw std::overflow_error("BigNat wider than 128 bits");
  u128 v = 0;
  for (size_t i = limbs_.size(); i-- > 0;) v = (v << 64) | limbs_[i];
  return v;
}
double BigNat::to_double() const {  // limb-wise, as BigNat::to_double (bignat.cpp:56-60)
  double v = 0.0;
  for (size_t i = limbs_.size(); i-- > 0;) v = v * 18446744073709551616.0 + (double)limbs_[i];
  return v;
}
std::string BigNat::to_decimal() const {
  if (is_zero()) return "0";
  std::string s;
  BigNat v = *this;
  const BigNat ten(10);
  while (!v.is_zero()) {
    DivModResult d = divmod(v, ten);
    s.push_back((char)('0' + d.rem.to_u64()));
    v = d.quot;
  }
  return std::string(s.rbegin(), s.rend());
}
std::vector<uint8_t> BigNat::to_bytes_be() const {
  std::vector<uint8_t> out;
  for (size_t i = (bit_length() + 7) / 8; i-- > 0;) out.push_back((uint8_t)(limbs_[i / 8] >> (8 * (i % 8))));
  return out;
}
std::vector<uint32_t> BigNat::to_u32(size_t width) const {
  std::vector<uint32_t> w(width, 0);
  for (size_t i = 0; i < width && i / 2 < limbs_.size(); i++) w[i] = (uint32_t)(limbs_[i / 2] >> (32 * (i % 2)));
  return w;
}
BigNat BigNat::from_u32(const uint32_t* w, size_t n) {
  std::vector<u64> l((n + 1) / 2, 0);
  for (size_t i = 0; i < n; i++) l[i / 2] |= (u64)w[i] << (32 * (i % 2));
  return from_limbs(std::move(l));
}
int cmp(const BigNat& a, const BigNat& b) {
  if (a.limbs_.size() != b.limbs_.size()) return a.limbs_.size() < b.limbs_.size() ? -1 : 1;
  for (size_t i = a.limbs_.size(); i-- > 0;)
    if (a.limbs_[i] != b.limbs_[i]) return a.limbs_[i] < b.limbs_[i] ? -1 : 1;
  return 0;
}
BigNat operator+(const BigNat& a, const BigNat& b) { return from_h(to_h(a) + to_h(b)); }
BigNat operator-(const BigNat& a, const BigNat& b) {
  if (a < b) throw std::invalid_argument("BigNat subtraction underflow");
  return from_h(to_h(a) - to_h(b));
}
BigNat operator*(const BigNat& a, const BigNat& b) { return from_h(to_h(a) * to_h(b)); }
BigNat operator<<(const BigNat& a, size_t s) { return from_h(to_h(a) << s); }
BigNat operator>>(const BigNat& a, size_t s) { return from_h(to_h(a) >> s); }
DivModResult divmod(const BigNat& a, const BigNat& b) {
  if (b.is_zero()) throw std::invalid_argument("division by zero");
  HBN q, r;
  pcb::divmod(to_h(a), to_h(b), q, r);
  return {from_h(q), from_h(r)};
}
BigNat mod(const BigNat& a, const BigNat& m) { return divmod(a, m).rem; }
BigNat gcd(BigNat a, BigNat b) { return from_h(pcb::gcd(to_h(a), to_h(b))); }
BigNat lcm(const BigNat& a, const BigNat& b) { return from_h(pcb::lcm(to_h(a), to_h(b))); }
std::optional<BigNat> mod_inverse(const BigNat& a, const BigNat& m) {
  HBN out;
  if (!pcb::mod_inverse(to_h(a), to_h(m), out)) return std::nullopt;
  return from_h(out);
}
BigNat pow_mod(const BigNat& b, const BigNat& e, const BigNat& m) {
  if (m == BigNat(1)) return BigNat();
  return from_h(pcb::pow_mod(pcb::mod(to_h(b), to_h(m)), to_h(e), to_h(m)));
}

// ---- Rng (bignat.cpp:388-412) ---------------------------------------------------------------
u64 Rng::next() {
  pcb::HRng h(state);
  const u64 v = h.next();
  state = h.state;
  return v;
}
u64 Rng::below(u64 bound) {
  if (bound <= 1) return 0;
  const u64 mask = ~0ull >> __builtin_clzll(bound - 1);
  for (;;) {
    const u64 v = next() & mask;
    if (v < bound) return v;
  }
}
double Rng::unit() { return (double)(next() >> 11) * 0x1.0p-53; }
double Rng::gaussian() {
  double u1 = unit(), u2 = unit();
  while (u1 <= 0.0) u1 = unit();
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586477 * u2);
}
BigNat random_bits(Rng& rng, size_t bits) {
  pcb::HRng h(rng.state);
  BigNat v = from_h(pcb::random_bits(h, bits));
  rng.state = h.state;
  return v;
}
BigNat random_below(Rng& rng, const BigNat& bound) {
  if (bound.is_zero()) throw std::invalid_argument("random_below: zero bound");
  pcb::HRng h(rng.state);
  BigNat v = from_h(pcb::random_below(h, to_h(bound)));
  rng.state = h.state;
  return v;
}
bool is_probable_prime(const BigNat& n, Rng& rng, int rounds) {
  pcb::HRng h(rng.state);
  const bool r = pcb::is_probable_prime(to_h(n), h, rounds);
  rng.state = h.state;
  return r;
}
BigNat random_prime(Rng& rng, size_t bits, int mr_rounds) {
  pcb::HRng h(rng.state);
  BigNat p = from_h(pcb::random_prime(h, bits, mr_rounds));
  rng.state = h.state;
  return p;
}

// ---- keys -----------------------------------------------------------------------------------
KeyPair keygen(Rng& rng, size_t key_bits, GMode gmode) {
  if (key_bits != 64 && key_bits != 1024 && key_bits != 2048 && key_bits != 4096)
    throw std::invalid_argument("key_bits must be 64, 1024, 2048 or 4096");
  const size_t L = key_bits / 32, H = L / 2;
  std::vector<uint32_t> n(L), p(H), q(H);
  u64 st = rng.state;
  check(pcb_keygen(&st, (uint32_t)key_bits, n.data(), p.data(), q.data()), "keygen");
  rng.state = st;
  KeyPair k = finish_binomial(BigNat::from_u32(p.data(), H), BigNat::from_u32(q.data(), H), key_bits);
  if (gmode == GMode::random_g) {
    // the reference seeds the generator search with the stream's last draw, rng.next() at
    // paillier.cpp:120, which pcb_keygen has consumed: its output is the mix of the final state
    pcb::HRng h(st - 0x9e3779b97f4a7c15ull);
    finish_random_g(k, h.next());
  }
  return k;
}

KeyPair keypair_from_primes(const BigNat& p, const BigNat& q, GMode gmode, u64 g_seed) {
  (void)g_seed;
  if (p == q || p < BigNat(2) || q < BigNat(2)) throw std::invalid_argument("need two distinct primes");
  KeyPair k = finish_binomial(p, q, (p * q).bit_length());
  if (gmode == GMode::random_g) finish_random_g(k, g_seed);
  return k;
}

CrtShare crt_share(const KeyPair& k) { return CrtShare{k.crt.p2, k.crt.phi_p2}; }

// Key record: "PB" magic, version 1, the binomial flag, key_bits (u32 BE), then n, p, q as
// (u32 BE byte count, big-endian magnitude); the rest is re-derived (and n == p q checked).
namespace {
void put_u32(std::vector<uint8_t>& o, uint32_t v) {
  for (int s = 24; s >= 0; s -= 8) o.push_back((uint8_t)(v >> s));
}
uint32_t get_u32(const std::vector<uint8_t>& d, size_t& off) {
  if (off + 4 > d.size()) throw std::runtime_error("truncated key record");
  const uint32_t v = ((uint32_t)d[off] << 24) | ((uint32_t)d[off + 1] << 16) | ((uint32_t)d[off + 2] << 8) | d[off + 3];
  off += 4;
  return v;
}
void put_big(std::vector<uint8_t>& o, const BigNat& v) {
  std::vector<uint8_t> b = v.to_bytes_be();
  put_u32(o, (uint32_t)b.size());
  o.insert(o.end(), b.begin(), b.end());
}
BigNat get_big(const std::vector<uint8_t>& d, size_t& off) {
  const uint32_t len = get_u32(d, off);
  if (off + len > d.size()) throw std::runtime_error("truncated key record");
  BigNat v = BigNat::from_bytes_be(d.data() + off, len);
  off += len;
  return v;
}
}  // namespace

std::vector<uint8_t> serialize_keypair(const KeyPair& k) {
  std::vector<uint8_t> o = {'P', 'B', 1, (uint8_t)(k.pub.binomial_g ? 1 : 0)};
  put_u32(o, (uint32_t)k.pub.key_bits);
  put_big(o, k.pub.n);
  put_big(o, k.prv.p);
  put_big(o, k.prv.q);
  if (!k.pub.binomial_g) put_big(o, k.pub.g);
  return o;
}

KeyPair parse_keypair(const std::vector<uint8_t>& d) {
  if (d.size() < 8 || d[0] != 'P' || d[1] != 'B') throw std::runtime_error("not a key record");
  if (d[2] != 1) throw std::runtime_error("unknown key record version");
  if (d[3] > 1) throw std::runtime_error("corrupt key record: generator flag");
  size_t off = 4;
  const uint32_t bits = get_u32(d, off);
  const BigNat n = get_big(d, off), p = get_big(d, off), q = get_big(d, off);
  BigNat g;
  if (d[3] == 0) g = get_big(d, off);
  if (off != d.size()) throw std::runtime_error("trailing bytes in key record");
  if (p * q != n) throw std::runtime_error("corrupt key record: n != p*q");
  KeyPair k = finish_binomial(p, q, bits);
  if (d[3] == 0) {  // the recorded generator: mu from it (paillier.cpp:90-92)
    const HBN hn = to_h(n), hn2 = hn * hn, hg = to_h(g);
    if (hg >= hn2 || pcb::gcd(hg, hn) != HBN(1)) throw std::runtime_error("corrupt key record: g");
    HBN l, r, mu;
    pcb::divmod(pcb::pow_mod(hg, to_h(k.prv.epsilon), hn2) - HBN(1), hn, l, r);
    if (!pcb::mod_inverse(l, hn, mu)) throw std::runtime_error("corrupt key record: g");
    k.pub.g = g;
    k.pub.binomial_g = false;
    k.prv.mu = from_h(mu);
    k.crt.g_p2 = mod(g, k.crt.p2);
    k.crt.g_q2 = mod(g, k.crt.q2);
  }
  return k;
}

// ---- Paillier ---------------------------------------------------------------------------------
Paillier::Paillier(PublicKey pub, Engine engine) : pub_(std::move(pub)), engine_(engine) {
  if (pub_.n.is_zero()) throw std::invalid_argument("empty public key");
  if (pub_.n2.is_zero()) pub_.n2 = pub_.n * pub_.n;
  L_ = (pub_.n.bit_length() + 31) / 32;
  std::vector<uint32_t> n = pub_.n.to_u32(L_);
  pcb_ctx* c = nullptr;
  check(pcb_ctx_create(&c, device_index(), n.data(), (uint32_t)L_, nullptr, nullptr, 0), "context");
  ctx_ = c;
  set_generator();
}

void Paillier::set_generator() {
  if (pub_.binomial_g) return;
  std::vector<uint32_t> g = pub_.g.to_u32(2 * L_);
  check(pcb_ctx_set_generator((pcb_ctx*)ctx_, g.data(), (uint32_t)(2 * L_)), "generator");
}

Paillier::Paillier(const KeyPair& keys, Engine engine)
    : pub_(keys.pub), has_prv_(true), prv_(keys.prv), crt_(keys.crt), engine_(engine) {
  if (pub_.n.is_zero()) throw std::invalid_argument("empty public key");
  if (pub_.n2.is_zero()) pub_.n2 = pub_.n * pub_.n;
  L_ = (pub_.n.bit_length() + 31) / 32;
  const size_t w = std::max((prv_.p.bit_length() + 31) / 32, (prv_.q.bit_length() + 31) / 32);
  std::vector<uint32_t> n = pub_.n.to_u32(L_), p = prv_.p.to_u32(w), q = prv_.q.to_u32(w);
  pcb_ctx* c = nullptr;
  check(pcb_ctx_create(&c, device_index(), n.data(), (uint32_t)L_, p.data(), q.data(), (uint32_t)w), "context");
  ctx_ = c;
  set_generator();
}

Paillier::~Paillier() {
  if (ctx_) pcb_ctx_destroy((pcb_ctx*)ctx_);
}

const PrivateKey& Paillier::prv() const {
  need_private("no private key loaded");
  return prv_;
}
const CrtContext& Paillier::crt() const {
  need_private("no private key loaded");
  return crt_;
}
void Paillier::need_private(const char* what) const {
  if (!has_prv_) throw std::logic_error(what);
}
void Paillier::bump_bits_or_throw(u32 bits) const {  // paillier.cpp:245-251
  if (bits >= pub_.n.bit_length()) throw std::overflow_error("homomorphic accumulation exceeds plaintext space");
}

BigNat Paillier::sample_r(Rng& rng) const {
  std::vector<uint32_t> r(L_);
  u64 st = rng.state;
  check(pcb_sample_r((pcb_ctx*)ctx_, &st, 1, r.data(), nullptr), "sample_r");
  rng.state = st;
  return BigNat::from_u32(r.data(), L_);
}

std::vector<BigNat> Paillier::enc_batch(const std::vector<BigNat>& ms, const std::vector<BigNat>& rs, bool use_crt,
                                        bool count_g) {
  const size_t cnt = ms.size();
  if (cnt == 0) return {};
  if (use_crt) need_private("split encryption needs p and q");
  for (const BigNat& m : ms)  // wider than n: the reference's check_plaintext throws first
    if (m >= pub_.n) throw std::invalid_argument("plaintext not below n");
  for (const BigNat& r : rs)
    if (r.is_zero() || r >= pub_.n) throw std::invalid_argument("randomness not in [1, n)");
  std::vector<uint32_t> m(cnt * L_), r(cnt * L_), c(cnt * 2 * L_);
  for (size_t i = 0; i < cnt; i++) {
    std::vector<uint32_t> a = ms[i].to_u32(L_), b = rs[i].to_u32(L_);
    std::memcpy(&m[i * L_], a.data(), L_ * 4);
    std::memcpy(&r[i * L_], b.data(), L_ * 4);
  }
  std::vector<int32_t> st(cnt);
  // a private context computes the direct form through the CRT halves (same residue,
  // test_paillier.cpp:63-78); a public one runs the n^2 path
  check(pcb_encrypt((pcb_ctx*)ctx_, m.data(), (uint32_t)L_, r.data(), cnt, c.data(), use_crt ? 1 : 0, st.data(),
                    nullptr),
        "encrypt");
  check_elems(st, "encrypt");
  std::vector<BigNat> out(cnt);
  for (size_t i = 0; i < cnt; i++) out[i] = BigNat::from_u32(&c[i * 2 * L_], 2 * L_);
  if (use_crt)
    pow_half_ += 2 * cnt;  // two half_pow per element (paillier.cpp:339-342)
  else
    pow_full_ += cnt;      // r^n mod n^2 (paillier.cpp:325)
  if (count_g && !pub_.binomial_g) {  // g^m: one full power, or one per CRT side (paillier.cpp:253-271)
    if (use_crt)
      pow_half_ += 2 * cnt;
    else
      pow_full_ += cnt;
  }
  return out;
}

std::vector<BigNat> Paillier::dec_batch(const std::vector<Ciphertext>& cs, bool use_crt) {
  need_private("no private key loaded");
  const size_t cnt = cs.size();
  if (cnt == 0) return {};
  for (const Ciphertext& c : cs)
    if (c.value >= pub_.n2) throw std::invalid_argument("ciphertext not below n^2");
  std::vector<uint32_t> c(cnt * 2 * L_), m(cnt * L_);
  for (size_t i = 0; i < cnt; i++) {
    std::vector<uint32_t> a = cs[i].value.to_u32(2 * L_);
    std::memcpy(&c[i * 2 * L_], a.data(), 2 * L_ * 4);
  }
  std::vector<int32_t> st(cnt);
  check(pcb_decrypt((pcb_ctx*)ctx_, c.data(), cnt, m.data(), use_crt ? 1 : 0, st.data(), nullptr), "decrypt");
  check_elems(st, "decrypt");
  std::vector<BigNat> out(cnt);
  for (size_t i = 0; i < cnt; i++) out[i] = BigNat::from_u32(&m[i * L_], L_);
  if (use_crt)
    pow_half_ += 2 * cnt;  // paillier.cpp:357-358
  else
    pow_full_ += cnt;      // paillier.cpp:349
  return out;
}

Ciphertext Paillier::encrypt_with_r(const BigNat& m, const BigNat& r) {
  return Ciphertext{enc_batch({m}, {r}, false)[0], (u32)m.bit_length()};
}
Ciphertext Paillier::crt_encrypt_with_r(const BigNat& m, const BigNat& r) {
  need_private("split encryption needs p and q");
  return Ciphertext{enc_batch({m}, {r}, true)[0], (u32)m.bit_length()};
}
// r is drawn before the argument checks, as paillier.cpp:316-318, 330-332 (the Rng advances
// even when the plaintext is then rejected)
Ciphertext Paillier::encrypt(const BigNat& m, Rng& rng) { return encrypt_with_r(m, sample_r(rng)); }
Ciphertext Paillier::crt_encrypt(const BigNat& m, Rng& rng) { return crt_encrypt_with_r(m, sample_r(rng)); }
BigNat Paillier::decrypt(const Ciphertext& c) { return dec_batch({c}, false)[0]; }
BigNat Paillier::crt_decrypt(const Ciphertext& c) { return dec_batch({c}, true)[0]; }

RnFactor Paillier::make_rn_factor(const BigNat& r) {
  // r^n mod n^2 = Enc(0; r) on the device; the split residues are its reductions mod p^2, q^2
  if (r.is_zero() || r >= pub_.n) throw std::invalid_argument("randomness not in [1, n)");
  RnFactor f;
  f.r = r;
  f.full = enc_batch({BigNat()}, {r}, false, false)[0];
  if (has_prv_) {
    f.half_p2 = mod(f.full, crt_.p2);
    f.half_q2 = mod(f.full, crt_.q2);
    pow_half_ += 2;  // paillier.cpp:378-382
  }
  return f;
}

Ciphertext Paillier::encrypt_with_factor(const BigNat& m, const RnFactor& f) {
  if (f.full.is_zero()) throw std::invalid_argument("factor missing r^n");
  if (m >= pub_.n) throw std::invalid_argument("plaintext not below n");
  std::vector<uint32_t> mm = m.to_u32(L_), rn = f.full.to_u32(2 * L_), c(2 * L_);
  int32_t st = 0;
  check(pcb_encrypt_rn((pcb_ctx*)ctx_, mm.data(), (uint32_t)L_, rn.data(), 1, c.data(), &st, nullptr), "encrypt");
  if (st) throw_status(st, "encrypt");
  if (!pub_.binomial_g) pow_full_ += 1;  // g^m (paillier.cpp:388)
  return Ciphertext{BigNat::from_u32(c.data(), 2 * L_), (u32)m.bit_length()};
}

Ciphertext Paillier::crt_encrypt_with_factor(const BigNat& m, const RnFactor& f) {
  need_private("split encryption needs p and q");
  if (f.half_p2.is_zero() && f.half_q2.is_zero()) throw std::invalid_argument("factor missing split residues");
  Ciphertext c = encrypt_with_factor(m, f);  // the same residue (paillier.cpp:391-400 == 384-389)
  if (!pub_.binomial_g) {  // ledger of the split form: g on both sides (paillier.cpp:397-398)
    pow_full_ -= 1;
    pow_half_ += 2;
  }
  return c;
}

Ciphertext Paillier::finish_split_encrypt(const BigNat& m, const BigNat& p2_g_power, const BigNat& r) {
  need_private("split encryption needs p and q");
  if (m >= pub_.n) throw std::invalid_argument("plaintext not below n");
  if (r.is_zero() || r >= pub_.n) throw std::invalid_argument("randomness not in [1, n)");
  std::vector<uint32_t> mm = m.to_u32(L_), g = mod(p2_g_power, pub_.n2).to_u32(2 * L_), rr = r.to_u32(L_), c(2 * L_);
  int32_t st = 0;
  check(pcb_finish_split_encrypt((pcb_ctx*)ctx_, mm.data(), (uint32_t)L_, g.data(), (uint32_t)(2 * L_), rr.data(), 1,
                                 c.data(), &st, nullptr),
        "finish_split_encrypt");
  if (st) throw_status(st, "finish_split_encrypt");
  pow_half_ += pub_.binomial_g ? 2 : 3;  // both r halves (+ the q-side g power, paillier.cpp:410-413)
  return Ciphertext{BigNat::from_u32(c.data(), 2 * L_), (u32)m.bit_length()};
}

Ciphertext Paillier::finish_split_encrypt_with_factor(const BigNat& m, const BigNat& p2_g_power, const RnFactor& f) {
  if (f.half_p2.is_zero() && f.half_q2.is_zero()) throw std::invalid_argument("factor missing split residues");
  need_private("split encryption needs p and q");
  if (f.full.is_zero()) {  // a factor carrying only its halves: recompute from r
    Ciphertext c = finish_split_encrypt(m, p2_g_power, f.r);
    pow_half_ -= 2;  // the factor's r^n halves are reused (paillier.cpp:416-426)
    return c;
  }
  if (m >= pub_.n) throw std::invalid_argument("plaintext not below n");
  std::vector<uint32_t> mm = m.to_u32(L_), g = mod(p2_g_power, pub_.n2).to_u32(2 * L_), rn = f.full.to_u32(2 * L_),
                        c(2 * L_);
  int32_t st = 0;
  check(pcb_finish_split_encrypt_rn((pcb_ctx*)ctx_, mm.data(), (uint32_t)L_, g.data(), (uint32_t)(2 * L_), rn.data(), 1,
                                    c.data(), &st, nullptr),
        "finish_split_encrypt_with_factor");
  if (st) throw_status(st, "finish_split_encrypt_with_factor");
  if (!pub_.binomial_g) pow_half_ += 1;  // the q-side g power (paillier.cpp:424)
  return Ciphertext{BigNat::from_u32(c.data(), 2 * L_), (u32)m.bit_length()};
}

BigNat Paillier::decrypt_with_half(const Ciphertext& c, const BigNat& p2_power) {
  need_private("no private key loaded");
  if (c.value >= pub_.n2) throw std::invalid_argument("ciphertext not below n^2");
  std::vector<uint32_t> cc = c.value.to_u32(2 * L_), pw = mod(p2_power, pub_.n2).to_u32(2 * L_), m(L_);
  int32_t st = 0;
  check(pcb_decrypt_with_half((pcb_ctx*)ctx_, cc.data(), pw.data(), (uint32_t)(2 * L_), 1, m.data(), &st, nullptr),
        "decrypt_with_half");
  if (st) throw_status(st, "decrypt_with_half");
  pow_half_ += 1;
  return BigNat::from_u32(m.data(), L_);
}

Ciphertext Paillier::hom_add(const Ciphertext& a, const Ciphertext& b) {
  const u32 bits = std::max(a.plain_bits, b.plain_bits) + 1;
  bump_bits_or_throw(bits);
  std::vector<uint32_t> x = a.value.to_u32(2 * L_), y = b.value.to_u32(2 * L_), o(2 * L_);
  check(pcb_hom_add((pcb_ctx*)ctx_, x.data(), y.data(), 1, o.data(), nullptr), "hom_add");
  return Ciphertext{BigNat::from_u32(o.data(), 2 * L_), bits};
}

Ciphertext Paillier::hom_scalar_mul(const BigNat& k, const Ciphertext& c) {
  const u32 bits = k.is_zero() ? 0 : c.plain_bits + (u32)k.bit_length();
  bump_bits_or_throw(bits);
  if (k.bit_length() > 64) throw std::invalid_argument("hom_scalar_mul: scalars are at most 64 bits on the B200 path");
  const u64 kk = k.is_zero() ? 0 : k.to_u64();
  std::vector<uint32_t> x = c.value.to_u32(2 * L_), o(2 * L_);
  check(pcb_hom_scalar_mul((pcb_ctx*)ctx_, &kk, x.data(), 1, o.data(), nullptr), "hom_scalar_mul");
  pow_full_ += 1;
  return Ciphertext{BigNat::from_u32(o.data(), 2 * L_), bits};
}

std::vector<Ciphertext> Paillier::hom_matvec(const std::vector<Ciphertext>& alpha,
                                             const std::vector<std::vector<u64>>& expo,
                                             const std::vector<Ciphertext>& zv, unsigned window) {
  const size_t rows = alpha.size(), cols = zv.size();
  if (expo.size() != rows) throw std::invalid_argument("exponent row count");
  for (const auto& row : expo)
    if (row.size() != cols) throw std::invalid_argument("exponent row width");
  if (window < 1 || window > 8) throw std::invalid_argument("window in [1,8]");
  // plain_bits exactly as paillier.cpp:453-489
  u32 kbits = 0, zbits = 0;
  for (const auto& row : expo)
    for (u64 k : row) kbits = std::max(kbits, (u32)(k ? 64 - __builtin_clzll(k) : 0));
  for (const auto& c : zv) zbits = std::max(zbits, c.plain_bits);
  const u32 sum_bits = cols ? kbits + zbits + (u32)(64 - __builtin_clzll((u64)cols)) : 0;
  std::vector<Ciphertext> out(rows);
  if (rows == 0) return out;
  for (size_t i = 0; i < rows; i++) bump_bits_or_throw(std::max(alpha[i].plain_bits, sum_bits) + 1);
  const size_t W = 2 * L_;
  std::vector<uint32_t> a(rows * W), z(std::max<size_t>(cols, 1) * W), o(rows * W);
  std::vector<u64> e(rows * std::max<size_t>(cols, 1));
  for (size_t i = 0; i < rows; i++) {
    std::vector<uint32_t> t = alpha[i].value.to_u32(W);
    std::memcpy(&a[i * W], t.data(), W * 4);
    for (size_t j = 0; j < cols; j++) e[i * cols + j] = expo[i][j];
  }
  for (size_t j = 0; j < cols; j++) {
    std::vector<uint32_t> t = zv[j].value.to_u32(W);
    std::memcpy(&z[j * W], t.data(), W * 4);
  }
  check(pcb_hom_matvec((pcb_ctx*)ctx_, a.data(), e.data(), z.data(), rows, cols, window, o.data(), nullptr),
        "hom_matvec");
  for (size_t i = 0; i < rows; i++)
    out[i] = Ciphertext{BigNat::from_u32(&o[i * W], W), std::max(alpha[i].plain_bits, sum_bits) + 1};
  pow_full_ += rows;  // paillier.cpp:476
  return out;
}

std::vector<Ciphertext> Paillier::encrypt_vec(const std::vector<BigNat>& ms, Rng& rng, bool use_crt) {
  if (use_crt) need_private("split encryption needs p and q");
  const size_t cnt = ms.size();
  if (cnt == 0) return {};
  // the serial r draw of paillier.cpp:497-500, as one device batch (same stream, same state)
  std::vector<uint32_t> r(cnt * L_);
  u64 st = rng.state;
  check(pcb_sample_r((pcb_ctx*)ctx_, &st, cnt, r.data(), nullptr), "sample_r");
  rng.state = st;
  std::vector<BigNat> rs(cnt);
  for (size_t i = 0; i < cnt; i++) rs[i] = BigNat::from_u32(&r[i * L_], L_);
  std::vector<BigNat> cs = enc_batch(ms, rs, use_crt);
  std::vector<Ciphertext> out(cnt);
  for (size_t i = 0; i < cnt; i++) out[i] = Ciphertext{cs[i], (u32)ms[i].bit_length()};
  return out;
}

std::vector<BigNat> Paillier::decrypt_vec(const std::vector<Ciphertext>& cs, bool use_crt) {
  return dec_batch(cs, use_crt);
}

}  // namespace pcadmm
