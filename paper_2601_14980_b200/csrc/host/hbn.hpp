// hbn.hpp — host big naturals for one-time key work (keygen, Montgomery constants, CRT
// factors, exponent schedules).  Not on the batched hot path: every per-element operation runs
// on the GPU.  Little-endian u32 limbs, canonical (no high zero limbs; zero = empty).
//
// Mirrors the semantics of the reference's BigNat (/root/reference/proj/include/pcadmm/
// bignat.hpp:19-61) where keygen bit-exactness needs it (random_bits, random_below,
// random_prime, is_probable_prime consume the splitmix64 stream exactly like bignat.cpp:388-515).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace pcb {

class HBN {
 public:
  std::vector<uint32_t> w;  // LE limbs, normalised

  HBN() = default;
  explicit HBN(uint64_t v);
  static HBN from_limbs(const uint32_t* p, size_t n);
  static HBN from_u64_limbs(const std::vector<uint64_t>& l);
  void to_limbs(uint32_t* out, size_t n) const;  // zero-padded; caller ensures it fits
  std::vector<uint32_t> limbs(size_t n) const;

  bool is_zero() const { return w.empty(); }
  bool is_odd() const { return !w.empty() && (w[0] & 1u); }
  size_t bit_length() const;
  bool bit(size_t i) const;
  uint64_t low64() const;
  std::string to_hex() const;

  void normalize();
};

int cmp(const HBN& a, const HBN& b);
inline bool operator==(const HBN& a, const HBN& b) { return a.w == b.w; }
inline bool operator!=(const HBN& a, const HBN& b) { return a.w != b.w; }
inline bool operator<(const HBN& a, const HBN& b) { return cmp(a, b) < 0; }
inline bool operator<=(const HBN& a, const HBN& b) { return cmp(a, b) <= 0; }
inline bool operator>(const HBN& a, const HBN& b) { return cmp(a, b) > 0; }
inline bool operator>=(const HBN& a, const HBN& b) { return cmp(a, b) >= 0; }
HBN operator+(const HBN& a, const HBN& b);
HBN operator-(const HBN& a, const HBN& b);  // requires a >= b
HBN operator*(const HBN& a, const HBN& b);
HBN operator<<(const HBN& a, size_t bits);
HBN operator>>(const HBN& a, size_t bits);

void divmod(const HBN& a, const HBN& b, HBN& q, HBN& r);  // throws on b == 0
HBN mod(const HBN& a, const HBN& m);
HBN gcd(HBN a, HBN b);
HBN lcm(const HBN& a, const HBN& b);
bool mod_inverse(const HBN& a, const HBN& m, HBN& out);  // false if gcd != 1
HBN pow_mod(const HBN& b, const HBN& e, const HBN& m);   // host Montgomery (odd m) / plain

// splitmix64 — identical stream to pcadmm::Rng (bignat.cpp:388-394)
struct HRng {
  uint64_t state;
  explicit HRng(uint64_t s) : state(s) {}
  uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
};

HBN random_bits(HRng& rng, size_t bits);            // bignat.cpp:431-436
HBN random_below(HRng& rng, const HBN& bound);      // bignat.cpp:438-445
bool is_probable_prime(const HBN& n, HRng& rng, int rounds = 40);  // bignat.cpp:458-495
HBN random_prime(HRng& rng, size_t bits, int mr_rounds = 40);     // bignat.cpp:497-515

// Batched Miller-Rabin: x_i = a_i ^ d_i mod n_i for a batch of (odd) moduli -- the device
// evaluates it (prime.cu); the CPU tests plug pow_mod in.
struct MrBatch {
  std::vector<HBN> n, d, a;
};
using MrPow = bool (*)(const MrBatch& b, std::vector<HBN>& x, void* user);
// random_prime with the Miller-Rabin rounds evaluated in batches, consuming the rng EXACTLY like
// random_prime (so the primes, and the rng state after, are the reference's).  Speculation: every
// trial-division survivor of the next `lookahead` marches is assumed to fail its first round (the
// base draws are then fixed by the stream), all first rounds run as one batch, and the prefix up
// to the first survivor that passes is committed; its remaining rounds run as a second batch,
// rewinding the stream to the first failing round if it turns out composite.  Returns false if
// `pow` fails.
bool random_prime_batched(HRng& rng, size_t bits, int mr_rounds, int lookahead, MrPow pow, void* user, HBN& out);
bool keygen_batched(HRng& rng, size_t key_bits, MrPow pow, void* user, HBN& p, HBN& q);
// keygen restated (paillier.cpp:106-123, binomial g): returns false on an unsupported size.
// Consumes the rng exactly like the reference (including finish_keys' g_seed draw).
bool keygen(HRng& rng, size_t key_bits, HBN& p, HBN& q);

}  // namespace pcb
