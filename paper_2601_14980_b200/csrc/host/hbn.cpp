// hbn.cpp — host big naturals (see hbn.hpp).  One-time key work only.
#include "hbn.hpp"

#include <algorithm>
#include <stdexcept>

namespace pcb {

HBN::HBN(uint64_t v) {
  if (v) {
    w.push_back((uint32_t)v);
    if (v >> 32) w.push_back((uint32_t)(v >> 32));
  }
}

void HBN::normalize() {
  while (!w.empty() && w.back() == 0) w.pop_back();
}

HBN HBN::from_limbs(const uint32_t* p, size_t n) {
  HBN r;
  r.w.assign(p, p + n);
  r.normalize();
  return r;
}

HBN HBN::from_u64_limbs(const std::vector<uint64_t>& l) {
  HBN r;
  r.w.resize(2 * l.size());
  for (size_t i = 0; i < l.size(); i++) {
    r.w[2 * i] = (uint32_t)l[i];
    r.w[2 * i + 1] = (uint32_t)(l[i] >> 32);
  }
  r.normalize();
  return r;
}

void HBN::to_limbs(uint32_t* out, size_t n) const {
  for (size_t i = 0; i < n; i++) out[i] = i < w.size() ? w[i] : 0u;
}

std::vector<uint32_t> HBN::limbs(size_t n) const {
  std::vector<uint32_t> v(n);
  to_limbs(v.data(), n);
  return v;
}

size_t HBN::bit_length() const {
  if (w.empty()) return 0;
  return 32 * (w.size() - 1) + (32 - __builtin_clz(w.back()));
}

bool HBN::bit(size_t i) const {
  size_t k = i / 32;
  return k < w.size() && ((w[k] >> (i % 32)) & 1u);
}

uint64_t HBN::low64() const {
  uint64_t v = 0;
  if (w.size() > 0) v = w[0];
  if (w.size() > 1) v |= (uint64_t)w[1] << 32;
  return v;
}

std::string HBN::to_hex() const {
  if (w.empty()) return "0";
  static const char* d = "0123456789abcdef";
  std::string s;
  for (size_t i = w.size(); i-- > 0;)
    for (int b = 28; b >= 0; b -= 4) s.push_back(d[(w[i] >> b) & 15]);
  size_t nz = s.find_first_not_of('0');
  return s.substr(nz);
}

int cmp(const HBN& a, const HBN& b) {
  if (a.w.size() != b.w.size()) return a.w.size() < b.w.size() ? -1 : 1;
  for (size_t i = a.w.size(); i-- > 0;)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

HBN operator+(const HBN& a, const HBN& b) {
  HBN r;
  size_t n = std::max(a.w.size(), b.w.size());
  r.w.resize(n + 1);
  uint64_t c = 0;
  for (size_t i = 0; i < n; i++) {
    c += (uint64_t)(i < a.w.size() ? a.w[i] : 0) + (i < b.w.size() ? b.w[i] : 0);
    r.w[i] = (uint32_t)c;
    c >>= 32;
  }
  r.w[n] = (uint32_t)c;
  r.normalize();
  return r;
}

HBN operator-(const HBN& a, const HBN& b) {
  if (cmp(a, b) < 0) throw std::underflow_error("HBN subtraction underflow");
  HBN r;
  r.w.resize(a.w.size());
  int64_t br = 0;
  for (size_t i = 0; i < a.w.size(); i++) {
    int64_t d = (int64_t)a.w[i] - (i < b.w.size() ? b.w[i] : 0) - br;
    br = d < 0;
    r.w[i] = (uint32_t)(d + (br ? (int64_t)1 << 32 : 0));
  }
  r.normalize();
  return r;
}

HBN operator*(const HBN& a, const HBN& b) {
  if (a.is_zero() || b.is_zero()) return HBN();
  HBN r;
  r.w.assign(a.w.size() + b.w.size(), 0);
  for (size_t i = 0; i < a.w.size(); i++) {
    uint64_t c = 0;
    for (size_t j = 0; j < b.w.size(); j++) {
      c += (uint64_t)a.w[i] * b.w[j] + r.w[i + j];
      r.w[i + j] = (uint32_t)c;
      c >>= 32;
    }
    r.w[i + b.w.size()] = (uint32_t)c;
  }
  r.normalize();
  return r;
}

HBN operator<<(const HBN& a, size_t bits) {
  if (a.is_zero()) return HBN();
  size_t k = bits / 32, s = bits % 32;
  HBN r;
  r.w.assign(a.w.size() + k + 1, 0);
  for (size_t i = 0; i < a.w.size(); i++) {
    r.w[i + k] |= a.w[i] << s;
    if (s) r.w[i + k + 1] |= a.w[i] >> (32 - s);
  }
  r.normalize();
  return r;
}

HBN operator>>(const HBN& a, size_t bits) {
  size_t k = bits / 32, s = bits % 32;
  if (k >= a.w.size()) return HBN();
  HBN r;
  r.w.assign(a.w.size() - k, 0);
  for (size_t i = 0; i < r.w.size(); i++) {
    r.w[i] = a.w[i + k] >> s;
    if (s && i + k + 1 < a.w.size()) r.w[i] |= a.w[i + k + 1] << (32 - s);
  }
  r.normalize();
  return r;
}

// Knuth algorithm D on 32-bit limbs.
void divmod(const HBN& a, const HBN& b, HBN& q, HBN& r) {
  if (b.is_zero()) throw std::domain_error("HBN division by zero");
  if (cmp(a, b) < 0) {
    q = HBN();
    r = a;
    return;
  }
  if (b.w.size() == 1) {
    uint64_t d = b.w[0], rem = 0;
    HBN qq;
    qq.w.resize(a.w.size());
    for (size_t i = a.w.size(); i-- > 0;) {
      uint64_t cur = (rem << 32) | a.w[i];
      qq.w[i] = (uint32_t)(cur / d);
      rem = cur % d;
    }
    qq.normalize();
    q = qq;
    r = HBN(rem);
    return;
  }
  int sh = __builtin_clz(b.w.back());
  HBN u = a << sh, v = b << sh;
  size_t n = v.w.size(), m = u.w.size() - n;
  std::vector<uint32_t> un(u.w);
  un.push_back(0);
  const std::vector<uint32_t>& vn = v.w;
  std::vector<uint32_t> qv(m + 1, 0);
  for (size_t j = m + 1; j-- > 0;) {
    uint64_t top = ((uint64_t)un[j + n] << 32) | un[j + n - 1];
    uint64_t qhat = top / vn[n - 1], rhat = top % vn[n - 1];
    while (qhat >= (1ull << 32) || qhat * vn[n - 2] > ((rhat << 32) | un[j + n - 2])) {
      qhat--;
      rhat += vn[n - 1];
      if (rhat >= (1ull << 32)) break;
    }
    int64_t borrow = 0;
    uint64_t carry = 0;
    for (size_t i = 0; i < n; i++) {
      uint64_t p = qhat * vn[i] + carry;
      carry = p >> 32;
      int64_t t = (int64_t)un[i + j] - (int64_t)(uint32_t)p - borrow;
      un[i + j] = (uint32_t)t;
      borrow = t < 0;
    }
    int64_t t = (int64_t)un[j + n] - (int64_t)carry - borrow;
    un[j + n] = (uint32_t)t;
    if (t < 0) {
      qhat--;
      uint64_t c = 0;
      for (size_t i = 0; i < n; i++) {
        c += (uint64_t)un[i + j] + vn[i];
        un[i + j] = (uint32_t)c;
        c >>= 32;
      }
      un[j + n] += (uint32_t)c;
    }
    qv[j] = (uint32_t)qhat;
  }
  un.resize(n);
  HBN rr;
  rr.w = un;
  rr.normalize();
  r = rr >> sh;
  q.w = qv;
  q.normalize();
}

HBN mod(const HBN& a, const HBN& m) {
  HBN q, r;
  divmod(a, m, q, r);
  return r;
}

HBN gcd(HBN a, HBN b) {
  while (!b.is_zero()) {
    HBN r = mod(a, b);
    a = b;
    b = r;
  }
  return a;
}

HBN lcm(const HBN& a, const HBN& b) {
  if (a.is_zero() || b.is_zero()) return HBN();
  HBN q, r;
  divmod(a * b, gcd(a, b), q, r);
  return q;
}

bool mod_inverse(const HBN& a, const HBN& m, HBN& out) {
  HBN r0 = m, r1 = mod(a, m), t0, t1(1);
  bool n0 = false, n1 = false;
  while (!r1.is_zero()) {
    HBN qt, rm;
    divmod(r0, r1, qt, rm);
    HBN qt1 = qt * t1, t2;
    bool n2;
    if (n0 == n1) {
      if (cmp(t0, qt1) >= 0) {
        t2 = t0 - qt1;
        n2 = n0;
      } else {
        t2 = qt1 - t0;
        n2 = !n0;
      }
    } else {
      t2 = t0 + qt1;
      n2 = n0;
    }
    r0 = r1;
    r1 = rm;
    t0 = t1;
    n0 = n1;
    t1 = t2;
    n1 = n2;
  }
  if (!(r0 == HBN(1))) return false;
  out = n0 ? m - mod(t0, m) : mod(t0, m);
  return true;
}

namespace {
// Host Montgomery context for odd moduli (keygen's Miller-Rabin is the only heavy host user).
struct HMont {
  std::vector<uint32_t> m;
  uint32_t minv = 0;
  size_t s = 0;
  explicit HMont(const HBN& mod) : m(mod.w), s(mod.w.size()) {
    uint32_t inv = 1;
    for (int i = 0; i < 5; i++) inv *= 2u - m[0] * inv;
    minv = (uint32_t)(0u - inv);
  }
  // t = a*b*R^-1 mod m  (a, b < m, s limbs)
  void mul(const uint32_t* a, const uint32_t* b, uint32_t* out) const {
    std::vector<uint32_t> t(s + 2, 0);
    for (size_t i = 0; i < s; i++) {
      uint64_t c = 0;
      for (size_t j = 0; j < s; j++) {
        c += (uint64_t)a[j] * b[i] + t[j];
        t[j] = (uint32_t)c;
        c >>= 32;
      }
      c += t[s];
      t[s] = (uint32_t)c;
      t[s + 1] = (uint32_t)(c >> 32);
      uint32_t q = t[0] * minv;
      c = ((uint64_t)q * m[0] + t[0]) >> 32;
      for (size_t j = 1; j < s; j++) {
        c += (uint64_t)q * m[j] + t[j];
        t[j - 1] = (uint32_t)c;
        c >>= 32;
      }
      c += t[s];
      t[s - 1] = (uint32_t)c;
      t[s] = t[s + 1] + (uint32_t)(c >> 32);
      t[s + 1] = 0;
    }
    bool ge = t[s] != 0;
    if (!ge) {
      ge = true;
      for (size_t j = s; j-- > 0;)
        if (t[j] != m[j]) {
          ge = t[j] > m[j];
          break;
        }
    }
    if (ge) {
      int64_t br = 0;
      for (size_t j = 0; j < s; j++) {
        int64_t d = (int64_t)t[j] - m[j] - br;
        br = d < 0;
        t[j] = (uint32_t)d;
      }
    }
    for (size_t j = 0; j < s; j++) out[j] = t[j];
  }
};
}  // namespace

HBN pow_mod(const HBN& b, const HBN& e, const HBN& m) {
  if (m == HBN(1)) return HBN();
  if (e.is_zero()) return HBN(1);
  if (!m.is_odd()) {  // plain square-and-multiply (rare: only tests)
    HBN acc(1), base = mod(b, m);
    for (size_t i = e.bit_length(); i-- > 0;) {
      acc = mod(acc * acc, m);
      if (e.bit(i)) acc = mod(acc * base, m);
    }
    return acc;
  }
  HMont ctx(m);
  size_t s = ctx.s;
  HBN R2 = mod(HBN(1) << (64 * s), m);
  std::vector<uint32_t> r2 = R2.limbs(s), x = mod(b, m).limbs(s);
  std::vector<std::vector<uint32_t>> tab(16, std::vector<uint32_t>(s));
  std::vector<uint32_t> one(s, 0);
  one[0] = 1;
  ctx.mul(x.data(), r2.data(), tab[1].data());
  ctx.mul(one.data(), r2.data(), tab[0].data());
  for (int i = 2; i < 16; i++) ctx.mul(tab[i - 1].data(), tab[1].data(), tab[i].data());
  std::vector<uint32_t> acc = tab[0], tmp(s);
  size_t nb = e.bit_length(), nwin = (nb + 3) / 4;
  for (size_t wdx = nwin; wdx-- > 0;) {
    if (wdx != nwin - 1)
      for (int k = 0; k < 4; k++) {
        ctx.mul(acc.data(), acc.data(), tmp.data());
        acc.swap(tmp);
      }
    unsigned d = 0;
    for (int k = 0; k < 4; k++)
      if (e.bit(wdx * 4 + k)) d |= 1u << k;
    if (d) {
      ctx.mul(acc.data(), tab[d].data(), tmp.data());
      acc.swap(tmp);
    }
  }
  ctx.mul(acc.data(), one.data(), tmp.data());
  return HBN::from_limbs(tmp.data(), s);
}

HBN random_bits(HRng& rng, size_t bits) {
  std::vector<uint64_t> l((bits + 63) / 64);
  for (auto& x : l) x = rng.next();
  if (bits % 64) l.back() &= ~0ull >> (64 - bits % 64);
  return HBN::from_u64_limbs(l);
}

HBN random_below(HRng& rng, const HBN& bound) {
  if (bound.is_zero()) throw std::domain_error("random_below: zero bound");
  size_t bits = bound.bit_length();
  for (;;) {
    HBN v = random_bits(rng, bits);
    if (cmp(v, bound) < 0) return v;
  }
}

namespace {
const uint32_t kSmallPrimes[] = {
    3,   5,   7,   11,  13,  17,  19,  23,  29,  31,  37,  41,  43,  47,  53,  59,  61,  67,
    71,  73,  79,  83,  89,  97,  101, 103, 107, 109, 113, 127, 131, 137, 139, 149, 151, 157,
    163, 167, 173, 179, 181, 191, 193, 197, 199, 211, 223, 227, 229, 233, 239, 241, 251, 257,
    263, 269, 271, 277, 281, 283, 293, 307, 311, 313, 317, 331, 337, 347, 349, 353, 359, 367,
    373, 379, 383, 389, 397, 401, 409, 419, 421, 431, 433, 439, 443, 449, 457, 461, 463, 467,
    479, 487, 491, 499, 503, 509, 521, 523, 541};

uint32_t mod_small(const HBN& n, uint32_t d) {
  uint64_t r = 0;
  for (size_t i = n.w.size(); i-- > 0;) r = ((r << 32) | n.w[i]) % d;
  return (uint32_t)r;
}
}  // namespace

bool is_probable_prime(const HBN& n, HRng& rng, int rounds) {
  if (n.bit_length() <= 6) {
    uint64_t v = n.low64();
    if (v < 2) return false;
    for (uint64_t d = 2; d * d <= v; d++)
      if (v % d == 0) return false;
    return true;
  }
  if (!n.is_odd()) return false;
  for (uint32_t p : kSmallPrimes)
    if (mod_small(n, p) == 0) return n == HBN(p);
  HBN nm1 = n - HBN(1);
  size_t s = 0;
  HBN d = nm1;
  while (!d.is_odd()) {
    d = d >> 1;
    s++;
  }
  HBN three(3), two(2);
  for (int r = 0; r < rounds; r++) {
    HBN a = random_below(rng, n - three) + two;
    HBN x = pow_mod(a, d, n);
    if (x == HBN(1) || x == nm1) continue;
    bool witness = true;
    for (size_t i = 0; i + 1 < s; i++) {
      x = mod(x * x, n);
      if (x == nm1) {
        witness = false;
        break;
      }
    }
    if (witness) return false;
  }
  return true;
}

HBN random_prime(HRng& rng, size_t bits, int mr_rounds) {
  if (bits < 2) throw std::domain_error("random_prime: need >= 2 bits");
  for (;;) {
    HBN cand = random_bits(rng, bits);
    std::vector<uint32_t> l = cand.limbs((bits + 63) / 64 * 2);
    l[(bits - 1) / 32] |= 1u << ((bits - 1) % 32);
    l[0] |= 1u;
    cand = HBN::from_limbs(l.data(), l.size());
    for (int step = 0; step < 64; step++) {
      if (is_probable_prime(cand, rng, mr_rounds)) return cand;
      cand = cand + HBN(2);
      if (cand.bit_length() != bits) break;
    }
  }
}

namespace {
// trial division exactly as is_probable_prime's prefix (bignat.cpp:471-473) for n > 6 bits:
// false = composite (n is never one of the small primes at these widths)
bool survives_trial_division(const HBN& n) {
  for (uint32_t p : kSmallPrimes)
    if (mod_small(n, p) == 0) return n == HBN(p);
  return true;
}
// the witness loop of one round given x = a^d mod n (bignat.cpp:483-493): true = n passes
bool round_passes(HBN x, const HBN& n, size_t s) {
  const HBN nm1 = n - HBN(1);
  if (x == HBN(1) || x == nm1) return true;
  for (size_t i = 0; i + 1 < s; i++) {
    x = mod(x * x, n);
    if (x == nm1) return true;
  }
  return false;
}
struct Spec {
  size_t march, step;  // which candidate
  HBN n, d;
  size_t s;
  HRng after;  // stream state right after this survivor's first base draw
};
}  // namespace

bool random_prime_batched(HRng& rng, size_t bits, int mr_rounds, int lookahead, MrPow pow, void* user, HBN& out) {
  if (bits < 2) throw std::domain_error("random_prime: need >= 2 bits");
  if (bits <= 64 || mr_rounds <= 0) {  // tiny widths / no rounds: nothing worth batching
    out = random_prime(rng, bits, mr_rounds);
    return true;
  }
  const HBN three(3), two(2);
  // a march = the candidates of one random_bits draw (random_prime's inner loop)
  auto march_of = [&](HRng& r) {
    HBN cand = random_bits(r, bits);
    std::vector<uint32_t> l = cand.limbs((bits + 63) / 64 * 2);
    l[(bits - 1) / 32] |= 1u << ((bits - 1) % 32);
    l[0] |= 1u;
    cand = HBN::from_limbs(l.data(), l.size());
    std::vector<HBN> cs;
    for (int step = 0; step < 64; step++) {
      cs.push_back(cand);
      cand = cand + HBN(2);
      if (cand.bit_length() != bits) break;
    }
    return cs;
  };
  std::vector<HBN> pending;  // the committed march still being examined
  size_t pending_from = 0;
  for (;;) {
    HRng r = rng;
    std::vector<std::vector<HBN>> marches;
    std::vector<Spec> sp;
    MrBatch b1;
    auto emit = [&](size_t m, size_t from) {
      for (size_t j = from; j < marches[m].size(); j++) {
        const HBN& n = marches[m][j];
        if (!survives_trial_division(n)) continue;
        Spec x{m, j, n, n - HBN(1), 0, r};
        while (!x.d.is_odd()) {
          x.d = x.d >> 1;
          x.s++;
        }
        b1.a.push_back(random_below(r, n - three) + two);
        b1.n.push_back(n);
        b1.d.push_back(x.d);
        x.after = r;
        sp.push_back(std::move(x));
      }
    };
    if (!pending.empty()) {
      marches.push_back(pending);
      emit(0, pending_from);
    }
    for (int m = 0; m < lookahead; m++) {
      marches.push_back(march_of(r));
      emit(marches.size() - 1, 0);
    }
    std::vector<HBN> x1;
    if (!b1.n.empty() && !pow(b1, x1, user)) return false;
    size_t k = 0;
    while (k < sp.size() && !round_passes(x1[k], sp[k].n, sp[k].s)) k++;
    if (k == sp.size()) {  // every survivor fails its first round: all of it is committed
      rng = r;
      pending.clear();
      continue;
    }
    // committed up to survivor k's first base draw; rounds 2.. of its candidate in one batch
    rng = sp[k].after;
    HRng r2 = rng;
    MrBatch b2;
    std::vector<HRng> snap;
    for (int t = 1; t < mr_rounds; t++) {
      b2.a.push_back(random_below(r2, sp[k].n - three) + two);
      b2.n.push_back(sp[k].n);
      b2.d.push_back(sp[k].d);
      snap.push_back(r2);
    }
    std::vector<HBN> x2;
    if (!b2.n.empty() && !pow(b2, x2, user)) return false;
    size_t t = 0;
    while (t < b2.n.size() && round_passes(x2[t], sp[k].n, sp[k].s)) t++;
    if (t == b2.n.size()) {
      if (!snap.empty()) rng = snap.back();
      out = sp[k].n;
      return true;
    }
    rng = snap[t];  // composite at round t + 2: continue its march after it
    pending = marches[sp[k].march];
    pending_from = sp[k].step + 1;
  }
}

bool keygen_batched(HRng& rng, size_t key_bits, MrPow pow, void* user, HBN& p, HBN& q) {
  if (key_bits != 64 && key_bits != 1024 && key_bits != 2048 && key_bits != 4096) return false;
  size_t half = key_bits / 2;
  for (int attempt = 0; attempt < 64; attempt++) {  // keygen's loop, paillier.cpp:110-121
    HBN pp, qq;
    if (!random_prime_batched(rng, half, 40, 16, pow, user, pp)) return false;
    if (!random_prime_batched(rng, half, 40, 16, pow, user, qq)) return false;
    if (pp == qq) continue;
    HBN diff = pp > qq ? pp - qq : qq - pp;
    if (diff.bit_length() < half - 7) continue;
    if ((pp * qq).bit_length() != key_bits) continue;
    (void)rng.next();  // finish_keys' g_seed draw (paillier.cpp:120)
    p = pp;
    q = qq;
    return true;
  }
  throw std::runtime_error("key generation attempt budget exhausted");
}

bool keygen(HRng& rng, size_t key_bits, HBN& p, HBN& q) {
  if (key_bits != 64 && key_bits != 1024 && key_bits != 2048 && key_bits != 4096) return false;
  size_t half = key_bits / 2;
  for (int attempt = 0; attempt < 64; attempt++) {
    HBN pp = random_prime(rng, half);
    HBN qq = random_prime(rng, half);
    if (pp == qq) continue;
    HBN diff = pp > qq ? pp - qq : qq - pp;
    if (diff.bit_length() < half - 7) continue;
    if ((pp * qq).bit_length() != key_bits) continue;
    (void)rng.next();  // finish_keys(p, q, gmode, rng.next(), key_bits) — paillier.cpp:120
    p = pp;
    q = qq;
    return true;
  }
  throw std::runtime_error("key generation attempt budget exhausted");
}

}  // namespace pcb
