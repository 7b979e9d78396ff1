"""CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the GPU path.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs may import it; the product
(paper_2601_14980_b200) never does.  Python ints carry the big-integer arithmetic (any exact
algorithm gives the same residues); Python floats are IEEE binary64 with the reference's operation
order, so the quantizers are bit-exact with the x86-64 reference build (no FMA contraction there).

Pinned against: the compiled reference (oracle/_ref/libpcref.so, built from /root/reference by
oracle/Makefile) through the committed golden vectors in tests/golden/ (oracle/gen_golden.py),
and the reference's own known-answer tests restated in tests/test_oracle_golden.py
(toy key p=5, q=7 from test_paillier.cpp:27-61; pow_mod KATs test_bignat.cpp:178-180;
Gamma KATs test_quantize.cpp:11-34).

Every function cites the reference file:line it restates (paths under /root/reference/proj).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


# --------------------------------------------------------------------------------------------
# splitmix64 Rng — bignat.hpp:107-114, bignat.cpp:388-412
# --------------------------------------------------------------------------------------------
class Rng:
    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:  # bignat.cpp:388-394
        self.state = (self.state + GAMMA) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def below(self, bound: int) -> int:  # bignat.cpp:396-404
        if bound <= 1:
            return 0
        mask = MASK64 >> (64 - (bound - 1).bit_length()) if bound > 1 else 0
        while True:
            v = self.next() & mask
            if v < bound:
                return v

    def unit(self) -> float:  # bignat.cpp:406
        return float(self.next() >> 11) * (2.0 ** -53)

    def gaussian(self) -> float:  # bignat.cpp:408-412
        u1, u2 = self.unit(), self.unit()
        while u1 <= 0:
            u1 = self.unit()
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586477 * u2)


def random_bits(rng: Rng, bits: int) -> int:  # bignat.cpp:431-436
    words = (bits + 63) // 64
    v = 0
    for i in range(words):
        w = rng.next()
        if i == words - 1 and bits % 64:
            w &= MASK64 >> (64 - bits % 64)
        v |= w << (64 * i)
    return v


def random_below(rng: Rng, bound: int) -> int:  # bignat.cpp:438-445
    if bound == 0:
        raise ValueError("random_below: zero bound")
    bits = bound.bit_length()
    while True:
        v = random_bits(rng, bits)
        if v < bound:
            return v


SMALL_PRIMES = [p for p in range(3, 542) if all(p % d for d in range(2, int(p ** 0.5) + 1))]  # bignat.cpp:448-455


def is_probable_prime(n: int, rng: Rng, rounds: int = 40) -> bool:  # bignat.cpp:458-495
    if n.bit_length() <= 6:
        if n < 2:
            return False
        d = 2
        while d * d <= n:
            if n % d == 0:
                return False
            d += 1
        return True
    if n % 2 == 0:
        return False
    for p in SMALL_PRIMES:
        if n % p == 0:
            return n == p
    nm1 = n - 1
    s, d = 0, nm1
    while d % 2 == 0:
        d //= 2
        s += 1
    for _ in range(rounds):
        a = random_below(rng, n - 3) + 2
        x = pow(a, d, n)
        if x == 1 or x == nm1:
            continue
        witness = True
        for _ in range(s - 1):
            x = x * x % n
            if x == nm1:
                witness = False
                break
        if witness:
            return False
    return True


def random_prime(rng: Rng, bits: int, mr_rounds: int = 40) -> int:  # bignat.cpp:497-515
    if bits < 2:
        raise ValueError("random_prime: need >= 2 bits")
    while True:
        cand = random_bits(rng, bits) | (1 << (bits - 1)) | 1
        for _ in range(64):
            if is_probable_prime(cand, rng, mr_rounds):
                return cand
            cand += 2
            if cand.bit_length() != bits:
                break


# --------------------------------------------------------------------------------------------
# keys — paillier.cpp:43-130 (binomial g = n + 1, the default GMode)
# --------------------------------------------------------------------------------------------
@dataclass
class KeyPair:
    n: int
    p: int
    q: int
    key_bits: int
    g: int = 0
    n2: int = 0
    eps: int = 0  # lcm(p-1, q-1)
    mu: int = 0
    crt: dict = field(default_factory=dict)


def _lcm(a: int, b: int) -> int:
    return a // math.gcd(a, b) * b


def finish_keys(p: int, q: int, key_bits: int) -> KeyPair:  # paillier.cpp:63-104 (binomial branch)
    n = p * q
    eps = _lcm(p - 1, q - 1)
    mu = pow(eps % n, -1, n)  # (eps mod n)^-1 mod n, paillier.cpp:78
    kp = KeyPair(n=n, p=p, q=q, key_bits=key_bits, g=n + 1, n2=n * n, eps=eps, mu=mu)
    p2, q2 = p * p, q * q
    kp.crt = dict(  # make_crt, paillier.cpp:43-60
        p2=p2, q2=q2, phi_p2=p2 - p, phi_q2=q2 - q, p2_inv_q2=pow(p2 % q2, -1, q2),
        n_mod_phi_p2=n % (p2 - p), n_mod_phi_q2=n % (q2 - q),
        eps_mod_phi_p2=eps % (p2 - p), eps_mod_phi_q2=eps % (q2 - q))
    return kp


def keygen(rng: Rng, key_bits: int) -> KeyPair:  # paillier.cpp:106-123
    if key_bits not in (64, 1024, 2048, 4096):
        raise ValueError("key_bits must be 64, 1024, 2048 or 4096")
    half = key_bits // 2
    for _ in range(64):
        p = random_prime(rng, half)
        q = random_prime(rng, half)
        if p == q:
            continue
        if abs(p - q).bit_length() < half - 7:
            continue
        if (p * q).bit_length() != key_bits:
            continue
        rng.next()  # finish_keys(p, q, gmode, rng.next(), key_bits), paillier.cpp:120
        return finish_keys(p, q, key_bits)
    raise RuntimeError("key generation attempt budget exhausted")


def keypair_from_primes(p: int, q: int) -> KeyPair:  # paillier.cpp:125-130
    if p == q or p < 2 or q < 2:
        raise ValueError("need two distinct primes")
    return finish_keys(p, q, (p * q).bit_length())


# --------------------------------------------------------------------------------------------
# Paillier — paillier.cpp:233-516.  Errors raise the reference's exception classes, mapped to
# the pcb_status codes by STATUS_OF.
# --------------------------------------------------------------------------------------------
class PlaintextRange(ValueError): ...      # invalid_argument paillier.cpp:242
class RandomnessRange(ValueError): ...     # invalid_argument paillier.cpp:322-323
class CipherRange(ValueError): ...         # invalid_argument paillier.cpp:348, 356
class NotUnit(RuntimeError): ...           # runtime_error paillier.cpp:36, 39
class Overflow(OverflowError): ...         # overflow_error paillier.cpp:250
class Shape(ValueError): ...               # invalid_argument (shape / window)


STATUS_OF = {PlaintextRange: 1, RandomnessRange: 2, CipherRange: 3, NotUnit: 4, Overflow: 5, Shape: 7}


def sample_r(kp: KeyPair, rng: Rng) -> int:  # paillier.cpp:233-239
    while True:
        r = random_below(rng, kp.n)
        if r == 0:
            continue
        if math.gcd(r, kp.n) == 1:
            return r


def encrypt_with_r(kp: KeyPair, m: int, r: int) -> int:  # paillier.cpp:320-328 (binomial g)
    if m >= kp.n:
        raise PlaintextRange("plaintext not below n")
    if r == 0 or r >= kp.n:
        raise RandomnessRange("randomness not in [1, n)")
    return (1 + m * kp.n) % kp.n2 * pow(r, kp.n, kp.n2) % kp.n2


def crt_encrypt_with_r(kp: KeyPair, m: int, r: int) -> int:  # paillier.cpp:334-344
    if m >= kp.n:
        raise PlaintextRange("plaintext not below n")
    if r == 0 or r >= kp.n:
        raise RandomnessRange("randomness not in [1, n)")
    c = kp.crt
    cp = (1 + m * kp.n) % c["p2"] * pow(r % c["p2"], c["n_mod_phi_p2"], c["p2"]) % c["p2"]
    cq = (1 + m * kp.n) % c["q2"] * pow(r % c["q2"], c["n_mod_phi_q2"], c["q2"]) % c["q2"]
    return combine_halves(kp, cp, cq)


def combine_halves(kp: KeyPair, cp: int, cq: int) -> int:  # paillier.cpp:307-314
    c = kp.crt
    return cp + c["p2"] * ((cq - cp % c["q2"]) % c["q2"] * c["p2_inv_q2"] % c["q2"])


def l_function(x: int, n: int) -> int:  # paillier.cpp:34-41
    if x == 0 or (x - 1) % n != 0:
        raise NotUnit("ciphertext outside the multiplicative group")
    return (x - 1) // n


def decrypt(kp: KeyPair, c: int) -> int:  # paillier.cpp:346-352
    if c >= kp.n2:
        raise CipherRange("ciphertext not below n^2")
    return l_function(pow(c, kp.eps, kp.n2), kp.n) * kp.mu % kp.n


def crt_decrypt(kp: KeyPair, c: int) -> int:  # paillier.cpp:354-361
    if c >= kp.n2:
        raise CipherRange("ciphertext not below n^2")
    cc = kp.crt
    xp = pow(c % cc["p2"], cc["eps_mod_phi_p2"], cc["p2"])
    xq = pow(c % cc["q2"], cc["eps_mod_phi_q2"], cc["q2"])
    return l_function(combine_halves(kp, xp, xq), kp.n) * kp.mu % kp.n


def bump_bits_or_throw(kp: KeyPair, bits: int) -> None:  # paillier.cpp:245-251
    if bits >= kp.n.bit_length():
        raise Overflow("homomorphic accumulation exceeds plaintext space")


def hom_add(kp: KeyPair, a: int, a_bits: int, b: int, b_bits: int) -> tuple[int, int]:  # paillier.cpp:428-432
    bits = max(a_bits, b_bits) + 1
    bump_bits_or_throw(kp, bits)
    return a * b % kp.n2, bits


def hom_scalar_mul(kp: KeyPair, k: int, c: int, c_bits: int) -> tuple[int, int]:  # paillier.cpp:434-439
    bits = 0 if k == 0 else c_bits + k.bit_length()
    bump_bits_or_throw(kp, bits)
    return pow(c, k, kp.n2), bits


def hom_matvec(kp: KeyPair, alpha, alpha_bits, expo, zv, zv_bits, window: int = 6):  # paillier.cpp:441-493
    rows, cols = len(alpha), len(zv)
    if len(expo) != rows or any(len(r) != cols for r in expo):
        raise Shape("exponent shape")
    if window < 1 or window > 8:
        raise Shape("window in [1,8]")
    max_bits = max((k.bit_length() for row in expo for k in row), default=0)
    zvb = max(zv_bits, default=0)
    sum_bits = max_bits + zvb + cols.bit_length() if cols else 0
    out, out_bits = [], []
    for i in range(rows):
        acc = 1
        for j in range(cols):
            acc = acc * pow(zv[j], expo[i][j], kp.n2) % kp.n2
        bits = max(alpha_bits[i], sum_bits) + 1
        bump_bits_or_throw(kp, bits)
        out.append(alpha[i] * acc % kp.n2)
        out_bits.append(bits)
    return out, out_bits


# --------------------------------------------------------------------------------------------
# quantize — quantize.cpp:8-129
# --------------------------------------------------------------------------------------------
def c_round(x: float) -> float:
    """libm round(): half away from zero, exact on binary64 (x - floor(x) is exact)."""
    if x >= 0:
        f = math.floor(x)
        return f + 1.0 if x - f >= 0.5 else f
    return -c_round(-x)


def check_spec(zmin: float, zmax: float, delta: float) -> None:  # quantize.cpp:8-15
    if not (math.isfinite(zmin) and math.isfinite(zmax)) or zmax <= zmin:
        raise Shape("quantization window is empty or non-finite")
    if not (delta >= 1.0) or delta > 9.0e15:
        raise Shape("delta outside [1, 9e15]")


def clamp_in(v: float, zmin: float, zmax: float, clamps: list | None) -> float:  # quantize.cpp:17-29
    if not math.isfinite(v):
        raise Shape("non-finite value into quantizer")
    if v < zmin:
        if clamps is not None:
            clamps[0] += 1
        return zmin
    if v > zmax:
        if clamps is not None:
            clamps[1] += 1
        return zmax
    return v


def gamma2(v: float, zmin: float, zmax: float, delta: float, clamps: list | None = None) -> int:  # quantize.cpp:31-35
    check_spec(zmin, zmax, delta)
    t = delta * ((clamp_in(v, zmin, zmax, clamps) - zmin) / (zmax - zmin))
    return int(c_round(t))


def gamma1(v: float, zmin: float, zmax: float, delta: float, clamps: list | None = None) -> int:  # quantize.cpp:37-41
    check_spec(zmin, zmax, delta)
    r = zmax - zmin
    d = (clamp_in(v, zmin, zmax, clamps) - zmin) / (r * r)
    return int(c_round(delta * delta * d))


def degamma2(q: int, zmin: float, zmax: float, delta: float) -> float:  # quantize.cpp:43-45
    return zmin + float(q) * ((zmax - zmin) / delta)


def combined_quantized_update(q_alpha, q_b, q_z, q_negv):  # quantize.cpp:66-82
    rows, cols = len(q_alpha), len(q_z)
    out = []
    for i in range(rows):
        acc = q_alpha[i]
        for j in range(cols):
            acc += q_b[i][j] * (q_z[j] + q_negv[j])
        out.append(acc & ((1 << 128) - 1))
    return out


def u128_to_double(q: int) -> float:
    """__floatuntidf: correctly rounded u128 -> binary64 (Python int -> float rounds to nearest even)."""
    return float(q)


def inverse_quantize_x(q, q_b_rowsum, q_z, q_negv, zmin, zmax, delta):  # quantize.cpp:84-112
    check_spec(zmin, zmax, delta)
    cols = len(q_z)
    step = (zmax - zmin) / delta
    step2 = step * step
    sum_zv = 0.0
    for j in range(cols):
        sum_zv += 2.0 * zmin + step * (float(q_z[j]) + float(q_negv[j]))
    out = []
    for i in range(len(q)):
        rowsum_b = float(cols) * zmin + step * float(q_b_rowsum[i])
        out.append(u128_to_double(q[i]) * step2 + zmin * (1.0 + 2.0 * rowsum_b + sum_zv)
                   - 2.0 * zmin * zmin * float(cols))
    return out


def widen_bounds(lo: float, hi: float, margin: float, delta: float):  # quantize.cpp:114-129
    if not (math.isfinite(lo) and math.isfinite(hi)) or hi < lo:
        raise Shape("bad value extremes")
    if margin < 1.0:
        raise Shape("margin below 1")
    if hi - lo < 1e-12:
        lo -= 0.5
        hi += 0.5
    pad = (margin - 1.0) * (hi - lo) / 2.0
    zmin, zmax = lo - pad, hi + pad
    check_spec(zmin, zmax, delta)
    return zmin, zmax


def bignat_to_double(q: int) -> float:  # BigNat::to_double, bignat.cpp:56-60 (limb-wise, not correctly rounded)
    v = 0.0
    limbs = []
    while q:
        limbs.append(q & MASK64)
        q >>= 64
    for w in reversed(limbs):
        v = v * 18446744073709551616.0 + float(w)
    return v


def check_update_range(q: int, zmin: float, zmax: float, delta: float, cols: int) -> bool:  # protocol.cpp:20-27
    cap = delta * delta / (zmax - zmin) + float(cols) * delta * 2.0 * delta
    return not (q.bit_length() > 127 or bignat_to_double(q) > cap * 1.000001 + 4.0)


def soft_threshold(v: float, kappa: float) -> float:  # admm.cpp:18-22
    if v > kappa:
        return v - kappa
    if v < -kappa:
        return v + kappa
    return 0.0
