"""RNS Montgomery arithmetic restated in numpy — TEST INFRASTRUCTURE ONLY (never imported by the
product).  It is the checker for paper_2601_14980_b200/csrc/rns.cu, the residue-number-system
core that replaces the carry-chain Montgomery product for the CRT halves (mod p^2, q^2) of
Paillier Enc/Dec (reference: Paillier::half_pow / crt_encrypt_with_r / crt_decrypt,
/root/reference/proj/src/paillier.cpp:275-305, 330-361).  Any exact algorithm gives the same
residues, so the check is against Python pow() and the reference's golden vectors.

Algorithm (Bajard-Imbert RNS Montgomery; approximate first base extension, exact second):
  bases B = {m_i}, B' = {m'_j}, k primes each, all < 2^30; M = prod m_i, M' = prod m'_j;
  per-prime values are lazy Montgomery residues  x~ = x 2^32 mod m  in [0, 2m);
  REDC(T) = (T + ((T mod 2^32) (-m^-1) mod 2^32) m) / 2^32  (< 2m for T < 4m^2).
  MM(x, y) = x y M^-1 mod N (lazy, < (2k+2) N):
    1. t~ = REDC(x~ y~)                                    (both bases)
    2. xi_i = REDC(t~_i C1_i),  C1_i = -N^-1 M_i^-1 mod m_i           (plain, lazy)
    3. qh'_j = REDC(sum_i xi_i W1_ji),  W1_ji = M_i 2^32 mod m'_j      (GEMM 1)
       = q + alpha M in B', alpha < 2k
    4. r~'_j = REDC(t~'_j C2_j) + REDC(qh'_j C3_j) (-2m' if >= 2m'),
       C2 = M^-1 2^32, C3 = N M^-1 2^64 (mod m'_j)
       fused form (rnsx.cu rx_e1, round 2): GEMM 1 on W1'_ji = M_i C3_j mod m'_j gives
       V'_j = sum_i xi_i W1'_ji = qh'_j C3_j 2^32 (mod m'_j), and r~'_j = REDC(t~'_j C2_j + V'_j)
       in one REDC (t~' C2 + V' < 2 m'^2 + 2^49, so the result stays < 2m')
    5. xi'_j = REDC(r~'_j C4_j), C4 = M'_j^-1;  beta = floor(sum_j xi'_j / m'_j + 2^-20)
       (rnsx.cu, round 2: S is an FP32 over-estimate -- terms f32(2^23 + (xi' >> 8)) * f32(2^8 / m'),
       the 2^23 parts subtracted once -- plus 2^-8: S_true lies in [beta, beta + 2^-24) and the FP32
       error is ~2^-12.5, so any estimate in [S_true, S_true + 1 - 2^-24) floors to beta)
    6. r~_i = REDC(sum_j xi'_j W2_ij + beta W2_ik),  W2_ij = M'_j 2^64 mod m_i,
       W2_ik = -M' 2^64 mod m_i                                       (GEMM 2, exact)
  The GEMMs run on int8 tensor cores: each 32-bit operand is split into 4 bytes on both sides,
  D_b = sum over (i, a) of byte_a(xi_i) byte_b(W^(a)_ji) with W^(a) = W 2^(8a) mod m (int32
  exact: 4(k+1) 255^2 < 2^31), and V = sum_b D_b 2^(8b) < 2^49 feeds REDC.
"""
from __future__ import annotations

import numpy as np

K_PRIMES = 72
PRIME_BITS = 30
MASK32 = (1 << 32) - 1


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17):  # deterministic for n < 3.4e14
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def rns_primes(k: int = K_PRIMES, bits: int = PRIME_BITS):
    """The 2k largest primes below 2^bits, descending: B = first k, B' = next k."""
    out, c = [], (1 << bits) - 1
    while len(out) < 2 * k:
        if _is_prime(c):
            out.append(c)
        c -= 2
    return out[:k], out[k:]


class RnsCtx:
    def __init__(self, N: int, k: int = K_PRIMES):
        self.N, self.k = N, k
        B, Bp = rns_primes(k)
        self.B, self.Bp = B, Bp
        M = 1
        for m in B:
            M *= m
        Mp = 1
        for m in Bp:
            Mp *= m
        self.M, self.Mp = M, Mp
        assert M > (2 * k + 2) ** 2 * N and Mp > (1 << 24) * (2 * k + 2) * N
        self.mB = np.array(B, np.uint64)
        self.mBp = np.array(Bp, np.uint64)
        self.minvB = np.array([(-pow(m, -1, 1 << 32)) % (1 << 32) for m in B], np.uint64)
        self.minvBp = np.array([(-pow(m, -1, 1 << 32)) % (1 << 32) for m in Bp], np.uint64)
        Ninv = [pow(N, -1, m) for m in B]
        self.C1 = np.array([(-Ninv[i] * pow(M // m, -1, m)) % m for i, m in enumerate(B)], np.uint64)
        self.W1 = np.array([[(M // mi) * (1 << 32) % mj for mi in B] for mj in Bp], np.uint64)  # [j][i]
        self.C2 = np.array([pow(M, -1, m) * (1 << 32) % m for m in Bp], np.uint64)
        self.C3 = np.array([N * pow(M, -1, m) * (1 << 64) % m for m in Bp], np.uint64)
        self.C4 = np.array([pow(Mp // m, -1, m) for m in Bp], np.uint64)
        C3i = [N * pow(M, -1, m) * (1 << 64) % m for m in Bp]
        self.W1f = np.array([[(M // mi) * c3 % mj for mi in B] for mj, c3 in zip(Bp, C3i)], np.uint64)
        self.fused = True  # the fused GEMM-1 epilogue of rnsx.cu (step 4, fused form)
        self.invBp = np.array([1.0 / m for m in Bp], np.float64)
        W2 = [[(Mp // mj) * (1 << 64) % mi for mj in Bp] + [(-Mp * (1 << 64)) % mi] for mi in B]
        self.W2 = np.array(W2, np.uint64)  # [i][j], column k = beta coefficient
        # constants in RNS (lazy Montgomery per prime): M^2 mod N (to-Montgomery), 2^(32 S) M^2 mod N
        self.R2N = self.to_rns(M * M % N)

    # ---- per-prime helpers -------------------------------------------------------------------
    @staticmethod
    def redc(T, m, minv):
        u = ((T & MASK32) * minv) & MASK32
        return (T + u * m) >> np.uint64(32)

    def to_rns(self, x: int):
        """Integer x (0 <= x < M) -> (xB~, xBp~) lazy Montgomery residues (here: canonical)."""
        a = np.array([(x % m) * (1 << 32) % m for m in self.B], np.uint64)
        b = np.array([(x % m) * (1 << 32) % m for m in self.Bp], np.uint64)
        return a, b

    def from_rns(self, xb) -> int:
        """Exact integer from the B' residues (lazy Montgomery form accepted)."""
        _, b = xb
        r = [int(v) * pow(1 << 32, -1, m) % m for v, m in zip(b, self.Bp)]
        x = 0
        for v, m in zip(r, self.Bp):
            Mj = self.Mp // m
            x += v * pow(Mj, -1, m) % m * Mj
        return x % self.Mp

    def gemm_bytes(self, xi, W, mods):
        """sum_i xi_i W_ji exactly as the tensor-core byte split computes it, then REDC per j."""
        k_in = xi.shape[0]
        a_bytes = np.stack([(xi >> np.uint64(8 * a)) & np.uint64(255) for a in range(4)], 1)  # [i][a]
        Wa = np.stack([(W * np.uint64(1 << (8 * a))) % mods[:, None] for a in range(4)], 2)  # [j][i][a]
        D = []
        for b in range(4):
            wb = (Wa >> np.uint64(8 * b)) & np.uint64(255)                                   # [j][i][a]
            D.append(np.einsum("ia,jia->j", a_bytes.astype(np.int64), wb.astype(np.int64)))
        for d in D:
            assert d.max() < (1 << 31)
        V = sum(d.astype(np.uint64) << np.uint64(8 * b) for b, d in enumerate(D))
        assert k_in <= W.shape[1]
        return V

    def mm(self, x, y):
        (xa, xb), (ya, yb) = x, y
        mB, mBp = self.mB, self.mBp
        ta = self.redc(xa * ya, mB, self.minvB)
        tb = self.redc(xb * yb, mBp, self.minvBp)
        xi = self.redc(ta * self.C1, mB, self.minvB)
        if self.fused:
            r1 = self.redc(tb * self.C2 + self.gemm_bytes(xi, self.W1f, mBp), mBp, self.minvBp)
        else:
            qh = self.redc(self.gemm_bytes(xi, self.W1, mBp), mBp, self.minvBp)
            r1 = self.redc(tb * self.C2, mBp, self.minvBp) + self.redc(qh * self.C3, mBp, self.minvBp)
            r1 = np.where(r1 >= 2 * mBp, r1 - 2 * mBp, r1)
        xip = self.redc(r1 * self.C4, mBp, self.minvBp)
        if self.fused:  # rnsx.cu rx_e1: FP32 over-estimate, 2^-8 bias (one-sided bound, see module doc)
            f = ((xip >> np.uint64(8)) | np.uint64(0x4B000000)).astype(np.uint32).view(np.float32)
            inv8 = (256.0 / self.mBp.astype(np.float64)).astype(np.float32)
            sp = np.float32(0.0)
            for a, b in zip(f, inv8):
                sp = np.float32(sp + np.float32(a * b))
            cthr = np.float32(0.0)
            for b in inv8:
                cthr = np.float32(cthr + np.float32(np.float32(8388608.0) * b))
            beta = int(np.floor(np.float32(np.float32(sp - cthr) + np.float32(0.00390625))))
        else:
            S = float(np.sum(xip.astype(np.float64) * self.invBp))
            beta = int(np.floor(S + 2.0 ** -20))
        assert beta == int(sum(int(a) * ((self.Mp // int(m)) % self.Mp) for a, m in zip(xip, self.mBp)) // self.Mp)
        xiext = np.concatenate([xip, np.array([beta], np.uint64)])
        ra = self.redc(self.gemm_bytes(xiext, self.W2, mB), mB, self.minvB)
        for v, m in ((ra, mB), (r1, mBp)):
            assert (v < 2 * m).all()
        return ra, r1

    def pow(self, base: int, e: int) -> int:
        """base^e mod N through the RNS Montgomery product (square and multiply)."""
        x = self.mm(self.to_rns(base), self.R2N)  # base M mod N
        acc = self.mm(self.to_rns(1), self.R2N)   # M mod N
        for bit in bin(e)[2:]:
            acc = self.mm(acc, acc)
            if bit == "1":
                acc = self.mm(acc, x)
        acc = self.mm(acc, self.to_rns(1))
        v = self.from_rns(acc)
        assert v < (2 * self.k + 2) * self.N
        return v % self.N
