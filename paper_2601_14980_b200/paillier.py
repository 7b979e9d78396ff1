"""Host-side mirror of the reference's hot-path API over the C ABI (include/pcb200.h).

Names, argument meaning and error behaviour follow pcadmm (paths under /root/reference/proj):
  Rng                  bignat.hpp:107-114   (splitmix64; host-side, feeds keygen / sample_r)
  keygen               paillier.cpp:106-123 (pcb_keygen: bit-exact key + Rng state)
  keypair_from_primes  paillier.cpp:125-130
  Ciphertext           paillier.hpp:71-74   (value + plain_bits bookkeeping, kept on the host)
  Paillier             paillier.hpp:104-181 (every batch op is one CUDA pipeline; no CPU fallback)

Exceptions map the reference's: invalid_argument -> ValueError, runtime_error -> RuntimeError,
overflow_error -> OverflowError, logic_error -> LogicError.
Batched tensor entry points (encrypt_batch / decrypt_batch / ...) keep data on the GPU as
fixed-width little-endian u32 limb tensors (torch.int32 views) for the hot path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L

MASK64 = (1 << 64) - 1


class LogicError(RuntimeError):
    """pcadmm's std::logic_error (private operation without the private key)."""


def _raise_for(code: int, what: str = "") -> None:
    if code == L.PCB_OK:
        return
    msg = L.lib().pcb_status_str(code).decode() + (f" ({what})" if what else "")
    if code in (L.PCB_E_PLAINTEXT_RANGE, L.PCB_E_RANDOMNESS_RANGE, L.PCB_E_CIPHER_RANGE, L.PCB_E_SHAPE):
        raise ValueError(msg)
    if code == L.PCB_E_NOT_UNIT:
        raise RuntimeError(msg)
    if code == L.PCB_E_OVERFLOW:
        raise OverflowError(msg)
    if code == L.PCB_E_NO_PRIVATE:
        raise LogicError(msg)
    raise L.PcbError(code, what)


class Rng:
    """splitmix64, identical stream to pcadmm::Rng (bignat.cpp:388-394)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def unit(self) -> float:
        return float(self.next() >> 11) * (2.0 ** -53)


@dataclass
class KeyPair:
    n: int
    p: int
    q: int
    key_bits: int

    @property
    def n2(self) -> int:
        return self.n * self.n


@dataclass
class PublicKey:
    n: int
    key_bits: int


@dataclass
class RnFactor:
    """pcadmm::RnFactor (paillier.hpp:78-82): r, r^n mod n^2 and its residues mod p^2 / q^2."""

    r: int
    full: int
    half_p2: int
    half_q2: int


@dataclass
class Ciphertext:
    value: int
    plain_bits: int = 0


def keygen(rng: Rng, key_bits: int, device: int | None = None) -> KeyPair:
    """pcadmm::keygen(rng, key_bits, GMode::binomial); advances rng exactly like the reference.
    device: run the Miller-Rabin rounds in batches on that CUDA device (pcb_keygen_speculative,
    same key and rng state); None: the host search (pcb_keygen)."""
    nl = (key_bits + 31) // 32
    hl = (key_bits // 2 + 31) // 32
    st = C.c_uint64(rng.state)
    n = np.zeros(nl, np.uint32)
    p = np.zeros(hl, np.uint32)
    q = np.zeros(hl, np.uint32)
    if device is not None:
        _raise_for(L.lib().pcb_keygen_speculative(C.byref(st), key_bits, int(device), n.ctypes.data_as(L._u32p),
                                                  p.ctypes.data_as(L._u32p), q.ctypes.data_as(L._u32p)), "keygen")
    else:
        _raise_for(L.lib().pcb_keygen(C.byref(st), key_bits, n.ctypes.data_as(L._u32p), p.ctypes.data_as(L._u32p),
                                      q.ctypes.data_as(L._u32p)), "keygen")
    rng.state = st.value
    return KeyPair(L.limbs_to_int(n), L.limbs_to_int(p), L.limbs_to_int(q), key_bits)


def random_prime(rng: Rng, bits: int, device: int | None = None) -> int:
    """pcadmm::random_prime(rng, bits, 40) (bignat.cpp:497-515); device as keygen."""
    st = C.c_uint64(rng.state)
    out = np.zeros((bits + 31) // 32, np.uint32)
    if device is not None:
        _raise_for(L.lib().pcb_random_prime_speculative(C.byref(st), bits, int(device), out.ctypes.data_as(L._u32p)),
                   "random_prime")
    else:
        _raise_for(L.lib().pcb_random_prime(C.byref(st), bits, out.ctypes.data_as(L._u32p)), "random_prime")
    rng.state = st.value
    return L.limbs_to_int(out)


def _wire_put(out: bytearray, v: int) -> None:
    """wire_put (bignat.cpp:414-418): u32 BE byte length, then the minimal big-endian magnitude."""
    b = v.to_bytes((v.bit_length() + 7) // 8, "big") if v else b""
    out += len(b).to_bytes(4, "big") + b


def _wire_get(data: bytes, off: int) -> tuple[int, int]:
    if off + 4 > len(data):
        raise RuntimeError("truncated integer field")
    n = int.from_bytes(data[off:off + 4], "big")
    if off + 4 + n > len(data):
        raise RuntimeError("truncated integer field")
    return int.from_bytes(data[off + 4:off + 4 + n], "big"), off + 4 + n


def serialize_keypair(kp: KeyPair) -> bytes:
    """serialize_keypair (paillier.cpp:152-166), binomial g: 'p' 'k' 1 1, u32 BE key_bits, then
    wire_put of n, g = n + 1, p, q, epsilon = lcm(p - 1, q - 1), mu = epsilon^-1 mod n."""
    import math

    eps = (kp.p - 1) * (kp.q - 1) // math.gcd(kp.p - 1, kp.q - 1)
    out = bytearray(b"pk\x01\x01") + int(kp.key_bits).to_bytes(4, "big")
    for v in (kp.n, kp.n + 1, kp.p, kp.q, eps, pow(eps % kp.n, -1, kp.n)):
        _wire_put(out, v)
    return bytes(out)


def parse_keypair(data: bytes) -> KeyPair:
    """parse_keypair (paillier.cpp:168-191) for binomial-g records; the same errors (RuntimeError)."""
    if len(data) < 4 or data[0:2] != b"pk":
        raise RuntimeError("not a key record")
    if data[2] != 1:
        raise RuntimeError("unknown key record version")
    if data[3] == 0:
        raise NotImplementedError("random-g key records: load them through the C++ drop-in (pcadmm::parse_keypair)")
    if len(data) < 8:
        raise RuntimeError("truncated key record")
    key_bits = int.from_bytes(data[4:8], "big")
    off = 8
    vals = []
    for _ in range(6):
        v, off = _wire_get(data, off)
        vals.append(v)
    n, g, p, q = vals[:4]
    if p * q != n:
        raise RuntimeError("corrupt key record: n != p*q")
    if g != n + 1:
        raise RuntimeError("corrupt key record: g mismatch")
    return KeyPair(n, p, q, key_bits)


def keypair_from_primes(p: int, q: int) -> KeyPair:
    """pcadmm::keypair_from_primes (binomial g)."""
    if p == q or p < 2 or q < 2:
        raise ValueError("need two distinct primes")
    return KeyPair(p * q, p, q, (p * q).bit_length())


def _torch():
    import torch

    return torch


class Paillier:
    """A key + its device context (pcadmm::Paillier, paillier.hpp:104-181)."""

    def __init__(self, keys: KeyPair | PublicKey, device: int = 0):
        self.device = device
        n = keys.n
        self.n = n
        self.n2 = n * n
        self.key_bits = keys.key_bits
        self.L = (n.bit_length() + 31) // 32
        self._has_prv = isinstance(keys, KeyPair)
        self._p, self._q = (keys.p, keys.q) if self._has_prv else (0, 0)
        nl = L.int_to_limbs(n, self.L)
        ctx = C.c_void_p()
        if self._has_prv:
            w = max((keys.p.bit_length() + 31) // 32, (keys.q.bit_length() + 31) // 32)
            pl, ql = L.int_to_limbs(keys.p, w), L.int_to_limbs(keys.q, w)
            rc = L.lib().pcb_ctx_create(C.byref(ctx), device, nl.ctypes.data_as(L._u32p), self.L,
                                        pl.ctypes.data_as(L._u32p), ql.ctypes.data_as(L._u32p), w)
        else:
            rc = L.lib().pcb_ctx_create(C.byref(ctx), device, nl.ctypes.data_as(L._u32p), self.L, None, None, 0)
        _raise_for(rc, "context")
        self._ctx = ctx

    def __del__(self):
        ctx = getattr(self, "_ctx", None)
        if ctx and L is not None and L._lib is not None:  # module globals are gone at interpreter exit
            L._lib.pcb_ctx_destroy(ctx)
            self._ctx = None

    # ---- introspection ------------------------------------------------------------------
    def has_private(self) -> bool:
        return self._has_prv

    def crt_half_words(self) -> int:
        """u32 words per element of a CRT half on the device (the context's S: the kernel width
        that holds p^2, q^2 and n), e.g. pcb_decrypt_half_q's output row."""
        l2 = (max((self._p * self._p).bit_length(), (self._q * self._q).bit_length()) + 31) // 32
        need = max(l2, self.L)
        for w in (32, 64, 96, 128):
            if need <= w:
                return w
        raise ValueError("no CRT half width for this key")

    def counters(self) -> tuple[int, int]:
        """(pow_full, pow_half) — pcadmm::OpCount (paillier.hpp:84-87)."""
        a, b = C.c_uint64(), C.c_uint64()
        L.lib().pcb_ctx_counters(self._ctx, C.byref(a), C.byref(b))
        return a.value, b.value

    def reset_counters(self) -> None:
        L.lib().pcb_ctx_reset_counters(self._ctx)

    def _need_prv(self):
        if not self._has_prv:
            raise LogicError("no private key loaded")

    # ---- batched tensor API (device-resident) --------------------------------------------
    def sample_r_batch(self, rng: Rng, count: int):
        """count x sample_r(rng) on the GPU -> int32 tensor (count, L); rng advanced."""
        torch = _torch()
        out = torch.empty((count, self.L), dtype=torch.int32, device=f"cuda:{self.device}")
        st = C.c_uint64(rng.state)
        _raise_for(L.lib().pcb_sample_r(self._ctx, C.byref(st), count, L.ptr(out), self._stream()), "sample_r")
        rng.state = st.value
        return out

    def skip_r(self, rng: Rng, count: int, chunk: int = 1 << 20) -> None:
        """Advance rng past `count` sample_r draws (the accepted-candidate count is data
        dependent, so the state after them is found by drawing them on the GPU, in chunks into
        one scratch buffer).  Rank k of a job whose single r stream is sliced over ranks calls
        skip_r(rng, k * n) and then draws its own n."""
        torch = _torch()
        if count <= 0:
            return
        buf = torch.empty((min(count, chunk), self.L), dtype=torch.int32, device=f"cuda:{self.device}")
        left = count
        while left:
            k = min(left, chunk)
            st = C.c_uint64(rng.state)
            _raise_for(L.lib().pcb_sample_r(self._ctx, C.byref(st), k, L.ptr(buf), self._stream()), "sample_r")
            rng.state = st.value
            left -= k

    def _stream(self):
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def encrypt_batch(self, m, r, use_crt: bool = True, status=None):
        """m: (count, m_limbs) int32/uint32 limbs, r: (count, L) -> c: (count, 2L).  Device or host."""
        torch = _torch()
        count, ml = m.shape
        dev = m.is_cuda if hasattr(m, "is_cuda") else False
        if dev:
            c = torch.empty((count, 2 * self.L), dtype=torch.int32, device=m.device)
        else:
            c = np.zeros((count, 2 * self.L), np.uint32)
        if use_crt:
            self._need_prv()
        rc = L.lib().pcb_encrypt(self._ctx, L.ptr(m), ml, L.ptr(r), count, L.ptr(c), 1 if use_crt else 0,
                                 L.ptr(status), self._stream() if dev else None)
        _raise_for(rc, "encrypt")
        return c

    def encrypt_rn_batch(self, m, rn, status=None):
        """Online encryption with precomputed randomness rn = r^n mod n^2 (= encrypt_batch(0, r)):
        c = (1 + m n) rn mod n^2, equal to encrypt_batch(m, r)."""
        torch = _torch()
        count, ml = m.shape
        dev = m.is_cuda if hasattr(m, "is_cuda") else False
        c = torch.empty((count, 2 * self.L), dtype=torch.int32, device=m.device) if dev else \
            np.zeros((count, 2 * self.L), np.uint32)
        _raise_for(L.lib().pcb_encrypt_rn(self._ctx, L.ptr(m), ml, L.ptr(rn), count, L.ptr(c), L.ptr(status),
                                          self._stream() if dev else None), "encrypt_rn")
        return c

    def finish_split_encrypt_rn_batch(self, m, p2_g_power, rn, status=None):
        """Paillier::finish_split_encrypt_with_factor (paillier.cpp:416-426) with the factor's
        rn = r^n mod n^2: c = CRT(p2_g_power mod p^2, (1 + m n) mod q^2) rn mod n^2."""
        torch = _torch()
        self._need_prv()
        count, ml = m.shape
        dev = m.is_cuda if hasattr(m, "is_cuda") else False
        c = torch.empty((count, 2 * self.L), dtype=torch.int32, device=m.device) if dev else \
            np.zeros((count, 2 * self.L), np.uint32)
        _raise_for(L.lib().pcb_finish_split_encrypt_rn(self._ctx, L.ptr(m), ml, L.ptr(p2_g_power), p2_g_power.shape[1],
                                                       L.ptr(rn), count, L.ptr(c), L.ptr(status),
                                                       self._stream() if dev else None), "finish_split_encrypt_rn")
        return c

    def decrypt_batch(self, c, use_crt: bool = True, status=None):
        torch = _torch()
        self._need_prv()
        count = c.shape[0]
        dev = c.is_cuda if hasattr(c, "is_cuda") else False
        if dev:
            m = torch.empty((count, self.L), dtype=torch.int32, device=c.device)
        else:
            m = np.zeros((count, self.L), np.uint32)
        rc = L.lib().pcb_decrypt(self._ctx, L.ptr(c), count, L.ptr(m), 1 if use_crt else 0, L.ptr(status),
                                 self._stream() if dev else None)
        _raise_for(rc, "decrypt")
        return m

    def quantize_encrypt_batch(self, v, z_min: float, z_max: float, delta: float, r, fine: bool = False):
        """Fused Gamma2/Gamma1 + CRT encryption (quantize.cpp:31-41 then crt_encrypt_with_r).
        Returns (c, q, clamps) with q the quantized integers (u64, or u128 as (lo, hi))."""
        torch = _torch()
        self._need_prv()
        count = v.shape[0]
        dev = v.is_cuda if hasattr(v, "is_cuda") else False
        if dev:
            c = torch.empty((count, 2 * self.L), dtype=torch.int32, device=v.device)
            q = torch.empty((count, 2) if fine else (count,), dtype=torch.int64, device=v.device)
        else:
            c = np.zeros((count, 2 * self.L), np.uint32)
            q = np.zeros((count, 2) if fine else (count,), np.uint64)
        cl = (C.c_uint64 * 2)()
        rc = L.lib().pcb_quantize_encrypt(self._ctx, L.ptr(v), count, z_min, z_max, delta, 1 if fine else 0,
                                          L.ptr(r), 1, L.ptr(c), L.ptr(q), cl, self._stream() if dev else None)
        _raise_for(rc, "quantize_encrypt")
        return c, q, (cl[0], cl[1])

    # ---- reference-shaped scalar / vector API (Python ints) ---------------------------------
    def _enc_list(self, ms, rs, use_crt):
        count = len(ms)
        if count == 0:
            return []
        M = L.ints_to_limbs(ms, self.L)
        R = L.ints_to_limbs(rs, self.L)
        st = np.zeros(count, np.int32)
        c = self.encrypt_batch(M, R, use_crt, status=st)
        bad = np.nonzero(st)[0]
        if len(bad):
            _raise_for(int(st[bad[0]]), f"element {int(bad[0])}")
        return [Ciphertext(v, int(m).bit_length()) for v, m in zip(L.limbs_to_ints(c), ms)]

    def sample_r(self, rng: Rng) -> int:
        """Paillier::sample_r (paillier.cpp:233-239), one value."""
        out = np.zeros((1, self.L), np.uint32)
        st = C.c_uint64(rng.state)
        _raise_for(L.lib().pcb_sample_r(self._ctx, C.byref(st), 1, L.ptr(out), None), "sample_r")
        rng.state = st.value
        return L.limbs_to_int(out[0])

    def encrypt_with_r(self, m: int, r: int) -> Ciphertext:
        return self._enc_list([m], [r], use_crt=False)[0]

    def crt_encrypt_with_r(self, m: int, r: int) -> Ciphertext:
        self._need_prv()
        return self._enc_list([m], [r], use_crt=True)[0]

    def make_rn_factor(self, r: int) -> "RnFactor":
        """Paillier::make_rn_factor (paillier.cpp:371-383): r^n mod n^2 (= Enc(0; r)) and, with the
        private key, its residues mod p^2 / q^2."""
        if not 0 < r < self.n:
            raise ValueError("randomness not in [1, n)")
        full = self._enc_list([0], [r], use_crt=self._has_prv)[0].value
        if not self._has_prv:
            return RnFactor(r, full, 0, 0)
        return RnFactor(r, full, full % (self._p * self._p), full % (self._q * self._q))

    def encrypt_with_factor(self, m: int, f: "RnFactor") -> Ciphertext:
        """encrypt_with_factor (paillier.cpp:385-389): c = (1 + m n) f.full mod n^2, one multiply."""
        if not f.full:
            raise ValueError("factor missing r^n")
        W = 2 * self.L
        st = np.zeros(1, np.int32)
        c = self.encrypt_rn_batch(L.ints_to_limbs([m], self.L), L.ints_to_limbs([f.full], W), status=st)
        _raise_for(int(st[0]), "element 0")
        return Ciphertext(L.limbs_to_int(c[0]), int(m).bit_length())

    def crt_encrypt_with_factor(self, m: int, f: "RnFactor") -> Ciphertext:
        """crt_encrypt_with_factor (paillier.cpp:391-400): the same residue as encrypt_with_factor."""
        self._need_prv()
        if not f.half_p2 or not f.half_q2:
            raise ValueError("factor missing split residues")
        return self.encrypt_with_factor(m, f)

    def finish_split_encrypt_with_factor(self, m: int, p2_g_power: int, f: "RnFactor") -> Ciphertext:
        """finish_split_encrypt_with_factor (paillier.cpp:416-426) through pcb_finish_split_encrypt_rn."""
        self._need_prv()
        if not f.half_p2 or not f.half_q2:
            raise ValueError("factor missing split residues")
        W = 2 * self.L
        st = np.zeros(1, np.int32)
        c = self.finish_split_encrypt_rn_batch(L.ints_to_limbs([m], self.L),
                                               L.ints_to_limbs([int(p2_g_power) % self.n2], W),
                                               L.ints_to_limbs([f.full], W), status=st)
        _raise_for(int(st[0]), "element 0")
        return Ciphertext(L.limbs_to_int(c[0]), int(m).bit_length())

    def encrypt_vec(self, ms, rng: Rng, use_crt: bool) -> list[Ciphertext]:
        """Paillier::encrypt_vec (paillier.cpp:495-507): r drawn serially (here: on the GPU, same
        stream), then one batched encryption."""
        if use_crt:
            self._need_prv()
        rs = []
        if ms:
            out = np.zeros((len(ms), self.L), np.uint32)
            st = C.c_uint64(rng.state)
            _raise_for(L.lib().pcb_sample_r(self._ctx, C.byref(st), len(ms), L.ptr(out), None), "sample_r")
            rng.state = st.value
            rs = L.limbs_to_ints(out)
        return self._enc_list(list(ms), rs, use_crt)

    def _dec_list(self, cs, use_crt):
        self._need_prv()
        vals = [c.value if isinstance(c, Ciphertext) else int(c) for c in cs]
        if not vals:
            return []
        if any(v.bit_length() > 64 * self.L for v in vals):
            raise ValueError("ciphertext not below n^2")
        Cl = L.ints_to_limbs(vals, 2 * self.L)
        st = np.zeros(len(vals), np.int32)
        m = self.decrypt_batch(Cl, use_crt, status=st)
        bad = np.nonzero(st)[0]
        if len(bad):
            _raise_for(int(st[bad[0]]), f"element {int(bad[0])}")
        return L.limbs_to_ints(m)

    def decrypt(self, c) -> int:
        return self._dec_list([c], use_crt=False)[0]

    def crt_decrypt(self, c) -> int:
        return self._dec_list([c], use_crt=True)[0]

    def decrypt_vec(self, cs, use_crt: bool) -> list[int]:
        return self._dec_list(cs, use_crt)

    # ---- collaborative variant (paper Alg. 3, paillier.cpp:363-426; protocol.cpp:11-18) ---------
    def decrypt_with_half(self, c, p2_power: int) -> int:
        """Paillier::decrypt_with_half: the p^2 side comes from an edge (delegated_power)."""
        self._need_prv()
        v = c.value if isinstance(c, Ciphertext) else int(c)
        if v.bit_length() > 64 * self.L:
            raise ValueError("ciphertext not below n^2")
        W = 2 * self.L
        p2 = int(p2_power) % (self.n * self.n)  # the GPU path reduces mod p^2; any representative < n^2
        Cl, Pl = L.ints_to_limbs([v], W), L.ints_to_limbs([p2], W)
        m = np.zeros((1, self.L), np.uint32)
        st = np.zeros(1, np.int32)
        _raise_for(L.lib().pcb_decrypt_with_half(self._ctx, L.ptr(Cl), L.ptr(Pl), W, 1, L.ptr(m), L.ptr(st), None),
                   "decrypt_with_half")
        _raise_for(int(st[0]), "element 0")
        return L.limbs_to_int(m[0])

    def finish_split_encrypt(self, m: int, p2_g_power: int, r: int) -> Ciphertext:
        """Paillier::finish_split_encrypt: the p^2-side g-power comes from an edge."""
        self._need_prv()
        W = 2 * self.L
        M, R = L.ints_to_limbs([m], self.L), L.ints_to_limbs([r], self.L)
        G = L.ints_to_limbs([int(p2_g_power) % (self.n * self.n)], W)
        c = np.zeros((1, W), np.uint32)
        st = np.zeros(1, np.int32)
        _raise_for(L.lib().pcb_finish_split_encrypt(self._ctx, L.ptr(M), self.L, L.ptr(G), W, L.ptr(R), 1, L.ptr(c),
                                                    L.ptr(st), None), "finish_split_encrypt")
        _raise_for(int(st[0]), "element 0")
        return Ciphertext(L.limbs_to_int(c[0]), int(m).bit_length())

    @staticmethod
    def obfuscate_exponent(value: int, n_eps: int, mask: int) -> int:
        """protocol.cpp:11-13: value + mask * n_eps (host-side integer)."""
        return int(value) + (int(mask) & MASK64) * int(n_eps)

    # ---- homomorphic operations (paillier.cpp:428-493) ----------------------------------------
    def _nbits(self) -> int:
        return self.n.bit_length()

    def _bump(self, bits: int) -> None:
        """bump_bits_or_throw (paillier.cpp:245-251)."""
        if bits >= self._nbits():
            raise OverflowError("homomorphic accumulation exceeds plaintext space")

    def _cw(self, cs):
        vals = [c.value if isinstance(c, Ciphertext) else int(c) for c in cs]
        return L.ints_to_limbs(vals, 2 * self.L)

    def hom_add_batch(self, a, b):
        """out_i = a_i b_i mod n^2 on (count, 2L) limb arrays / tensors."""
        dev = hasattr(a, "is_cuda") and a.is_cuda
        out = _torch().empty_like(a) if dev else np.zeros_like(a)
        _raise_for(L.lib().pcb_hom_add(self._ctx, L.ptr(a), L.ptr(b), a.shape[0], L.ptr(out),
                                       self._stream() if dev else None), "hom_add")
        return out

    def hom_scalar_mul_batch(self, k, c):
        dev = hasattr(c, "is_cuda") and c.is_cuda
        out = _torch().empty_like(c) if dev else np.zeros_like(c)
        _raise_for(L.lib().pcb_hom_scalar_mul(self._ctx, L.ptr(k), L.ptr(c), c.shape[0], L.ptr(out),
                                              self._stream() if dev else None), "hom_scalar_mul")
        return out

    def aggregate_batch(self, c):
        """prod_i c_i mod n^2 (balanced product tree on the GPU) -> (2L,) limbs."""
        dev = hasattr(c, "is_cuda") and c.is_cuda
        out = _torch().empty((2 * self.L,), dtype=c.dtype, device=c.device) if dev else np.zeros(2 * self.L, np.uint32)
        _raise_for(L.lib().pcb_aggregate(self._ctx, L.ptr(c), c.shape[0], L.ptr(out),
                                         self._stream() if dev else None), "aggregate")
        return out

    def hom_add(self, a: Ciphertext, b: Ciphertext) -> Ciphertext:
        """Paillier::hom_add (paillier.cpp:428-432): bits = max + 1, overflow guard."""
        bits = max(a.plain_bits, b.plain_bits) + 1
        self._bump(bits)
        out = self.hom_add_batch(self._cw([a]), self._cw([b]))
        return Ciphertext(L.limbs_to_int(out[0]), bits)

    def hom_scalar_mul(self, k: int, c: Ciphertext) -> Ciphertext:
        """Paillier::hom_scalar_mul (paillier.cpp:434-439), k < 2^64."""
        bits = 0 if k == 0 else c.plain_bits + int(k).bit_length()
        self._bump(bits)
        out = self.hom_scalar_mul_batch(np.array([k], np.uint64), self._cw([c]))
        return Ciphertext(L.limbs_to_int(out[0]), bits)

    def hom_matvec_batch(self, alpha, expo, zv, window: int = 6):
        """out_i = alpha_i prod_j zv_j^expo[i][j] mod n^2 on limb arrays; expo (rows, cols) uint64."""
        rows = alpha.shape[0]
        cols = zv.shape[0]
        dev = hasattr(alpha, "is_cuda") and alpha.is_cuda
        out = _torch().empty_like(alpha) if dev else np.zeros_like(alpha)
        _raise_for(L.lib().pcb_hom_matvec(self._ctx, L.ptr(alpha), L.ptr(expo), L.ptr(zv), rows, cols, window,
                                          L.ptr(out), self._stream() if dev else None), "hom_matvec")
        return out

    def hom_matvec(self, alpha, expo, zv, window: int = 6) -> list[Ciphertext]:
        """Paillier::hom_matvec (paillier.cpp:441-493) incl. shape checks and plain_bits rules."""
        rows, cols = len(alpha), len(zv)
        if len(expo) != rows:
            raise ValueError("exponent row count")
        if any(len(r) != cols for r in expo):
            raise ValueError("exponent row width")
        if window < 1 or window > 8:
            raise ValueError("window in [1,8]")
        max_bits = max((int(k).bit_length() for r in expo for k in r), default=0)
        zv_bits = max((c.plain_bits for c in zv), default=0)
        sum_bits = max_bits + zv_bits + cols.bit_length() if cols else 0
        bits = [max(a.plain_bits, sum_bits) + 1 for a in alpha]
        for b in bits:
            self._bump(b)
        if rows == 0:
            return []
        E = np.array(expo, dtype=np.uint64).reshape(rows, cols)
        out = self.hom_matvec_batch(self._cw(alpha), E, self._cw(zv) if cols else np.zeros((0, 2 * self.L), np.uint32),
                                    window)
        return [Ciphertext(v, b) for v, b in zip(L.limbs_to_ints(out), bits)]

    def edge_step_batch(self, alpha, expo, zc, vc, window: int = 6):
        """protocol.cpp:264-271: range check, zv = hom_add(z, v), then hom_matvec (square block)."""
        cols = zc.shape[0]
        dev = hasattr(alpha, "is_cuda") and alpha.is_cuda
        out = _torch().empty_like(alpha) if dev else np.zeros_like(alpha)
        _raise_for(L.lib().pcb_edge_step(self._ctx, L.ptr(alpha), L.ptr(expo), L.ptr(zc), L.ptr(vc), cols, window,
                                         L.ptr(out), self._stream() if dev else None), "edge_step")
        return out

    def edge_step_blocks_batch(self, sizes, alpha, expo, zc, vc, window: int = 6):
        """pcb_edge_step_blocks: the edge steps of len(sizes) square blocks in one batch (block k's
        rows / columns are the next sizes[k] ciphertexts; expo holds the sizes[k]^2 exponents of
        each block back to back, row-major)."""
        sz = np.ascontiguousarray(np.asarray(sizes, dtype=np.uint32))
        dev = hasattr(alpha, "is_cuda") and alpha.is_cuda
        out = _torch().empty_like(alpha) if dev else np.zeros_like(alpha)
        _raise_for(L.lib().pcb_edge_step_blocks(self._ctx, len(sz), sz.ctypes.data, L.ptr(alpha), L.ptr(expo),
                                                L.ptr(zc), L.ptr(vc), window, L.ptr(out),
                                                self._stream() if dev else None), "edge_step_blocks")
        return out

    def aggregate(self, cs) -> Ciphertext:
        """prod c_i mod n^2; plain_bits follows a balanced hom_add tree (depth ceil(log2 count))."""
        cs = list(cs)
        bits = max(c.plain_bits for c in cs) + (len(cs) - 1).bit_length()
        self._bump(bits)
        out = self.aggregate_batch(self._cw(cs))
        return Ciphertext(L.limbs_to_int(out), bits)


class CrtShare:
    """An edge's share of the private key (paillier.hpp:64-66: p^2 and phi(p^2)) on the device."""

    def __init__(self, p2: int, phi_p2: int, device: int = 0):
        self.p2, self.phi_p2 = int(p2), int(phi_p2)
        self.S = (self.p2.bit_length() + 31) // 32
        a = L.int_to_limbs(self.p2, self.S)
        b = L.int_to_limbs(self.phi_p2, self.S)
        h = C.c_void_p()
        _raise_for(L.lib().pcb_share_create(C.byref(h), device, a.ctypes.data_as(L._u32p), self.S,
                                            b.ctypes.data_as(L._u32p), self.S), "share")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and L is not None and L._lib is not None:
            L._lib.pcb_share_destroy(h)
            self._h = None

    def delegated_power_tensor(self, base, obf, stream=None):
        """Device tensors (int32 limb views): base (count, <= 2S), obf (count, k) -> (count, S)
        tensor of (base mod p^2)^(obf mod phi(p^2)) mod p^2, exponent reduction on the device."""
        torch = _torch()
        out = torch.empty((base.shape[0], self.S), dtype=torch.int32, device=base.device)
        _raise_for(L.lib().pcb_delegated_power(self._h, L.ptr(base), base.shape[1], L.ptr(obf), obf.shape[1],
                                               base.shape[0], L.ptr(out), stream), "delegated_power")
        return out

    def delegated_power_fermat_tensor(self, base, u_mont, stream=None):
        """Device tensors: base (count, <= 2S), u_mont (count, S/2: u R mod p) -> (count, S) tensor of
        (base mod p^2)^(u (p - 1)) mod p^2 (pcb_delegated_power_fermat: one |p|-bit chain)."""
        torch = _torch()
        out = torch.empty((base.shape[0], self.S), dtype=torch.int32, device=base.device)
        _raise_for(L.lib().pcb_delegated_power_fermat(self._h, L.ptr(base), base.shape[1], L.ptr(u_mont),
                                                      base.shape[0], L.ptr(out), stream), "delegated_power_fermat")
        return out

    def fermat_factor(self, obf: int):
        """(u R mod p) limbs when obf mod phi(p^2) = u (p - 1) with u != 0 (the Fermat form), else None."""
        p = self.p2 - self.phi_p2
        if p * p != self.p2 or self.S not in (64, 96, 128):  # the widths pcb_delegated_power_fermat serves
            return None
        u, w = divmod(int(obf) % self.phi_p2, p - 1)
        if w or not u:
            return None
        return L.int_to_limbs(u * (1 << (16 * self.S)) % p, self.S // 2)

    def delegated_power_binomial_tensor(self, n_limbs, obf, stream=None):
        """delegated_power with base g = n + 1 for every element (n_limbs: the n limbs, a device
        tensor or host array): 1 + (obf mod phi(p^2)) n mod p^2, no exponentiation, same bits."""
        torch = _torch()
        out = torch.empty((obf.shape[0], self.S), dtype=torch.int32, device=obf.device)
        _raise_for(L.lib().pcb_delegated_power_binomial(self._h, L.ptr(n_limbs), n_limbs.shape[-1], L.ptr(obf),
                                                        obf.shape[1], obf.shape[0], L.ptr(out), stream),
                   "delegated_power_binomial")
        return out

    def delegated_power_batch(self, base, obf):
        """base: (count, <= 2S) limbs, obf: (count, k) limbs -> (count, S) limbs of
        (base mod p^2)^(obf mod phi(p^2)) mod p^2."""
        base = np.ascontiguousarray(base, np.uint32)
        obf = np.ascontiguousarray(obf, np.uint32)
        out = np.zeros((base.shape[0], self.S), np.uint32)
        _raise_for(L.lib().pcb_delegated_power(self._h, L.ptr(base), base.shape[1], L.ptr(obf), obf.shape[1],
                                               base.shape[0], L.ptr(out), None), "delegated_power")
        return out


def crt_share(kp: KeyPair, device: int = 0) -> CrtShare:
    """pcadmm::crt_share (paillier.hpp:95): what the master hands an edge in the collaborative variant."""
    p2 = kp.p * kp.p
    return CrtShare(p2, p2 - kp.p, device)


def delegated_power(base: int, obf: int, share: CrtShare) -> int:
    """protocol.cpp:15-18, one value."""
    W = 2 * share.S
    out = share.delegated_power_batch(L.ints_to_limbs([int(base) % (1 << (32 * W))], W),
                                      L.ints_to_limbs([int(obf)], max(1, (int(obf).bit_length() + 31) // 32)))
    return L.limbs_to_int(out[0])

