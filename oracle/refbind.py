"""ctypes binding of oracle/_ref/libpcref.so — the UNMODIFIED reference hot path compiled from
/root/reference by oracle/Makefile.  TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's
cpu_baseline and --impl reference legs).  Values cross as fixed-width LE u32 limb arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libpcref.so"

_vp, _u32p, _u64p, _i32p, _f64p = C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p
_SIGS = {
    "pcref_keygen": (C.c_void_p, [C.c_uint64, C.c_uint32, C.c_int, C.POINTER(C.c_uint64)]),
    "pcref_from_primes": (C.c_void_p, [_u32p, _u32p, C.c_uint32, C.c_int, C.c_uint64]),
    "pcref_free": (None, [_vp]),
    "pcref_n_bits": (C.c_uint32, [_vp]),
    "pcref_get": (C.c_int, [_vp, C.c_int, _u32p, C.c_uint32]),
    "pcref_serialize": (C.c_size_t, [_vp, C.c_void_p, C.c_size_t]),
    "pcref_parse": (C.c_void_p, [C.c_void_p, C.c_size_t]),
    "pcref_sample_r": (None, [_vp, C.POINTER(C.c_uint64), C.c_size_t, _u32p, C.c_uint32]),
    "pcref_encrypt": (None, [_vp, C.c_int, _u32p, C.c_uint32, _u32p, C.c_uint32, C.c_size_t, _u32p, C.c_uint32,
                             _i32p, C.c_int]),
    "pcref_decrypt": (None, [_vp, C.c_int, _u32p, C.c_uint32, C.c_size_t, _u32p, C.c_uint32, _i32p, C.c_int]),
    "pcref_decrypt_with_half": (None, [_vp, _u32p, C.c_uint32, _u32p, C.c_uint32, C.c_size_t, _u32p, C.c_uint32,
                                       _i32p]),
    "pcref_finish_split_encrypt": (None, [_vp, _u32p, C.c_uint32, _u32p, C.c_uint32, _u32p, C.c_uint32, C.c_size_t,
                                          _u32p, C.c_uint32, _i32p]),
    "pcref_hom_add": (None, [_vp, _u32p, _u32p, _u32p, _u32p, C.c_size_t, C.c_uint32, _u32p, _u32p, _i32p]),
    "pcref_hom_scalar_mul": (None, [_vp, _u64p, _u32p, _u32p, C.c_size_t, C.c_uint32, _u32p, _u32p, _i32p]),
    "pcref_hom_matvec": (C.c_int, [_vp, _u32p, _u32p, _u64p, _u32p, _u32p, C.c_size_t, C.c_size_t, C.c_uint32,
                                   C.c_uint32, _u32p, _u32p, C.c_int]),
    "pcref_counters": (None, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "pcref_gamma2": (C.c_int, [_f64p, C.c_size_t, C.c_double, C.c_double, C.c_double, _u64p, _u64p]),
    "pcref_gamma1": (C.c_int, [_f64p, C.c_size_t, C.c_double, C.c_double, C.c_double, _u64p, _u64p]),
    "pcref_combined_update": (None, [_u64p, _u64p, _u64p, _u64p, C.c_size_t, C.c_size_t, _u64p]),
    "pcref_inverse_quantize_x": (None, [_u64p, _u64p, _u64p, _u64p, C.c_size_t, C.c_size_t, C.c_double,
                                        C.c_double, C.c_double, _f64p]),
    "pcref_widen_bounds": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]),
}
_lib = None


def available() -> bool:
    return REF_SO.exists()


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle)")
        L = C.CDLL(str(REF_SO))
        for k, (res, args) in _SIGS.items():
            f = getattr(L, k)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def a(x: np.ndarray):
    return C.c_void_p(x.ctypes.data) if x is not None else None


def limbs(vals, n):
    out = np.zeros((len(vals), n), np.uint32)
    for i, v in enumerate(vals):
        out[i] = np.frombuffer(int(v).to_bytes(4 * n, "little"), np.uint32)
    return out


def ints(arr):
    return [int.from_bytes(np.ascontiguousarray(r, np.uint32).tobytes(), "little") for r in np.atleast_2d(arr)]


class RefKey:
    """A reference KeyPair + Paillier instance (paillier.hpp:54-58, 104-181)."""

    def __init__(self, handle):
        if not handle:
            raise ValueError("reference key construction failed")
        self.h = C.c_void_p(handle)
        self.bits = lib().pcref_n_bits(self.h)
        self.L = (self.bits + 31) // 32

    @classmethod
    def keygen(cls, seed: int, bits: int):
        st = C.c_uint64(seed)
        k = cls(lib().pcref_keygen(seed, bits, 1, C.byref(st)))
        k.rng_state_after = st.value
        return k

    @classmethod
    def from_primes(cls, p: int, q: int):
        w = max(p.bit_length(), q.bit_length()) // 32 + 1
        P, Q = limbs([p], w), limbs([q], w)
        return cls(lib().pcref_from_primes(a(P), a(Q), w, 1, 1))

    def get(self, which: int, width: int | None = None) -> int:
        width = width or 2 * self.L + 2
        out = np.zeros(width, np.uint32)
        lib().pcref_get(self.h, which, a(out), width)
        return ints(out)[0]

    @property
    def n(self): return self.get(0)
    @property
    def p(self): return self.get(1)
    @property
    def q(self): return self.get(2)

    def serialize(self) -> bytes:
        n = lib().pcref_serialize(self.h, None, 0)
        buf = np.zeros(n, np.uint8)
        lib().pcref_serialize(self.h, a(buf), n)
        return buf.tobytes()

    def sample_r(self, state: int, count: int):
        st = C.c_uint64(state)
        out = np.zeros((count, self.L), np.uint32)
        lib().pcref_sample_r(self.h, C.byref(st), count, a(out), self.L)
        return out, st.value

    def encrypt(self, m: np.ndarray, r: np.ndarray, crt: bool = True, threads: int = 1):
        m = np.ascontiguousarray(m, np.uint32)
        r = np.ascontiguousarray(r, np.uint32)
        n = m.shape[0]
        c = np.zeros((n, 2 * self.L), np.uint32)
        st = np.zeros(n, np.int32)
        lib().pcref_encrypt(self.h, 1 if crt else 0, a(m), m.shape[1], a(r), r.shape[1], n, a(c), 2 * self.L, a(st),
                            threads)
        return c, st

    def decrypt(self, c: np.ndarray, crt: bool = True, threads: int = 1):
        c = np.ascontiguousarray(c, np.uint32)
        n = c.shape[0]
        m = np.zeros((n, self.L), np.uint32)
        st = np.zeros(n, np.int32)
        lib().pcref_decrypt(self.h, 1 if crt else 0, a(c), c.shape[1], n, a(m), self.L, a(st), threads)
        return m, st

    def decrypt_with_half(self, c: np.ndarray, p2: np.ndarray):
        c, p2 = np.ascontiguousarray(c, np.uint32), np.ascontiguousarray(p2, np.uint32)
        n = c.shape[0]
        m = np.zeros((n, self.L), np.uint32)
        st = np.zeros(n, np.int32)
        lib().pcref_decrypt_with_half(self.h, a(c), c.shape[1], a(p2), p2.shape[1], n, a(m), self.L, a(st))
        return m, st

    def finish_split_encrypt(self, m: np.ndarray, g: np.ndarray, r: np.ndarray):
        m, g, r = (np.ascontiguousarray(v, np.uint32) for v in (m, g, r))
        n = m.shape[0]
        c = np.zeros((n, 2 * self.L), np.uint32)
        st = np.zeros(n, np.int32)
        lib().pcref_finish_split_encrypt(self.h, a(m), m.shape[1], a(g), g.shape[1], a(r), r.shape[1], n, a(c),
                                         2 * self.L, a(st))
        return c, st

    def __del__(self):
        try:
            lib().pcref_free(self.h)
        except Exception:
            pass


def gamma2(v, zmin, zmax, delta):
    v = np.ascontiguousarray(v, np.float64)
    out = np.zeros(len(v), np.uint64)
    cl = np.zeros(2, np.uint64)
    rc = lib().pcref_gamma2(a(v), len(v), zmin, zmax, delta, a(out), a(cl))
    return out, cl, rc


def gamma1(v, zmin, zmax, delta):
    v = np.ascontiguousarray(v, np.float64)
    out = np.zeros(2 * len(v), np.uint64)
    cl = np.zeros(2, np.uint64)
    rc = lib().pcref_gamma1(a(v), len(v), zmin, zmax, delta, a(out), a(cl))
    return out.reshape(-1, 2), cl, rc
