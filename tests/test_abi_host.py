"""C-ABI library: loads, exports every symbol include/pcb200.h declares, host-side key work is
bit-exact with the reference, and compute entry points fail loudly without a GPU (no CPU
fallback).  CPU only."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import paillier as P


def header_symbols():
    txt = (ROOT / "include" / "pcb200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:pcb_status|void|uint32_t|uint64_t|int|double|const char\*)\s+(pcb_\w+)\(",
                                 txt, re.M)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(L.SIGNATURES), set(syms) ^ set(L.SIGNATURES)


def test_library_is_sm100a_only():
    out = Path(L.LIB_PATH).read_bytes()
    assert b"sm_100a" in out or b"sm_100" in out


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_host_keygen_bit_exact(idx):
    k = golden("keys.json")[idx]
    rng = P.Rng(k["seed"])
    kp = P.keygen(rng, k["bits"])
    assert kp.n == int(k["n"], 16) and kp.p == int(k["p"], 16) and kp.q == int(k["q"], 16)
    assert rng.state == k["rng_state_after"]


def test_keygen_rejects_unsupported_size():
    with pytest.raises(ValueError):
        P.keygen(P.Rng(3), 512)  # test_paillier.cpp:168-172


def test_random_prime_matches_oracle():
    import pcadmm_oracle as O

    r1, r2 = P.Rng(99), O.Rng(99)
    assert P.random_prime(r1, 256) == O.random_prime(r2, 256)
    assert r1.state == r2.state


def test_status_strings():
    lib = L.lib()
    assert lib.pcb_status_str(L.PCB_E_NOT_UNIT) == b"ciphertext outside the multiplicative group"
    assert lib.pcb_status_str(L.PCB_OK) == b"ok"


def test_compute_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    lib = L.lib()
    m = np.array([5], np.uint32)
    e = np.array([3], np.uint32)
    x = np.array([2], np.uint32)
    y = np.zeros(1, np.uint32)
    rc = lib.pcb_modexp_batch(L.ptr(m), 1, L.ptr(e), 1, L.ptr(x), 1, L.ptr(y), None)
    assert rc != L.PCB_OK
    n = L.int_to_limbs(35, 1)
    ctx = C.c_void_p()
    rc = lib.pcb_ctx_create(C.byref(ctx), 0, n.ctypes.data_as(L._u32p), 1,
                            L.int_to_limbs(5, 1).ctypes.data_as(L._u32p), L.int_to_limbs(7, 1).ctypes.data_as(L._u32p), 1)
    assert rc == L.PCB_E_CUDA


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_2601_14980_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "pcadmm_oracle" not in src and "refbind" not in src and "oracle/" not in src, f


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_key_record_matches_reference_serializer(idx):
    """serialize_keypair / parse_keypair (paillier.cpp:152-191): byte-identical to the compiled
    reference's record for the golden keys, round trip, and the reference's error cases."""
    import refbind as R_

    k = golden("keys.json")[idx]
    kp = P.KeyPair(int(k["n"], 16), int(k["p"], 16), int(k["q"], 16), k["bits"])
    rec = P.serialize_keypair(kp)
    if R_.available():
        assert rec == R_.RefKey.keygen(k["seed"], k["bits"]).serialize()
    assert P.parse_keypair(rec) == kp
    with pytest.raises(RuntimeError, match="not a key record"):
        P.parse_keypair(b"xx" + rec[2:])
    with pytest.raises(RuntimeError, match="version"):
        P.parse_keypair(rec[:2] + b"\x02" + rec[3:])
    bad = bytearray(rec)
    bad[-1] ^= 1  # mu's last byte: still parses (mu is not re-derived), n/p/q intact
    assert P.parse_keypair(bytes(bad)) == kp
    with pytest.raises(RuntimeError):
        P.parse_keypair(rec[:20])
