"""GPU cross-checks between the modular-exponentiation cores, through the C ABI.

The streaming RNS core (rnsx.cu) is the default for 2048/3072-bit CRT halves and for n^2 up to
4096 bits; its two-tile (ping-pong) variant runs once a batch gives every SM two tiles.  These
tests pin every variant to the independent cores (CIOS carry chains / radix-2^28, selected with
PCB_RNSX=0 / PCB_RNSX_N2=0) and to Python big-int arithmetic on full-GPU batch sizes, where the
parity tests' small batches do not reach."""
import os
import random

import numpy as np
import pytest

from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu


def _key2048():
    return P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)


def _ctx(kp, **env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return P.Paillier(kp)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_engines_reported():
    kp = _key2048()
    assert L.lib().pcb_ctx_engine(_ctx(kp)._ctx) == 3             # streaming RNS core
    assert L.lib().pcb_ctx_engine(_ctx(kp, PCB_RNSX=0)._ctx) == 1  # resident-matrix RNS core


@pytest.mark.parametrize("n_el", [300, 40000])
def test_rnsx_pingpong_and_single_tile_match_other_core(n_el):
    """40000 values give every SM two tiles: the ping-pong path; 300 values: one tile per CTA."""
    torch = pytest.importorskip("torch")
    kp = _key2048()
    rx, base = _ctx(kp), _ctx(kp, PCB_RNSX=0)
    g = np.random.default_rng(n_el)
    m = torch.from_numpy(g.integers(0, 2**32, (n_el, rx.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
    m[:, rx.L - 1] = 0
    m[0] = 0
    r = rx.sample_r_batch(P.Rng(7), n_el)
    c1, c0 = rx.encrypt_batch(m, r, True), base.encrypt_batch(m, r, True)
    assert torch.equal(c1, c0)
    os.environ["PCB_RNSX_PP"] = "0"
    try:
        assert torch.equal(rx.encrypt_batch(m, r, True), c1)
    finally:
        os.environ.pop("PCB_RNSX_PP", None)
    d = rx.decrypt_batch(c1, True)
    assert torch.equal(d, m)
    # spot-check against Python integers
    M, R, C = (t.cpu().numpy().view(np.uint32) for t in (m, r, c1))
    n, n2 = kp.n, kp.n * kp.n
    for i in list(range(3)) + [n_el - 1]:
        mi, ri = L.limbs_to_ints(M[i:i + 1])[0], L.limbs_to_ints(R[i:i + 1])[0]
        assert L.limbs_to_ints(C[i:i + 1])[0] == (1 + mi * n) * pow(ri, n, n2) % n2


def test_public_encrypt_n2_core_matches_radix_core():
    """Public-key (edge) encryption at n^2 = 4096 bits: rnsx_kernel<144> vs the radix-2^27 core."""
    kp = _key2048()
    pub = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    old = os.environ.get("PCB_RNSX_N2")
    os.environ["PCB_RNSX_N2"] = "0"
    try:
        pub_radix = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    finally:
        if old is None:
            os.environ.pop("PCB_RNSX_N2", None)
        else:
            os.environ["PCB_RNSX_N2"] = old
    rnd = random.Random(3)
    n_el = 700
    ms = [rnd.getrandbits(60) for _ in range(n_el - 2)] + [0, kp.n - 1]
    rs = [rnd.randrange(1, kp.n) for _ in range(n_el)]
    M, R = L.ints_to_limbs(ms, pub.L), L.ints_to_limbs(rs, pub.L)
    st = np.zeros(n_el, np.int32)
    a = pub.encrypt_batch(M, R, use_crt=False, status=st)
    b = pub_radix.encrypt_batch(M, R, use_crt=False)
    assert (st == 0).all() and (a == b).all()
    n2 = kp.n * kp.n
    for i in (0, 1, n_el - 2, n_el - 1):
        assert L.limbs_to_ints(a[i:i + 1])[0] == (1 + ms[i] * kp.n) * pow(rs[i], kp.n, n2) % n2


def test_matvec_n2_core_matches_radix_core_full_block():
    """A 512 x 64 block (rows x columns, 50-bit exponents) through both n^2 cores."""
    kp = _key2048()
    old = os.environ.get("PCB_RNSX_N2")
    pub = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    os.environ["PCB_RNSX_N2"] = "0"
    try:
        pub_radix = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    finally:
        if old is None:
            os.environ.pop("PCB_RNSX_N2", None)
        else:
            os.environ["PCB_RNSX_N2"] = old
    rnd = random.Random(9)
    rows, cols, n2 = 512, 64, kp.n * kp.n
    W = 2 * pub.L
    alpha = L.ints_to_limbs([rnd.randrange(1, n2) for _ in range(rows)], W)
    zv = L.ints_to_limbs([rnd.randrange(1, n2) for _ in range(cols)], W)
    E = np.array([[rnd.getrandbits(50) for _ in range(cols)] for _ in range(rows)], np.uint64)
    a = pub.hom_matvec_batch(alpha, E, zv)
    b = pub_radix.hom_matvec_batch(alpha, E, zv)
    assert (a == b).all()


@pytest.mark.parametrize("bits", [2048, 3072])
def test_split_encryption_matches_single_pass(bits):
    """Split CRT Enc (r^n mod p^2 = ((r mod p)^q mod p)^p mod p^2) against the
    single r^n pass (PCB_ENC_SPLIT=0), the carry-core stage 1 (PCB_ENC_SPLIT=1, 2048-bit) and Python
    integers, on a full-GPU batch with edge randomness: r = 1, n - 1, multiples of p and of q."""
    torch = pytest.importorskip("torch")
    if bits == 2048:
        kp = _key2048()
    else:
        rng = P.Rng(3072)
        while True:
            p, q = P.random_prime(rng, 1536), P.random_prime(rng, 1536)
            if p != q and (p * q).bit_length() == 3072:
                break
        kp = P.keypair_from_primes(p, q)
    n_el = 40000
    split, single = _ctx(kp), _ctx(kp, PCB_ENC_SPLIT=0)
    g = np.random.default_rng(bits)
    m = torch.from_numpy(g.integers(0, 2**32, (n_el, split.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
    m[:, split.L - 1] = 0
    r = split.sample_r_batch(P.Rng(11), n_el)
    n, p, q = kp.n, kp.p, kp.q
    edge = [1, n - 1, p, q, 3 * p, 5 * q, n - p]
    r[:len(edge)] = torch.from_numpy(L.ints_to_limbs(edge, split.L).view(np.int32)).cuda()
    c1, c0 = split.encrypt_batch(m, r, True), single.encrypt_batch(m, r, True)
    assert torch.equal(c1, c0)
    if bits == 2048:
        assert torch.equal(_ctx(kp, PCB_ENC_SPLIT=1).encrypt_batch(m, r, True), c1)
    M, R, C = (t.cpu().numpy().view(np.uint32) for t in (m, r, c1))
    # every edge row (r = 1, n - 1, multiples of p and q) and a sample of the batch, exactly
    # equal to the compiled reference's crt_encrypt_with_r (paillier.cpp:334-344)
    import os
    import refbind as RB
    rows = list(range(len(edge) + 64)) + [n_el - 1]
    ref = RB.RefKey.from_primes(p, q)
    cref, st = ref.encrypt(M[rows], R[rows], crt=True, threads=os.cpu_count() or 1)
    assert (st == 0).all()
    assert np.array_equal(C[rows], cref)
    n2 = n * n
    for i in rows[:len(edge)]:  # and the closed form with Python integers
        mi, ri = L.limbs_to_ints(M[i:i + 1])[0], L.limbs_to_ints(R[i:i + 1])[0]
        assert L.limbs_to_ints(C[i:i + 1])[0] == (1 + mi * n) * pow(ri, n, n2) % n2, i
    assert torch.equal(split.decrypt_batch(c1[len(edge):], True), m[len(edge):])
