"""Every batched entry point at every key size the reference handles (1024, 2048 and 4096 from
keygen; 3072 via keypair_from_primes) against the compiled reference
(oracle/_ref/libpcref.so) on the same key and inputs: sample_r, CRT and public-key encryption,
CRT and direct decryption, hom_matvec, the collaborative finish_split_encrypt / decrypt_with_half,
and hom_add / hom_scalar_mul / aggregate against Python integers."""
import math
import os
import random

import numpy as np
import pytest

import refbind as R_
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1


def _key(bits):
    if bits == 3072:
        rng = P.Rng(3072)
        while True:
            p, q = P.random_prime(rng, 1536, device=0), P.random_prime(rng, 1536, device=0)
            if p != q and (p * q).bit_length() == 3072:
                return P.keypair_from_primes(p, q), R_.RefKey.from_primes(p, q)
    kp = P.keygen(P.Rng(bits + 1), bits, device=0)
    return kp, R_.RefKey.from_primes(kp.p, kp.q)


@pytest.fixture(scope="module", params=[1024, 2048, 3072, 4096])
def sized(request):
    return request.param, *_key(request.param)


def test_encrypt_decrypt_and_r_stream(sized):
    bits, kp, ref = sized
    ph = P.Paillier(kp)
    assert ref.n == kp.n
    count = 150
    rnd = random.Random(bits)
    ms = [rnd.randrange(0, kp.n) for _ in range(count - 2)] + [0, kp.n - 1]
    M = L.ints_to_limbs(ms, ph.L)
    r_ref, _ = ref.sample_r(bits, count)
    assert np.array_equal(ph.sample_r_batch(P.Rng(bits), count).cpu().numpy().view(np.uint32), r_ref)
    for crt in (True, False):
        cref, st = ref.encrypt(M, r_ref, crt=crt, threads=THREADS)
        assert (st == 0).all()
        assert np.array_equal(ph.encrypt_batch(M, np.ascontiguousarray(r_ref), use_crt=crt), cref), crt
        mref, st = ref.decrypt(cref, crt=crt, threads=THREADS)
        assert (st == 0).all()
        assert np.array_equal(ph.decrypt_batch(np.ascontiguousarray(cref), use_crt=crt), mref), crt
        assert L.limbs_to_ints(mref) == ms


def test_homomorphic_entries(sized):
    bits, kp, ref = sized
    edge = P.Paillier(P.PublicKey(kp.n, bits))
    n2 = kp.n * kp.n
    rnd = random.Random(bits + 7)
    a = [rnd.randrange(1, n2) for _ in range(24)]
    b = [rnd.randrange(1, n2) for _ in range(24)]
    ks = [rnd.getrandbits(64) for _ in range(24)]
    A, B = L.ints_to_limbs(a, 2 * edge.L), L.ints_to_limbs(b, 2 * edge.L)
    assert L.limbs_to_ints(edge.hom_add_batch(A, B)) == [x * y % n2 for x, y in zip(a, b)]
    assert L.limbs_to_ints(edge.hom_scalar_mul_batch(np.array(ks, np.uint64), A)) == \
        [pow(x, k, n2) for x, k in zip(a, ks)]
    assert L.limbs_to_ints(edge.aggregate_batch(A).reshape(1, -1))[0] == math.prod(a) % n2
    rows, cols = 5, 9
    E = np.array([[rnd.getrandbits(50) for _ in range(cols)] for _ in range(rows)], np.uint64)
    out = edge.hom_matvec_batch(A[:rows].copy(), E, B[:cols].copy())
    o = np.zeros((rows, 2 * edge.L), np.uint32)
    assert R_.lib().pcref_hom_matvec(ref.h, R_.a(np.ascontiguousarray(A[:rows])), None, R_.a(E),
                                     R_.a(np.ascontiguousarray(B[:cols])), None, rows, cols, 6, 2 * edge.L, R_.a(o),
                                     None, 1) == 0
    assert np.array_equal(out, o)


def test_collaborative_entries(sized):
    """finish_split_encrypt / decrypt_with_half (paillier.cpp:363-414) vs the compiled reference;
    the collaborative share needs p^2 above 1024 bits (keys of 2048 bits and more)."""
    bits, kp, ref = sized
    if bits < 2048:
        pytest.skip("the delegated p^2 side needs a 2048-bit or larger key")
    ph = P.Paillier(kp)
    p2 = kp.p * kp.p
    rnd = random.Random(bits + 11)
    count = 40
    ms = [rnd.getrandbits(60) for _ in range(count)]
    rs = [rnd.randrange(1, kp.n) for _ in range(count)]
    gp = [rnd.randrange(0, p2) for _ in range(count)]  # any p^2-side g power the edge returns
    W = 2 * ph.L
    M, R, G = L.ints_to_limbs(ms, ph.L), L.ints_to_limbs(rs, ph.L), L.ints_to_limbs(gp, W)
    c = np.zeros((count, W), np.uint32)
    st = np.zeros(count, np.int32)
    assert L.lib().pcb_finish_split_encrypt(ph._ctx, L.ptr(M), ph.L, L.ptr(G), W, L.ptr(R), count, L.ptr(c),
                                           L.ptr(st), None) == 0 and not st.any()
    cref, st_ref = ref.finish_split_encrypt(M, G, R)
    assert not st_ref.any() and np.array_equal(c, cref)
    px = [rnd.randrange(1, p2) for _ in range(count)]
    PX = L.ints_to_limbs(px, W)
    m = np.zeros((count, ph.L), np.uint32)
    st = np.zeros(count, np.int32)
    L.lib().pcb_decrypt_with_half(ph._ctx, L.ptr(c), L.ptr(PX), W, count, L.ptr(m), L.ptr(st), None)
    mref, st_ref = ref.decrypt_with_half(c, PX)
    assert np.array_equal(st, st_ref) and np.array_equal(m[st == 0], mref[st_ref == 0])
