"""4096-bit keys -- the largest size the reference's keygen accepts (paillier.cpp:107-109) -- on the
device: the key from the batched Miller-Rabin keygen equals the compiled reference's keygen on the
same seed; CRT encryption (split form: r^q mod p on rnsx_kernel<72>, (1 + m n) u^p mod p^2 on
rnsx_kernel<144>), the public-key n^2 = 8192-bit encryption (radix core), CRT decryption, the
r streams and the homomorphic operations are bit-identical to the compiled reference
(oracle/_ref/libpcref.so) or to Python integers."""
import os
import random

import numpy as np
import pytest

import refbind as R_
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1
SEED = 4096


@pytest.fixture(scope="module")
def keys():
    kp = P.keygen(P.Rng(SEED), 4096, device=0)
    ref = R_.RefKey.keygen(SEED, 4096)
    return kp, ref


def test_keygen_4096_equals_reference(keys):
    kp, ref = keys
    assert (kp.n, kp.p, kp.q) == (ref.n, ref.p, ref.q) and kp.n.bit_length() == 4096
    r = P.Rng(SEED)
    P.keygen(r, 4096, device=0)
    assert r.state == ref.rng_state_after


def test_crt_and_public_encryption_and_decryption_match_reference(keys):
    kp, ref = keys
    ph = P.Paillier(kp)
    assert ph.L == 128
    count = 300  # > 2 tiles of the RNS core
    rnd = random.Random(7)
    ms = [rnd.getrandbits(60) for _ in range(count - 3)] + [0, 1, kp.n - 1]
    M = L.ints_to_limbs(ms, ph.L)
    r_ref, st_ref = ref.sample_r(2, count)
    r_dev = ph.sample_r_batch(P.Rng(2), count).cpu().numpy().view(np.uint32)
    assert np.array_equal(r_dev, r_ref)
    for crt in (True, False):
        cref, st = ref.encrypt(M, r_ref, crt=crt, threads=THREADS)
        assert (st == 0).all()
        c = ph.encrypt_batch(M, np.ascontiguousarray(r_ref), use_crt=crt)
        assert np.array_equal(c, cref), f"crt={crt}"
    mref, st = ref.decrypt(cref, crt=True, threads=THREADS)
    assert (st == 0).all()
    m = ph.decrypt_batch(np.ascontiguousarray(cref))
    assert np.array_equal(m, mref) and L.limbs_to_ints(m) == ms


def test_homomorphic_operations_and_aggregate(keys):
    kp, _ = keys
    ph = P.Paillier(kp)
    edge = P.Paillier(P.PublicKey(kp.n, 4096))
    n2 = kp.n * kp.n
    rnd = random.Random(11)
    ms = [rnd.getrandbits(40) for _ in range(40)]
    r = ph.sample_r_batch(P.Rng(5), 40).cpu().numpy().view(np.uint32)
    c = ph.encrypt_batch(L.ints_to_limbs(ms, ph.L), np.ascontiguousarray(r))
    cs = L.limbs_to_ints(c)
    s = edge.hom_add_batch(c[:20], c[20:])
    assert L.limbs_to_ints(s) == [(a * b) % n2 for a, b in zip(cs[:20], cs[20:])]
    ks = [rnd.getrandbits(50) for _ in range(20)]
    sm = edge.hom_scalar_mul_batch(np.array(ks, dtype=np.uint64), c[:20])
    assert L.limbs_to_ints(sm) == [pow(a, k, n2) for a, k in zip(cs[:20], ks)]
    agg = edge.aggregate_batch(c)
    d = ph.decrypt_batch(np.ascontiguousarray(agg.reshape(1, -1)))
    assert L.limbs_to_ints(d)[0] == sum(ms) % kp.n


@pytest.mark.parametrize("variant", ["basic", "collab"])
def test_session_4096_bit_exact_vs_shadow(keys, variant):
    """The encrypted ADMM session on a 4096-bit key (both variants; the collaborative one delegates
    the 4096-bit p^2 side to the edges) is bit-identical to the reference's shadow pipeline."""
    import admm_oracle as AO
    from paper_2601_14980_b200 import admm as ADMM

    kp, _ = keys
    iters = 3
    a, y, _ = AO.gen_gaussian_problem(24, 40, 0.1, 2)
    sizes = AO.split_columns(40, 2)
    fac, at = [], 0
    for c in sizes:
        fac.append(AO.node_factor(a[:, at:at + c], y, 1.0, 2))
        at += c
    spec = AO.session_bounds(a, y, 1.0, 1.0, iters, sizes, 1.5, 1e15, fac)
    res = ADMM.EncryptedSession(kp, ADMM.SessionConfig(nodes=2, iters=iters, variant=variant)).run(
        a, y, factors=fac, spec=spec)
    trace, z, v = AO.shadow_session_ref(fac, sizes, spec, 1.0, 1.0, iters)
    assert all(np.array_equal(res.x_trace[t], trace[t]) for t in range(iters))
    assert np.array_equal(res.z, z) and np.array_equal(res.v, v)
