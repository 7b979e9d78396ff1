"""GPU parity for the public-key / homomorphic operations modulo n^2 (radix-2^r kernels), through
the C ABI, against the reference's golden vectors and Python big-int arithmetic."""
import random

import numpy as np
import pytest

import pcadmm_oracle as O
from conftest import golden
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu


def H(x):
    return int(x, 16)


def key(idx):
    k = golden("keys.json")[idx]
    return P.KeyPair(H(k["n"]), H(k["p"]), H(k["q"]), k["bits"])


@pytest.fixture(scope="module", params=[0, 1, 2], ids=["k64", "k1024", "k2048"])
def kk(request):
    kp = key(request.param)
    return request.param, kp, P.Paillier(kp), P.Paillier(P.PublicKey(kp.n, kp.key_bits))


def test_public_key_encrypt_matches_reference(kk):
    idx, kp, ph, pub = kk
    e = golden("encrypt.json")[idx]
    ms, rs, cs = [H(v) for v in e["m"]], [H(v) for v in e["r"]], [H(v) for v in e["c"]]
    st = np.zeros(len(ms), np.int32)
    c = pub.encrypt_batch(L.ints_to_limbs(ms, pub.L), L.ints_to_limbs(rs, pub.L), use_crt=False, status=st)
    assert (st == 0).all()
    assert L.limbs_to_ints(c) == cs  # encrypt_with_r == crt_encrypt_with_r (test_paillier.cpp:63-78)
    # error statuses of the public path
    st = np.zeros(3, np.int32)
    pub.encrypt_batch(L.ints_to_limbs([H(v) for v in e["bad_m"]], pub.L),
                      L.ints_to_limbs([H(v) for v in e["bad_r"]], pub.L), use_crt=False, status=st)
    assert st.tolist() == e["bad_status"]
    # decrypting the public-path ciphertexts with the private context
    assert ph.decrypt_vec([P.Ciphertext(v) for v in L.limbs_to_ints(c)], True) == ms


def test_public_context_refuses_private_ops(kk):
    idx, kp, ph, pub = kk
    with pytest.raises(P.LogicError):
        pub.decrypt(5)
    with pytest.raises(P.LogicError):
        pub.crt_encrypt_with_r(3, 2)


def test_hom_add_matches_bigint(kk):
    idx, kp, ph, pub = kk
    rnd = random.Random(idx)
    n2 = kp.n2
    a = [rnd.randrange(n2) for _ in range(257)] + [0, 1, n2 - 1]
    b = [rnd.randrange(n2) for _ in range(257)] + [n2 - 1, n2 - 1, n2 - 1]
    out = pub.hom_add_batch(L.ints_to_limbs(a, 2 * pub.L), L.ints_to_limbs(b, 2 * pub.L))
    assert L.limbs_to_ints(out) == [x * y % n2 for x, y in zip(a, b)]


def test_hom_add_decrypts_to_sum_and_guard(kk):
    idx, kp, ph, pub = kk
    rng = P.Rng(5)
    m1, m2 = 123456789, 987654321
    c1, c2 = ph.encrypt_vec([m1, m2], rng, True)
    s = pub.hom_add(c1, c2)
    assert ph.crt_decrypt(s) == (m1 + m2) % kp.n
    assert s.plain_bits == max(c1.plain_bits, c2.plain_bits) + 1
    big = P.Ciphertext(c1.value, kp.n.bit_length() - 1)
    with pytest.raises(OverflowError):  # bump_bits_or_throw (paillier.cpp:245-251)
        pub.hom_add(big, big)


def test_hom_scalar_mul_matches_bigint(kk):
    idx, kp, ph, pub = kk
    rnd = random.Random(10 + idx)
    n2 = kp.n2
    cs = [rnd.randrange(1, n2) for _ in range(200)]
    ks = [0, 1, 2, 3, 15, 16, 2**64 - 1, 2**63] + [rnd.getrandbits(64) for _ in range(192)]
    out = pub.hom_scalar_mul_batch(np.array(ks, np.uint64), L.ints_to_limbs(cs, 2 * pub.L))
    assert L.limbs_to_ints(out) == [pow(c, k, n2) for c, k in zip(cs, ks)]


def test_hom_scalar_mul_reference_semantics():
    # test_paillier.cpp:102-115 on the toy key
    ph = P.Paillier(P.keypair_from_primes(5, 7))
    rng = P.Rng(19)
    for m in (0, 1, 2, 5, 11):
        c = ph.encrypt_vec([m], rng, True)[0]
        for k in (0, 1, 2, 3):
            if k * m >= 35 or (m >= 8 and k >= 2):
                continue
            assert ph.crt_decrypt(ph.hom_scalar_mul(k, c)) == k * m
    c = ph.encrypt_vec([30], rng, True)[0]
    with pytest.raises(OverflowError):
        ph.hom_scalar_mul(64, c)


@pytest.mark.parametrize("count", [1, 2, 31, 32, 33, 1000, 1057])
def test_aggregate_product_tree(count):
    kp = key(1)
    pub = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    rnd = random.Random(count)
    cs = [rnd.randrange(1, kp.n2) for _ in range(count)]
    out = pub.aggregate_batch(L.ints_to_limbs(cs, 2 * pub.L))
    want = 1
    for c in cs:
        want = want * c % kp.n2
    assert L.limbs_to_int(out) == want


def test_aggregate_decrypts_to_sum():
    kp = key(2)
    ph = P.Paillier(kp)
    ms = [i * 1000003 for i in range(300)]
    cs = ph.encrypt_vec(ms, P.Rng(3), True)
    agg = ph.aggregate(cs)
    assert ph.crt_decrypt(agg) == sum(ms) % kp.n


def test_matvec_reference_recurrence_64bit():
    # test_paillier.cpp:285-321: rows 5, cols 4, 14-bit exponents, a zero entry and a zero row
    rng = P.Rng(77)
    kp = P.keygen(rng, 64)
    ph = P.Paillier(kp)
    ork = O.Rng(77)
    O.keygen(ork, 64)
    n = kp.n
    rows, cols = 5, 4
    alpha_m = [ork.below(1 << 20) for _ in range(rows)]
    zv_m = [ork.below(1 << 16) for _ in range(cols)]
    expo = [[ork.below(1 << 14) for _ in range(cols)] for _ in range(rows)]
    expo[2][1] = 0
    expo[4] = [0, 0, 0, 0]
    rng.state = ork.state
    alpha = ph.encrypt_vec(alpha_m, rng, True)
    zv = ph.encrypt_vec(zv_m, rng, True)
    for window in (1, 3, 6):
        ph.reset_counters()
        out = ph.hom_matvec(alpha, expo, zv, window)
        assert ph.counters()[0] == rows
        for i in range(rows):
            want = alpha_m[i]
            for j in range(cols):
                want = (want + expo[i][j] * zv_m[j] % n) % n
            assert ph.crt_decrypt(out[i]) == want
            assert out[i].plain_bits < n.bit_length()
    ragged = [list(r) for r in expo]
    ragged[1].pop()
    with pytest.raises(ValueError):
        ph.hom_matvec(alpha, ragged, zv)
    with pytest.raises(ValueError):
        ph.hom_matvec(alpha, expo, zv, 9)


@pytest.mark.parametrize("idx,rows,cols", [(1, 17, 23), (2, 9, 40), (2, 33, 96)])  # 96: partial tree 6 -> 3
def test_matvec_matches_bigint_and_reference(idx, rows, cols):
    kp = key(idx)
    pub = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    rnd = random.Random(rows * cols)
    n2 = kp.n2
    alpha = [rnd.randrange(1, n2) for _ in range(rows)]
    zv = [rnd.randrange(1, n2) for _ in range(cols)]
    expo = [[rnd.getrandbits(50) for _ in range(cols)] for _ in range(rows)]
    expo[0] = [0] * cols
    E = np.array(expo, np.uint64)
    out = pub.hom_matvec_batch(L.ints_to_limbs(alpha, 2 * pub.L), E, L.ints_to_limbs(zv, 2 * pub.L))
    got = L.limbs_to_ints(out)
    for i in range(rows):
        want = alpha[i]
        for j in range(cols):
            want = want * pow(zv[j], expo[i][j], n2) % n2
        assert got[i] == want
    import refbind as R_

    if R_.available():
        import ctypes as C

        ref = R_.RefKey.keygen(golden("keys.json")[idx]["seed"], kp.key_bits)
        A, Z = L.ints_to_limbs(alpha, 2 * pub.L), L.ints_to_limbs(zv, 2 * pub.L)
        o = np.zeros_like(A)
        rc = R_.lib().pcref_hom_matvec(ref.h, R_.a(A), None, R_.a(E), R_.a(Z), None, rows, cols, 6, 2 * pub.L,
                                       R_.a(o), None, 1)
        assert rc == 0 and (o == out).all()


def test_edge_step_matches_bigint():
    kp = key(1)
    ph = P.Paillier(kp)
    rnd = random.Random(5)
    cols = 12
    zc = [rnd.randrange(1, kp.n2) for _ in range(cols)]
    vc = [rnd.randrange(1, kp.n2) for _ in range(cols)]
    alpha = [rnd.randrange(1, kp.n2) for _ in range(cols)]
    E = np.array([[rnd.getrandbits(50) for _ in range(cols)] for _ in range(cols)], np.uint64)
    W = 2 * ph.L
    out = ph.edge_step_batch(L.ints_to_limbs(alpha, W), E, L.ints_to_limbs(zc, W), L.ints_to_limbs(vc, W))
    got = L.limbs_to_ints(out)
    for i in range(cols):
        want = alpha[i]
        for j in range(cols):
            want = want * pow(zc[j] * vc[j] % kp.n2, int(E[i, j]), kp.n2) % kp.n2
        assert got[i] == want
    bad = list(zc)
    bad[3] = kp.n2  # protocol.cpp:264-266
    with pytest.raises(ValueError):
        ph.edge_step_batch(L.ints_to_limbs(alpha, W), E, L.ints_to_limbs(bad, W), L.ints_to_limbs(vc, W))


@pytest.mark.parametrize("idx,sizes", [(0, [1, 7, 3]), (1, [5, 3, 4]), (2, [6, 6])])
def test_edge_step_blocks_match_bigint(idx, sizes):
    """pcb_edge_step_blocks == pcb_edge_step per block (unequal sizes exercise the padding)."""
    kp = key(idx)
    ph = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    rnd = random.Random(11 + idx)
    n2, W, tot = kp.n2, 2 * ph.L, sum(sizes)
    zc = [rnd.randrange(1, n2) for _ in range(tot)]
    vc = [rnd.randrange(1, n2) for _ in range(tot)]
    alpha = [rnd.randrange(1, n2) for _ in range(tot)]
    Es = [np.array([[rnd.getrandbits(rnd.choice([1, 20, 53])) for _ in range(c)] for _ in range(c)], np.uint64)
          for c in sizes]
    expo = np.concatenate([e.reshape(-1) for e in Es])
    out = ph.edge_step_blocks_batch(sizes, L.ints_to_limbs(alpha, W), expo, L.ints_to_limbs(zc, W),
                                    L.ints_to_limbs(vc, W))
    got = L.limbs_to_ints(out)
    at = 0
    for c, E in zip(sizes, Es):
        single = L.limbs_to_ints(ph.edge_step_batch(L.ints_to_limbs(alpha[at:at + c], W), np.ascontiguousarray(E),
                                                    L.ints_to_limbs(zc[at:at + c], W),
                                                    L.ints_to_limbs(vc[at:at + c], W)))
        for i in range(c):
            want = alpha[at + i]
            for j in range(c):
                want = want * pow(zc[at + j] * vc[at + j] % n2, int(E[i, j]), n2) % n2
            assert got[at + i] == want == single[i]
        at += c


def test_encrypt_rn_equals_encrypt(kk):
    """Offline/online split: pcb_encrypt_rn(m, pcb_encrypt(0, r)) == pcb_encrypt(m, r) (== the
    reference's crt_encrypt_with_r golden ciphertexts), on private and public contexts."""
    idx, kp, ph, pub = kk
    e = golden("encrypt.json")[idx]
    ms, rs, cs = [H(v) for v in e["m"]], [H(v) for v in e["r"]], [H(v) for v in e["c"]]
    R = L.ints_to_limbs(rs, ph.L)
    rn = ph.encrypt_batch(L.ints_to_limbs([0] * len(rs), 1), R, use_crt=True)
    assert L.limbs_to_ints(rn) == [pow(r, kp.n, kp.n2) for r in rs]
    for ctx in (ph, pub):
        st = np.zeros(len(ms), np.int32)
        c = ctx.encrypt_rn_batch(L.ints_to_limbs(ms, ctx.L), rn, status=st)
        assert (st == 0).all() and L.limbs_to_ints(c) == cs
    bad_m = [kp.n, kp.n + 5, 3, 4]
    bad_rn = [5, 5, 0, kp.n2]
    st = np.zeros(4, np.int32)
    c = pub.encrypt_rn_batch(L.ints_to_limbs(bad_m, pub.L), L.ints_to_limbs(bad_rn, 2 * pub.L), status=st)
    assert st.tolist() == [1, 1, 2, 2]  # PLAINTEXT_RANGE, RANDOMNESS_RANGE
    assert not L.limbs_to_ints(c)[0] and not L.limbs_to_ints(c)[3]
