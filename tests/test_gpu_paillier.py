"""GPU parity tests: the CUDA path, called through the C ABI, against the compiled reference's
golden vectors and the CPU restatement (oracle).  Bit-exact for every ciphertext, plaintext,
r value, status and quantized integer."""
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
def ctx(request):
    kp = key(request.param)
    return request.param, kp, P.Paillier(kp)


def test_encrypt_matches_reference_golden(ctx):
    idx, kp, ph = ctx
    e = golden("encrypt.json")[idx]
    ms, rs, cs = [H(v) for v in e["m"]], [H(v) for v in e["r"]], [H(v) for v in e["c"]]
    M, R = L.ints_to_limbs(ms, ph.L), L.ints_to_limbs(rs, ph.L)
    st = np.zeros(len(ms), np.int32)
    c = ph.encrypt_batch(M, R, use_crt=True, status=st)
    assert (st == 0).all()
    assert L.limbs_to_ints(c) == cs
    # the direct (encrypt_with_r) form is bit-identical (test_paillier.cpp:63-78)
    c2 = ph.encrypt_batch(M, R, use_crt=False, status=st)
    assert L.limbs_to_ints(c2) == cs


def test_encrypt_error_statuses_match_reference(ctx):
    idx, kp, ph = ctx
    e = golden("encrypt.json")[idx]
    M = L.ints_to_limbs([H(v) for v in e["bad_m"]], ph.L)
    R = L.ints_to_limbs([H(v) for v in e["bad_r"]], ph.L)
    st = np.zeros(len(e["bad_m"]), np.int32)
    c = ph.encrypt_batch(M, R, status=st)
    assert st.tolist() == e["bad_status"]
    assert not c.any()
    with pytest.raises(ValueError):
        ph.crt_encrypt_with_r(kp.n, 5)  # paillier.cpp:242
    with pytest.raises(ValueError):
        ph.crt_encrypt_with_r(3, 0)  # paillier.cpp:322-323


def test_decrypt_matches_reference_golden(ctx):
    idx, kp, ph = ctx
    d = golden("decrypt.json")[idx]
    cs = [H(v) for v in d["c"]]
    Cl = L.ints_to_limbs(cs, 2 * ph.L)
    for crt in (True, False):
        st = np.zeros(len(cs), np.int32)
        m = ph.decrypt_batch(Cl, use_crt=crt, status=st)
        assert st.tolist() == d["status"]
        assert L.limbs_to_ints(m) == [H(v) for v in d["m"]]


def test_decrypt_exceptions(ctx):
    idx, kp, ph = ctx
    with pytest.raises(RuntimeError):
        ph.decrypt(kp.n)  # multiple of n: outside the group (test_paillier.cpp:151-152)
    with pytest.raises(RuntimeError):
        ph.crt_decrypt(0)
    with pytest.raises(ValueError):
        ph.crt_decrypt(kp.n2 + 5)  # paillier.cpp:356


def test_sample_r_stream_matches_reference(ctx):
    idx, kp, ph = ctx
    s = golden("sample_r.json")[idx]
    rng = P.Rng(s["seed"])
    r = ph.sample_r_batch(rng, s["count"]).cpu().numpy().view(np.uint32)
    assert L.limbs_to_ints(r) == [H(v) for v in s["r"]]
    assert rng.state == s["state_after"]


def test_sample_r_long_stream_matches_oracle():
    kp = key(1)
    ph = P.Paillier(kp)
    okp = O.finish_keys(kp.p, kp.q, kp.key_bits)
    rng, orng = P.Rng(777), O.Rng(777)
    # split into several GPU calls: the stream state must carry across
    got = []
    for cnt in (1, 300, 1699):
        got += L.limbs_to_ints(ph.sample_r_batch(rng, cnt).cpu().numpy().view(np.uint32))
    want = [O.sample_r(okp, orng) for _ in range(2000)]
    assert got == want and rng.state == orng.state


def test_toy_key_exhaustive():
    g = golden("toy.json")
    ph = P.Paillier(P.keypair_from_primes(5, 7))
    M, R = L.ints_to_limbs(g["m"], 1), L.ints_to_limbs(g["r"], 1)
    c = ph.encrypt_batch(M, R)
    assert L.limbs_to_ints(c) == g["c"]
    m = ph.decrypt_batch(np.ascontiguousarray(c))
    assert L.limbs_to_ints(m) == g["m"]


@pytest.mark.parametrize("bits", [1024, 2048])
def test_random_batch_round_trip_and_oracle(bits):
    torch = pytest.importorskip("torch")
    kp = P.keygen(P.Rng(bits), bits)
    ph = P.Paillier(kp)
    okp = O.finish_keys(kp.p, kp.q, bits)
    rnd = random.Random(bits)
    n = 3000
    ms = [rnd.getrandbits(50) for _ in range(n // 2)] + [rnd.randrange(kp.n) for _ in range(n - n // 2)]
    R = ph.sample_r_batch(P.Rng(5), n)
    M = torch.from_numpy(L.ints_to_limbs(ms, ph.L).view(np.int32)).cuda()
    c = ph.encrypt_batch(M, R)
    m = ph.decrypt_batch(c)
    assert L.limbs_to_ints(m.cpu().numpy().view(np.uint32)) == ms
    rs = L.limbs_to_ints(R.cpu().numpy().view(np.uint32))
    cs = L.limbs_to_ints(c.cpu().numpy().view(np.uint32))
    for i in range(0, n, 97):
        assert cs[i] == O.crt_encrypt_with_r(okp, ms[i], rs[i])


def test_encrypt_vec_decrypt_vec_api():
    kp = key(1)
    ph = P.Paillier(kp)
    okp = O.finish_keys(kp.p, kp.q, kp.key_bits)
    ms = [0, 1, 2**60, kp.n - 1]
    r1, r2 = P.Rng(9), O.Rng(9)
    cs = ph.encrypt_vec(ms, r1, use_crt=True)
    want = [O.crt_encrypt_with_r(okp, m, O.sample_r(okp, r2)) for m in ms]
    assert [c.value for c in cs] == want and r1.state == r2.state
    assert [c.plain_bits for c in cs] == [m.bit_length() for m in ms]
    assert ph.decrypt_vec(cs, use_crt=True) == ms
    # same seed, same ciphertexts (test_paillier.cpp:273-277)
    assert [c.value for c in ph.encrypt_vec(ms, P.Rng(9), True)] == want


def test_counters_follow_reference_ledger():
    ph = P.Paillier(key(0))
    ph.reset_counters()
    ph.crt_encrypt_with_r(3, 2)
    assert ph.counters() == (0, 2)  # binomial g: two half_pow (test_paillier.cpp:221-223)
    ph.reset_counters()
    ph.encrypt_with_r(3, 2)
    assert ph.counters() == (1, 0)
    ph.reset_counters()
    c = ph.crt_encrypt_with_r(3, 2)
    ph.reset_counters()
    ph.crt_decrypt(c)
    assert ph.counters() == (0, 2)
    ph.reset_counters()
    ph.decrypt(c)
    assert ph.counters() == (1, 0)


def test_quantize_encrypt_matches_reference_gammas():
    q = golden("quantize.json")
    kp = key(2)
    ph = P.Paillier(kp)
    okp = O.finish_keys(kp.p, kp.q, kp.key_bits)
    vals = np.array([float.fromhex(v) for v in q["v"]], np.float64)
    n = len(vals)
    R = ph.sample_r_batch(P.Rng(4), n)
    rs = L.limbs_to_ints(R.cpu().numpy().view(np.uint32))
    import torch

    V = torch.from_numpy(vals).cuda()
    for fine, key_ in ((False, "g2"), (True, "g1")):
        c, qv, cl = ph.quantize_encrypt_batch(V, q["zmin"], q["zmax"], q["delta"], R, fine=fine)
        qn = qv.cpu().numpy().view(np.uint64)
        got = [int(a) | (int(b) << 64) for a, b in qn] if fine else [int(x) for x in qn]
        assert got == q[key_]
        assert list(cl) == q["clamps1" if fine else "clamps2"]
        cs = L.limbs_to_ints(c.cpu().numpy().view(np.uint32))
        for i in range(0, n, 9):
            assert cs[i] == O.crt_encrypt_with_r(okp, got[i], rs[i])


@pytest.mark.parametrize("bits", [64, 512, 1024, 2048, 3072])
def test_modexp_batch_vs_pow(bits):
    rnd = random.Random(bits)
    limbs = (bits + 31) // 32
    m = rnd.getrandbits(bits) | (1 << (bits - 1)) | 1
    lib = L.lib()
    for e in (0, 1, 2, 3, 65537, rnd.getrandbits(bits)):
        xs = [rnd.getrandbits(bits) for _ in range(67)] + [0, 1, m - 1]
        X = L.ints_to_limbs(xs, limbs)
        Y = np.zeros_like(X)
        E = L.int_to_limbs(e, max(1, (e.bit_length() + 31) // 32))
        M = L.int_to_limbs(m, limbs)
        rc = lib.pcb_modexp_batch(L.ptr(M), limbs, L.ptr(E), len(E), L.ptr(X), len(xs), L.ptr(Y), None)
        assert rc == 0
        assert L.limbs_to_ints(Y) == [pow(x, e, m) for x in xs]


def key3072():
    """cfg4 key: keypair_from_primes(random_prime(1536) x 2), redrawn until n has 3072 bits
    (the reference keygen rejects 3072, paillier.cpp:107-109)."""
    rng = P.Rng(3072)
    while True:
        p, q = P.random_prime(rng, 1536), P.random_prime(rng, 1536)
        if p != q and (p * q).bit_length() == 3072:
            return P.keypair_from_primes(p, q)


def test_3072_bit_crt_encrypt_decrypt_vs_oracle():
    torch = pytest.importorskip("torch")
    kp = key3072()
    ph = P.Paillier(kp)
    okp = O.finish_keys(kp.p, kp.q, 3072)
    n = 200
    rnd = random.Random(3)
    ms = [rnd.getrandbits(50) for _ in range(n - 3)] + [0, 1, kp.n - 1]
    R = ph.sample_r_batch(P.Rng(2), n)
    rs = L.limbs_to_ints(R.cpu().numpy().view(np.uint32))
    M = torch.from_numpy(L.ints_to_limbs(ms, ph.L).view(np.int32)).cuda()
    c = ph.encrypt_batch(M, R)
    cs = L.limbs_to_ints(c.cpu().numpy().view(np.uint32))
    for i in list(range(0, n, 23)) + [n - 1, n - 2]:
        assert cs[i] == O.crt_encrypt_with_r(okp, ms[i], rs[i])
    m = ph.decrypt_batch(c)
    assert L.limbs_to_ints(m.cpu().numpy().view(np.uint32)) == ms
    # public-key path at 6144-bit n^2 (radix-2^27 core, 240 limbs): bit-identical to CRT Enc
    pub = P.Paillier(P.PublicKey(kp.n, 3072))
    c_pub = pub.encrypt_batch(M.cpu().numpy().view(np.uint32)[:8].copy(), R.cpu().numpy().view(np.uint32)[:8].copy(),
                              use_crt=False)
    assert (c_pub == c.cpu().numpy().view(np.uint32)[:8]).all()
    # homomorphic aggregation at 6144 bits decrypts to the plaintext sum (cfg4)
    agg = ph.aggregate_batch(c[:50])
    s = ph.decrypt_batch(agg.reshape(1, -1))
    assert L.limbs_to_ints(s.cpu().numpy().view(np.uint32))[0] == sum(ms[:50]) % kp.n


def test_3072_bit_matches_compiled_reference():
    import refbind as R_

    if not R_.available():
        pytest.skip("oracle/_ref not built")
    kp = key3072()
    ref = R_.RefKey.from_primes(kp.p, kp.q)
    ph = P.Paillier(kp)
    rnd = random.Random(4)
    ms = [rnd.getrandbits(50) for _ in range(16)]
    r, _ = ref.sample_r(2, 16)
    cref, st = ref.encrypt(L.ints_to_limbs(ms, ph.L), r, crt=True)
    assert (st == 0).all()
    c = ph.encrypt_batch(L.ints_to_limbs(ms, ph.L), np.ascontiguousarray(r))
    assert (c == cref).all()
    mref, _ = ref.decrypt(cref, crt=True)
    assert (ph.decrypt_batch(np.ascontiguousarray(c)) == mref).all()
