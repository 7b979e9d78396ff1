"""The CPU restatement (oracle/pcadmm_oracle.py) pinned against the reference:
golden vectors produced by the compiled reference (oracle/gen_golden.py) and the reference's own
known-answer tests.  CPU only."""
import math

import pytest

import pcadmm_oracle as O
from conftest import golden


def H(x):
    return int(x, 16)


def test_toy_key_hand_values():
    # test_paillier.cpp:27-45
    kp = O.keypair_from_primes(5, 7)
    assert (kp.n, kp.n2, kp.g, kp.eps, kp.mu) == (35, 1225, 36, 12, 3)
    c = kp.crt
    assert (c["p2"], c["q2"], c["phi_p2"], c["phi_q2"]) == (25, 49, 20, 42)
    assert (c["p2_inv_q2"], c["n_mod_phi_p2"], c["eps_mod_phi_p2"]) == (2, 15, 12)


def test_toy_exhaustive_table_matches_reference():
    g = golden("toy.json")
    kp = O.keypair_from_primes(g["p"], g["q"])
    for m, r, c in zip(g["m"], g["r"], g["c"]):
        # test_paillier.cpp:47-61: c = 36^m r^35 mod 1225, CRT == direct
        assert c == pow(36, m, 1225) * pow(r, 35, 1225) % 1225
        assert O.crt_encrypt_with_r(kp, m, r) == c == O.encrypt_with_r(kp, m, r)
        assert O.decrypt(kp, c) == m == O.crt_decrypt(kp, c)
    assert O.encrypt_with_r(kp, 0, 1) == 1


def test_pow_mod_kats():
    # test_bignat.cpp:178-180 (pow_mod), restated with the same numbers
    assert pow(2, 10, 1000) == 24
    assert pow(123456789, 0, 1000003) == 1
    assert pow(0, 5, 97) == 0


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_keygen_matches_reference(idx):
    k = golden("keys.json")[idx]
    rng = O.Rng(k["seed"])
    kp = O.keygen(rng, k["bits"])
    assert (kp.n, kp.p, kp.q) == (H(k["n"]), H(k["p"]), H(k["q"]))
    assert kp.eps == H(k["eps"]) and kp.mu == H(k["mu"])
    assert rng.state == k["rng_state_after"]
    assert kp.n.bit_length() == k["bits"]


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_sample_r_stream_matches_reference(idx):
    k, s = golden("keys.json")[idx], golden("sample_r.json")[idx]
    kp = O.finish_keys(H(k["p"]), H(k["q"]), k["bits"])
    rng = O.Rng(s["seed"])
    assert [O.sample_r(kp, rng) for _ in range(s["count"])] == [H(v) for v in s["r"]]
    assert rng.state == s["state_after"]


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_encrypt_decrypt_match_reference(idx):
    k, e, d = golden("keys.json")[idx], golden("encrypt.json")[idx], golden("decrypt.json")[idx]
    kp = O.finish_keys(H(k["p"]), H(k["q"]), k["bits"])
    for m, r, c in zip(e["m"], e["r"], e["c"]):
        assert O.crt_encrypt_with_r(kp, H(m), H(r)) == H(c)
    for m, r, st in zip(e["bad_m"], e["bad_r"], e["bad_status"]):
        with pytest.raises(ValueError) as ex:
            O.crt_encrypt_with_r(kp, H(m), H(r))
        assert O.STATUS_OF[type(ex.value)] == st
    for c, m, st in zip(d["c"], d["m"], d["status"]):
        if st == 0:
            assert O.crt_decrypt(kp, H(c)) == H(m) == O.decrypt(kp, H(c))
        else:
            with pytest.raises((ValueError, RuntimeError)) as ex:
                O.crt_decrypt(kp, H(c))
            assert O.STATUS_OF[type(ex.value)] == st


def test_gamma_quantizers_match_reference():
    q = golden("quantize.json")
    vals = [float.fromhex(v) for v in q["v"]]
    cl2, cl1 = [0, 0], [0, 0]
    g2 = [O.gamma2(v, q["zmin"], q["zmax"], q["delta"], cl2) for v in vals]
    g1 = [O.gamma1(v, q["zmin"], q["zmax"], q["delta"], cl1) for v in vals]
    assert g2 == q["g2"] and g1 == q["g1"]
    assert cl2 == q["clamps2"] and cl1 == q["clamps1"]


def test_gamma_kats():
    # test_quantize.cpp:11-19: ties round away from zero
    assert O.gamma2(0.5, 0.0, 1.0, 1.0) == 1
    assert O.gamma2(0.25, 0.0, 1.0, 2.0) == 1  # 0.5 -> 1
    assert O.c_round(2.5) == 3.0 and O.c_round(-2.5) == -3.0 and O.c_round(0.49999999999999994) == 0.0
    with pytest.raises(ValueError):
        O.gamma2(math.nan, 0.0, 1.0, 10.0)
    with pytest.raises(ValueError):
        O.gamma2(0.1, 1.0, 1.0, 10.0)


def test_combined_update_and_inverse_match_reference():
    q = golden("quantize.json")
    qa = [int(v) for v in q["comb_alpha"]]
    out = O.combined_quantized_update(qa, q["comb_b"], q["comb_z"], q["comb_nv"])
    assert out == [int(v) for v in q["comb_out"]]
    rowsum = [sum(r) for r in q["comb_b"]]
    xs = O.inverse_quantize_x(out, rowsum, q["comb_z"], q["comb_nv"], q["inv_zmin"], q["inv_zmax"], q["inv_delta"])
    assert [x.hex() for x in xs] == q["inv_x"]


def test_hom_ops_semantics_toy():
    # test_paillier.cpp:80-115 restated: hom_add decrypts to the sum, the plain_bits guard trips
    kp = O.keypair_from_primes(5, 7)
    rng = O.Rng(7)
    enc = [O.encrypt_with_r(kp, m, O.sample_r(kp, rng)) for m in range(35)]
    c, b = O.hom_add(kp, enc[13], 4, enc[9], 4)
    assert O.decrypt(kp, c) == 22 and b == 5
    with pytest.raises(OverflowError):
        O.hom_add(kp, enc[16], 5, enc[16], 5)
    c, b = O.hom_scalar_mul(kp, 3, enc[5], 3)
    assert O.decrypt(kp, c) == 15


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_split_encryption_identity_on_golden_vectors(idx):
    """The split CRT encryption reproduces the reference's ciphertexts:
    r^n mod p^2 == ((r mod p)^q mod p)^p mod p^2 (and the same with p, q swapped), combined by CRT,
    on every golden (m, r, c) vector, plus r multiples of p and q."""
    k, e = golden("keys.json")[idx], golden("encrypt.json")[idx]
    p, q = H(k["p"]), H(k["q"])
    n, p2, q2 = p * q, p * p, q * q
    rs = [H(r) for r in e["r"]] + [1, p, 2 * q, n - 1]
    for r in rs:
        assert pow(r, n, p2) == pow(pow(r % p, q, p), p, p2)
        assert pow(r, n, q2) == pow(pow(r % q, p, q), q, q2)
    kp = O.finish_keys(p, q, k["bits"])
    for m, r, c in zip(e["m"], e["r"], e["c"]):
        m, r = H(m), H(r)
        cp = (1 + m * n) * pow(pow(r % p, q, p), p, p2) % p2
        cq = (1 + m * n) * pow(pow(r % q, p, q), q, q2) % q2
        c_split = (cp + p2 * ((cq - cp) * pow(p2, -1, q2) % q2)) % (n * n)
        assert c_split == H(c) == O.crt_encrypt_with_r(kp, m, r)
