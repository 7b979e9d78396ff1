"""Collaborative variant (paper Alg. 3) through the C ABI on the GPU, against the
compiled reference (Paillier::decrypt_with_half / finish_split_encrypt, paillier.cpp:363-414) and
the restated edge-side worker delegated_power (protocol.cpp:15-18: base^(obf mod phi(p^2)) mod p^2
with obf = obfuscate_exponent(value, n eps, mask), protocol.cpp:11-13)."""
import random

import numpy as np
import pytest

import refbind as R_
from conftest import golden
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu


def _lcm(a, b):
    import math

    return a * b // math.gcd(a, b)


@pytest.fixture(scope="module")
def key2048():
    k = golden("keys.json")[2]
    return P.KeyPair(int(k["n"], 16), int(k["p"], 16), int(k["q"], 16), k["bits"]), k["seed"]


def test_finish_split_encrypt_and_decrypt_with_half(key2048):
    kp, seed = key2048
    ph = P.Paillier(kp)
    n, p, q = kp.n, kp.p, kp.q
    n2, p2 = n * n, p * p
    eps = _lcm(p - 1, q - 1)
    phi_p2 = p2 - p
    g = n + 1
    rnd = random.Random(17)
    count = 300  # > 2 tiles: every CTA path
    ms = [rnd.getrandbits(50) for _ in range(count - 2)] + [0, n - 1]
    rs = [rnd.randrange(1, n) for _ in range(count)]
    masks = [rnd.getrandbits(64) for _ in range(count)]
    # edge: delegated g-powers of the obfuscated plaintexts (protocol.cpp:248-249)
    gp = [pow(g % p2, (m + k * n * eps) % phi_p2, p2) for m, k in zip(ms, masks)]
    W = 2 * ph.L
    M, R, G = L.ints_to_limbs(ms, ph.L), L.ints_to_limbs(rs, ph.L), L.ints_to_limbs(gp, W)
    c = np.zeros((count, W), np.uint32)
    st = np.zeros(count, np.int32)
    rc = L.lib().pcb_finish_split_encrypt(ph._ctx, L.ptr(M), ph.L, L.ptr(G), W, L.ptr(R), count, L.ptr(c),
                                          L.ptr(st), None)
    assert rc == 0 and (st == 0).all()
    # == the basic CRT encryption (the obfuscation cancels: g^(n eps) = 1 mod p^2)
    cb = ph.encrypt_batch(M, R, use_crt=True)
    assert (c == cb).all()
    # edge: delegated decryption power of each ciphertext (protocol.cpp:226, 492)
    cs = L.limbs_to_ints(c)
    px = [pow(cv % p2, (eps + k * n * eps) % phi_p2, p2) for cv, k in zip(cs, masks)]
    PX = L.ints_to_limbs(px, W)
    m = np.zeros((count, ph.L), np.uint32)
    st[:] = 0
    rc = L.lib().pcb_decrypt_with_half(ph._ctx, L.ptr(c), L.ptr(PX), W, count, L.ptr(m), L.ptr(st), None)
    assert rc == 0 and (st == 0).all()
    assert L.limbs_to_ints(m) == ms
    # the compiled reference gives the same ciphertexts / plaintexts
    if R_.available():
        ref = R_.RefKey.keygen(seed, kp.key_bits)
        cref, sref = ref.finish_split_encrypt(M, G, R)
        assert (sref == 0).all() and (cref == c).all()
        mref, sref = ref.decrypt_with_half(c, PX)
        assert (sref == 0).all() and (mref == m).all()
    # single-value mirrors and the obfuscation helper
    ob = P.Paillier.obfuscate_exponent(ms[0], n * eps, masks[0])
    assert ob == ms[0] + masks[0] * n * eps
    ct = ph.finish_split_encrypt(ms[0], pow(g % p2, ob % phi_p2, p2), rs[0])
    assert ct.value == cs[0]
    assert ph.decrypt_with_half(ct, px[0]) == ms[0]


def test_collab_error_statuses(key2048):
    kp, _ = key2048
    ph = P.Paillier(kp)
    W = 2 * ph.L
    n2 = kp.n * kp.n
    # c >= n^2 -> invalid_argument (paillier.cpp:365); non-unit p-half -> runtime_error (L check)
    C_ = L.ints_to_limbs([n2 + 5, 5], W)  # n^2 + 5 is out of range; 5 with a zero p-half is a non-unit
    PX = L.ints_to_limbs([1, 0], W)  # p-half 0: x = CRT(0, ...) not = 1 mod p
    m = np.zeros((2, ph.L), np.uint32)
    st = np.zeros(2, np.int32)
    assert L.lib().pcb_decrypt_with_half(ph._ctx, L.ptr(C_), L.ptr(PX), W, 2, L.ptr(m), L.ptr(st), None) == 0
    assert st[0] == L.PCB_E_CIPHER_RANGE and st[1] == L.PCB_E_NOT_UNIT
    # m >= n and r = 0 -> invalid_argument (paillier.cpp:409-411)
    M = L.ints_to_limbs([kp.n, 3], ph.L)
    R = L.ints_to_limbs([5, 0], ph.L)
    G = L.ints_to_limbs([1, 1], W)
    c = np.zeros((2, W), np.uint32)
    assert L.lib().pcb_finish_split_encrypt(ph._ctx, L.ptr(M), ph.L, L.ptr(G), W, L.ptr(R), 2, L.ptr(c), L.ptr(st),
                                            None) == 0
    assert st[0] == L.PCB_E_PLAINTEXT_RANGE and st[1] == L.PCB_E_RANDOMNESS_RANGE and not c.any()


def test_delegated_power_edge_worker(key2048):
    """The edge side of Alg. 3: per-element exponents on the RNS core, only {p^2, phi(p^2)} known."""
    kp, _ = key2048
    share = P.crt_share(kp)
    p2, phi = kp.p * kp.p, kp.p * kp.p - kp.p
    n2, eps = kp.n * kp.n, _lcm(kp.p - 1, kp.q - 1)
    rnd = random.Random(23)
    count = 260
    bases = [rnd.randrange(0, n2) for _ in range(count - 4)] + [0, 1, p2, kp.n + 1]
    obfs = [P.Paillier.obfuscate_exponent(rnd.getrandbits(50), kp.n * eps, rnd.getrandbits(64))
            for _ in range(count - 3)] + [0, phi, 3 * phi + 5]
    W = 2 * share.S
    ow = max(1, max(o.bit_length() for o in obfs) // 32 + 1)
    out = share.delegated_power_batch(L.ints_to_limbs(bases, W), L.ints_to_limbs(obfs, ow))
    got = L.limbs_to_ints(out)
    for i in range(count):
        assert got[i] == pow(bases[i] % p2, obfs[i] % phi, p2), i
    assert P.delegated_power(bases[5], obfs[5], share) == got[5]


def test_collab_session_equals_basic():
    """The collaborative session (delegated p^2 powers, finish_split_encrypt, decrypt_with_half)
    gives the same trajectory as the basic one (test_protocol.cpp:173, 202)."""
    import admm_oracle as AO
    from paper_2601_14980_b200 import admm as ADMM

    a, y, _ = AO.gen_gaussian_problem(24, 40, 0.1, 4)
    sizes = AO.split_columns(40, 2)
    fac, at = [], 0
    for c in sizes:
        fac.append(AO.node_factor(a[:, at:at + c], y, 1.0, 2))
        at += c
    spec = AO.session_bounds(a, y, 1.0, 1.0, 3, sizes, 1.5, 1e15, fac)
    keys = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
    basic = ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=2, iters=3)).run(a, y, factors=fac, spec=spec)
    collab = ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=2, iters=3, variant="collab")).run(
        a, y, factors=fac, spec=spec)
    for t in range(3):
        assert collab.x_trace[t].tolist() == basic.x_trace[t].tolist(), t
    assert collab.z.tolist() == basic.z.tolist() and collab.v.tolist() == basic.v.tolist()


def test_collab_session_masks_exponents_and_ledger():
    """Reference fidelity of the collaborative session: the mask stream is Rng(seed ^ "maskmask")
    (protocol.cpp:334) -- one draw_mask per edge for obf_dec at session init (352-353), then per
    iteration and block c_k masks for z and c_k for -v (440-446) -- and the obfuscated exponents
    the edges receive are q + mask * n eps (protocol.cpp:11-13), computed on the device.  Ledger
    (test_protocol.cpp:179-195, binomial g): the master pays 5 half-exponentiations per element
    and iteration (2 x 2 r halves + 1 decrypt_with_half; basic: 6), the edges 3 delegated powers."""
    import math

    import torch

    import admm_oracle as AO
    from paper_2601_14980_b200 import admm as ADMM

    iters, seed = 2, 7
    a, y, _ = AO.gen_gaussian_problem(24, 40, 0.1, 4)
    sizes = AO.split_columns(40, 2)
    fac, at = [], 0
    for c in sizes:
        fac.append(AO.node_factor(a[:, at:at + c], y, 1.0, 2))
        at += c
    spec = AO.session_bounds(a, y, 1.0, 1.0, iters, sizes, 1.5, 1e15, fac)
    keys = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
    sess = ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=2, iters=iters, variant="collab", seed=seed))
    sess.capture = {"iters": iters}
    sess.master.reset_counters()
    res = sess.run(a, y, factors=fac, spec=spec)
    n_tot = sum(sizes)
    # the exponents: replay the reference's mask stream with Python integers
    eps = (keys.p - 1) * (keys.q - 1) // math.gcd(keys.p - 1, keys.q - 1)
    n_eps = keys.n * eps
    rng = P.Rng(seed ^ 0x6D61736B6D61736B)
    obf_dec = [eps + ADMM.draw_mask(rng) * n_eps for _ in range(2)]
    assert obf_dec == sess.obf_dec
    for t in range(iters):
        q = sess.capture["q"][t].cpu().numpy().view(np.uint64)
        obf = L.limbs_to_ints(sess.capture["obf"][t].cpu().numpy().view(np.uint32))
        masks = [ADMM.draw_mask(rng) for _ in range(2 * n_tot)]
        o = 0
        for c in sizes:  # block: c masks for z, then c for -v; batch rows [z_all ; -v_all]
            for i in range(c):
                assert obf[o + i] == int(q[o + i]) + masks[2 * o + i] * n_eps
                assert obf[n_tot + o + i] == int(q[n_tot + o + i]) + masks[2 * o + c + i] * n_eps
            o += c
    # ledger
    # the master role = its online context + the offline r^n precompute (the 2 x 2 r halves)
    assert res.master.pow_half == 5 * n_tot * iters and sess.delegated_pows == 3 * n_tot * iters
    assert res.edges.delegated_pows == 3 * n_tot * iters
    basic = ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=2, iters=iters, seed=seed)).run(
        a, y, factors=fac, spec=spec)
    for t in range(iters):
        assert res.x_trace[t].tolist() == basic.x_trace[t].tolist()


def test_binomial_delegated_power_equals_the_exponentiation(key2048):
    """pcb_delegated_power_binomial (g = n + 1: 1 + (obf mod phi(p^2)) n mod p^2) is bit-identical to
    the generic delegated_power (protocol.cpp:15-18) for masked, bare and edge exponents."""
    import torch

    kp, _ = key2048
    share = P.crt_share(kp)
    n, p2 = kp.n, kp.p * kp.p
    eps = _lcm(kp.p - 1, kp.q - 1)
    phi = p2 - kp.p
    rnd = random.Random(23)
    obfs = [rnd.getrandbits(60) + rnd.getrandbits(64) * n * eps for _ in range(200)]
    obfs += [0, 1, phi, phi - 1, phi + 1, 5 * phi, n * eps, rnd.getrandbits(60)]
    ow = max(o.bit_length() for o in obfs) // 32 + 1
    O = torch.from_numpy(L.ints_to_limbs(obfs, ow).view(np.int32)).cuda()
    W = 2 * share.S
    G = torch.from_numpy(np.tile(L.int_to_limbs(n + 1, W), (len(obfs), 1)).view(np.int32)).cuda()
    nd = torch.from_numpy(L.int_to_limbs(n, (n.bit_length() + 31) // 32).view(np.int32)).cuda()
    got = share.delegated_power_binomial_tensor(nd, O)
    want = share.delegated_power_tensor(G, O)
    assert torch.equal(got, want)
    vals = L.limbs_to_ints(got.cpu().numpy().view(np.uint32))
    assert vals == [pow(n + 1, o % phi, p2) for o in obfs]


def test_decrypt_half_q_is_the_masters_crt_half(key2048):
    """pcb_decrypt_half_q: the q^2 chain of decrypt_with_half (paillier.cpp:366), which the
    collaborative session runs while the edge works on the p^2 side.  eps mod phi(q^2) = u (q - 1), so
    the chain is c^(q-1) mod q^2 and u is folded into the finish (half_pow, paillier.cpp:275-305)."""
    import torch

    kp, _ = key2048
    ph = P.Paillier(kp)
    n, p, q = kp.n, kp.p, kp.q
    q2 = q * q
    e = _lcm(p - 1, q - 1) % (q2 - q)
    rnd = random.Random(23)
    count = 130  # two tiles, the second ragged
    cs = [rnd.randrange(1, n * n) for _ in range(count - 2)] + [1, n * n - 1]
    W, S = 2 * ph.L, ph.crt_half_words()
    c = torch.from_numpy(L.ints_to_limbs(cs, W).view(np.int32)).cuda()
    yq = torch.zeros((count, S), dtype=torch.int32, device="cuda")
    f0, h0 = ph.counters()
    assert L.lib().pcb_decrypt_half_q(ph._ctx, L.ptr(c), count, L.ptr(yq), None) == 0
    torch.cuda.synchronize()
    got = L.limbs_to_ints(yq.cpu().numpy().view(np.uint32))
    u, w = divmod(e, q - 1)
    assert w == 0 and u != 0
    assert got == [pow(x % q2, q - 1, q2) for x in cs]
    assert [1 + q * ((((g - 1) // q) * u) % q) if g else 0 for g in got] == [pow(x % q2, e, q2) for x in cs]
    assert ph.counters() == (f0, h0 + count)  # one half per element
    # host pointers are refused (device-only asynchronous form)
    assert L.lib().pcb_decrypt_half_q(ph._ctx, c.cpu().numpy().ctypes.data, count, L.ptr(yq), None) != 0


def test_delegated_power_fermat_equals_generic(key2048):
    """pcb_delegated_power_fermat (one |p|-bit chain + 1 + p (L_p(s) u mod p)) == pcb_delegated_power
    for exponents u (p - 1), the form of the collaborative obf_dec = eps (1 + mask n); bases include
    multiples of p (result 0) and 1."""
    import torch

    kp, _ = key2048
    share = P.crt_share(kp)
    p, q, n = kp.p, kp.q, kp.n
    p2 = p * p
    eps = _lcm(p - 1, q - 1)
    rnd = random.Random(29)
    count = 140
    bases = [rnd.randrange(1, n * n) for _ in range(count - 4)] + [p, 3 * p * q, 1, n * n - 1]
    obfs = [eps * (1 + rnd.getrandbits(64) * n) for _ in range(count)]
    W, S = 2 * share.S, share.S
    B = torch.from_numpy(L.ints_to_limbs(bases, W).view(np.int32)).cuda()
    facs = [share.fermat_factor(o) for o in obfs]
    assert all(f is not None for f in facs)
    U = torch.from_numpy(np.stack(facs).view(np.int32)).cuda()
    got = L.limbs_to_ints(share.delegated_power_fermat_tensor(B, U).cpu().numpy().view(np.uint32))
    ow = max((o.bit_length() + 31) // 32 for o in obfs)
    O = torch.from_numpy(L.ints_to_limbs(obfs, ow).view(np.int32)).cuda()
    ref = L.limbs_to_ints(share.delegated_power_tensor(B, O).cpu().numpy().view(np.uint32))
    torch.cuda.synchronize()
    assert got == ref
    assert got[:3] == [pow(b % p2, o % (p2 - p), p2) for b, o in zip(bases[:3], obfs[:3])]
    assert got[count - 4] == 0 and got[count - 3] == 0 and got[count - 2] == 1
    # an exponent that is not a multiple of p - 1 has no Fermat form
    assert share.fermat_factor(eps + 1) is None


def test_decrypt_update_half_async_matches_sync_and_flags(key2048):
    """pcb_decrypt_update_blocks_half_async, with the q side computed inside or handed over from
    pcb_decrypt_half_q, == the synchronous pcb_decrypt_update_blocks_half (decrypt_with_half +
    range gate + update, protocol.cpp:20-27, 488-511): same x / z / v, and the range failure lands in
    the device flag instead of the return code."""
    import ctypes as C

    import torch

    kp, _ = key2048
    ph = P.Paillier(kp)
    share = P.crt_share(kp)
    lib = L.lib()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    n, p, q = kp.n, kp.p, kp.q
    eps = _lcm(p - 1, q - 1)
    cols = 8
    zmin, zmax, delta = -2.0, 2.0, 1e15
    cap = delta * delta / (zmax - zmin) + float(cols) * delta * 2.0 * delta
    lim = int(cap * 1.000001 + 4.0)
    qs = [0, 12345, lim - (1 << 40), 99, lim + (1 << 50), 7, 1 << 127, 5]
    r = ph.sample_r_batch(P.Rng(3), cols)
    c = ph.encrypt_batch(torch.from_numpy(L.ints_to_limbs(qs, ph.L).view(np.int32)).cuda(), r)
    W = 2 * ph.L
    obf = eps * (1 + 4242 * n)  # an edge's obf_dec (protocol.cpp:352-353)
    U = torch.from_numpy(np.tile(share.fermat_factor(obf), (cols, 1)).view(np.int32)).cuda()
    px = torch.zeros((cols, W), dtype=torch.int32, device="cuda")
    px[:, :share.S] = share.delegated_power_fermat_tensor(c, U)
    yq = torch.empty((cols, ph.crt_half_words()), dtype=torch.int32, device="cuda")
    assert lib.pcb_decrypt_half_q(ph._ctx, L.ptr(c), cols, L.ptr(yq), stream) == 0
    rowsum = torch.full((cols,), 1000, dtype=torch.int64, device="cuda")
    qz = torch.full((cols,), 10, dtype=torch.int64, device="cuda")
    qn = torch.full((cols,), 20, dtype=torch.int64, device="cuda")
    one = np.array([cols], np.uint32)
    outs = []
    for mode in ("sync", "async", "async_q"):
        x = torch.full((cols,), 7.0, dtype=torch.float64, device="cuda")
        z, vv = x.clone(), x.clone()
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        if mode == "sync":
            rc = lib.pcb_decrypt_update_blocks_half(ph._ctx, 1, one.ctypes.data, L.ptr(c), L.ptr(px), L.ptr(rowsum),
                                                    L.ptr(qz), L.ptr(qn), zmin, zmax, delta, 1.0, L.ptr(x), L.ptr(z),
                                                    L.ptr(vv), None, stream)
            assert rc == L.PCB_E_RANGE_UPDATE
        else:
            rc = lib.pcb_decrypt_update_blocks_half_async(
                ph._ctx, 1, one.ctypes.data, L.ptr(c), L.ptr(px), L.ptr(yq) if mode == "async_q" else None,
                L.ptr(rowsum), L.ptr(qz), L.ptr(qn), zmin, zmax, delta, 1.0, L.ptr(x), L.ptr(z), L.ptr(vv),
                L.ptr(err), stream)
            torch.cuda.synchronize()
            assert rc == 0 and int(err.item()) == L.PCB_E_RANGE_UPDATE
        outs.append((x.cpu(), z.cpu(), vv.cpu()))
    for a_, b_, c_ in zip(*outs):
        assert torch.equal(a_, b_) and torch.equal(a_, c_)
    # the accepted rows were updated, the rejected ones (qs above the cap) kept 7.0
    assert outs[0][0][0].item() != 7.0 and outs[0][0][4].item() == 7.0 and outs[0][0][6].item() == 7.0
    # host pointers are refused by the asynchronous form
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    assert lib.pcb_decrypt_update_blocks_half_async(
        ph._ctx, 1, one.ctypes.data, c.cpu().numpy().ctypes.data, L.ptr(px), None, L.ptr(rowsum), L.ptr(qz),
        L.ptr(qn), zmin, zmax, delta, 1.0, L.ptr(x), L.ptr(z), L.ptr(vv), L.ptr(err), stream) != 0
