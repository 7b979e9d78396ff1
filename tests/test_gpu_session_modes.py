"""The reference SessionConfig surface beyond the defaults (protocol.hpp:17-41) and the master's
phase timers, on the GPU:

  * pooled randomness (r_mode / pool_size, protocol.cpp:382-391): same trajectory as fresh
    randomness, enc_state ciphertexts = Enc(q; pool[pool_at++ % pool_size]) against the compiled
    reference, and the exponentiation ledger of test_protocol.cpp:244-279 (fresh 6 halves per
    element and iteration; pooled 1 full + 2 halves per factor plus 2 halves per decryption;
    pooled collaborative 1 half per decryption);
  * use_crt = false (protocol.cpp:313, 410): the same ciphertexts and trajectory, ledger in fulls;
  * mask_bits (protocol.cpp:86-93): width 0 sends the exponents bare, a narrower width draws
    shifted masks, the trajectory never changes (test_protocol.cpp:198-204);
  * engine = coeff_fft runs the same lane (test_protocol.cpp:300-313); argument errors;
  * t_pre_s / t_loc_s / t_comm_s / t_master_s decompose the loop span within 1%
    (test_protocol.cpp:316-339);
  * pcb_finish_split_encrypt_rn (finish_split_encrypt_with_factor, paillier.cpp:416-426).
"""
import os
import random

import numpy as np
import pytest

import admm_oracle as AO
import refbind as RB
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import admm as ADMM
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1
SEED = 1
ITERS = 5
NODES = 3
COLS = 8  # total_cols of test_protocol.cpp:246


@pytest.fixture(scope="module")
def bench():
    a, y, _ = AO.gen_gaussian_problem(12, COLS, 0.25, 3)
    sizes = AO.split_columns(COLS, NODES)
    fac, at = [], 0
    for c in sizes:
        fac.append(AO.node_factor(a[:, at:at + c], y, 1.0, NODES))
        at += c
    spec = AO.session_bounds(a, y, 1.0, 1.0, ITERS, sizes, 1.5, 1e6, fac)
    keys = P.keygen(P.Rng(31), 2048)  # the collaborative share needs a 2048/3072-bit key
    return a, y, sizes, fac, spec, keys


def _run(bench, capture=0, **kw):
    a, y, sizes, fac, spec, keys = bench
    sess = ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=NODES, iters=ITERS, seed=SEED, delta=1e6, **kw))
    if capture:
        sess.capture = {"iters": capture}
    return sess, sess.run(a, y, factors=fac, spec=spec)


def _same_trace(r1, r2):
    return all(np.array_equal(p, q) for p, q in zip(r1.x_trace, r2.x_trace)) and len(r1.x_trace) == len(r2.x_trace) \
        and np.array_equal(r1.z, r2.z) and np.array_equal(r1.v, r2.v)


def test_pooled_keeps_trajectory_and_drops_the_count(bench):
    a, y, sizes, fac, spec, keys = bench
    _, rf = _run(bench)
    sp, rp = _run(bench, capture=2, r_mode="pooled", pool_size=4)
    _, rpc = _run(bench, r_mode="pooled", pool_size=4, variant="collab")
    trace, z, v = AO.shadow_session_ref(fac, sizes, spec, 1.0, 1.0, ITERS)
    assert all(np.array_equal(rf.x_trace[t], trace[t]) for t in range(ITERS))
    assert _same_trace(rf, rp) and _same_trace(rf, rpc)
    per_iter = COLS * ITERS
    assert (rf.master.pow_full, rf.master.pow_half) == (0, 6 * per_iter)
    assert (rp.master.pow_full, rp.master.pow_half) == (4, 2 * 4 + 2 * per_iter)
    assert (rpc.master.pow_full, rpc.master.pow_half) == (4, 2 * 4 + 1 * per_iter)
    # edges: alpha encryption 1 full per element (binomial g), one full per matvec row
    # (test_protocol.cpp:187-194); collaborative: 3 delegated powers per element and iteration
    assert rf.edges.pow_full == COLS + COLS * ITERS and rf.edges.delegated_pows == 0
    assert rpc.edges.pow_full == COLS + COLS * ITERS and rpc.edges.delegated_pows == 3 * per_iter

    # the pooled enc_state ciphertexts: Enc(q; r) with r = pool[(t 2N + position) % pool_size],
    # the pool = the first pool_size draws of Rng(seed) (protocol.cpp:385-391, 411-414)
    ref = RB.RefKey.from_primes(keys.p, keys.q)
    pool, _ = ref.sample_r(SEED, 4)
    offs = np.cumsum([0] + sizes[:-1])
    for t in range(2):
        ct = sp.capture["ct"][t].cpu().numpy().view(np.uint32)
        q = sp.capture["q"][t].cpu().numpy().view(np.uint64)
        for kk, c in enumerate(sizes):
            o = int(offs[kk])
            pos = t * 2 * COLS + 2 * o + np.arange(2 * c)
            ms = np.concatenate([q[o:o + c], q[COLS + o:COLS + o + c]]).astype(np.uint64)
            cref, st = ref.encrypt(np.ascontiguousarray(ms.view(np.uint32).reshape(2 * c, 2)), pool[pos % 4], crt=True,
                                   threads=THREADS)
            assert (st == 0).all()
            assert np.array_equal(ct[o:o + c], cref[:c]) and np.array_equal(ct[COLS + o:COLS + o + c], cref[c:]), (t, kk)


def test_use_crt_false_same_ciphertexts_ledger_in_fulls(bench):
    sf, rf = _run(bench, capture=ITERS)
    sd, rd = _run(bench, capture=ITERS, use_crt=False)
    assert _same_trace(rf, rd)
    for t in range(ITERS):  # encrypt_with_r == crt_encrypt_with_r (paillier.cpp:318-343)
        assert np.array_equal(sf.capture["ct"][t].cpu().numpy(), sd.capture["ct"][t].cpu().numpy())
    per_iter = COLS * ITERS
    assert (rd.master.pow_full, rd.master.pow_half) == (3 * per_iter, 0)
    _, rdp = _run(bench, use_crt=False, r_mode="pooled", pool_size=3)
    assert _same_trace(rf, rdp)
    assert (rdp.master.pow_full, rdp.master.pow_half) == (3 + per_iter, 2 * 3)


def test_mask_width_changes_exponents_not_the_trajectory(bench):
    a, y, sizes, fac, spec, keys = bench
    s64, r64 = _run(bench, capture=1, variant="collab")
    s0, r0 = _run(bench, capture=1, variant="collab", mask_bits=0)
    s16, r16 = _run(bench, capture=1, variant="collab", mask_bits=16)
    assert _same_trace(r64, r0) and _same_trace(r64, r16)
    # bare exponents: obf == q (the test hook of protocol.cpp:86)
    q0 = s0.capture["q"][0].cpu().numpy().view(np.uint64)
    obf0 = L.limbs_to_ints(s0.capture["obf"][0].cpu().numpy().view(np.uint32))
    assert obf0 == [int(v) for v in q0]
    # 16-bit masks: the mask stream after the per-edge obf_dec draws, block order z then -v
    rng = P.Rng(SEED ^ 0x6D61736B6D61736B)
    for _ in range(NODES):
        ADMM.draw_mask(rng, 16)
    masks = ADMM.draw_masks(rng, 2 * COLS, 16)
    assert int(masks.max()) < 1 << 16 and (masks > 0).all()
    perm = s16.rperm.cpu().numpy()
    q16 = s16.capture["q"][0].cpu().numpy().view(np.uint64)
    obf16 = L.limbs_to_ints(s16.capture["obf"][0].cpu().numpy().view(np.uint32))
    assert obf16 == [int(qv) + int(m) * s16.n_eps for qv, m in zip(q16, masks[perm])]
    assert max(obf0).bit_length() < max(obf16).bit_length() < max(
        L.limbs_to_ints(s64.capture["obf"][0].cpu().numpy().view(np.uint32))).bit_length()


def test_engine_and_argument_errors(bench):
    _, rp = _run(bench)
    _, rc = _run(bench, engine="coeff_fft")
    assert _same_trace(rp, rc)
    a, y, sizes, fac, spec, keys = bench
    for kw, msg in [({"r_mode": "pooled", "pool_size": 0}, "pool size below 1"),
                    ({"variant": "collab", "mask_bits": 65}, "mask width above 64"),
                    ({"engine": "fft"}, "unknown engine"), ({"r_mode": "reuse"}, "unknown randomness mode")]:
        with pytest.raises(ValueError, match=msg):
            ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=NODES, iters=1, **kw)).run(a, y, factors=fac,
                                                                                          spec=spec)


@pytest.mark.parametrize("variant", ["basic", "collab"])
def test_master_phase_timers_decompose_the_loop_span(bench, variant):
    _, r = _run(bench, variant=variant)
    assert len(r.t_loc_s) == ITERS and len(r.t_comm_s) == ITERS
    assert r.t_pre_s > 0
    acc = r.t_pre_s
    for t in range(ITERS):
        assert r.t_loc_s[t] >= 0.0 and r.t_comm_s[t] > 0.0  # the edge step always takes device time
        acc += r.t_loc_s[t] + r.t_comm_s[t]
    assert abs(r.t_master_s - acc) <= 0.01 * r.t_master_s


def test_faithful_driver_pooled_and_timers(bench):
    import torch

    a, y, sizes, fac, spec, keys = bench
    _, rf = _run(bench)
    cfg = ADMM.SessionConfig(nodes=NODES, iters=ITERS, seed=SEED, delta=1e6, r_mode="pooled", pool_size=4)
    drv = ADMM.FaithfulDriver(ADMM.FaithfulGpuBackend(keys, 0, 0), cfg)
    res = drv.run(torch.as_tensor(a, device="cuda"), torch.as_tensor(y, device="cuda"),
                  [(torch.as_tensor(b, device="cuda"), torch.as_tensor(al, device="cuda")) for b, al in fac], spec)
    assert _same_trace(rf, res)
    per_iter = COLS * ITERS
    assert (res.master.pow_full, res.master.pow_half) == (4, 2 * 4 + 2 * per_iter)
    acc = res.t_pre_s + sum(res.t_loc_s) + sum(res.t_comm_s)
    assert abs(res.t_master_s - acc) <= 0.01 * res.t_master_s


def test_finish_split_encrypt_rn_matches_the_r_form():
    """finish_split_encrypt_with_factor == finish_split_encrypt with the factor's r (paillier.cpp:
    402-426), = CRT(gp mod p^2, (1 + m n) mod q^2) rn mod n^2; rn = 0 fails that element."""
    keys = P.keygen(P.Rng(77), 2048)
    ph = P.Paillier(keys)
    n, p, q = keys.n, keys.p, keys.q
    n2, p2, q2 = n * n, p * p, q * q
    rnd = random.Random(5)
    count = 260
    ms = [rnd.getrandbits(60) for _ in range(count - 1)] + [n - 1]
    rs = [rnd.randrange(1, n) for _ in range(count)]
    gps = [rnd.randrange(0, n2) for _ in range(count)]  # any edge reply, honest or not
    W = 2 * ph.L
    M, R, G = L.ints_to_limbs(ms, ph.L), L.ints_to_limbs(rs, ph.L), L.ints_to_limbs(gps, W)
    rn = ph.encrypt_batch(np.zeros((count, 1), np.uint32), R, use_crt=True)
    c_rn = ph.finish_split_encrypt_rn_batch(M, G, rn)
    c_r = np.zeros((count, W), np.uint32)
    st = np.zeros(count, np.int32)
    assert L.lib().pcb_finish_split_encrypt(ph._ctx, L.ptr(M), ph.L, L.ptr(G), W, L.ptr(R), count, L.ptr(c_r),
                                           L.ptr(st), None) == 0 and (st == 0).all()
    assert np.array_equal(c_rn, c_r)
    inv = pow(p2, -1, q2)
    for i in range(0, count, 37):
        cp, cq = gps[i] % p2, (1 + ms[i] * n) % q2
        crt = cp + p2 * (((cq - cp) * inv) % q2)
        assert L.limbs_to_ints(c_rn[i:i + 1])[0] == crt * pow(rs[i], n, n2) % n2
    rn[3] = 0
    st = np.zeros(count, np.int32)
    c_bad = ph.finish_split_encrypt_rn_batch(M, G, rn, status=st)
    assert st[3] == L.PCB_E_RANDOMNESS_RANGE and (np.delete(st, 3) == 0).all()
    assert not c_bad[3].any() and np.array_equal(np.delete(c_bad, 3, 0), np.delete(c_r, 3, 0))


def test_tight_window_clamps_are_counted(bench):
    """test_protocol.cpp:353-369: a window far too narrow for the factors clamps (and counts it);
    the properly sized one on the same problem reports none."""
    a, y, sizes, fac, spec, keys = bench
    cfg = ADMM.SessionConfig(nodes=NODES, iters=2, seed=SEED, delta=1e6)
    r = ADMM.EncryptedSession(keys, cfg).run(a, y, factors=fac, spec=(-0.02, 0.02, 1e6))
    assert r.clamps > 0
    r_ok = ADMM.EncryptedSession(keys, cfg).run(a, y, factors=fac, spec=spec)
    assert r_ok.clamps == 0
    with pytest.raises(ValueError, match="window"):
        ADMM.EncryptedSession(keys, cfg).run(a, y, factors=fac, spec=(1.0, 1.0, 1e6))


def test_rn_factor_api(bench):
    """make_rn_factor / encrypt_with_factor / crt_encrypt_with_factor /
    finish_split_encrypt_with_factor (paillier.cpp:371-426) in the Python mirror: the factor forms
    give the r forms' ciphertexts; a factor without r^n or residues is rejected."""
    a, y, sizes, fac, spec, keys = bench
    ph = P.Paillier(keys)
    rng = P.Rng(12)
    for m in (0, 1, 123456789, keys.n - 1):
        r = ph.sample_r(rng)
        f = ph.make_rn_factor(r)
        assert f.full == pow(r, keys.n, keys.n2) and f.half_p2 == f.full % (keys.p ** 2)
        want = ph.crt_encrypt_with_r(m, r)
        assert ph.encrypt_with_factor(m, f) == want and ph.crt_encrypt_with_factor(m, f) == want
        g = pow(keys.n + 1, m, keys.p ** 2)
        assert ph.finish_split_encrypt_with_factor(m, g, f) == ph.finish_split_encrypt(m, g, r)
    with pytest.raises(ValueError):
        ph.make_rn_factor(0)
    with pytest.raises(ValueError):
        ph.encrypt_with_factor(5, P.RnFactor(3, 0, 0, 0))
    with pytest.raises(ValueError):
        ph.crt_encrypt_with_factor(5, P.RnFactor(3, 7, 0, 0))
