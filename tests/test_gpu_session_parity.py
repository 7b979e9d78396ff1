"""Round-2 parity pins for the encrypted ADMM session and the branches round 1 left unchecked.

  * the 2048-bit session at cfg3's shape (N=4096, M=512, K=8 blocks of 512) and cfg1 (1024-bit,
    N=256, M=128, K=4) for all 50 iterations, bit-identical to the reference's integer shadow
    pipeline (acceptance.cpp:214-281) whose per-element integer work runs in the COMPILED
    reference (oracle/_ref/libpcref.so: gamma1/gamma2, combined_quantized_update,
    inverse_quantize_x);
  * the session's ciphertexts themselves: the edges' alpha-hat (public-key encrypt_vec with the
    edge stream Rng(seed ^ mix*k), protocol.cpp:207-212, 74, 351) and the master's enc_state
    (crt encrypt_vec with the master stream Rng(seed), protocol.cpp:333, 410, 467-476), compared
    with the reference library on the same key and streams;
  * pcb_sample_r on a PUBLIC-key context (binary-gcd acceptance, rstream.cu) against the
    reference's Paillier::sample_r (paillier.cpp:233-239), including a toy key where rejections
    (r = 0, gcd(r, n) != 1) are frequent;
  * the range gate check_update_range (protocol.cpp:20-27): PCB_E_RANGE_UPDATE exactly where the
    restated gate rejects.
"""
import ctypes as C
import os

import numpy as np
import pytest

import admm_oracle as AO
import pcadmm_oracle as O
import refbind as RB
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import admm as ADMM
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 1
SEED = 1
KEY_SEED = SEED ^ 0x6B657967656E2E2E  # experiments.cpp:61-64


def _factors(a, y, sizes, rho=1.0):
    f, at = [], 0
    for c in sizes:
        f.append(AO.node_factor(a[:, at:at + c], y, rho, len(sizes)))
        at += c
    return f


def _problem(m, n, k, iters, seed=SEED):
    a, y, _ = AO.gen_gaussian_problem(m, n, 0.1, seed)
    sizes = AO.split_columns(n, k)
    fac = _factors(a, y, sizes)
    spec = AO.session_bounds(a, y, 1.0, 1.0, iters, sizes, 1.5, 1e15, fac)
    return a, y, sizes, fac, spec


def _run(bits, m, n, k, iters, capture=0):
    a, y, sizes, fac, spec = _problem(m, n, k, iters)
    keys = P.keygen(P.Rng(KEY_SEED), bits)
    sess = ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=k, iters=iters, seed=SEED))
    if capture:
        sess.capture = {"iters": capture}
    res = sess.run(a, y, factors=fac, spec=spec)
    return keys, sess, res, (a, y, sizes, fac, spec)


def _assert_trajectory(res, fac, sizes, spec, iters):
    trace, z, v = AO.shadow_session_ref(fac, sizes, spec, 1.0, 1.0, iters)
    for t in range(iters):
        assert np.array_equal(res.x_trace[t], trace[t]), f"x differs at iteration {t}"
    assert np.array_equal(res.z, z) and np.array_equal(res.v, v)


def test_shadow_ref_matches_scalar_shadow():
    """The compiled-reference shadow equals the scalar restatement (pins the fast path)."""
    a, y, sizes, fac, spec = _problem(20, 30, 3, 4)
    t1, z1, v1 = AO.shadow_session(fac, sizes, spec, 1.0, 1.0, 4)
    t2, z2, v2 = AO.shadow_session_ref(fac, sizes, spec, 1.0, 1.0, 4)
    assert all(list(p) == q.tolist() for p, q in zip(t1, t2)) and z1 == z2.tolist() and v1 == v2.tolist()


def test_cfg3_shape_2048_bit_exact():
    """cfg3 (N=4096, M=512, K=8, 2048-bit key, Delta=1e15): 3 iterations bit-identical."""
    iters = 3
    _, _, res, (a, y, sizes, fac, spec) = _run(2048, 512, 4096, 8, iters)
    _assert_trajectory(res, fac, sizes, spec, iters)


def test_cfg1_all_50_iterations():
    """cfg1 (N=256, M=128, K=4, 1024-bit): every one of the 50 iterations bit-identical, and the
    session with its own (GPU) node factors tracks the plaintext split recurrence
    (test_protocol.cpp:145-149: MSE < 1e-10)."""
    iters = 50
    keys, _, res, (a, y, sizes, fac, spec) = _run(1024, 128, 256, 4, iters)
    _assert_trajectory(res, fac, sizes, spec, iters)
    res2 = ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=4, iters=iters, seed=SEED)).run(a, y)
    xs, _, _, objs = AO.lasso_admm_split(a, y, 1.0, 1.0, iters, sizes)
    for t in range(iters):
        assert np.mean((res2.x_trace[t] - xs[t]) ** 2) < 1e-10, t
    assert abs(res2.objective[-1] - objs[-1]) / objs[-1] < 1e-5


@pytest.mark.parametrize("bits,m,n,k", [(1024, 128, 256, 4), (2048, 64, 384, 3)])
def test_session_ciphertexts_match_reference(bits, m, n, k):
    """alpha-hat and the first two iterations' enc_state ciphertexts, every element, against the
    reference library (same key, same edge/master splitmix64 streams, same quantized values)."""
    iters = 2
    keys, sess, res, (a, y, sizes, fac, spec) = _run(bits, m, n, k, iters, capture=iters)
    ref = RB.RefKey.from_primes(keys.p, keys.q)
    assert ref.n == keys.n
    Lw = ref.L
    # --- alpha-hat: edge k encrypts Gamma1(alpha_k) with the public key and Rng(seed ^ mix*k)
    ah = sess.alpha_hat.cpu().numpy().view(np.uint32)
    at = 0
    for kk, c in enumerate(sizes):
        seed_k = SEED ^ ((ADMM.EDGE_SEED_MIX * (kk + 1)) & ADMM.MASK64)
        r, _ = ref.sample_r(seed_k, c)
        qa, _, rc = RB.gamma1(np.asarray(fac[kk][1], np.float64), *spec)
        assert rc == 0
        m_limbs = np.ascontiguousarray(qa.view(np.uint32).reshape(c, 4))
        cref, st = ref.encrypt(m_limbs, r, crt=False, threads=THREADS)
        assert (st == 0).all()
        assert np.array_equal(ah[at:at + c], cref), f"alpha-hat of edge {kk + 1}"
        at += c
    # --- enc_state: per iteration, per block, z_k then -v_k, r drawn from Rng(seed) in that order
    _, _, _, qtr = AO.shadow_session_ref(fac, sizes, spec, 1.0, 1.0, iters, capture_q=True)
    state = SEED
    offs = np.cumsum([0] + sizes[:-1])
    for t in range(iters):
        rall, state = ref.sample_r(state, 2 * n)
        ct = sess.capture["ct"][t].cpu().numpy().view(np.uint32)
        q = sess.capture["q"][t].cpu().numpy().view(np.uint64)
        for kk, c in enumerate(sizes):
            o = int(offs[kk])
            q_z, q_nv = qtr[t][kk]
            assert np.array_equal(q[o:o + c], q_z) and np.array_equal(q[n + o:n + o + c], q_nv), (t, kk)
            ms = np.concatenate([q_z, q_nv]).astype(np.uint64)
            ml = np.ascontiguousarray(ms.view(np.uint32).reshape(2 * c, 2))
            cref, st = ref.encrypt(ml, rall[2 * o:2 * o + 2 * c], crt=True, threads=THREADS)
            assert (st == 0).all()
            assert np.array_equal(ct[o:o + c], cref[:c]), f"enc z, iteration {t}, block {kk + 1}"
            assert np.array_equal(ct[n + o:n + o + c], cref[c:]), f"enc -v, iteration {t}, block {kk + 1}"
    assert ref.L == Lw


@pytest.mark.parametrize("which", ["toy", "k64", "k1024", "k2048"])
def test_sample_r_public_key_matches_reference(which):
    """Public-key pcb_sample_r (gcd(r, n) == 1 by binary gcd on the GPU) == Paillier::sample_r."""
    if which == "toy":
        p, q, bits = 5, 7, 6
    else:
        kp = P.keygen(P.Rng(77), {"k64": 64, "k1024": 1024, "k2048": 2048}[which])
        p, q, bits = kp.p, kp.q, kp.key_bits
    ref = RB.RefKey.from_primes(p, q)
    pub = P.Paillier(P.PublicKey(p * q, bits))
    count = 3000 if which == "toy" else 2000
    for seed in (2, 0x9E3779B97F4A7C15 ^ 5):
        rng = P.Rng(seed)
        R = pub.sample_r_batch(rng, count).cpu().numpy().view(np.uint32)
        rref, st_ref = ref.sample_r(seed, count)
        assert np.array_equal(R, rref[:, :pub.L])
        assert rng.state == st_ref
    if which == "toy":  # the toy stream really rejects (multiples of 5 and 7, and 0)
        rng = O.Rng(2)
        raw = [O.random_below(rng, 35) for _ in range(200)]
        assert any(v == 0 or v % 5 == 0 or v % 7 == 0 for v in raw)


def test_range_gate_reports_range_update():
    """check_update_range (protocol.cpp:20-27) on the GPU's Dec epilogue: values around the cap,
    at 2^127 and 2^128 report PCB_E_RANGE_UPDATE exactly where the restated gate rejects; the
    accepted rows are updated, the rejected rows keep x/z/v."""
    import torch

    kp = P.keygen(P.Rng(KEY_SEED), 1024)
    ph = P.Paillier(kp)
    zmin, zmax, delta, cols = -2.0, 2.0, 1e15, 8
    cap = delta * delta / (zmax - zmin) + float(cols) * delta * 2.0 * delta
    lim = int(cap * 1.000001 + 4.0)
    qs = [0, 12345, lim - (1 << 40), lim, lim + (1 << 50), (1 << 127) - 1, 1 << 127, (1 << 128) + 7]
    assert len(qs) == cols
    expect_ok = [O.check_update_range(q, zmin, zmax, delta, cols) for q in qs]
    assert not all(expect_ok) and any(expect_ok)
    r = ph.sample_r_batch(P.Rng(3), cols)
    M = torch.from_numpy(L.ints_to_limbs(qs, ph.L).view(np.int32)).cuda()
    c = ph.encrypt_batch(M, r)
    rowsum = torch.full((cols,), 1000, dtype=torch.int64, device="cuda")
    q_z = torch.full((cols,), 10, dtype=torch.int64, device="cuda")
    q_nv = torch.full((cols,), 20, dtype=torch.int64, device="cuda")
    x = torch.full((cols,), 7.0, dtype=torch.float64, device="cuda")
    z, v = x.clone(), x.clone()
    st = torch.zeros(cols, dtype=torch.int32, device="cuda")
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = L.lib().pcb_decrypt_update(ph._ctx, L.ptr(c), cols, L.ptr(rowsum), L.ptr(q_z), L.ptr(q_nv), zmin, zmax,
                                    delta, 1.0, L.ptr(x), L.ptr(z), L.ptr(v), L.ptr(st), stream)
    torch.cuda.synchronize()
    assert rc == L.PCB_E_RANGE_UPDATE
    got = st.cpu().tolist()
    assert got == [0 if ok else L.PCB_E_RANGE_UPDATE for ok in expect_ok]
    xs = x.cpu().tolist()
    for i, ok in enumerate(expect_ok):
        if not ok:
            assert xs[i] == 7.0
    # the Python session raises the reference's ProtocolError analogue on the first bad element
    with pytest.raises(L.PcbError):
        P._raise_for(rc, "update")


def test_null_status_reports_first_failure():
    """With status = NULL every batch entry point returns the first failing element's code (the
    reference throws there, paillier.cpp:242, 322-323, 348) instead of silently returning 0."""
    import torch

    kp = P.keygen(P.Rng(KEY_SEED), 2048)
    ph = P.Paillier(kp)
    n = 300
    r = ph.sample_r_batch(P.Rng(4), n)
    ms = [i * 977 for i in range(n)]
    M = torch.from_numpy(L.ints_to_limbs(ms, ph.L).view(np.int32)).cuda()
    c = ph.encrypt_batch(M, r)  # all valid: no error
    assert L.limbs_to_ints(ph.decrypt_batch(c).cpu().numpy().view(np.uint32)) == ms
    bad = M.clone()
    bad[123] = torch.from_numpy(L.ints_to_limbs([kp.n], ph.L).view(np.int32))[0].cuda()  # m == n
    with pytest.raises(ValueError):
        ph.encrypt_batch(bad, r)
    r0 = r.clone()
    r0[7] = 0  # r == 0
    with pytest.raises(ValueError):
        ph.encrypt_batch(M, r0)
    cb = c.clone()
    cb[200] = torch.from_numpy(L.ints_to_limbs([kp.n * kp.n + 5], 2 * ph.L).view(np.int32))[0].cuda()  # c >= n^2
    with pytest.raises(ValueError):
        ph.decrypt_batch(cb)
    cn = c.clone()
    cn[5] = torch.from_numpy(L.ints_to_limbs([3 * kp.p], 2 * ph.L).view(np.int32))[0].cuda()  # not a unit
    with pytest.raises(RuntimeError):
        ph.decrypt_batch(cn)
    with pytest.raises(ValueError):
        ph.encrypt_rn_batch(bad, ph.encrypt_batch(torch.zeros_like(M[:, :1]), r))


def test_async_iteration_entries_match_sync_and_flag_errors():
    """pcb_quantize_async / pcb_edge_step_blocks_async / pcb_decrypt_update_blocks_async (no host
    sync, errors in a device flag) give the synchronous forms' results, and flag the reference's
    failures: non-finite value (quantize.cpp:18-19), ciphertext >= n^2 (protocol.cpp:264-266),
    update above the range cap (protocol.cpp:20-27)."""
    import torch

    kp = P.keygen(P.Rng(KEY_SEED), 1024)
    ph, pub = P.Paillier(kp), P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    lib = L.lib()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = np.random.default_rng(3)
    spec = (-3.0, 3.0, 1e15)
    # quantize
    v = torch.from_numpy(g.uniform(-4, 4, 500)).cuda()
    q1 = torch.empty(500, dtype=torch.int64, device="cuda")
    q2 = torch.empty_like(q1)
    cl = (C.c_uint64 * 2)()
    assert lib.pcb_quantize(L.ptr(v), 500, *spec, 0, L.ptr(q1), cl, stream) == 0
    cld = torch.zeros(2, dtype=torch.int64, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    assert lib.pcb_quantize_async(L.ptr(v), 500, *spec, 0, L.ptr(q2), L.ptr(cld), L.ptr(err), stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(q1, q2) and cld.tolist() == [cl[0], cl[1]] and int(err.item()) == 0
    v[17] = float("nan")
    assert lib.pcb_quantize_async(L.ptr(v), 500, *spec, 0, L.ptr(q2), L.ptr(cld), L.ptr(err), stream) == 0
    torch.cuda.synchronize()
    assert int(err.item()) == L.PCB_E_SHAPE
    # edge step over 2 blocks of 24
    sizes = np.array([24, 24], np.uint32)
    n2 = kp.n * kp.n
    W = 2 * ph.L
    mk = lambda k: torch.from_numpy(L.ints_to_limbs([int(x) for x in g.integers(1, 2**62, k)], W).view(np.int32)).cuda()  # noqa: E731
    alpha, zc, vc = mk(48), mk(48), mk(48)
    expo = torch.from_numpy(g.integers(0, 10**15, 2 * 24 * 24, dtype=np.uint64).view(np.int64)).cuda()
    o1 = torch.empty((48, W), dtype=torch.int32, device="cuda")
    o2 = torch.empty_like(o1)
    assert lib.pcb_edge_step_blocks(pub._ctx, 2, sizes.ctypes.data, L.ptr(alpha), L.ptr(expo), L.ptr(zc), L.ptr(vc),
                                    6, L.ptr(o1), stream) == 0
    err.zero_()
    assert lib.pcb_edge_step_blocks_async(pub._ctx, 2, sizes.ctypes.data, L.ptr(alpha), L.ptr(expo), 50, L.ptr(zc),
                                          L.ptr(vc), 6, L.ptr(o2), L.ptr(err), stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and int(err.item()) == 0
    zc[30] = torch.from_numpy(L.ints_to_limbs([n2 + 1], W).view(np.int32))[0].cuda()
    assert lib.pcb_edge_step_blocks_async(pub._ctx, 2, sizes.ctypes.data, L.ptr(alpha), L.ptr(expo), 50, L.ptr(zc),
                                          L.ptr(vc), 6, L.ptr(o2), L.ptr(err), stream) == 0
    torch.cuda.synchronize()
    assert int(err.item()) == L.PCB_E_CIPHER_RANGE
    # decrypt + update: the range gate
    cols = 8
    zmin, zmax, delta = -2.0, 2.0, 1e15
    cap = delta * delta / (zmax - zmin) + float(cols) * delta * 2.0 * delta
    lim = int(cap * 1.000001 + 4.0)
    qs = [0, 12345, lim - (1 << 40), 99, lim + (1 << 50), 7, 1 << 127, 5]
    r = ph.sample_r_batch(P.Rng(3), cols)
    c = ph.encrypt_batch(torch.from_numpy(L.ints_to_limbs(qs, ph.L).view(np.int32)).cuda(), r)
    rowsum = torch.full((cols,), 1000, dtype=torch.int64, device="cuda")
    qz = torch.full((cols,), 10, dtype=torch.int64, device="cuda")
    qn = torch.full((cols,), 20, dtype=torch.int64, device="cuda")
    outs = []
    for fn in ("sync", "async"):
        x = torch.full((cols,), 7.0, dtype=torch.float64, device="cuda")
        z, vv = x.clone(), x.clone()
        err.zero_()
        one = np.array([cols], np.uint32)
        if fn == "sync":
            st = torch.zeros(cols, dtype=torch.int32, device="cuda")
            rc = lib.pcb_decrypt_update_blocks(ph._ctx, 1, one.ctypes.data, L.ptr(c), L.ptr(rowsum), L.ptr(qz),
                                               L.ptr(qn), zmin, zmax, delta, 1.0, L.ptr(x), L.ptr(z), L.ptr(vv),
                                               L.ptr(st), stream)
            assert rc == L.PCB_E_RANGE_UPDATE
        else:
            rc = lib.pcb_decrypt_update_blocks_async(ph._ctx, 1, one.ctypes.data, L.ptr(c), L.ptr(rowsum), L.ptr(qz),
                                                     L.ptr(qn), zmin, zmax, delta, 1.0, L.ptr(x), L.ptr(z), L.ptr(vv),
                                                     L.ptr(err), stream)
            torch.cuda.synchronize()
            assert rc == 0 and int(err.item()) == L.PCB_E_RANGE_UPDATE
        outs.append((x.cpu(), z.cpu(), vv.cpu()))
    for a_, b_ in zip(*outs):
        assert torch.equal(a_, b_)


def test_faithful_driver_gpu_backend_bit_exact():
    """Faithful-trust session (FaithfulDriver + FaithfulGpuBackend: the private context exists on
    rank 0 only, edges hold public contexts) -- one rank here -- bit-identical to the shadow."""
    import torch

    iters = 4
    a, y, sizes, fac, spec = _problem(128, 256, 4, iters)
    keys = P.keygen(P.Rng(KEY_SEED), 2048)
    cfg = ADMM.SessionConfig(nodes=4, iters=iters, seed=SEED)
    drv = ADMM.FaithfulDriver(ADMM.FaithfulGpuBackend(keys, 0, 0), cfg)
    res = drv.run(torch.as_tensor(a, device="cuda"), torch.as_tensor(y, device="cuda"),
                  [(torch.as_tensor(b, device="cuda"), torch.as_tensor(al, device="cuda")) for b, al in fac], spec)
    _assert_trajectory(res, fac, sizes, spec, iters)
