"""The multi-rank session driver (paper_2601_14980_b200/admm.py ShardedDriver) with world_size 2
over gloo on CPU: block ownership, the shared stream order, the objective all-reduce and the final
assembly must give exactly the single-rank trajectory.  The encrypted block step needs a GPU, so
these tests plug the reference's integer shadow step (oracle) into the driver's hooks."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import admm_oracle as AO
import pcadmm_oracle as O
from paper_2601_14980_b200 import admm as ADMM


class ShadowDriver(ADMM.ShardedDriver):
    """ShardedDriver whose block step is the reference's crypto-free integer pipeline
    (acceptance.cpp:214-281) — the value the encrypted step must reproduce bit-exactly."""

    def setup_block(self, k):
        b_bar, alpha = self.factors[k]
        c = self.sizes[k]
        zmin, zmax, delta = self.spec
        self.q_alpha = getattr(self, "q_alpha", {})
        self.q_b = getattr(self, "q_b", {})
        self.q_alpha[k] = [O.gamma1(float(x), zmin, zmax, delta) for x in alpha]
        self.q_b[k] = [[O.gamma2(float(b_bar[i, j]), zmin, zmax, delta) for j in range(c)] for i in range(c)]
        self.stream_calls = []
        return 0

    def advance_stream(self, k):
        self.stream_calls.append(k)

    def step_block(self, k, t):
        zmin, zmax, delta = self.spec
        o, c = self.offs[k], self.sizes[k]
        z = self.z[o:o + c].tolist()
        v = self.v[o:o + c].tolist()
        q_z = [O.gamma2(zz, zmin, zmax, delta) for zz in z]
        q_nv = [O.gamma2(-vv, zmin, zmax, delta) for vv in v]
        q = O.combined_quantized_update(self.q_alpha[k], self.q_b[k], q_z, q_nv)
        xk = O.inverse_quantize_x(q, [sum(r) for r in self.q_b[k]], q_z, q_nv, zmin, zmax, delta)
        kappa = self.cfg.lam / self.cfg.rho
        for i in range(c):
            xv = xk[i] + v[i]
            zz = O.soft_threshold(xv, kappa)
            self.x[o + i] = xk[i]
            self.z[o + i] = zz
            self.v[o + i] = xv - zz
        return 0


def problem():
    a, y, _ = AO.gen_gaussian_problem(10, 18, 0.2, 7)
    sizes = AO.split_columns(18, 4)
    factors, at = [], 0
    for c in sizes:
        factors.append(AO.node_factor(a[:, at:at + c], y, 1.0, 4))
        at += c
    spec = AO.session_bounds(a, y, 1.0, 1.0, 6, sizes, 1.5, 1e15, factors)
    return a, y, factors, spec


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, y, factors, spec = problem()
    cfg = ADMM.SessionConfig(nodes=4, iters=6)
    d = ShadowDriver(cfg, rank=rank, world=world)
    res = d.run_blocks(torch.from_numpy(a), torch.from_numpy(y), factors, spec)
    q.put((rank, d.mine, d.stream_calls, res.x_trace, res.objective, res.z.tolist()))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_driver_matches_single_rank_and_shadow():
    a, y, factors, spec = problem()
    single = ShadowDriver(ADMM.SessionConfig(nodes=4, iters=6)).run_blocks(
        torch.from_numpy(a), torch.from_numpy(y), factors, spec)
    trace, z, v = AO.shadow_session(factors, AO.split_columns(18, 4), spec, 1.0, 1.0, 6)
    assert [list(t) for t in single.x_trace] == trace  # driver == reference pipeline, bit-exact
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    (r0, mine0, calls0, tr0, obj0, z0), (r1, mine1, calls1, tr1, obj1, z1) = out
    assert mine0 == [0, 1] and mine1 == [2, 3]          # block k -> rank floor(k G / K)
    assert calls0 == calls1 == [0, 1, 2, 3] * 6          # every rank walks the stream in block order
    for t in range(6):
        assert np.array_equal(tr0[t], single.x_trace[t]) and np.array_equal(tr1[t], single.x_trace[t])
    assert z0 == z1 == single.z.tolist()
    assert np.allclose(obj0, single.objective, rtol=1e-12) and obj0 == obj1


# ---- faithful trust (private key on rank 0 only): the exchange logic of FaithfulDriver ------------
class OracleFaithfulBackend:
    """FaithfulDriver backend with the ciphertext arithmetic in Python integers (the oracle's
    restatement of the reference, 1024-bit key): the driver's broadcast / all-gather and its
    block bookkeeping are exercised on CPU over gloo exactly as on NCCL."""

    def __init__(self, kp, rank):
        from paper_2601_14980_b200 import _lib as L

        self.L_ = L
        self.kp = kp if rank == 0 else None
        self.pub_n = kp.n
        self.n2 = kp.n * kp.n
        self.Lw = (kp.n.bit_length() + 31) // 32
        self.width = 2 * self.Lw
        self.device = torch.device("cpu")
        self.okp = O.finish_keys(kp.p, kp.q, kp.key_bits) if rank == 0 else None

    def sync(self):
        pass

    def _ct(self, vals):
        return torch.from_numpy(self.L_.ints_to_limbs(vals, self.width).view(np.int32).copy())

    def _ints(self, t):
        return self.L_.limbs_to_ints(t.numpy().view(np.uint32))

    def setup_edges(self, mine, factors, sizes, spec, cfg):
        zmin, zmax, delta = spec
        self.mine, self.blk = mine, {}
        rows, alpha_hat = [], []
        for k in mine:
            b_bar, alpha = factors[k]
            c = sizes[k]
            q_b = [[O.gamma2(float(b_bar[i, j]), zmin, zmax, delta) for j in range(c)] for i in range(c)]
            rng = O.Rng(cfg.seed ^ ((ADMM.EDGE_SEED_MIX * (k + 1)) & ADMM.MASK64))
            ah = []
            for i in range(c):
                while True:  # sample_r with the public key (paillier.cpp:233-239)
                    r = O.random_below(rng, self.pub_n)
                    if r and math.gcd(r, self.pub_n) == 1:
                        break
                m = O.gamma1(float(alpha[i]), zmin, zmax, delta)
                ah.append((1 + m * self.pub_n) % self.n2 * pow(r, self.pub_n, self.n2) % self.n2)
            self.blk[k] = (q_b, ah)
            rows.extend(sum(r_) for r_ in q_b)
        return torch.tensor(rows, dtype=torch.int64), 0

    def setup_master(self, sizes, spec, cfg):
        self.rng = O.Rng(cfg.seed)
        self.sizes, self.spec, self.kappa = sizes, spec, cfg.lam / cfg.rho

    def master_encrypt(self, z, v, t):
        zmin, zmax, delta = self.spec
        n = len(z)
        qz = [O.gamma2(float(a), zmin, zmax, delta) for a in z.tolist()]
        qv = [O.gamma2(-float(a), zmin, zmax, delta) for a in v.tolist()]
        cz, cv = [0] * n, [0] * n
        o = 0
        for c in self.sizes:  # block k: c draws for z, then c for -v (protocol.cpp:467-468)
            for i in range(c):
                cz[o + i] = O.crt_encrypt_with_r(self.okp, qz[o + i], O.sample_r(self.okp, self.rng))
            for i in range(c):
                cv[o + i] = O.crt_encrypt_with_r(self.okp, qv[o + i], O.sample_r(self.okp, self.rng))
            o += c
        return self._ct(cz + cv), (qz, qv)

    def edge_step(self, mine, sizes, offs, ct):
        cts = self._ints(ct)
        n = len(cts) // 2
        out = []
        for k in mine:
            q_b, ah = self.blk[k]
            o, c = offs[k], sizes[k]
            zv = [cts[o + j] * cts[n + o + j] % self.n2 for j in range(c)]
            for i in range(c):
                acc = ah[i]
                for j in range(c):
                    acc = acc * pow(zv[j], q_b[i][j], self.n2) % self.n2
                out.append(acc)
        return self._ct(out) if out else torch.zeros((0, self.width), dtype=torch.int32)

    def master_update(self, upd, q, rowsum, sizes, spec, cfg, x, z, v):
        zmin, zmax, delta = spec
        qz, qv = q
        ups = self._ints(upd)
        rs = rowsum.tolist()
        o = 0
        for c in sizes:
            qs = [O.crt_decrypt(self.okp, ups[o + i]) for i in range(c)]
            for qq in qs:
                assert O.check_update_range(qq, zmin, zmax, delta, c)
            xk = O.inverse_quantize_x(qs, rs[o:o + c], qz[o:o + c], qv[o:o + c], zmin, zmax, delta)
            for i in range(c):
                xv = xk[i] + float(v[o + i])
                zz = O.soft_threshold(xv, self.kappa)
                x[o + i], z[o + i], v[o + i] = xk[i], zz, xv - zz
            o += c

    def check_iteration(self, t):
        return 0


FAITHFUL_ITERS = 3


def faithful_problem():
    from paper_2601_14980_b200 import paillier as P

    a, y, factors, spec = problem()
    kp = P.keygen(P.Rng(11), 1024)
    return a, y, factors, spec, kp


def faithful_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, y, factors, spec, kp = faithful_problem()
    cfg = ADMM.SessionConfig(nodes=4, iters=FAITHFUL_ITERS)
    d = ADMM.FaithfulDriver(OracleFaithfulBackend(kp, rank), cfg, rank=rank, world=world)
    res = d.run(torch.from_numpy(a), torch.from_numpy(y), factors, spec)
    q.put((rank, d.mine, [t.tolist() for t in res.x_trace], None if res.z is None else res.z.tolist()))
    dist.destroy_process_group()


def test_faithful_two_rank_exchange_matches_single_rank_and_shadow():
    """Private key on rank 0 only: broadcast of enc_state, edge steps on the owning ranks,
    all-gather of enc_update -> rank 0's trajectory equals the single-rank run and the
    reference's integer shadow pipeline bit for bit; the edge rank never holds the key."""
    a, y, factors, spec, kp = faithful_problem()
    cfg = ADMM.SessionConfig(nodes=4, iters=FAITHFUL_ITERS)
    single = ADMM.FaithfulDriver(OracleFaithfulBackend(kp, 0), cfg).run(torch.from_numpy(a), torch.from_numpy(y),
                                                                          factors, spec)
    trace, z, v = AO.shadow_session(factors, AO.split_columns(18, 4), spec, 1.0, 1.0, FAITHFUL_ITERS)
    assert [list(t) for t in single.x_trace] == trace
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=faithful_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    (r0, mine0, tr0, z0), (r1, mine1, tr1, z1) = out
    assert mine0 == [0, 1] and mine1 == [2, 3]
    assert tr0 == trace and z0 == z and tr1 == [] and z1 is None


def test_rank_slices_and_fold_partials():
    """Slicing one job-wide stream over ranks (bench.py cfg2/cfg4) and the aggregation exchange
    (per-rank partial product -> all-gather -> fold) reproduce the single-rank values."""
    for total in (0, 1, 7, 1 << 20, 4194304 + 3):
        for world in (1, 2, 3, 8):
            sl = [ADMM.rank_slice(total, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sum(c for _, c in sl) == total
            assert all(sl[r][0] + sl[r][1] == sl[r + 1][0] for r in range(world - 1))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=fold_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    kp, cs, n2 = fold_setup()
    want = 1
    for c in cs:
        want = want * c % n2
    assert out[0][1] == out[1][1] == want


def fold_setup():
    kp = O.keygen(O.Rng(5), 64)
    rng = O.Rng(9)
    cs = [O.crt_encrypt_with_r(kp, i * 3 + 1, O.sample_r(kp, rng)) for i in range(37)]
    return kp, cs, kp.n * kp.n


def fold_worker(rank, world, port, q):
    from paper_2601_14980_b200 import _lib as L

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    kp, cs, n2 = fold_setup()
    off, cnt = ADMM.rank_slice(len(cs), world, rank)
    part = 1
    for c in cs[off:off + cnt]:
        part = part * c % n2
    W = 4

    def fold(parts):
        acc = 1
        for v_ in L.limbs_to_ints(parts.numpy().view(np.uint32)):
            acc = acc * v_ % n2
        return torch.from_numpy(L.ints_to_limbs([acc], W).view(np.int32).copy())

    t = torch.from_numpy(L.ints_to_limbs([part], W).view(np.int32).copy())
    tot = ADMM.fold_partials(t, world, None, fold)
    q.put((rank, L.limbs_to_ints(tot.numpy().view(np.uint32))[0]))
    dist.destroy_process_group()
