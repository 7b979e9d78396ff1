"""The multi-rank session driver (paper_2601_14980_b200/admm.py ShardedDriver) with world_size 2
over gloo on CPU: block ownership, the shared stream order, the objective all-reduce and the final
assembly must give exactly the single-rank trajectory.  The encrypted block step needs a GPU, so
these tests plug the reference's integer shadow step (oracle) into the driver's hooks."""
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
