"""Resident 3P-ADMM-PC2 session on the GPU (basic variant, fresh randomness, CRT master).

Mirrors the per-iteration hot loop of the reference's run_session
(/root/reference/proj/src/protocol.cpp:309-526 master_loop, 181-293 edge_run) with every array
resident in HBM:

  master, per block k (protocol.cpp:425-511):
      pcb_quantize_encrypt(z_k)  and  pcb_quantize_encrypt(-v_k)   Gamma2 + CRT Enc, r from the
                                                                   master stream Rng(seed)
  edge k (protocol.cpp:257-275):
      pcb_edge_step(alpha_hat_k, Gamma2(B_k), zc, vc)             hom_add + hom_matvec (public key)
  master:
      pcb_decrypt_update(...)                                     Dec, range gate, inverse
                                                                   quantization, soft threshold

Setup per edge (protocol.cpp:186-220): node factors (FP64 on the GPU via torch.linalg.solve —
host linear algebra in the reference, Eigen LDLT), Gamma1(alpha) encrypted with the PUBLIC key
and the edge stream Rng(seed ^ 0x9e37...*k), Gamma2(B) rows and their sums.

Multi-GPU: edge blocks are sharded over ranks (block k -> rank
floor(k*G/K)); every rank runs the master and edge work of its own blocks.  The master r stream is
one serial stream in block order, so every rank advances it through all blocks (pcb_sample_r is
cheap next to an encryption) and uses only its own slice: ciphertexts are identical to the
single-GPU session.  Per iteration the objective's A z partials are summed with one NCCL
all-reduce, and x/z/v blocks are all-gathered at the end.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .paillier import KeyPair, Paillier, PublicKey, Rng, _raise_for

EDGE_SEED_MIX = 0x9E3779B97F4A7C15  # protocol.cpp:74, edge seed = seed ^ (mix * k)
MASK64 = (1 << 64) - 1


@dataclass
class SessionConfig:
    """pcadmm::SessionConfig defaults (protocol.hpp:24-41) for the basic variant."""

    nodes: int = 3
    iters: int = 100
    rho: float = 1.0
    lam: float = 1.0
    delta: float = 1e15
    margin: float = 1.5
    window: int = 6
    seed: int = 1
    over_k: bool = False  # YScaling::full


@dataclass
class SessionResult:
    x: np.ndarray = None
    z: np.ndarray = None
    v: np.ndarray = None
    x_trace: list = field(default_factory=list)
    objective: list = field(default_factory=list)
    clamps: int = 0
    spec: tuple = None
    iter_seconds: list = field(default_factory=list)


def split_columns(cols: int, k: int) -> list[int]:
    """admm.cpp:77-83."""
    if cols < 1 or k < 1 or k > cols:
        raise ValueError("cannot split columns across nodes")
    sizes = [cols // k] * k
    for i in range(cols % k):
        sizes[i] += 1
    return sizes


def node_factor(a_k, y, rho: float, k_total: int, over_k: bool = False):
    """admm.cpp:63-75 in FP64 on the GPU: B = rho (A^T A + rho I)^-1, alpha = (A^T A + rho I)^-1 A^T y."""
    import torch

    n = a_k.shape[1]
    normal = a_k.T @ a_k + rho * torch.eye(n, dtype=torch.float64, device=a_k.device)
    y_s = y / float(k_total) if over_k else y
    b_bar = rho * torch.linalg.solve(normal, torch.eye(n, dtype=torch.float64, device=a_k.device))
    alpha = torch.linalg.solve(normal, a_k.T @ y_s)
    return b_bar, alpha


def session_bounds(factors, sizes, rho, lam, iters, margin, delta):
    """protocol.cpp:29-70 (plaintext rehearsal of the block recurrence) + widen_bounds."""
    import torch

    lo = hi = 0.0
    for b_bar, alpha in factors:
        lo = min(lo, float(alpha.min()), float(b_bar.min()))
        hi = max(hi, float(alpha.max()), float(b_bar.max()))
    n = sum(sizes)
    dev = factors[0][0].device
    z = torch.zeros(n, dtype=torch.float64, device=dev)
    v = torch.zeros(n, dtype=torch.float64, device=dev)
    kappa = lam / rho
    for _ in range(iters):
        at = 0
        for (b_bar, alpha), c in zip(factors, sizes):
            zk, vk = z[at:at + c], v[at:at + c]
            xk = alpha + b_bar @ (zk - vk)
            xv = xk + vk
            znew = torch.where(xv > kappa, xv - kappa, torch.where(xv < -kappa, xv + kappa, torch.zeros_like(xv)))
            v[at:at + c] = vk + (xk - znew)
            z[at:at + c] = znew
            lo = min(lo, float(znew.min()), float((-v[at:at + c]).min()))
            hi = max(hi, float(znew.max()), float((-v[at:at + c]).max()))
            at += c
    # widen_bounds (quantize.cpp:114-129)
    if hi - lo < 1e-12:
        lo -= 0.5
        hi += 0.5
    pad = (margin - 1.0) * (hi - lo) / 2.0
    return lo - pad, hi + pad, delta


class ShardedDriver:
    """Backend-independent part of a session: block ownership, the per-iteration loop over blocks
    in reference order, the objective all-reduce and the final assembly of x/z/v over ranks.
    Subclasses provide setup_block(k) and step_block(k, t) (the encrypted hot path on the GPU;
    tests plug a plaintext step in to exercise the multi-rank logic on CPU with gloo)."""

    def __init__(self, cfg: SessionConfig, rank: int = 0, world: int = 1, group=None, device: str = "cpu"):
        self.cfg, self.rank, self.world, self.group = cfg, rank, world, group
        self.dev = device

    def owner(self, k: int) -> int:
        return k * self.world // self.cfg.nodes

    # hooks ------------------------------------------------------------------------------------
    def setup_block(self, k: int) -> int:  # returns clamp count
        raise NotImplementedError

    def advance_stream(self, k: int) -> None:  # keep shared streams in reference order
        pass

    def step_block(self, k: int, t: int) -> int:  # updates x/z/v slices of block k; returns clamps
        raise NotImplementedError

    # driver -----------------------------------------------------------------------------------
    def run_blocks(self, a, y, factors, spec, record_trace: bool = True) -> SessionResult:
        import time

        import torch

        cfg = self.cfg
        n = a.shape[1]
        self.sizes = split_columns(n, cfg.nodes)
        self.offs = np.cumsum([0] + self.sizes[:-1]).tolist()
        self.factors, self.spec = factors, spec
        self.mine = [k for k in range(cfg.nodes) if self.owner(k) == self.rank]
        res = SessionResult(spec=spec)
        self.x = torch.zeros(n, dtype=torch.float64, device=self.dev)
        self.z = torch.zeros(n, dtype=torch.float64, device=self.dev)
        self.v = torch.zeros(n, dtype=torch.float64, device=self.dev)
        for k in self.mine:
            res.clamps += self.setup_block(k)
        for t in range(cfg.iters):
            if self.dev != "cpu":
                torch.cuda.synchronize(self.dev)
            t0 = time.perf_counter()
            for k in range(cfg.nodes):
                self.advance_stream(k)
                if k in self.mine:
                    res.clamps += self.step_block(k, t)
            # objective on z (admm.cpp:31-34): A z partial sums over this rank's blocks
            az = torch.zeros(a.shape[0], dtype=torch.float64, device=self.dev)
            l1 = torch.zeros(1, dtype=torch.float64, device=self.dev)
            for k in self.mine:
                o, c = self.offs[k], self.sizes[k]
                az += a[:, o:o + c] @ self.z[o:o + c]
                l1 += self.z[o:o + c].abs().sum()
            if self.world > 1:
                import torch.distributed as dist

                dist.all_reduce(az, group=self.group)
                dist.all_reduce(l1, group=self.group)
            r = az - y
            res.objective.append(0.5 * float(r @ r) + cfg.lam * float(l1))
            if self.dev != "cpu":
                torch.cuda.synchronize(self.dev)
            res.iter_seconds.append(time.perf_counter() - t0)
            if record_trace:
                res.x_trace.append(self._gather(self.x.clone()))
        res.x, res.z, res.v = (self._gather(t_).cpu().numpy() for t_ in (self.x, self.z, self.v))
        res.x_trace = [xt.cpu().numpy() for xt in res.x_trace]
        return res

    def _gather(self, vec):
        """Every block lives on exactly one rank: zero the others and sum (one all-reduce)."""
        if self.world == 1:
            return vec
        import torch.distributed as dist

        for k in range(self.cfg.nodes):
            if k not in self.mine:
                vec[self.offs[k]:self.offs[k] + self.sizes[k]] = 0
        dist.all_reduce(vec, group=self.group)
        return vec


class EncryptedSession(ShardedDriver):
    """One rank's share of an encrypted session.  keys: the master's KeyPair (edges get the
    PublicKey only)."""

    def __init__(self, keys: KeyPair, cfg: SessionConfig, device: int = 0, rank: int = 0, world: int = 1,
                 group=None):
        super().__init__(cfg, rank, world, group, device=f"cuda:{device}")
        self.device = device
        self.master = Paillier(keys, device=device)
        self.edge = Paillier(PublicKey(keys.n, keys.key_bits), device=device)
        self.L = self.master.L
        self.lib = L.lib()

    def _stream(self):
        import torch

        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _quantize(self, v, spec, fine):
        import torch

        q = torch.empty((v.shape[0], 2) if fine else (v.shape[0],), dtype=torch.int64, device=v.device)
        cl = (C.c_uint64 * 2)()
        _raise_for(self.lib.pcb_quantize(L.ptr(v), v.shape[0], spec[0], spec[1], spec[2], 1 if fine else 0,
                                         L.ptr(q), cl, self._stream()), "quantize")
        return q, cl[0] + cl[1]

    def run(self, a, y, factors=None, spec=None, record_trace: bool = True) -> SessionResult:
        import torch

        cfg = self.cfg
        dev = torch.device(self.dev)
        a = torch.as_tensor(a, dtype=torch.float64, device=dev)
        y = torch.as_tensor(y, dtype=torch.float64, device=dev)
        sizes = split_columns(a.shape[1], cfg.nodes)
        offs = np.cumsum([0] + sizes[:-1]).tolist()
        if factors is None:
            factors = [node_factor(a[:, o:o + c], y, cfg.rho, cfg.nodes, cfg.over_k) for o, c in zip(offs, sizes)]
        else:
            factors = [(torch.as_tensor(b, dtype=torch.float64, device=dev),
                        torch.as_tensor(al, dtype=torch.float64, device=dev)) for b, al in factors]
        if spec is None:
            spec = session_bounds(factors, sizes, cfg.rho, cfg.lam, cfg.iters, cfg.margin, cfg.delta)
        self.rng_r = Rng(cfg.seed)
        self.kappa = cfg.lam / cfg.rho
        self.rbuf = torch.empty((2 * max(sizes), self.L), dtype=torch.int32, device=dev)
        self.blk = {}
        return self.run_blocks(a, y, factors, spec, record_trace)

    def setup_block(self, k: int) -> int:
        """Edge setup (protocol.cpp:186-220): Gamma2(B) rows + sums, Enc_pk(Gamma1(alpha))."""
        import torch

        cfg, spec = self.cfg, self.spec
        b_bar, alpha = self.factors[k]
        c = self.sizes[k]
        st = self._stream()
        q_b, cl_b = self._quantize(b_bar.reshape(-1).contiguous(), spec, fine=False)
        q_b = q_b.reshape(c, c)
        erng = Rng(cfg.seed ^ ((EDGE_SEED_MIX * (k + 1)) & MASK64))
        r_a = self.edge.sample_r_batch(erng, c)
        alpha_hat = torch.empty((c, 2 * self.L), dtype=torch.int32, device=self.dev)
        cla = (C.c_uint64 * 2)()
        _raise_for(self.lib.pcb_quantize_encrypt(self.edge._ctx, L.ptr(alpha.contiguous()), c, spec[0], spec[1],
                                                 spec[2], 1, L.ptr(r_a), 0, L.ptr(alpha_hat), None, cla, st),
                   "alpha encryption")
        self.blk[k] = dict(q_b=q_b.contiguous(), rowsum=q_b.sum(dim=1).contiguous(), alpha_hat=alpha_hat)
        return cl_b + cla[0] + cla[1]

    def advance_stream(self, k: int) -> None:
        """Master r stream: c draws for z, then c for -v (encrypt_state x 2, protocol.cpp:467-468),
        drawn on every rank so each rank's slice matches the single-stream reference."""
        c = self.sizes[k]
        s = C.c_uint64(self.rng_r.state)
        _raise_for(self.lib.pcb_sample_r(self.master._ctx, C.byref(s), 2 * c, L.ptr(self.rbuf), self._stream()),
                   "sample_r")
        self.rng_r.state = s.value

    def step_block(self, k: int, t: int) -> int:
        import torch

        cfg, spec, st = self.cfg, self.spec, self._stream()
        o, c = self.offs[k], self.sizes[k]
        W = 2 * self.L
        b = self.blk[k]
        zc = torch.empty((c, W), dtype=torch.int32, device=self.dev)
        vc = torch.empty((c, W), dtype=torch.int32, device=self.dev)
        q_z = torch.empty(c, dtype=torch.int64, device=self.dev)
        q_nv = torch.empty(c, dtype=torch.int64, device=self.dev)
        nv = (-self.v[o:o + c]).contiguous()
        zk = self.z[o:o + c].contiguous()
        cl1, cl2 = (C.c_uint64 * 2)(), (C.c_uint64 * 2)()
        _raise_for(self.lib.pcb_quantize_encrypt(self.master._ctx, L.ptr(zk), c, spec[0], spec[1], spec[2], 0,
                                                 L.ptr(self.rbuf[:c]), 1, L.ptr(zc), L.ptr(q_z), cl1, st), "Enc z")
        _raise_for(self.lib.pcb_quantize_encrypt(self.master._ctx, L.ptr(nv), c, spec[0], spec[1], spec[2], 0,
                                                 L.ptr(self.rbuf[c:2 * c]), 1, L.ptr(vc), L.ptr(q_nv), cl2, st),
                   "Enc -v")
        upd = torch.empty((c, W), dtype=torch.int32, device=self.dev)
        _raise_for(self.lib.pcb_edge_step(self.edge._ctx, L.ptr(b["alpha_hat"]), L.ptr(b["q_b"]), L.ptr(zc), L.ptr(vc),
                                          c, cfg.window, L.ptr(upd), st), "edge step")
        _raise_for(self.lib.pcb_decrypt_update(self.master._ctx, L.ptr(upd), c, L.ptr(b["rowsum"]), L.ptr(q_z),
                                               L.ptr(q_nv), spec[0], spec[1], spec[2], self.kappa,
                                               L.ptr(self.x[o:o + c]), L.ptr(self.z[o:o + c]),
                                               L.ptr(self.v[o:o + c]), None, st), "master update")
        return cl1[0] + cl1[1] + cl2[0] + cl2[1]
