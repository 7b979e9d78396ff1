"""Resident 3P-ADMM-PC2 session on the GPU (basic variant, fresh randomness, CRT master).

Mirrors the per-iteration hot loop of the reference's run_session
(/root/reference/proj/src/protocol.cpp:309-526 master_loop, 181-293 edge_run) with every array
resident in HBM:

  master, per block k (protocol.cpp:425-511):
      Gamma2 + CRT Enc of z_k and -v_k, r from the master stream Rng(seed)
  edge k (protocol.cpp:257-275):
      hom_add + hom_matvec with the public key
  master:
      Dec, range gate, inverse quantization, soft threshold

Blocks are independent inside an iteration (block k reads only its own z_k, v_k), so one
iteration is a few batched calls over all blocks a rank owns — pcb_quantize + pcb_encrypt_rn
on [z ; -v], pcb_edge_step_blocks, pcb_decrypt_update_blocks — with the master r stream drawn
once per iteration in reference order and permuted into batch order.  Encryption is split
offline/online: rn = r^n mod n^2 for iteration t+1 (the expensive modexps; the r stream does not
depend on the data) is computed on a side stream while iteration t's edge step runs, and the
online part is c = (1 + m n) rn mod n^2.  Ciphertexts and the x/z/v trajectory are
bit-identical to the block-at-a-time reference loop.

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
import os
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
    variant: str = "basic"  # "collab": paper Alg. 3, the p^2 side of every Enc/Dec delegated to the edges
    # RandomnessMode (protocol.hpp:17-22): "fresh" draws r per encryption from Rng(seed); "pooled"
    # draws pool_size r once, precomputes their r^n and cycles them (pool[pool_at++ % pool_size],
    # protocol.cpp:382-391) -- ciphertexts change, plaintexts and the trajectory do not
    r_mode: str = "fresh"
    pool_size: int = 16
    mask_bits: int = 64  # exponent mask width of the collaborative variant; 0 sends exponents bare
    use_crt: bool = True  # master arithmetic of the basic variant (the collaborative one is always split)
    engine: str = "packed"  # Engine::packed | coeff_fft: one CUDA lane; the reference pins both to equal results

    def validate(self) -> None:
        """The argument errors run_session raises (protocol.cpp:384, 86-88; protocol.hpp:24-41)."""
        if self.nodes < 1:
            raise ValueError("need at least one node")  # protocol.cpp:533
        if self.iters < 1:
            raise ValueError("need at least one iteration")  # protocol.cpp:534
        if self.variant not in ("basic", "collab"):
            raise ValueError(f"unknown protocol variant {self.variant!r}")
        if self.r_mode not in ("fresh", "pooled"):
            raise ValueError(f"unknown randomness mode {self.r_mode!r}")
        if self.r_mode == "pooled" and self.pool_size < 1:
            raise ValueError("pool size below 1")
        if self.mask_bits > 64 or self.mask_bits < 0:
            raise ValueError("mask width above 64")
        if self.engine not in ("packed", "coeff_fft"):
            raise ValueError(f"unknown engine {self.engine!r}")


@dataclass
class RoleStats:
    """pcadmm::RoleStats (protocol.hpp:43-46): the exponentiation ledger of one protocol role under
    the reference's booking rules (paillier.cpp OpCount), and the edge-side delegated powers."""

    pow_full: int = 0
    pow_half: int = 0
    delegated_pows: int = 0


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
    # master-side phase accounting (protocol.hpp:58-64, protocol.cpp:316-329, 392, 515-525): t_pre_s
    # from loop entry through setup and the randomness pool; each iteration splits into the time the
    # master waits on the edges / the exchange (t_comm_s) and the local remainder (t_loc_s);
    # t_pre_s + sum(t_loc_s + t_comm_s) == t_master_s up to the loop's own bookkeeping
    t_pre_s: float = 0.0
    t_loc_s: list = field(default_factory=list)
    t_comm_s: list = field(default_factory=list)
    t_master_s: float = 0.0
    master: RoleStats = None
    edges: RoleStats = None  # this rank's edges together
    profile: dict = None  # RNS-core launches of the profiled iterations (ShardedDriver.profile_iters)


def check_spec(spec) -> None:
    """check_spec (quantize.cpp:8-15) / run_session's window check (protocol.cpp:535-536)."""
    import math

    z_min, z_max, delta = spec
    if not (math.isfinite(z_min) and math.isfinite(z_max)) or z_max <= z_min:
        raise ValueError("quantization window is empty or non-finite")
    if not (delta >= 1.0) or delta > 9.0e15:
        raise ValueError("delta outside [1, 9e15]")


def draw_mask(rng: Rng, bits: int = 64) -> int:
    """draw_mask (protocol.cpp:86-93): a non-zero mask of `bits` bits (0 = masking off)."""
    if bits == 0:
        return 0
    if bits > 64:
        raise ValueError("mask width above 64")
    while True:
        m = rng.next() if bits == 64 else rng.next() >> (64 - bits)
        if m:
            return m


def draw_masks(rng: Rng, count: int, bits: int = 64) -> np.ndarray:
    """count x draw_mask(rng, bits) as a u64 array: the counter form of splitmix64, with the
    serial retry on a zero draw (probability 2^-bits) kept exact; bits = 0 draws nothing."""
    if bits == 0:
        return np.zeros(count, dtype=np.uint64)
    if bits > 64:
        raise ValueError("mask width above 64")
    GAMMA = 0x9E3779B97F4A7C15
    with np.errstate(over="ignore"):
        z = np.uint64(rng.state) + np.arange(1, count + 1, dtype=np.uint64) * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        if bits < 64:
            z = z >> np.uint64(64 - bits)
    if count and not (z == 0).any():
        rng.state = (rng.state + count * GAMMA) & MASK64
        return z
    return np.array([draw_mask(rng, bits) for _ in range(count)], dtype=np.uint64)


def split_columns(cols: int, k: int) -> list[int]:
    """admm.cpp:77-83."""
    if cols < 1 or k < 1 or k > cols:
        raise ValueError("cannot split columns across nodes")
    sizes = [cols // k] * k
    for i in range(cols % k):
        sizes[i] += 1
    return sizes


def node_factors(a, y, sizes, rho: float, k_total: int, over_k: bool = False):
    """node_factor (admm.cpp:63-75) of every block of the column split at once, on the device
    (pcb_node_factors: FP64 Gram, blocked Cholesky, triangular inverse on DMMA, csrc/factor.cu):
    [(B_k = rho (A_k^T A_k + rho I)^-1, alpha_k = (A_k^T A_k + rho I)^-1 A_k^T y_s)], y_s = y / K
    under over_k.  a: (rows, cols) FP64 CUDA tensor, blocks = consecutive column ranges."""
    import torch

    a = a.contiguous() if a.stride(1) != 1 else a
    y = y.contiguous()
    rows, cols = a.shape
    sz = np.asarray(sizes, dtype=np.uint32)
    b = torch.empty(int((sz.astype(np.uint64) ** 2).sum()), dtype=torch.float64, device=a.device)
    al = torch.empty(cols, dtype=torch.float64, device=a.device)
    st = C.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)
    # a column window of a wider row-major matrix is fine: rows keep unit stride, lda = stride(0)
    _raise_for(L.lib().pcb_node_factors(C.c_void_p(a.data_ptr()), rows, cols, a.stride(0), L.ptr(y), len(sz), sz.ctypes.data,
                                        float(rho), int(k_total), 1 if over_k else 0, L.ptr(b), L.ptr(al), st),
               "node_factors")
    out, mo, co = [], 0, 0
    for c in sz.tolist():
        out.append((b[mo:mo + c * c].view(c, c), al[co:co + c]))
        mo += c * c
        co += c
    return out


def node_factor(a_k, y, rho: float, k_total: int, over_k: bool = False):
    """admm.cpp:63-75 for one block: B = rho (A^T A + rho I)^-1, alpha = (A^T A + rho I)^-1 A^T y_s."""
    return node_factors(a_k, y, [a_k.shape[1]], rho, k_total, over_k)[0]


def session_bounds(factors, sizes, rho, lam, iters, margin, delta):
    """protocol.cpp:29-70 (plaintext rehearsal of the block recurrence) + widen_bounds, on the
    device: the blocks of an iteration are independent, so they advance together as one batched
    matvec over the zero-padded stack of node factors (padding rows stay 0, and 0 is already in
    the running bounds), with the running min / max kept on the device -- one read-back at the end."""
    import torch

    dev = factors[0][0].device
    K, cmax = len(sizes), max(sizes)
    B = torch.zeros((K, cmax, cmax), dtype=torch.float64, device=dev)
    al = torch.zeros((K, cmax), dtype=torch.float64, device=dev)
    for k, ((b_bar, alpha), c) in enumerate(zip(factors, sizes)):
        B[k, :c, :c] = b_bar
        al[k, :c] = alpha
    zero = torch.zeros((), dtype=torch.float64, device=dev)
    lo = torch.minimum(zero, torch.minimum(al.min(), B.min()))
    hi = torch.maximum(zero, torch.maximum(al.max(), B.max()))
    z = torch.zeros((K, cmax), dtype=torch.float64, device=dev)
    v = torch.zeros((K, cmax), dtype=torch.float64, device=dev)
    kappa = lam / rho
    for _ in range(iters):
        x = al + torch.bmm(B, (z - v).unsqueeze(2)).squeeze(2)
        xv = x + v
        z = torch.where(xv > kappa, xv - kappa, torch.where(xv < -kappa, xv + kappa, torch.zeros_like(xv)))
        v = v + (x - z)
        lo = torch.minimum(lo, torch.minimum(z.min(), (-v).min()))
        hi = torch.maximum(hi, torch.maximum(z.max(), (-v).max()))
    lo, hi = float(lo), float(hi)
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

    def check_iteration(self, t: int) -> int:
        """After the iteration's device work has completed: raise deferred errors, return clamps
        counted on the device (backends whose steps never synchronise)."""
        return 0

    def iteration_wait(self, t: int) -> float:
        """Seconds of iteration t the master spent waiting on edge work (the reference's
        carrier-blocked time covers the edges' compute, protocol.cpp:319-329); read after the
        iteration's device work has completed.  Collectives are timed by the driver itself."""
        return 0.0

    def role_stats(self, res: SessionResult) -> None:
        """Fill res.master / res.edges (backends that keep a ledger)."""

    def setup_all(self) -> int:
        """Setup of every block this rank owns (default: one block at a time)."""
        return sum(self.setup_block(k) for k in self.mine)

    def step_all(self, t: int) -> int:
        """One iteration over all blocks in reference order (default: one block at a time).
        Blocks are independent inside an iteration (x_k, z_k, v_k depend only on block k's own
        state, protocol.cpp:486-511), so a backend may batch them."""
        clamps = 0
        for k in range(self.cfg.nodes):
            self.advance_stream(k)
            if k in self.mine:
                clamps += self.step_block(k, t)
        return clamps

    # driver -----------------------------------------------------------------------------------
    def run_blocks(self, a, y, factors, spec, record_trace: bool = True) -> SessionResult:
        import time

        import torch

        cfg = self.cfg
        cfg.validate()
        check_spec(spec)
        sync = (lambda: torch.cuda.synchronize(self.dev)) if self.dev != "cpu" else (lambda: None)
        m0 = time.perf_counter()
        n = a.shape[1]
        self.sizes = split_columns(n, cfg.nodes)
        self.offs = np.cumsum([0] + self.sizes[:-1]).tolist()
        self.factors, self.spec = factors, spec
        self.mine = [k for k in range(cfg.nodes) if self.owner(k) == self.rank]
        res = SessionResult(spec=spec)
        self.x = torch.zeros(n, dtype=torch.float64, device=self.dev)
        self.z = torch.zeros(n, dtype=torch.float64, device=self.dev)
        self.v = torch.zeros(n, dtype=torch.float64, device=self.dev)
        res.clamps += self.setup_all()
        sync()
        res.t_pre_s = time.perf_counter() - m0
        prof = getattr(self, "profile_iters", None)  # (first, last): RNS-core launch profile of those iterations
        for t in range(cfg.iters):
            if prof and t == prof[0]:
                L.lib().pcb_profile_begin()
            it0 = time.perf_counter()
            t0 = time.perf_counter()
            comm = 0.0
            res.clamps += self.step_all(t)
            # objective on z (admm.cpp:31-34): A z partial sums over this rank's blocks
            az = torch.zeros(a.shape[0], dtype=torch.float64, device=self.dev)
            l1 = torch.zeros(1, dtype=torch.float64, device=self.dev)
            for k in self.mine:
                o, c = self.offs[k], self.sizes[k]
                az += a[:, o:o + c] @ self.z[o:o + c]
                l1 += self.z[o:o + c].abs().sum()
            if self.world > 1:
                import torch.distributed as dist

                sync()
                c0 = time.perf_counter()
                dist.all_reduce(az, group=self.group)
                dist.all_reduce(l1, group=self.group)
                sync()
                comm += time.perf_counter() - c0
            r = az - y
            res.objective.append(0.5 * float(r @ r) + cfg.lam * float(l1))
            sync()
            res.clamps += self.check_iteration(t)
            res.iter_seconds.append(time.perf_counter() - t0)
            comm += self.iteration_wait(t)
            if record_trace:
                c0 = time.perf_counter()
                xt = self._gather(self.x.clone())
                if self.world > 1:
                    comm += time.perf_counter() - c0
                res.x_trace.append(xt)
            res.t_comm_s.append(comm)
            res.t_loc_s.append(time.perf_counter() - it0 - comm)
            if prof and t == prof[1]:
                ms, nl, alg = C.c_double(), C.c_uint64(), C.c_double()
                _raise_for(L.lib().pcb_profile_end(C.byref(ms), C.byref(nl), C.byref(alg)), "profile")
                res.profile = {"kernel_ms": ms.value, "launches": int(nl.value),
                               "int8_macs": L.lib().pcb_profile_int8_macs(), "iterations": prof[1] - prof[0] + 1}
        res.t_master_s = time.perf_counter() - m0
        self.role_stats(res)
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
        # offline randomness rn = r^n mod n^2 runs on its own stream and context (the master's
        # private key; separate internal side streams, so it never queues behind the master's Dec)
        self.pre = Paillier(keys, device=device)
        self.edge = Paillier(PublicKey(keys.n, keys.key_bits), device=device)
        self.L = self.master.L
        self.lib = L.lib()
        # capture = {"iters": T}: keep the quantized state and the enc_state ciphertexts of the first
        # T iterations (tests compare them with the reference's encrypt_vec, protocol.cpp:410, 473)
        self.capture = None
        # the iteration's critical path (online Enc -> edge step -> Dec + update) runs at high
        # stream priority; the offline r^n precompute of the next iteration only fills idle SMs
        _raise_for(self.lib.pcb_ctx_set_priority(self.master._ctx, 1), "priority")
        _raise_for(self.lib.pcb_ctx_set_priority(self.edge._ctx, 1), "priority")
        _raise_for(self.lib.pcb_ctx_set_priority(self.pre._ctx, 0), "priority")
        self.delegated_pows = 0  # RoleStats.delegated_pows of this rank's edges (protocol.hpp:43-46)
        self.adj_full = self.adj_half = 0  # ledger bookings the device path does not do itself (role_stats)
        cfg.validate()
        if cfg.variant == "collab":
            # the edges' CrtShare {p^2, phi(p^2)} (paillier.hpp:64-66), n eps, and the mask stream
            # Rng(seed ^ "maskmask") of protocol.cpp:334: first one draw_mask per edge for its
            # decryption exponent obf_dec (session_init, 352-353), then per iteration and block c_k
            # masks for z and c_k for -v (440-446).  Every rank walks the whole stream.
            import math

            from .paillier import crt_share

            self.share = crt_share(keys, device)
            lam = (keys.p - 1) * (keys.q - 1) // math.gcd(keys.p - 1, keys.q - 1)
            self.n_eps = keys.n * int(lam)
            self.eps = int(lam)
            self.mask_rng = Rng(cfg.seed ^ 0x6D61736B6D61736B)
            self.obf_dec = [self.eps + draw_mask(self.mask_rng, cfg.mask_bits) * self.n_eps for _ in range(cfg.nodes)]

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

    def _quantize_async(self, v, spec):
        """Gamma2 on the device; clamps accumulate in clamps_dev, failures in err (no host sync)."""
        import torch

        q = torch.empty((v.shape[0],), dtype=torch.int64, device=v.device)
        _raise_for(self.lib.pcb_quantize_async(L.ptr(v), v.shape[0], spec[0], spec[1], spec[2], 0, L.ptr(q),
                                               L.ptr(self.clamps_dev), L.ptr(self.err), self._stream()), "quantize")
        return q

    def check_iteration(self, t: int) -> int:
        """One read of the device flags per iteration (the stream is already synchronised by the
        objective): the reference throws at the first bad element (ProtocolError /
        invalid_argument / runtime_error, protocol.cpp:20-27, 264-266; paillier.cpp:322-356)."""
        if self.n_own == 0:
            return 0
        code = int(self.err.item())
        if code:
            _raise_for(code, f"iteration {t}")
        if int(self.bad.item()):
            raise ValueError("encryption argument out of range (crt_encrypt_with_r, paillier.cpp:322-323)")
        total = int(self.clamps_dev.sum().item())
        new, self.clamps_seen = total - self.clamps_seen, total
        return new

    def run(self, a, y, factors=None, spec=None, record_trace: bool = True) -> SessionResult:
        import torch

        cfg = self.cfg
        dev = torch.device(self.dev)
        a = torch.as_tensor(a, dtype=torch.float64, device=dev)
        y = torch.as_tensor(y, dtype=torch.float64, device=dev)
        sizes = split_columns(a.shape[1], cfg.nodes)
        offs = np.cumsum([0] + sizes[:-1]).tolist()
        if factors is None:
            factors = node_factors(a, y, sizes, cfg.rho, cfg.nodes, cfg.over_k)
        else:
            factors = [(torch.as_tensor(b, dtype=torch.float64, device=dev),
                        torch.as_tensor(al, dtype=torch.float64, device=dev)) for b, al in factors]
        if spec is None:
            spec = session_bounds(factors, sizes, cfg.rho, cfg.lam, cfg.iters, cfg.margin, cfg.delta)
        self.rng_r = Rng(cfg.seed)
        self.kappa = cfg.lam / cfg.rho
        return self.run_blocks(a, y, factors, spec, record_trace)

    def setup_all(self) -> int:
        """Edge setup of every owned block in one batch (protocol.cpp:186-220 per edge):
        Gamma2(B_k) + row sums, and Enc_pk(Gamma1(alpha_k)) with edge k's own r stream."""
        import torch

        cfg, spec, st = self.cfg, self.spec, self._stream()
        own = self.mine
        self.own_sizes = np.array([self.sizes[k] for k in own], dtype=np.uint32)
        n_own = int(self.own_sizes.sum())
        self.own_lo = self.offs[own[0]] if own else 0
        self.n_own = n_own
        # streams, events and the master r-stream buffers exist on every rank, including one that
        # owns no block (world > nodes): it still advances the shared r stream each iteration
        self.pstream = torch.cuda.Stream(device=self.device, priority=0)  # least priority (offline work)
        self.mstream = torch.cuda.Stream(device=self.device, priority=-1)  # critical path
        self.qstream = torch.cuda.Stream(device=self.device, priority=-1)  # collab: the master's own Dec half
        # the offline r^n runs pre_ahead() iterations ahead: 2 queues it behind the edge step, so it
        # fills the SMs a latency-bound decryption (fewer tiles than SMs) leaves idle (three rn
        # slots); 1 runs the next iteration's beside the edge step, better once the decryption fills
        # the GPU itself (profiles/r02_pre_ahead_ab.txt: cfg3 2, cfg5 1)
        self.pre_ahead = pre_ahead(n_own, torch.cuda.get_device_properties(self.device).multi_processor_count)
        nslot = self.pre_ahead + 1
        self.nslot = nslot
        self.edge_done = torch.cuda.Event()
        self.rn_ready = [torch.cuda.Event() for _ in range(nslot)]
        self.enc_done = torch.cuda.Event()
        self.rall = torch.empty((2 * sum(self.sizes), self.L), dtype=torch.int32, device=self.dev)
        self.rn = [torch.empty((2 * n_own, 2 * self.L), dtype=torch.int32, device=self.dev) for _ in range(nslot)]
        # per-element statuses of the asynchronous encryptions, checked once per iteration after
        # the update's own stream synchronisation (no extra host sync on the critical path)
        self.st_pre = [torch.zeros(2 * n_own, dtype=torch.int32, device=self.dev) for _ in range(nslot)]
        self.st_enc = torch.zeros(2 * n_own, dtype=torch.int32, device=self.dev)
        self.bad = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # asynchronous iteration (pcb_*_async): first failing element's code, clamps on the device
        self.err = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.clamps_dev = torch.zeros(2, dtype=torch.int64, device=self.dev)
        self.clamps_seen = 0
        self.rperm = torch.zeros(0, dtype=torch.int64, device=self.dev)
        self.ev_wait = []  # (start, end) events around edge work the master waits on, this iteration
        self._build_pool()
        if n_own == 0:
            return 0
        b_all = torch.cat([self.factors[k][0].reshape(-1) for k in own]).contiguous()
        q_b, cl_b = self._quantize(b_all, spec, fine=False)
        rows, at = [], 0
        for c in self.own_sizes.tolist():
            rows.append(q_b[at:at + c * c].reshape(c, c).sum(dim=1))
            at += c * c
        self.expo = q_b
        # bit length bound of every Gamma2(B) exponent (constant over the session): the edge step
        # then needs no per-call OR-reduction and read-back
        self.expo_bits = int(q_b.max().item()).bit_length() if q_b.numel() else 1
        self.rowsum = torch.cat(rows).contiguous()
        r_a = torch.empty((n_own, self.L), dtype=torch.int32, device=self.dev)
        at = 0
        for k in own:
            c = self.sizes[k]
            erng = Rng(cfg.seed ^ ((EDGE_SEED_MIX * (k + 1)) & MASK64))
            s_ = C.c_uint64(erng.state)
            _raise_for(self.lib.pcb_sample_r(self.edge._ctx, C.byref(s_), c, L.ptr(r_a[at:at + c]), st), "sample_r")
            at += c
        alpha = torch.cat([self.factors[k][1] for k in own]).contiguous()
        self.alpha_hat = torch.empty((n_own, 2 * self.L), dtype=torch.int32, device=self.dev)
        cla = (C.c_uint64 * 2)()
        _raise_for(self.lib.pcb_quantize_encrypt(self.edge._ctx, L.ptr(alpha), n_own, spec[0], spec[1], spec[2], 1,
                                                 L.ptr(r_a), 0, L.ptr(self.alpha_hat), None, cla, st),
                   "alpha encryption")
        # master r stream layout: block k draws c_k for z then c_k for -v (protocol.cpp:467-468);
        # the batch encrypts [z_own ; -v_own], so gather the owned draws into that order.
        perm_z, perm_v = [], []
        for k in own:
            o, c = self.offs[k], self.sizes[k]
            perm_z.extend(range(2 * o, 2 * o + c))
            perm_v.extend(range(2 * o + c, 2 * o + 2 * c))
        self.rperm = torch.tensor(perm_z + perm_v, dtype=torch.int64, device=self.dev)
        self.m0 = torch.zeros((2 * n_own, 1), dtype=torch.int32, device=self.dev)
        return cl_b + cla[0] + cla[1]


    def _build_pool(self) -> None:
        """Pooled randomness (protocol.cpp:382-388): pool_size r from the master stream Rng(seed),
        each made into an RnFactor once -- r^n mod n^2 (= Enc(0; r)) on the device.  Every rank
        builds the same pool (it is pool_size elements); the ledger books it once, on rank 0, as
        make_rn_factor does (1 full + 2 halves per factor, paillier.cpp:371-383)."""
        import torch

        cfg = self.cfg
        if cfg.r_mode != "pooled":
            return
        P, st = cfg.pool_size, self._stream()
        self.pool_r = torch.empty((P, self.L), dtype=torch.int32, device=self.dev)
        s_ = C.c_uint64(self.rng_r.state)
        _raise_for(self.lib.pcb_sample_r(self.master._ctx, C.byref(s_), P, L.ptr(self.pool_r), st), "sample_r")
        self.rng_r.state = s_.value
        self.pool_rn = torch.empty((P, 2 * self.L), dtype=torch.int32, device=self.dev)
        m0 = torch.zeros((P, 1), dtype=torch.int32, device=self.dev)
        _raise_for(self.lib.pcb_encrypt(self.master._ctx, L.ptr(m0), 1, L.ptr(self.pool_r), P, L.ptr(self.pool_rn), 1,
                                        None, st), "make_rn_factor")
        # pcb_encrypt(use_crt) booked 2 halves per factor; make_rn_factor also books its full
        if self.rank == 0:
            self.adj_full += P
        else:
            self.adj_half -= 2 * P
        self.pool_at = 0

    def _precompute(self, slot: int) -> None:
        """Offline half of the next iteration's encryptions on the side stream: draw the master r
        stream for ALL blocks (reference order), keep this rank's draws in batch order, and
        rn = r^n mod n^2 = Enc(0; r)."""
        import torch

        ps = self.pstream
        ps.wait_event(self.enc_done)  # the slot was last read by an earlier online encryption
        if self.pre_ahead == 2 and self._edge_launched:
            ps.wait_event(self.edge_done)
        with torch.cuda.stream(ps):
            st = C.c_void_p(ps.cuda_stream)
            if self.cfg.r_mode == "pooled":
                # next_factor() in reference order: this iteration's draws sit at stream positions
                # pool_at + [0, 2N); block k's z draws at 2 off_k + i, its -v draws after them
                if self.n_own:
                    idx = torch.remainder(self.rperm + self.pool_at, self.cfg.pool_size)
                    torch.index_select(self.pool_rn, 0, idx, out=self.rn[slot])
                self.pool_at += self.rall.shape[0]
                self.rn_ready[slot].record(ps)
                return
            s_ = C.c_uint64(self.rng_r.state)
            _raise_for(self.lib.pcb_sample_r(self.pre._ctx, C.byref(s_), self.rall.shape[0], L.ptr(self.rall), st),
                       "sample_r")
            self.rng_r.state = s_.value
            # both variants: rn = r^n mod n^2, data-independent, so it is computed here, off the
            # critical path (the collaborative finish_split_encrypt then takes it as its factor)
            if self.n_own:
                r_in = self.rall.index_select(0, self.rperm).contiguous()
                _raise_for(self.lib.pcb_encrypt(self.pre._ctx, L.ptr(self.m0), 1, L.ptr(r_in), r_in.shape[0],
                                                L.ptr(self.rn[slot]), 1 if self.cfg.use_crt else 0,
                                                L.ptr(self.st_pre[slot]), st), "offline encryption")
            self.rn_ready[slot].record(ps)

    def _collab_setup(self):
        """Device-resident constants of the collaborative variant for this rank's blocks."""
        import torch

        n = self.n_own
        S = self.share.S
        self.ne_words = (self.n_eps.bit_length() + 31) // 32
        self.ow = self.ne_words + 3  # value (< 2^64) + mask (< 2^64) * n_eps
        self.neps_dev = torch.from_numpy(L.int_to_limbs(self.n_eps, self.ne_words).view(np.int32)).to(self.dev)
        g = L.int_to_limbs(self.master.n + 1, 2 * S).view(np.int32)
        self.gbase = torch.from_numpy(np.tile(g, (2 * n, 1))).to(self.dev)  # g for every delegated g power
        self.n_dev = torch.from_numpy(L.int_to_limbs(self.master.n, self.L).view(np.int32)).to(self.dev)
        rows = []
        for k in self.mine:  # each edge's obf_dec, repeated over its block's rows
            rows.append(np.tile(L.int_to_limbs(self.obf_dec[k], self.ow), (self.sizes[k], 1)))
        self.obf_dec_rows = torch.from_numpy(np.concatenate(rows).view(np.int32)).to(self.dev) if rows else None
        # obf_dec = eps (1 + mask n) is a multiple of p - 1: the edges' Dec powers take the Fermat form
        # (one |p|-bit chain, pcb_delegated_power_fermat), bit-identical to the generic power
        fac = [self.share.fermat_factor(self.obf_dec[k]) for k in self.mine]
        self.u_mont_rows = None
        if rows and all(f is not None for f in fac) and os.environ.get("PCB_COLLAB_GENERIC_DEC") != "1":
            self.u_mont_rows = torch.from_numpy(np.concatenate(
                [np.tile(f, (self.sizes[k], 1)) for f, k in zip(fac, self.mine)]).view(np.int32)).to(self.dev)
        self.obf_buf = torch.empty((2 * n, self.ow), dtype=torch.int32, device=self.dev)

    def _iteration_masks(self):
        """This iteration's masks for all blocks in reference order (block k: c_k for z, then c_k
        for -v), this rank's draws gathered into batch order [z_own ; -v_own] (like the r stream)."""
        import torch

        m = draw_masks(self.mask_rng, 2 * sum(self.sizes), self.cfg.mask_bits)
        idx = self.rperm.cpu().numpy()
        return torch.from_numpy(m[idx].view(np.int64)).to(self.dev)

    def _collab_encrypt(self, q, r, ct):
        """Alg. 3 encryption, device-resident: obfuscate_exponent(q, n eps, mask) on the master
        (protocol.cpp:11-13, 440-446), the edge's delegated g powers (protocol.cpp:244-249), then the
        master's finish_split_encrypt (paillier.cpp:402-414) with the same r stream as the basic
        variant (protocol.cpp:285-288)."""
        st = self._stream()
        n2 = q.shape[0]
        if not hasattr(self, "gbase"):
            self._collab_setup()
        mask = self._iteration_masks()
        _raise_for(self.lib.pcb_obfuscate_exponent(L.ptr(q), 2, L.ptr(mask), L.ptr(self.neps_dev), self.ne_words, n2,
                                                   L.ptr(self.obf_buf), self.ow, st), "obfuscate_exponent")
        ev = self._wait_begin()
        if os.environ.get("PCB_COLLAB_GENERIC_GPOW") == "1":  # the generic exponentiation (A/B)
            gp = self.share.delegated_power_tensor(self.gbase, self.obf_buf, st)
        else:  # g = n + 1: the binomial collapse, bit-identical (pcb_delegated_power_binomial)
            gp = self.share.delegated_power_binomial_tensor(self.n_dev, self.obf_buf, st)
        self._wait_end(ev)
        self.delegated_pows += n2
        # r: the factor r^n mod n^2 (pooled: protocol.cpp:401-403; fresh: finish_split_encrypt with r,
        # paillier.cpp:402-414, whose two r half_pows ran -- and were counted -- in the offline
        # precompute, _precompute), so the online step is finish_split_encrypt_with_factor
        _raise_for(self.lib.pcb_finish_split_encrypt_rn(self.master._ctx, L.ptr(q), 2, L.ptr(gp), gp.shape[1],
                                                        L.ptr(r), n2, L.ptr(ct), L.ptr(self.st_enc), st),
                   "finish_split_encrypt_with_factor")
        if self.capture is not None:
            self.capture.setdefault("obf", []).append(self.obf_buf.clone())
        return ct

    def _wait_begin(self):
        import torch

        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(self.device))
        return ev

    def _wait_end(self, ev0) -> None:
        import torch

        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(self.device))
        self.ev_wait.append((ev0, ev))

    def iteration_wait(self, t: int) -> float:
        """Device time of the edge work the master waited on this iteration: the edge step and,
        collaborative, the delegated g powers and Dec powers (events on the session stream)."""
        w = sum(a.elapsed_time(b) for a, b in self.ev_wait) / 1e3
        self.ev_wait = []
        return w

    def role_stats(self, res: SessionResult) -> None:
        """The master's ledger = the master and offline-precompute contexts' counters plus the
        bookings the device path does not do itself (pool build; decrypt_vec(use_crt = false) is
        one full per element, paillier.cpp:345-350, where the device always runs the CRT form)."""
        f1, h1 = self.master.counters()
        f2, h2 = self.pre.counters()
        res.master = RoleStats(f1 + f2 + self.adj_full, h1 + h2 + self.adj_half, 0)
        fe, he = self.edge.counters()
        res.edges = RoleStats(fe, he, self.delegated_pows)

    def _collab_dec_powers(self, upd):
        """Edge side of Alg. 3 decryption, device-resident: upd^(obf_dec_k mod phi(p^2)) mod p^2
        with the edge's own obf_dec (protocol.cpp:226-227, 288-291)."""
        import torch

        n = upd.shape[0]
        if self.u_mont_rows is not None:
            px = self.share.delegated_power_fermat_tensor(upd, self.u_mont_rows, self._stream())
        else:
            px = self.share.delegated_power_tensor(upd, self.obf_dec_rows, self._stream())
        self.delegated_pows += n
        full = torch.zeros((n, 2 * self.L), dtype=torch.int32, device=self.dev)
        full[:, : px.shape[1]] = px
        return full

    def step_all(self, t: int) -> int:
        """The iteration on the high-priority session stream, joined back to the caller's stream."""
        import torch

        cur = torch.cuda.current_stream(self.device)
        self.mstream.wait_stream(cur)
        with torch.cuda.stream(self.mstream):
            clamps = self._step_all(t)
        cur.wait_stream(self.mstream)
        return clamps

    def _step_all(self, t: int) -> int:
        """One iteration, all owned blocks batched: quantize [z ; -v] and encrypt online with the
        precomputed rn, launch the offline half of iteration t+1 on the side stream, then one edge
        step over the blocks and one Dec+update — all bit-equal to the block-at-a-time loop."""
        import torch

        cfg, spec, st = self.cfg, self.spec, self._stream()
        slot = t % self.nslot
        if t == 0:
            self._edge_launched = False
            self._precompute(slot)
            if self.pre_ahead == 2 and cfg.iters > 1:
                self._precompute(1)
        cur = torch.cuda.current_stream(self.device)
        cur.wait_event(self.rn_ready[slot])
        n = self.n_own
        clamps = 0
        if n and cfg.r_mode == "fresh":
            self.bad |= self.st_pre[slot].ne(0).any().to(torch.int32)
        if n:
            lo = self.own_lo
            W = 2 * self.L
            vin = torch.cat([self.z[lo:lo + n], -self.v[lo:lo + n]]).contiguous()
            if cfg.variant == "collab":
                q, clamps = self._quantize(vin, spec, fine=False)
            else:
                q = self._quantize_async(vin, spec)
            ct = torch.empty((2 * n, W), dtype=torch.int32, device=self.dev)
            if cfg.variant == "collab":
                ct = self._collab_encrypt(q, self.rn[slot], ct)
                self.bad |= self.st_enc.ne(0).any().to(torch.int32)
            else:
                _raise_for(self.lib.pcb_encrypt_rn(self.master._ctx, L.ptr(q), 2, L.ptr(self.rn[slot]), 2 * n,
                                                   L.ptr(ct), L.ptr(self.st_enc), st), "Enc z, -v")
                self.bad |= self.st_enc.ne(0).any().to(torch.int32)
            if self.capture is not None and t < self.capture.get("iters", 0):
                self.capture.setdefault("q", []).append(q.clone())
                self.capture.setdefault("ct", []).append(ct.clone())
        if not n and cfg.variant == "collab":
            draw_masks(self.mask_rng, 2 * sum(self.sizes), cfg.mask_bits)  # keep the shared mask stream in step
        self.enc_done.record(cur)
        if self.pre_ahead == 1 and t + 1 < cfg.iters:
            self._precompute((t + 1) % self.nslot)
        if n:
            upd = torch.empty((n, W), dtype=torch.int32, device=self.dev)
            sz = self.own_sizes
            ev = self._wait_begin()
            _raise_for(self.lib.pcb_edge_step_blocks_async(
                self.edge._ctx, len(sz), sz.ctypes.data, L.ptr(self.alpha_hat), L.ptr(self.expo), self.expo_bits,
                L.ptr(ct[:n]), L.ptr(ct[n:]), cfg.window, L.ptr(upd), L.ptr(self.err), st), "edge step")
            self.edge_done.record(cur)
            self._edge_launched = True
            if cfg.variant == "collab":  # edge: delegated Dec powers; master: decrypt_with_half + update
                # The master's own CRT half of decrypt_with_half needs only the update ciphertexts,
                # so it runs on its own stream while the edge computes the p^2 side (same results;
                # the edge's update is simply consumed before its delegated powers arrive).
                yq = torch.empty((n, self.master.crt_half_words()), dtype=torch.int32, device=self.dev)
                self.qstream.wait_stream(cur)
                _raise_for(self.lib.pcb_decrypt_half_q(self.master._ctx, L.ptr(upd), n, L.ptr(yq),
                                                       C.c_void_p(self.qstream.cuda_stream)), "decrypt_with_half (q)")
                px = self._collab_dec_powers(upd)
                self._wait_end(ev)
                cur.wait_stream(self.qstream)
                _raise_for(self.lib.pcb_decrypt_update_blocks_half_async(
                    self.master._ctx, len(sz), sz.ctypes.data, L.ptr(upd), L.ptr(px), L.ptr(yq), L.ptr(self.rowsum),
                    L.ptr(q[:n]), L.ptr(q[n:]), spec[0], spec[1], spec[2], self.kappa, L.ptr(self.x[lo:lo + n]),
                    L.ptr(self.z[lo:lo + n]), L.ptr(self.v[lo:lo + n]), L.ptr(self.err), st), "master update (collab)")
            else:
                self._wait_end(ev)
                if not cfg.use_crt:  # decrypt_vec(use_crt = false): one full each (paillier.cpp:345-350)
                    self.adj_full += n
                    self.adj_half -= 2 * n
                _raise_for(self.lib.pcb_decrypt_update_blocks_async(
                    self.master._ctx, len(sz), sz.ctypes.data, L.ptr(upd), L.ptr(self.rowsum), L.ptr(q[:n]),
                    L.ptr(q[n:]), spec[0], spec[1], spec[2], self.kappa, L.ptr(self.x[lo:lo + n]),
                    L.ptr(self.z[lo:lo + n]), L.ptr(self.v[lo:lo + n]), L.ptr(self.err), st), "master update")
        if self.pre_ahead == 2 and t + 2 < cfg.iters:
            self._precompute((t + 2) % self.nslot)
        return clamps


# ---- faithful trust: the private key on rank 0 only (north_star 5) -------------

def pre_ahead(n_own: int, nsm: int = 148) -> int:
    """How many iterations ahead EncryptedSession computes the offline r^n: 2 when the decryption of
    the n_own rows leaves SMs idle (two CRT halves of ceil(n_own / 128)-element tiles on fewer CTAs
    than SMs), else 1; PCB_PRE_AHEAD=1/2 forces it.  A run's last pre_ahead() iterations have no
    precompute left to overlap (bench.py runs PRE_AHEAD_MAX untimed tail iterations)."""
    env = os.environ.get("PCB_PRE_AHEAD")
    if env in ("1", "2"):
        return int(env)
    return 2 if 2 * ((n_own + 127) // 128) < nsm else 1


PRE_AHEAD_MAX = 2


def rank_slice(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal slice [offset, offset + count) of `total` items for `rank` (the first
    total % world ranks take one more): how a job-wide stream of values is sharded."""
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    return rank * base + min(rank, extra), count


def fold_partials(part, world: int, group, fold):
    """Aggregation exchange step: every rank holds its partial product
    (1 x W int32 limb tensor); all-gather the G partials (G x W x 4 bytes over NVLink with NCCL)
    and fold them with `fold` (G x W -> 1 x W, e.g. Paillier.aggregate_batch) on every rank."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return part.reshape(1, -1)
    parts = torch.empty((world, part.numel()), dtype=part.dtype, device=part.device)
    dist.all_gather_into_tensor(parts, part.reshape(1, -1).contiguous(), group=group)
    return fold(parts).reshape(1, -1)


class FaithfulDriver:
    """Faithful-trust 3P-ADMM-PC2 across ranks: rank 0 is the master and the only holder of the
    private key; edge k runs on rank floor(k G / K) with the public key.  Per iteration
    (protocol.cpp:425-511 master, 257-275 edge):

      rank 0      Gamma2 + Enc of [z ; -v] for every block, r from the master stream Rng(seed)
                  in reference order (block k: c_k draws for z, then c_k for -v)
      broadcast   the 2N enc_state ciphertexts (protocol.cpp:471-476) from rank 0
      every rank  the edge step of its own blocks: hom_add + hom_matvec (protocol.cpp:264-271)
      all-gather  the enc_update ciphertexts (protocol.cpp:273-275), padded per rank, reassembled
                  in block order on rank 0
      rank 0      Dec + range gate + inverse quantization + soft threshold (protocol.cpp:488-511)

    Setup: every edge quantizes its own node factor and encrypts Gamma1(alpha) with its own stream
    Rng(seed ^ mix k) (protocol.cpp:186-212); the Gamma2(B) row sums go to rank 0 (node_share,
    protocol.cpp:214-218) through one all-gather.  The ciphertext arithmetic is the backend's
    (FaithfulGpuBackend: the CUDA path; the CPU tests plug a Python-integer backend in), so the
    exchange logic here is the same for NCCL over NVLink and for gloo.  Rank 0's x / z / v equal
    the single-process session's bit for bit."""

    def __init__(self, backend, cfg: SessionConfig, rank: int = 0, world: int = 1, group=None):
        self.B, self.cfg, self.rank, self.world, self.group = backend, cfg, rank, world, group

    def owner(self, k: int) -> int:
        return k * self.world // self.cfg.nodes

    def _gather_rows(self, rows_own, n_max: int, width: int):
        """All-gather each rank's rows (n_own x width), padded to n_max, into block order."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return rows_own
        pad = torch.zeros((n_max, width), dtype=rows_own.dtype, device=rows_own.device)
        pad[: rows_own.shape[0]] = rows_own
        allr = torch.empty((self.world * n_max, width), dtype=rows_own.dtype, device=rows_own.device)
        dist.all_gather_into_tensor(allr, pad, group=self.group)
        out = []
        for r in range(self.world):
            n_r = sum(self.sizes[k] for k in range(self.cfg.nodes) if self.owner(k) == r)
            out.append(allr[r * n_max: r * n_max + n_r])
        return torch.cat(out)  # ranks own consecutive block ranges: rank order == block order

    def run(self, a, y, factors, spec, record_trace: bool = True) -> SessionResult:
        import torch
        import torch.distributed as dist

        import time

        cfg = self.cfg
        cfg.validate()
        if cfg.variant != "basic":
            raise ValueError("the faithful-trust driver runs the basic variant")
        check_spec(spec)
        m0 = time.perf_counter()
        n = a.shape[1]
        self.sizes = split_columns(n, cfg.nodes)
        self.offs = np.cumsum([0] + self.sizes[:-1]).tolist()
        self.mine = [k for k in range(cfg.nodes) if self.owner(k) == self.rank]
        n_max = max(sum(self.sizes[k] for k in range(cfg.nodes) if self.owner(k) == r) for r in range(self.world))
        B = self.B
        res = SessionResult(spec=spec)
        # edge setup of the own blocks; row sums to the master
        rowsum_own, clamps = B.setup_edges(self.mine, factors, self.sizes, spec, cfg)
        res.clamps += clamps
        rowsum = self._gather_rows(rowsum_own.reshape(-1, 1), n_max, 1).reshape(-1)
        if self.rank == 0:
            B.setup_master(self.sizes, spec, cfg)
        dev = B.device
        x = torch.zeros(n, dtype=torch.float64, device=dev)
        z = torch.zeros(n, dtype=torch.float64, device=dev)
        v = torch.zeros(n, dtype=torch.float64, device=dev)
        W = B.width
        B.sync()
        res.t_pre_s = time.perf_counter() - m0
        for t in range(cfg.iters):
            B.sync()
            t0 = time.perf_counter()
            if self.rank == 0:
                ct, q = B.master_encrypt(z, v, t)
            else:
                ct, q = torch.empty((2 * n, W), dtype=torch.int32, device=dev), None
            # the master waits from handing the enc_state frames over to holding every enc_update
            # (timed_send / timed_recv, protocol.cpp:319-329): broadcast, the edge steps, all-gather
            B.sync()
            c0 = time.perf_counter()
            if self.world > 1:
                dist.broadcast(ct, src=0, group=self.group)
            upd_own = B.edge_step(self.mine, self.sizes, self.offs, ct)
            upd = self._gather_rows(upd_own, n_max, W)
            B.sync()
            comm = time.perf_counter() - c0
            if self.rank == 0:
                B.master_update(upd, q, rowsum, self.sizes, spec, cfg, x, z, v)
                r = (a @ z) - y
                res.objective.append(0.5 * float(r @ r) + cfg.lam * float(z.abs().sum()))
                res.clamps += B.check_iteration(t)
            B.sync()
            res.iter_seconds.append(time.perf_counter() - t0)
            if record_trace and self.rank == 0:
                res.x_trace.append(x.clone())
            res.t_comm_s.append(comm)
            res.t_loc_s.append(time.perf_counter() - t0 - comm)
        res.t_master_s = time.perf_counter() - m0
        if hasattr(B, "role_stats"):
            B.role_stats(res, self.rank)
        if self.rank == 0:
            res.x, res.z, res.v = (t_.cpu().numpy() for t_ in (x, z, v))
            res.x_trace = [xt.cpu().numpy() for xt in res.x_trace]
        return res


class FaithfulGpuBackend:
    """The CUDA path under FaithfulDriver: the master's private context lives on rank 0 only; the
    edges use public contexts.  All calls are the asynchronous ABI forms on device tensors."""

    def __init__(self, keys, rank: int, device: int = 0):
        import torch

        self.device = torch.device(f"cuda:{device}")
        self.dev_index = device
        self.lib = L.lib()
        self.keys = keys if rank == 0 else None  # the private key never leaves rank 0
        self.edge = Paillier(PublicKey(keys.n, keys.key_bits), device=device)
        self.master = Paillier(keys, device=device) if rank == 0 else None
        self.L = self.edge.L
        self.width = 2 * self.L
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.clamps_dev = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.clamps_seen = 0

    def _st(self):
        import torch

        return C.c_void_p(torch.cuda.current_stream(self.dev_index).cuda_stream)

    def sync(self):
        """The critical path (the current stream, which the collectives join), not the offline
        precompute on its own stream: the phase timers measure what the master waits on."""
        import torch

        torch.cuda.current_stream(self.device).synchronize()

    def setup_edges(self, mine, factors, sizes, spec, cfg):
        import torch

        st = self._st()
        n_own = sum(sizes[k] for k in mine)
        self.n_own = n_own
        if n_own == 0:
            return torch.zeros(0, dtype=torch.int64, device=self.device), 0
        b_all = torch.cat([torch.as_tensor(factors[k][0], dtype=torch.float64, device=self.device).reshape(-1)
                           for k in mine]).contiguous()
        q_b = torch.empty(b_all.numel(), dtype=torch.int64, device=self.device)
        cl = (C.c_uint64 * 2)()
        _raise_for(self.lib.pcb_quantize(L.ptr(b_all), b_all.numel(), spec[0], spec[1], spec[2], 0, L.ptr(q_b), cl,
                                         st), "quantize B")
        rows, at = [], 0
        for k in mine:
            c = sizes[k]
            rows.append(q_b[at:at + c * c].reshape(c, c).sum(dim=1))
            at += c * c
        self.expo = q_b
        self.expo_bits = int(q_b.max().item()).bit_length() or 1
        r_a = torch.empty((n_own, self.L), dtype=torch.int32, device=self.device)
        at = 0
        for k in mine:
            erng = Rng(cfg.seed ^ ((EDGE_SEED_MIX * (k + 1)) & MASK64))
            s_ = C.c_uint64(erng.state)
            _raise_for(self.lib.pcb_sample_r(self.edge._ctx, C.byref(s_), sizes[k], L.ptr(r_a[at:at + sizes[k]]), st),
                       "sample_r")
            at += sizes[k]
        alpha = torch.cat([torch.as_tensor(factors[k][1], dtype=torch.float64, device=self.device)
                           for k in mine]).contiguous()
        self.alpha_hat = torch.empty((n_own, self.width), dtype=torch.int32, device=self.device)
        cla = (C.c_uint64 * 2)()
        _raise_for(self.lib.pcb_quantize_encrypt(self.edge._ctx, L.ptr(alpha), n_own, spec[0], spec[1], spec[2], 1,
                                                 L.ptr(r_a), 0, L.ptr(self.alpha_hat), None, cla, st), "alpha")
        self.own_sizes = np.array([sizes[k] for k in mine], dtype=np.uint32)
        return torch.cat(rows).contiguous(), int(cl[0] + cl[1] + cla[0] + cla[1])

    def setup_master(self, sizes, spec, cfg):
        import torch

        n = sum(sizes)
        self.n = n
        self.rng_r = Rng(cfg.seed)
        perm_z, perm_v = [], []
        offs = np.cumsum([0] + sizes[:-1]).tolist()
        for k in range(len(sizes)):
            o, c = offs[k], sizes[k]
            perm_z.extend(range(2 * o, 2 * o + c))
            perm_v.extend(range(2 * o + c, 2 * o + 2 * c))
        self.rperm = torch.tensor(perm_z + perm_v, dtype=torch.int64, device=self.device)
        self.rall = torch.empty((2 * n, self.L), dtype=torch.int32, device=self.device)
        self.st_enc = torch.zeros(2 * n, dtype=torch.int32, device=self.device)
        self.spec = spec
        self.kappa = cfg.lam / cfg.rho
        self.cfg = cfg
        self.adj_full = self.adj_half = 0
        if cfg.r_mode == "pooled":  # protocol.cpp:382-388, as EncryptedSession._build_pool
            P, st = cfg.pool_size, self._st()
            pool_r = torch.empty((P, self.L), dtype=torch.int32, device=self.device)
            s_ = C.c_uint64(self.rng_r.state)
            _raise_for(self.lib.pcb_sample_r(self.master._ctx, C.byref(s_), P, L.ptr(pool_r), st), "sample_r")
            self.rng_r.state = s_.value
            self.pool_rn = torch.empty((P, self.width), dtype=torch.int32, device=self.device)
            m0 = torch.zeros((P, 1), dtype=torch.int32, device=self.device)
            _raise_for(self.lib.pcb_encrypt(self.master._ctx, L.ptr(m0), 1, L.ptr(pool_r), P, L.ptr(self.pool_rn), 1,
                                            None, st), "make_rn_factor")
            self.adj_full += P  # make_rn_factor's full (paillier.cpp:376)
            self.pool_at = 0
        else:
            # fresh r: rn = r^n mod n^2 of the next iteration computed offline on a low-priority
            # stream and context (as EncryptedSession), the online Enc is one multiplication
            self.pre = Paillier(self.keys, device=self.dev_index)
            _raise_for(self.lib.pcb_ctx_set_priority(self.pre._ctx, 0), "priority")
            _raise_for(self.lib.pcb_ctx_set_priority(self.master._ctx, 1), "priority")
            self.pstream = torch.cuda.Stream(device=self.device, priority=0)
            # as EncryptedSession: two iterations ahead, behind the edge step, while the master's
            # decryption of the n rows leaves SMs idle (pre_ahead), else one ahead
            self.pre_ahead = pre_ahead(n, torch.cuda.get_device_properties(self.device).multi_processor_count)
            self.nslot = self.pre_ahead + 1
            self.rn = [torch.empty((2 * n, self.width), dtype=torch.int32, device=self.device)
                       for _ in range(self.nslot)]
            self.st_pre = [torch.zeros(2 * n, dtype=torch.int32, device=self.device) for _ in range(self.nslot)]
            self.pre_bad = torch.zeros((), dtype=torch.int32, device=self.device)
            self.m0 = torch.zeros((2 * n, 1), dtype=torch.int32, device=self.device)
            self.rn_ready = [torch.cuda.Event() for _ in range(self.nslot)]
            self.enc_done = torch.cuda.Event()
            self.enc_done.record(torch.cuda.current_stream(self.device))
            self.edge_done = None  # recorded when the edge step's updates reach the master
            self.t_enc = 0

    def master_encrypt(self, z, v, t):
        import torch

        st = self._st()
        spec = self.spec
        vin = torch.cat([z, -v]).contiguous()
        q = torch.empty(vin.numel(), dtype=torch.int64, device=self.device)
        _raise_for(self.lib.pcb_quantize_async(L.ptr(vin), vin.numel(), spec[0], spec[1], spec[2], 0, L.ptr(q),
                                               L.ptr(self.clamps_dev), L.ptr(self.err), st), "quantize")
        ct = torch.empty((vin.numel(), self.width), dtype=torch.int32, device=self.device)
        if self.cfg.r_mode == "pooled":  # crt_encrypt_with_factor / encrypt_with_factor (protocol.cpp:411-415)
            rn = self.pool_rn.index_select(0, torch.remainder(self.rperm + self.pool_at, self.cfg.pool_size))
            self.pool_at += vin.numel()
            _raise_for(self.lib.pcb_encrypt_rn(self.master._ctx, L.ptr(q), 2, L.ptr(rn), vin.numel(), L.ptr(ct),
                                               L.ptr(self.st_enc), st), "enc_state")
        else:
            slot = t % self.nslot
            self.t_enc = t
            if t == 0:
                self._precompute(slot)
                if self.pre_ahead == 2 and self.cfg.iters > 1:
                    self._precompute(1)
            cur = torch.cuda.current_stream(self.device)
            cur.wait_event(self.rn_ready[slot])
            self.pre_bad |= self.st_pre[slot].ne(0).any().to(torch.int32)
            _raise_for(self.lib.pcb_encrypt_rn(self.master._ctx, L.ptr(q), 2, L.ptr(self.rn[slot]), vin.numel(),
                                               L.ptr(ct), L.ptr(self.st_enc), st), "enc_state")
            self.enc_done.record(cur)
            if self.pre_ahead == 1 and t + 1 < self.cfg.iters:
                self._precompute((t + 1) % self.nslot)
        return ct, q

    def _precompute(self, slot):
        """The offline half of an iteration's enc_state (crt_encrypt_with_r, protocol.cpp:410): draw the
        master r stream in reference order, rn = Enc(0; r) = r^n mod n^2 on the low-priority stream."""
        import torch

        ps = self.pstream
        ps.wait_event(self.enc_done)  # the slot was last read by an earlier online encryption
        if self.edge_done is not None:
            ps.wait_event(self.edge_done)
        with torch.cuda.stream(ps):
            st = C.c_void_p(ps.cuda_stream)
            s_ = C.c_uint64(self.rng_r.state)
            _raise_for(self.lib.pcb_sample_r(self.pre._ctx, C.byref(s_), self.rall.shape[0], L.ptr(self.rall), st),
                       "sample_r")
            self.rng_r.state = s_.value
            r = self.rall.index_select(0, self.rperm).contiguous()
            _raise_for(self.lib.pcb_encrypt(self.pre._ctx, L.ptr(self.m0), 1, L.ptr(r), r.shape[0],
                                            L.ptr(self.rn[slot]), 1 if self.cfg.use_crt else 0,
                                            L.ptr(self.st_pre[slot]), st), "offline encryption")
            self.rn_ready[slot].record(ps)

    def edge_step(self, mine, sizes, offs, ct):
        import torch

        if self.n_own == 0:
            return torch.zeros((0, self.width), dtype=torch.int32, device=self.device)
        n = ct.shape[0] // 2
        lo = offs[mine[0]]
        zc = ct[lo:lo + self.n_own]
        vc = ct[n + lo:n + lo + self.n_own]
        upd = torch.empty((self.n_own, self.width), dtype=torch.int32, device=self.device)
        _raise_for(self.lib.pcb_edge_step_blocks_async(
            self.edge._ctx, len(self.own_sizes), self.own_sizes.ctypes.data, L.ptr(self.alpha_hat), L.ptr(self.expo),
            self.expo_bits, L.ptr(zc), L.ptr(vc), 6, L.ptr(upd), L.ptr(self.err), self._st()), "edge step")
        return upd

    def role_stats(self, res, rank: int) -> None:
        """Ledgers as EncryptedSession.role_stats: the master's on rank 0, each rank's edges."""
        if rank == 0:
            f, h = self.master.counters()
            if hasattr(self, "pre"):  # the offline r^n context (fresh r)
                f2, h2 = self.pre.counters()
                f, h = f + f2, h + h2
            res.master = RoleStats(f + self.adj_full, h + self.adj_half, 0)
        fe, he = self.edge.counters()
        res.edges = RoleStats(fe, he, 0)

    def master_update(self, upd, q, rowsum, sizes, spec, cfg, x, z, v):
        import torch

        n = self.n
        ahead2 = getattr(self, "pre_ahead", 1) == 2 and self.t_enc + 2 < cfg.iters
        if ahead2:  # the updates are here: iteration t+2's offline r^n goes beside the decryption
            if self.edge_done is None:
                self.edge_done = torch.cuda.Event()
            self.edge_done.record(torch.cuda.current_stream(self.device))
        if not cfg.use_crt:  # decrypt_vec(use_crt = false): one full each (paillier.cpp:345-350)
            self.adj_full += n
            self.adj_half -= 2 * n
        sz = np.array(sizes, dtype=np.uint32)
        _raise_for(self.lib.pcb_decrypt_update_blocks_async(
            self.master._ctx, len(sz), sz.ctypes.data, L.ptr(upd), L.ptr(rowsum), L.ptr(q[:n]), L.ptr(q[n:]),
            spec[0], spec[1], spec[2], self.kappa, L.ptr(x), L.ptr(z), L.ptr(v), L.ptr(self.err), self._st()),
            "master update")
        if ahead2:  # launched after the decryption, so its CTAs reach the SMs first
            self._precompute((self.t_enc + 2) % self.nslot)

    def check_iteration(self, t):
        code = int(self.err.item())
        if code:
            _raise_for(code, f"iteration {t}")
        if int(self.st_enc.ne(0).any().item()) or (hasattr(self, "pre_bad") and int(self.pre_bad.item())):
            raise ValueError("encryption argument out of range (crt_encrypt_with_r, paillier.cpp:322-323)")
        total = int(self.clamps_dev.sum().item())
        new, self.clamps_seen = total - self.clamps_seen, total
        return new
