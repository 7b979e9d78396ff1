"""bench.py — Paillier-2048 Enc+Dec microbench (BASELINE.json configs[1]) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 1048576]

One step = the hot path over one batch of 2^20 values: fused Gamma2-quantize + CRT encryption
(pcb_quantize_encrypt, r from the GPU sample_r stream) followed by CRT decryption
(pcb_decrypt) of the 2^20 ciphertexts.  `value` = Enc+Dec pairs per second for the whole job
(sum over ranks / max-over-ranks device time).  Prints ONE JSON line on rank 0.

Inputs: v_i = -6 + 12 * Rng(1).unit(), QuantSpec{-6, 6, 1e15}; r_i = the
sample_r stream of Rng(2) (rank k > 0 uses Rng(2 + k): the ranks shard independent batches);
key = keygen(Rng(1 ^ 0x6b657967656e2e2e), 2048) (experiments.cpp:61-64).

--impl reference times the reference's own CPU implementation (oracle/_ref/libpcref.so, compiled
from /root/reference by oracle/Makefile) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

KEY_SEED = 1 ^ 0x6B657967656E2E2E
SPEC = (-6.0, 6.0, 1e15)
METRIC = "Paillier-2048 Enc+Dec ops/s per GPU"
UNIT = "Enc+Dec pairs/s"
# canonical algorithmic work, |n| = 2048, s = 64
S = 64
MM = 2 * S * S + S
ENC_MAC = 2 * (2048 + 512) * MM + 4 * MM        # 42,303,744
DEC_MAC = 2 * (1024 + 256) * MM + 4 * MM        # 21,168,384


def splitmix_units(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """Draws offset .. offset+count-1 of Rng(seed).unit(), vectorised counter form of splitmix64
    (bignat.cpp:388-406); a rank's slice of the one job-wide stream."""
    with np.errstate(over="ignore"):
        j = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + j * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows if len(r) > 8 for k in range(4) if r[5 + k].strip() == "Active"})
        loaded = [x for x in sm if x > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def gen_problem_fast(m: int, n: int, sparsity: float, seed: int):
    """Vectorised gen_gaussian_problem (experiments.cpp:324-348): splitmix64 Box-Muller rows of A,
    partial-shuffle support.  numpy's log/cos may differ from libm in the last ulp (synthetic data;
    the encrypted session's parity is tested separately against the shadow pipeline)."""
    u = splitmix_units(seed, 2 * m * n)  # gaussian() draws u1, u2 in order (no u1 == 0 in practice)
    a = (np.sqrt(-2.0 * np.log(u[0::2])) * np.cos(6.283185307179586477 * u[1::2])).reshape(m, n)
    rng = np.random.default_rng(seed)
    x = np.zeros(n)
    idx = rng.choice(n, int(np.ceil(sparsity * n)), replace=False)
    x[idx] = rng.standard_normal(len(idx))
    return a, a @ x


def run_admm(args, rank: int, world: int, local: int):
    """cfg3: 3P-ADMM-PC2 LASSO N=4096, K=8 edge blocks (sharded over ranks), 2048-bit key, M=512."""
    import torch
    import torch.distributed as dist
    from paper_2601_14980_b200 import admm as ADMM
    from paper_2601_14980_b200 import paillier as P

    a, y = gen_problem_fast(512, 4096, 0.1, 1)
    keys = P.keygen(P.Rng(KEY_SEED), 2048, device=local)
    # untimed iterations at the end: every timed iteration then also runs the offline half of a
    # later one (steady state), as in a long session
    iters = args.admm_warmup + args.admm_iters + ADMM.PRE_AHEAD_MAX
    cfg = ADMM.SessionConfig(nodes=8, iters=iters)
    group = dist.group.WORLD if world > 1 else None
    sess = ADMM.EncryptedSession(keys, cfg, device=local, rank=rank, world=world, group=group)
    sess.profile_iters = (args.admm_warmup, args.admm_warmup + args.admm_iters - 1)
    t0 = time.perf_counter()
    res = sess.run(a, y, record_trace=True)  # x is gathered after the timed part of each iteration
    wall = time.perf_counter() - t0
    it = res.iter_seconds[args.admm_warmup:args.admm_warmup + args.admm_iters]
    t = torch.tensor([float(np.mean(it))], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = {"metric": "3P-ADMM-PC2 sec/iteration", "value": float(t.item()), "unit": "s/iteration",
           "higher_is_better": False,
           "config": {"workload": "cfg3 LASSO N=4096, M=512 (recorded choice), K=8 blocks, 2048-bit key, Delta=1e15",
                      "iterations_timed": args.admm_iters, "warmup_iterations": args.admm_warmup,
                      "blocks_per_gpu": 8 // world if 8 % world == 0 else None},
           "iter_seconds": [round(v, 5) for v in res.iter_seconds],
           "final_objective": res.objective[-1], "setup_plus_run_wall_s": wall,
           "phases": {"t_pre_s": res.t_pre_s, "t_master_s": res.t_master_s,
                      "t_loc_s": [round(v, 4) for v in res.t_loc_s], "t_comm_s": [round(v, 4) for v in res.t_comm_s]}}
    if res.profile and res.profile["kernel_ms"] > 0:
        # tensor roofline of the iteration's RNS-core launches (the hom_matvec programs at K = 144 dominate,
        # with the CRT Enc / Dec at K = 40 / 72): int8 ops issued / summed per-launch CUDA-event time
        here = os.path.dirname(os.path.abspath(__file__))
        mp_path = os.path.join(here, "MEASURED_PEAKS.json")
        mp = json.load(open(mp_path)) if os.path.exists(mp_path) else {}
        i8_peak = 2.0 * float(mp.get("bf16_tflops_sustained", mp.get("bf16_tflops", 1400.0)))
        ach = 2.0 * res.profile["int8_macs"] / (res.profile["kernel_ms"] / 1e3) / 1e12
        mv_path = os.path.join(here, "profiles", "r02_matvec_cfg3_ncu.json")
        mv = json.load(open(mv_path)) if os.path.exists(mv_path) else {}
        out["roofline"] = {"bound": "tensor", "achieved": ach, "peak": i8_peak, "unit": "TOPS (int8 dense)",
                           "frac": ach / i8_peak, "kernel": "pcb::rnsx_kernel<144> hom_matvec programs (+ <72>/<40> "
                           "CRT Enc/Dec)", "launches": res.profile["launches"],
                           "kernel_ms_per_iteration": res.profile["kernel_ms"] / res.profile["iterations"],
                           "traffic": mv.get("traffic_bytes_per_launch"), "ncu_pipes_matvec_B": mv.get("pipes")}
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = admm_cpu_leg(sess, res)
    return out


def run_admm_collab(args, rank: int, world: int, local: int):
    """cfg3 with the collaborative variant (paper Alg. 3): the p^2 side of every Enc / Dec is a
    delegated power on the edges (obfuscated exponents, device-side reduction), the master finishes
    with finish_split_encrypt / decrypt_with_half (protocol.cpp:425-511 collab branches)."""
    import torch
    import torch.distributed as dist
    from paper_2601_14980_b200 import admm as ADMM
    from paper_2601_14980_b200 import paillier as P

    a, y = gen_problem_fast(512, 4096, 0.1, 1)
    keys = P.keygen(P.Rng(KEY_SEED), 2048, device=local)
    # one more warm-up iteration than the basic line: the collaborative step runs on three streams,
    # and the stream-ordered scratch pool grows over its first iterations
    wu = args.admm_warmup + 1
    iters = wu + args.admm_collab_iters + ADMM.PRE_AHEAD_MAX
    cfg = ADMM.SessionConfig(nodes=8, iters=iters, variant="collab")
    group = dist.group.WORLD if world > 1 else None
    sess = ADMM.EncryptedSession(keys, cfg, device=local, rank=rank, world=world, group=group)
    res = sess.run(a, y, record_trace=False)
    it = res.iter_seconds[wu:wu + args.admm_collab_iters]
    t = torch.tensor([float(np.mean(it))], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"metric": "3P-ADMM-PC2 sec/iteration (collaborative variant, Alg. 3)", "value": float(t.item()),
            "unit": "s/iteration", "higher_is_better": False, "iter_seconds": [round(v, 5) for v in res.iter_seconds],
            "config": {"workload": "cfg3 LASSO N=4096, M=512, K=8 blocks, 2048-bit key, collaborative variant",
                       "iterations_timed": len(it), "warmup_iterations": wu}}


def run_admm_faithful(args, rank: int, world: int, local: int):
    """cfg3 in faithful-trust mode (FaithfulDriver): the private key on rank 0 only; rank 0
    encrypts and decrypts every block, the edge steps run on the block owners, ciphertexts cross
    ranks by NCCL broadcast / all-gather.  Reported separately: rank 0 serialises
    the whole master side."""
    import torch
    import torch.distributed as dist
    from paper_2601_14980_b200 import admm as ADMM
    from paper_2601_14980_b200 import paillier as P

    a, y = gen_problem_fast(512, 4096, 0.1, 1)
    keys = P.keygen(P.Rng(KEY_SEED), 2048, device=local)
    # one more warm-up iteration than the basic line (the scratch pool grows over the first
    # iterations on the three streams), and an untimed tail: every timed iteration precomputes
    wu = args.admm_warmup + 1
    iters = wu + args.admm_faithful_iters + ADMM.PRE_AHEAD_MAX
    cfg = ADMM.SessionConfig(nodes=8, iters=iters)
    dev = torch.device(f"cuda:{local}")
    at = torch.as_tensor(a, device=dev)
    yt = torch.as_tensor(y, device=dev)
    sizes = ADMM.split_columns(4096, 8)
    offs = np.cumsum([0] + sizes[:-1]).tolist()
    fac = [ADMM.node_factor(at[:, o:o + c], yt, 1.0, 8) for o, c in zip(offs, sizes)]
    spec = torch.tensor(ADMM.session_bounds(fac, sizes, 1.0, 1.0, iters, 1.5, 1e15), dtype=torch.float64, device=dev)
    if world > 1:
        dist.broadcast(spec, src=0)  # the master's QuantSpec (session_init, protocol.cpp:356-371)
    spec = tuple(float(v) for v in spec.tolist())
    drv = ADMM.FaithfulDriver(ADMM.FaithfulGpuBackend(keys, rank, local), cfg, rank=rank, world=world,
                              group=dist.group.WORLD if world > 1 else None)
    res = drv.run(at, yt, fac, spec, record_trace=False)
    it = res.iter_seconds[wu:wu + args.admm_faithful_iters]
    t = torch.tensor([float(np.mean(it))], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"metric": "3P-ADMM-PC2 sec/iteration (faithful trust: private key on rank 0)", "value": float(t.item()),
            "unit": "s/iteration", "higher_is_better": False, "iter_seconds": [round(v, 5) for v in res.iter_seconds],
            "config": {"workload": "cfg3 LASSO N=4096, M=512, K=8 blocks, 2048-bit key; enc_state broadcast + "
                                   "enc_update all-gather over NCCL", "iterations_timed": len(it),
                       "warmup_iterations": wu}}


def admm_cpu_leg(sess, res) -> dict:
    """cpu_baseline leg of the ADMM sub-line: the reference's CPU cost of one cfg3 iteration on
    this host (1 thread and all threads, admm_cpu_baseline), and the parity gate of the session's
    first two iterations against the reference's integer shadow pipeline run through the compiled
    reference (acceptance.cpp:214-281; oracle/admm_oracle.shadow_session_ref) on the same node
    factors and QuantSpec -- bit-identical x."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import admm_oracle as AO

    threads = os.cpu_count() or 1
    fac = [(b.double().cpu().numpy(), al.double().cpu().numpy()) for b, al in sess.factors]
    k = min(2, len(res.x_trace))
    trace, _, _ = AO.shadow_session_ref(fac, sess.sizes, sess.spec, sess.cfg.rho, sess.cfg.lam, k)
    same = all(np.array_equal(np.asarray(res.x_trace[t]), trace[t]) for t in range(k))
    one = admm_cpu_baseline(1)
    allc = admm_cpu_baseline(threads)
    return {"value": allc["value"], "unit": "s/iteration", "cores": threads, "kind": "reference",
            "value_1_thread": one["value"], "per_op_s": allc["per_op_s"], "per_op_s_1_thread": one["per_op_s"],
            "formula": allc["formula"], "host": host_cpu(),
            "sample": "per-op timings through oracle/_ref/libpcref.so: Enc/Dec on 4 x threads elements, hom_add on "
                      "64, hom_matvec 512 columns at two row counts (linear in rows)",
            "parity_vs_reference_shadow": {"iterations": k, "x_bit_identical": bool(same)}}


def run_cfg5(args, rank: int, world: int, local: int):
    """cfg5: 3P-ADMM-PC2 LASSO N=65536 sparse signal, M=10000, 64 edge blocks of 1024
    sharded over the ranks, 2048-bit key.  A is generated on the GPU (synthetic Gaussian, 5.2 GB FP64)."""
    import torch
    import torch.distributed as dist
    from paper_2601_14980_b200 import admm as ADMM
    from paper_2601_14980_b200 import paillier as P

    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(10000, 65536, dtype=torch.float64, device="cuda", generator=g)
    x = torch.zeros(65536, dtype=torch.float64, device="cuda")
    idx = torch.randperm(65536, device="cuda", generator=g)[:6554]
    x[idx] = torch.randn(6554, dtype=torch.float64, device="cuda", generator=g)
    y = a @ x
    keys = P.keygen(P.Rng(KEY_SEED), 2048, device=local)
    iters = args.admm_warmup + args.cfg5_iters + ADMM.PRE_AHEAD_MAX
    cfg = ADMM.SessionConfig(nodes=64, iters=iters)
    group = dist.group.WORLD if world > 1 else None
    sess = ADMM.EncryptedSession(keys, cfg, device=local, rank=rank, world=world, group=group)
    t0 = time.perf_counter()
    # the 64 node factors on the device (pcb_node_factors: FP64 Gram + blocked Cholesky +
    # triangular inverse on DMMA), timed on their own
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fac = ADMM.node_factors(a, y, ADMM.split_columns(65536, 64), cfg.rho, 64)
    e1.record()
    torch.cuda.synchronize()
    t_fac = e0.elapsed_time(e1) / 1e3
    res = sess.run(a, y, factors=fac, record_trace=True)  # x gathered after each iteration's timed part
    wall = time.perf_counter() - t0
    it = res.iter_seconds[args.admm_warmup:args.admm_warmup + args.cfg5_iters]
    t = torch.tensor([float(np.mean(it))], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    out = {"metric": "3P-ADMM-PC2 sec/iteration", "value": float(t.item()), "unit": "s/iteration",
           "higher_is_better": False, "iter_seconds": [round(v, 4) for v in res.iter_seconds],
           "config": {"workload": "cfg5 LASSO N=65536 (10% support), M=10000, K=64 blocks of 1024, 2048-bit key",
                      "iterations_timed": args.cfg5_iters, "blocks_per_gpu": 64 // world if 64 % world == 0 else None,
                      "data": "synthetic Gaussian A generated on the GPU"},
           "final_objective": res.objective[-1], "setup_plus_run_wall_s": wall, "node_factors_s": t_fac,
           "phases": {"t_pre_s": res.t_pre_s, "t_master_s": res.t_master_s,
                      "t_loc_s": [round(v, 4) for v in res.t_loc_s], "t_comm_s": [round(v, 4) for v in res.t_comm_s]}}
    if rank == 0 and not args.no_cpu_baseline:
        # parity gate: the first iteration against the reference's integer shadow pipeline run
        # through the compiled reference, on the session's node factors and QuantSpec
        sys.path.insert(0, str(ROOT / "oracle"))
        import admm_oracle as AO

        fac = [(b.double().cpu().numpy(), al.double().cpu().numpy()) for b, al in sess.factors]
        trace, _, _ = AO.shadow_session_ref(fac, sess.sizes, sess.spec, sess.cfg.rho, sess.cfg.lam, 1)
        out["parity_vs_reference_shadow"] = {"iterations": 1,
                                             "x_bit_identical": bool(np.array_equal(np.asarray(res.x_trace[0]),
                                                                                    trace[0]))}
    return out


def run_p4096(args, rank: int, world: int, local: int):
    """Paillier-4096 (the reference keygen's largest key, paillier.cpp:107-109; the n = 4096 column of
    PAPER.md Table II): key from keygen(Rng(4096), 4096) with the Miller-Rabin rounds batched on the
    device (same key as the reference's keygen), then CRT Enc + CRT Dec of this rank's slice of
    `p4096_n` values, CUDA-event timed after a warm-up pass, round trip checked."""
    import torch
    from paper_2601_14980_b200 import paillier as P

    kp = P.keygen(P.Rng(4096), 4096, device=local)
    ph = P.Paillier(kp, device=local)
    off, n = ADMM_slice(args.p4096_n, world, rank)
    vals = splitmix_units(13, n, offset=off)
    q64 = np.floor(vals * 2.0**60).astype(np.uint64)
    m = torch.zeros((n, ph.L), dtype=torch.int32, device="cuda")
    m[:, 0] = torch.from_numpy((q64 & 0xFFFFFFFF).astype(np.uint32).view(np.int32)).cuda()
    m[:, 1] = torch.from_numpy((q64 >> 32).astype(np.uint32).view(np.int32)).cuda()
    rr = P.Rng(17)
    ph.skip_r(rr, off)
    r = ph.sample_r_batch(rr, n)
    st = torch.zeros(n, dtype=torch.int32, device="cuda")
    w = min(n, 1 << 13)
    ph.decrypt_batch(ph.encrypt_batch(m[:w], r[:w], True, status=st[:w]), True, status=st[:w])  # warm-up
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    c = ph.encrypt_batch(m, r, True, status=st)
    e[1].record()
    d = ph.decrypt_batch(c, True, status=st)
    e[2].record()
    torch.cuda.synchronize()
    te, td = e[0].elapsed_time(e[1]) / 1e3, e[1].elapsed_time(e[2]) / 1e3
    ok = bool(torch.equal(d, m)) and int(st.ne(0).sum().item()) == 0
    t = torch.tensor([te + td], device="cuda")
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"metric": "Paillier-4096 Enc+Dec pairs/s", "value": args.p4096_n / float(t.item()),
            "unit": "Enc+Dec pairs/s", "higher_is_better": True, "enc_per_s": n / te, "dec_per_s": n / td,
            "parity_check": ok,
            "config": {"workload": "4096-bit key (keygen(Rng(4096), 4096)), CRT Enc + CRT Dec, values < 2^60",
                       "values_total": args.p4096_n, "values_per_gpu": n}}


def ADMM_slice(total: int, world: int, rank: int):
    from paper_2601_14980_b200 import admm as ADMM

    return ADMM.rank_slice(total, world, rank)


def run_cfg4(args, rank: int, world: int, local: int):
    """cfg4: Paillier-3072 CRT Enc + Dec of the job's `cfg4_n` values (default 2^22, BASELINE.json
    configs[3]) sliced over the ranks, then the homomorphic aggregation prod c_i mod n^2 (decrypting
    to sum m_i): per-rank product tree -> ncclAllGather of the G partial ciphertexts (G x 768 B) ->
    (G-1)-product fold on every rank (the one exchange step).  Rank k takes values
    [k n, (k+1) n) of the one splitmix stream and the matching slice of the one sample_r stream, so
    every ciphertext and the aggregate are those of the 1-GPU run.  CUDA-event time per phase after
    a warm-up pass on a 2^14 slice.  Key: keypair_from_primes(random_prime(1536) x 2), redrawn until
    n has 3072 bits."""
    import torch
    import torch.distributed as dist
    from paper_2601_14980_b200 import _lib as L
    from paper_2601_14980_b200 import paillier as P

    rng = P.Rng(3072)
    while True:
        p, q = P.random_prime(rng, 1536), P.random_prime(rng, 1536)
        if p != q and (p * q).bit_length() == 3072:
            break
    kp = P.keypair_from_primes(p, q)
    ph = P.Paillier(kp, device=local)
    off, n = ADMM_slice(args.cfg4_n, world, rank)
    vals = splitmix_units(7, n, offset=off) * 12.0 - 6.0
    q64 = np.round((vals + 6.0) / 12.0 * 1e15).astype(np.uint64)  # Gamma2-range plaintexts (< 2^50)
    m = torch.zeros((n, ph.L), dtype=torch.int32, device="cuda")
    m[:, 0] = torch.from_numpy((q64 & 0xFFFFFFFF).astype(np.uint32).view(np.int32)).cuda()
    m[:, 1] = torch.from_numpy((q64 >> 32).astype(np.uint32).view(np.int32)).cuda()
    rr = P.Rng(11)
    ph.skip_r(rr, off)
    r = ph.sample_r_batch(rr, n)
    torch.cuda.synchronize()
    w = min(n, 1 << 14)
    ph.decrypt_batch(ph.encrypt_batch(m[:w], r[:w], True), True)  # warm-up (kernel images, pools)

    def phase(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3, out

    t_enc, c = phase(lambda: ph.encrypt_batch(m, r, True))
    t_dec, d = phase(lambda: ph.decrypt_batch(c, True))
    ph.aggregate_batch(c[:w])

    from paper_2601_14980_b200 import admm as ADMM

    def agg():  # per-rank tree -> all-gather of the G partials (G x 768 B over NVLink) -> fold
        return ADMM.fold_partials(ph.aggregate_batch(c), world, dist.group.WORLD if world > 1 else None,
                                  ph.aggregate_batch)

    t_agg, tot = phase(agg)
    total = int(sum(int(v) for v in q64))
    if world > 1:
        tt = torch.tensor([total % (1 << 62), total >> 62], dtype=torch.int64, device="cuda")
        allt = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(allt, tt)
        total = sum(int(a[0]) + (int(a[1]) << 62) for a in allt)
    sm = ph.decrypt_batch(tot, True)
    ok = bool(torch.equal(d, m)) and L.limbs_to_ints(sm.cpu().numpy().view(np.uint32))[0] == total % kp.n
    t = torch.tensor([t_enc, t_dec, t_agg], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_enc, t_dec, t_agg = (float(v) for v in t.tolist())
    nn = args.cfg4_n
    return {"metric": "Paillier-3072 Enc+Dec pairs/s + aggregation (cfg4)", "value": nn / (t_enc + t_dec),
            "unit": "Enc+Dec pairs/s", "higher_is_better": True, "scaling": "strong",
            "enc_per_s": nn / t_enc, "dec_per_s": nn / t_dec, "aggregate_ciphertexts_per_s": nn / t_agg,
            "seconds": {"enc": t_enc, "dec": t_dec, "aggregate": t_agg}, "parity_check": ok,
            "config": {"workload": "cfg4: 3072-bit key, CRT Enc + CRT Dec + product tree at n^2 (6144-bit), "
                                   "per-rank tree + NCCL all-gather + fold",
                       "values_total": nn, "values_per_gpu": n}}


def cpu_reference_rate(key, vals: np.ndarray, target_s: float, threads: int, keep: bool = False) -> dict:
    """Reference CPU path (crt_encrypt_with_r + crt_decrypt via oracle/_ref/libpcref.so) on a
    bounded sample; returns pairs/s.  The sample grows until it runs >= target_s.  The sample is
    the head of the cfg2 workload: m = Gamma2(v_0..), r = the first draws of sample_r on Rng(2), so
    keep=True also returns the reference's ciphertexts for the bench's parity gate."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import refbind as R

    zmin, zmax, delta = SPEC
    q, _, _ = R.gamma2(vals, zmin, zmax, delta)
    n_el = max(threads, 8)
    while True:
        m = np.zeros((n_el, key.L), np.uint32)
        qq = q[:n_el].astype(np.uint64)
        m[:, 0] = (qq & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        m[:, 1] = (qq >> np.uint64(32)).astype(np.uint32)
        r, _ = key.sample_r(2, n_el)
        t0 = time.perf_counter()
        c, st = key.encrypt(m, r, crt=True, threads=threads)
        mm, sd = key.decrypt(c, crt=True, threads=threads)
        dt = time.perf_counter() - t0
        assert (st == 0).all() and (sd == 0).all() and (mm == m).all()
        if dt >= target_s or n_el >= len(vals):
            out = {"value": n_el / dt, "seconds": dt, "elements": n_el}
            if keep:
                out["c"], out["m"] = c, m
            return out
        n_el = min(len(vals), max(n_el * 2, int(n_el * target_s / max(dt, 1e-3) * 1.1)))


def host_cpu() -> dict:
    """The host the CPU baselines ran on (nproc, lscpu model, physical cores)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {a.strip(): b.strip() for a, b in (ln.split(":", 1) for ln in out.splitlines() if ":" in ln)}
        info["model"] = kv.get("Model name")
        cps, sock, tpc = (int(kv.get(k, "0") or 0) for k in ("Core(s) per socket", "Socket(s)", "Thread(s) per core"))
        info["physical_cores"] = cps * sock if cps and sock else None
        info["threads_per_core"] = tpc or None
    except Exception:  # noqa: BLE001 - informational only
        pass
    return info


def admm_cpu_baseline(threads: int, iters_blocks=(8, 512)) -> dict:
    """The reference's own CPU path for one cfg3 ADMM iteration (BASELINE.md §3 formula, the
    sequential per-link master loop of protocol.cpp:425-511 with the op ledger of
    test_protocol.cpp:179-195): per block of N_k = 512, 2 N_k CRT Enc + N_k (CRT Dec + hom_add) +
    one hom_matvec(512 x 512) at n^2, all through oracle/_ref/libpcref.so on `threads` OpenMP
    threads.  Each op is timed on a bounded sample (Enc/Dec: a few dozen elements; matvec: two row
    counts of the 512-column product, extrapolated linearly in rows: table + rows x row)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import refbind as R

    nblk, nk = iters_blocks
    key = R.RefKey.keygen(KEY_SEED, 2048)
    L = key.L
    rng = np.random.default_rng(3)
    ne = max(4 * threads, 16)
    m = np.zeros((ne, L), np.uint32)
    m[:, 0] = rng.integers(0, 2**32, ne, dtype=np.uint64).astype(np.uint32)
    r, _ = key.sample_r(2, ne)
    key.decrypt(key.encrypt(m[:threads], r[:threads], crt=True, threads=threads)[0], crt=True, threads=threads)  # warm
    t0 = time.perf_counter()
    c, st = key.encrypt(m, r, crt=True, threads=threads)
    t_enc = (time.perf_counter() - t0) / ne
    t0 = time.perf_counter()
    key.decrypt(c, crt=True, threads=threads)
    t_dec = (time.perf_counter() - t0) / ne
    lib = R.lib()
    W = 2 * L
    na = 64
    cc = np.ascontiguousarray(np.concatenate([c] * (na // ne + 1))[:na])
    out = np.zeros_like(cc)
    t0 = time.perf_counter()
    lib.pcref_hom_add(key.h, R.a(cc), R.a(cc), None, None, na, W, R.a(out), None, None)
    t_add = (time.perf_counter() - t0) / na
    cols = nk
    zv = np.ascontiguousarray(np.concatenate([c] * (cols // ne + 1))[:cols])
    expo = rng.integers(0, 10**15, (4 * threads, cols), dtype=np.uint64)
    tm = {}
    for rows in (threads, 2 * threads):
        al = np.ascontiguousarray(np.concatenate([c] * (rows // ne + 1))[:rows])
        ex = np.ascontiguousarray(expo[:rows])
        o = np.zeros((rows, W), np.uint32)
        t0 = time.perf_counter()
        rc = lib.pcref_hom_matvec(key.h, R.a(al), None, R.a(ex), R.a(zv), None, rows, cols, 6, W, R.a(o), None,
                                  threads)
        tm[rows] = time.perf_counter() - t0
        assert rc == 0
    t_row = (tm[2 * threads] - tm[threads]) / threads
    t_tab = max(tm[threads] - threads * t_row, 0.0)
    t_mv = t_tab + nk * t_row
    per_block = 2 * nk * t_enc + nk * (t_dec + t_add) + t_mv
    return {"value": nblk * per_block, "unit": "s/iteration", "threads": threads,
            "per_op_s": {"crt_encrypt_with_r": t_enc, "crt_decrypt": t_dec, "hom_add": t_add,
                         "hom_matvec_512x512": t_mv, "matvec_table": t_tab, "matvec_row": t_row},
            "formula": "8 x [2 N_k T_Enc + N_k (T_Dec + T_add) + T_matvec(N_k)], N_k = 512 (BASELINE.md §3)",
            "kind": "reference"}


def ref_key():
    sys.path.insert(0, str(ROOT / "oracle"))
    import refbind as R

    if not R.available():
        return None
    return R.RefKey.keygen(KEY_SEED, 2048)


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    key = ref_key()
    if key is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpcref.so not built"}))
        return
    vals = -6.0 + 12.0 * splitmix_units(1, 1 << 16)
    for _ in range(args.warmup):
        cpu_reference_rate(key, vals, 0.5, threads)
    rates, secs = [], []
    for _ in range(args.steps):
        r = cpu_reference_rate(key, vals, args.ref_seconds, threads)
        rates.append(r["value"])
        secs.append(r["seconds"])
    value = statistics.median(rates)
    sample = f"{r['elements']} of the 2^20 cfg2 values per step (Gamma2 plaintexts, sample_r(Rng(2)) r)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32-limb integer",
        "data": "synthetic", "config": {"workload": "cfg2 Paillier-2048 Enc+Dec microbench, bounded CPU sample",
                                       "key_bits": 2048},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--values", dest="n", type=int, default=1 << 20)
    ap.add_argument("--e2e-steps", type=int, default=2, help="timed end-to-end steps (>= 1)")
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--admm-iters", type=int, default=5, help="timed cfg3 ADMM iterations (0 = skip)")
    ap.add_argument("--admm-warmup", type=int, default=2)
    ap.add_argument("--admm-faithful-iters", type=int, default=3, help="timed faithful-trust cfg3 iterations (0 = skip)")
    ap.add_argument("--admm-collab-iters", type=int, default=3, help="timed collaborative-variant cfg3 iterations (0 = skip)")
    ap.add_argument("--cfg4-n", type=int, default=1 << 22, help="cfg4 3072-bit values per job, sliced over ranks (0 = skip)")
    ap.add_argument("--cfg5-iters", type=int, default=2, help="timed cfg5 ADMM iterations (N=65536, 64 blocks; 0 = skip)")
    ap.add_argument("--p4096-n", type=int, default=1 << 17, help="Paillier-4096 values per job (0 = skip)")
    args = ap.parse_args()
    args.e2e_steps = max(1, args.e2e_steps)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    # PCB_BENCH_BACKEND=gloo + PCB_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo (a one-GPU
    # rehearsal of the N-rank code path; its timings mean nothing)
    if os.environ.get("PCB_BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("PCB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    from paper_2601_14980_b200 import _lib as L
    from paper_2601_14980_b200 import paillier as P

    lib = L.lib()
    N = args.n
    zmin, zmax, delta = SPEC
    kp = P.keygen(P.Rng(KEY_SEED), 2048, device=local)
    ph = P.Paillier(kp, device=local)
    # rank k encrypts values [k N, (k+1) N) of the one job-wide cfg2 stream with the matching slice
    # of the one sample_r(Rng(2)) stream: the N-rank job computes the 1-rank job's ciphertexts
    vals_np = -6.0 + 12.0 * splitmix_units(1, N, offset=rank * N)
    V = torch.from_numpy(vals_np).cuda()
    rng_r = P.Rng(2)
    ph.skip_r(rng_r, rank * N)
    R = ph.sample_r_batch(rng_r, N)
    C_ = torch.empty((N, 2 * ph.L), dtype=torch.int32, device="cuda")
    M_ = torch.empty((N, ph.L), dtype=torch.int32, device="cuda")
    Q_ = torch.empty((N,), dtype=torch.int64, device="cuda")
    ST_ = torch.zeros((N,), dtype=torch.int32, device="cuda")  # per-element Dec statuses (no host sync)
    cl = (C.c_uint64 * 2)()
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def step():
        L.check(lib.pcb_quantize_encrypt(ph._ctx, L.ptr(V), N, zmin, zmax, delta, 0, L.ptr(R), 1, L.ptr(C_),
                                         L.ptr(Q_), cl, stream))
        L.check(lib.pcb_decrypt(ph._ctx, L.ptr(C_), N, L.ptr(M_), 1, L.ptr(ST_), stream))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    # correctness gate on this run's data: Dec(Enc(Gamma2(v))) == Gamma2(v)
    torch.cuda.synchronize()
    q = Q_.cpu().numpy().view(np.uint64)
    mm = M_.cpu().numpy().view(np.uint32)
    ok = bool((mm[:, 0].astype(np.uint64) | (mm[:, 1].astype(np.uint64) << np.uint64(32)) == q).all()
              and not mm[:, 2:].any() and not ST_.any().item())

    clocks = Clocks(local)
    launches0 = lib.pcb_launch_count()
    barrier()
    clocks.start()
    lib.pcb_profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    barrier()
    ms = C.c_double()
    nl = C.c_uint64()
    alg = C.c_double()
    L.check(lib.pcb_profile_end(C.byref(ms), C.byref(nl), C.byref(alg)))
    clk = clocks.stop()
    gpu_launches = lib.pcb_launch_count() - launches0
    t_ms = e0.elapsed_time(e1)
    t = torch.tensor([t_ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    ms_per_step = t_ms / args.steps
    value = world * N / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel, live CUDA-event per-launch times --------------------
    peak = max(lib.pcb_imad_peak(0, 2000, None), lib.pcb_imad_peak(1, 2000, None))
    achieved = alg.value / (ms.value / 1e3)
    side_share = ms.value / t_ms
    engine = lib.pcb_ctx_engine(ph._ctx)
    int8_macs = lib.pcb_profile_int8_macs()
    here = os.path.dirname(os.path.abspath(__file__))
    mp = json.load(open(os.path.join(here, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(here, "MEASURED_PEAKS.json")) else {}
    prof_path = os.path.join(here, "profiles", "r02_rnsx72_bench_ncu.json")
    prof = json.load(open(prof_path)) if os.path.exists(prof_path) else {}
    roof = None
    if engine == 3:
        kname = ("pcb::rnsx_kernel<72> (+ rnsx_kernel<40> for stage 1 of the split CRT Enc; streaming RNS Montgomery, "
                 "tcgen05 kind::i8 base extensions)")
        dtype = "u32 RNS residues (IMAD) + u8 byte planes on tcgen05 kind::i8 (s32 accumulate); FP64 quantizer"
        # tensor roofline: int8 ops issued by the kernels (2 per MAC, counted per tile-product from
        # the MMA slice shapes) / their CUDA-event time, against int8 dense = 2 x the measured bf16
        # dense peak; the kernels run inside a seconds-long step -> the SUSTAINED figure
        i8_ach = 2.0 * int8_macs / (ms.value / 1e3) / 1e12
        i8_peak = 2.0 * float(mp.get("bf16_tflops_sustained", mp.get("bf16_tflops", 1400.0)))
        roof = {"bound": "tensor", "achieved": i8_ach, "peak": i8_peak, "unit": "TOPS (int8 dense; 2 ops per MAC)",
                "frac": i8_ach / i8_peak, "traffic": prof.get("traffic_bytes_per_launch"),
                "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops_sustained (int8 dense = 2x bf16 dense on tcgen05); "
                               "of measured" if mp else "fallback 2 x 1400",
                "kernel": kname, "launches": int(nl.value), "kernel_ms": ms.value, "share_of_step": side_share,
                "int8_macs": int8_macs,
                "clock_matched_peak": {"value": 2.0 * 8188 * 148 * 1.965e9 / 1e12, "unit": "TOPS",
                                       "source": "tools/mma_mix.cu: 8188 int8 MAC/clk/SM at N = 256, x 148 SMs x "
                                                 "1965 MHz (the clock the bench runs at, `clocks` below)"},
                "ncu_pipes": prof.get("pipes"),
                "imad_canonical": {"achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TMAC32/s",
                                   "ratio": achieved / peak,
                                   "note": "canonical CIOS MAC32 of the reference algorithm per Enc/Dec (BASELINE.md "
                                           "2.1) per second over the measured IMAD.WIDE peak: an EFFECTIVE-THROUGHPUT "
                                           "ratio, not a utilisation (the RNS core and the split CRT encryption do "
                                           "less CUDA-core work than CIOS); the ncu pipe utilisation is ncu_pipes"}}
    else:
        kname = "pcb::side_kernel<64>" if engine != 1 else "pcb::rns_pow_kernel"
        dtype = "u32-limb integer (IMAD.WIDE.U32); FP64 quantizer"
        roof = {"bound": "imad", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TMAC32/s",
                "frac": achieved / peak, "traffic": None, "kernel": kname, "launches": int(nl.value),
                "kernel_ms": ms.value, "share_of_step": side_share}

    # ---- e2e through the C ABI with pinned HOST buffers (copies inside the timed region) ------
    hv = torch.from_numpy(vals_np).pin_memory()
    hc = torch.empty((N, 2 * ph.L), dtype=torch.int32).pin_memory()
    hm = torch.empty((N, ph.L), dtype=torch.int32).pin_memory()
    rdev = torch.empty((N, ph.L), dtype=torch.int32, device="cuda")
    rng_e2e = P.Rng(1000 + rank)

    def e2e_step():
        st = C.c_uint64(rng_e2e.state)
        L.check(lib.pcb_sample_r(ph._ctx, C.byref(st), N, L.ptr(rdev), stream))
        rng_e2e.state = st.value
        L.check(lib.pcb_quantize_encrypt(ph._ctx, L.ptr(hv), N, zmin, zmax, delta, 0, L.ptr(rdev), 1, L.ptr(hc),
                                         None, None, stream))
        L.check(lib.pcb_decrypt(ph._ctx, L.ptr(hc), N, L.ptr(hm), 1, None, stream))

    e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()
    barrier()
    e2e_s = (time.perf_counter() - t0) / args.e2e_steps
    te = torch.tensor([e2e_s], device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * N / float(te.item())
    h2d = N * (8 + 2 * ph.L * 4)          # values in; ciphertexts back in for decryption
    d2h = N * (2 * ph.L * 4 + ph.L * 4)   # ciphertexts out; plaintexts out

    admm = run_admm(args, rank, world, local) if args.admm_iters > 0 else None
    admm_f = run_admm_faithful(args, rank, world, local) if args.admm_faithful_iters > 0 else None
    admm_c = run_admm_collab(args, rank, world, local) if args.admm_collab_iters > 0 else None
    cfg4 = run_cfg4(args, rank, world, local) if args.cfg4_n > 0 else None
    cfg5 = run_cfg5(args, rank, world, local) if args.cfg5_iters > 0 else None
    p4096 = run_p4096(args, rank, world, local) if args.p4096_n > 0 else None

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        key = ref_key()
        if key is not None:
            threads = os.cpu_count() or 1
            r = cpu_reference_rate(key, vals_np[: 1 << 16], args.ref_seconds, threads, keep=True)
            r1 = cpu_reference_rate(key, vals_np[: 1 << 16], args.ref_seconds / 4, 1)
            # parity gate: the reference's ciphertexts of the sample == this run's C_ rows
            ne = r["elements"]
            ours_c = C_[:ne].cpu().numpy().view(np.uint32)
            ours_m = M_[:ne].cpu().numpy().view(np.uint32)
            cpu = {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "reference",
                   "value_1_thread": r1["value"], "host": host_cpu(),
                   "sample": f"{r['elements']} cfg2 elements (Enc+Dec) in {r['seconds']:.1f}s on {threads} OpenMP "
                             f"threads ({r1['elements']} in {r1['seconds']:.1f}s on 1 thread), "
                             f"oracle/_ref/libpcref.so",
                   "parity_vs_reference": {"elements": ne,
                                           "ciphertexts_identical": bool(np.array_equal(ours_c, r["c"])),
                                           "plaintexts_identical": bool(np.array_equal(ours_m, r["m"]))}}
            ok = ok and cpu["parity_vs_reference"]["ciphertexts_identical"] and \
                cpu["parity_vs_reference"]["plaintexts_identical"]
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": "cfg2: Paillier-2048 fused Gamma2-quantize+CRT-Enc then CRT-Dec of "
                                   + ("2^20 values" if N == 1 << 20 else f"{N} values (a reduced run)") + " per GPU",
                       "values_per_gpu": N, "key_bits": 2048,
                       "parallelism": f"dp{world} (rank k: slice k of one job-wide value and sample_r stream)",
                       "l2": "inputs+outputs 0.8 GB/step > 126 MB L2 (no flush needed)",
                       "enc_mac32_per_value": ENC_MAC, "dec_mac32_per_value": DEC_MAC},
            "parity_check": ok,
            "enc_dec_mac32_per_s": value * (ENC_MAC + DEC_MAC),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(gpu_launches),
            "clocks": clk,
            "admm": admm,
            "admm_faithful": admm_f,
            "admm_collab": admm_c,
            "cfg4": cfg4,
            "cfg5": cfg5,
            "p4096": p4096,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
