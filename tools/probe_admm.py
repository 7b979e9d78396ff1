"""Development probe: where an encrypted ADMM iteration spends its time (cfg3 block shape).

    python tools/probe_admm.py [--c 512] [--bits 2048]

Times, with a device synchronize around each call: CRT Enc / Dec latency vs batch size, the
edge step (hom_add + matvec) for one c x c block, and the master update.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_14980_b200 import _lib as L  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c", type=int, default=512)
    ap.add_argument("--bits", type=int, default=2048)
    a = ap.parse_args()
    lib = L.lib()
    kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), a.bits)
    ph = P.Paillier(kp)
    edge = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    Lw = ph.L
    rng = np.random.default_rng(1)
    for batch in (256, 512, 1024, 4096, 8192, 16384, 37888, 75776):
        m = torch.from_numpy(rng.integers(0, 2**31, (batch, Lw), dtype=np.int64).astype(np.uint32).view(np.int32)).cuda()
        m[:, Lw - 1] = 0
        r = ph.sample_r_batch(P.Rng(2), batch)
        te = timed(lambda: ph.encrypt_batch(m, r, True))
        c = ph.encrypt_batch(m, r, True)
        td = timed(lambda: ph.decrypt_batch(c, True))
        tp = timed(lambda: edge.encrypt_batch(m, r, False), reps=1) if batch <= 8192 else None
        emit(probe="latency", bits=a.bits, batch=batch, enc_s=te, dec_s=td, enc_per_s=batch / te,
             dec_per_s=batch / td, pub_enc_s=tp)
    c_ = a.c
    q_b = torch.from_numpy(rng.integers(0, 2**50, (c_, c_), dtype=np.int64)).cuda()
    m = torch.zeros((c_, Lw), dtype=torch.int32, device="cuda")
    m[:, 0] = torch.from_numpy(rng.integers(0, 2**31, c_).astype(np.int32)).cuda()
    r = ph.sample_r_batch(P.Rng(3), 3 * c_)
    alpha = edge.encrypt_batch(m, r[:c_], False)
    zc = ph.encrypt_batch(m, r[c_:2 * c_], True)
    vc = ph.encrypt_batch(m, r[2 * c_:], True)
    t_edge = timed(lambda: edge.edge_step_batch(alpha, q_b, zc, vc, 6), reps=2)
    t_mv = timed(lambda: edge.hom_matvec_batch(alpha, q_b, zc, 6), reps=2)
    upd = edge.edge_step_batch(alpha, q_b, zc, vc, 6)
    t_dec = timed(lambda: ph.decrypt_batch(upd, True))
    emit(probe="block", c=c_, bits=a.bits, edge_step_s=t_edge, matvec_s=t_mv, dec_upd_s=t_dec)


if __name__ == "__main__":
    main()
