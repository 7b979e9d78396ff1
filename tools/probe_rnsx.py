"""Development probe: streaming RNS core (PCB_RNSX=1 context) vs the default engine.
Bit-for-bit comparison of CRT Enc and Dec on the same inputs, and throughput of both.
usage: probe_rnsx.py BITS N [N ...]   (PROBE_ENV=VAR compares VAR=0 against VAR=1 instead of PCB_RNSX)"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402


def key(bits):
    if bits != 3072:
        return P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), bits)
    rng = P.Rng(3072)
    while True:
        p, q = P.random_prime(rng, 1536), P.random_prime(rng, 1536)
        if p != q and (p * q).bit_length() == 3072:
            return P.keypair_from_primes(p, q)


bits = int(sys.argv[1])
sizes = [int(a) for a in sys.argv[2:]] or [1024]
kp = key(bits)
VAR = os.environ.get("PROBE_ENV", "PCB_RNSX")
VALS = os.environ.get("PROBE_VALS", "0,1").split(",")
os.environ[VAR] = VALS[0]  # baseline: the previous default core for this key size
base = P.Paillier(kp)
os.environ[VAR] = VALS[1]
rx = P.Paillier(kp)
os.environ.pop(VAR, None)
from paper_2601_14980_b200 import _lib as L  # noqa: E402

eng = [L.lib().pcb_ctx_engine(base._ctx), L.lib().pcb_ctx_engine(rx._ctx)] if hasattr(base, "_ctx") else None


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best, out


for n_el in sizes:
    Lw = base.L
    rng = np.random.default_rng(5)
    m = torch.from_numpy(rng.integers(0, 2**32, (n_el, Lw), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
    m[:, Lw - 1] = 0
    r = base.sample_r_batch(P.Rng(2), n_el)
    te_b, cb = timed(lambda: base.encrypt_batch(m, r, True))
    te_r, cr = timed(lambda: rx.encrypt_batch(m, r, True))
    bad_c = int((cb != cr).any(dim=1).sum())
    td_b, mb = timed(lambda: base.decrypt_batch(cb, True))
    td_r, mr = timed(lambda: rx.decrypt_batch(cb, True))
    print(json.dumps(dict(bits=bits, n=n_el, engines=eng, enc_equal=bad_c == 0, enc_bad_rows=bad_c,
                          dec_equal=bool(torch.equal(mb, mr)), dec_roundtrip=bool(torch.equal(mr, m)),
                          enc_base_per_s=round(n_el / te_b), enc_rnsx_per_s=round(n_el / te_r),
                          dec_base_per_s=round(n_el / td_b), dec_rnsx_per_s=round(n_el / td_r))), flush=True)
