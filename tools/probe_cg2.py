"""cta_group::2 probe: public-key Enc at n^2 (K = 144) and 3072-bit CRT Enc/Dec (K = 112) with the
CTA-pair MMA (PCB_RNSX_CG2=1) vs one CTA per MMA; bit-exactness and throughput."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402


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


which = sys.argv[1]
n_el = int(sys.argv[2])
if which == "pub":
    kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
    ph = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
    rgen = P.Paillier(kp)
else:
    rng = P.Rng(3072)
    while True:
        p, q = P.random_prime(rng, 1536), P.random_prime(rng, 1536)
        if p != q and (p * q).bit_length() == 3072:
            kp = P.keypair_from_primes(p, q)
            break
    ph = rgen = P.Paillier(kp)
g = np.random.default_rng(5)
m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = rgen.sample_r_batch(P.Rng(2), n_el)
res, outs = {}, {}
for cg in ("0", "1"):
    os.environ["PCB_RNSX_CG2"] = cg
    te, c = timed(lambda: ph.encrypt_batch(m, r, which != "pub"))
    res[cg] = {"enc": round(n_el / te)}
    outs[cg] = c
    if which != "pub":
        td, d = timed(lambda: ph.decrypt_batch(c, True))
        res[cg]["dec"] = round(n_el / td)
        outs[cg + "d"] = d
same = bool(torch.equal(outs["0"], outs["1"]))
if which != "pub":
    same = same and bool(torch.equal(outs["0d"], outs["1d"]))
print(json.dumps(dict(which=which, n=n_el, equal=same, rates=res)), flush=True)
