"""Ping-pong probe: 2048-bit CRT Enc/Dec through rnsx with one tile (PCB_RNSX_PP=0) vs two tiles
in flight (PCB_RNSX_PP=1) per CTA; bit-exactness and throughput."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
ph = P.Paillier(kp)


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


for n_el in [int(a) for a in sys.argv[1:]] or [300, 65536]:
    g = np.random.default_rng(5)
    m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
    m[:, ph.L - 1] = 0
    r = ph.sample_r_batch(P.Rng(2), n_el)
    res = {}
    outs = {}
    for pp in ("0", "1"):
        os.environ["PCB_RNSX_PP"] = pp
        te, c = timed(lambda: ph.encrypt_batch(m, r, True))
        td, d = timed(lambda: ph.decrypt_batch(c, True))
        outs[pp] = (c, d)
        res[pp] = dict(enc=round(n_el / te), dec=round(n_el / td))
    same = bool(torch.equal(outs["0"][0], outs["1"][0])) and bool(torch.equal(outs["0"][1], outs["1"][1]))
    print(json.dumps(dict(n=n_el, equal=same, roundtrip=bool(torch.equal(outs["1"][1], m)), rates=res)), flush=True)
