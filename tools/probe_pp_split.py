"""Development probe: a launch-time switch (default PCB_RNSX_PP: one vs two tiles in flight) for
the split encryption's stages and for decryption, 2^20 values, 2048-bit key.
usage: probe_pp_split.py [N] [VAR] [v1,v2,...]"""
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
n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
g = np.random.default_rng(5)
m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = ph.sample_r_batch(P.Rng(2), n_el)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


var = sys.argv[2] if len(sys.argv) > 2 else "PCB_RNSX_PP"
vals = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "0"]
ref = None
for pp in vals:
    os.environ[var] = pp
    te, c = timed(lambda: ph.encrypt_batch(m, r, True))
    td, d = timed(lambda: ph.decrypt_batch(c, True))
    same = ref is None or bool(torch.equal(ref, c))
    ref = c if ref is None else ref
    print(json.dumps(dict(var=var, val=pp, n=n_el, enc_equal=same, enc_per_s=round(n_el / te), dec_per_s=round(n_el / td),
                          roundtrip=bool(torch.equal(d, m)))), flush=True)
