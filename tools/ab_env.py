"""A/B of a runtime switch of the RNS core (an environment variable read at every launch):
CRT Dec and CRT Enc of n 2048-bit values per setting, CUDA-event timed, best of 3, results
checked bit-exact against the first setting's.  usage: ab_env.py VAR v1,v2,... [n]"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

var, vals = sys.argv[1], sys.argv[2].split(",")
n_el = int(sys.argv[3]) if len(sys.argv) > 3 else 148 * 256 * 4
kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
ph = P.Paillier(kp)
g = np.random.default_rng(5)
m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = ph.sample_r_batch(P.Rng(2), n_el)
st = torch.zeros(n_el, dtype=torch.int32, device="cuda")
ref_c = None


def best(fn):
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), out


for rnd in range(2):
    for v in vals:
        os.environ[var] = v
        te, c = best(lambda: ph.encrypt_batch(m, r, True, status=st))
        td, d = best(lambda: ph.decrypt_batch(c, True, status=st))
        if ref_c is None:
            ref_c = c.clone()
        ok = bool(torch.equal(c, ref_c)) and bool(torch.equal(d, m))
        print(f"{var}={v}: Enc {te:.2f} ms  Dec {td:.2f} ms  pairs/s {n_el / (te + td) * 1e3:.0f}  exact={ok}", flush=True)
