"""Development probe: RNS/tensor-core CRT halves (PCB_RNS=1 context) vs the carry-chain core.
Bit-for-bit comparison of Enc and Dec on the same inputs, and throughput of both."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
os.environ["PCB_RNS"] = "0"
base = P.Paillier(kp)
os.environ["PCB_RNS"] = "1"
rns = P.Paillier(kp)
L = base.L
rng = np.random.default_rng(5)
m = torch.from_numpy(rng.integers(0, 2**32, (n_el, L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, L - 1] = 0
r = base.sample_r_batch(P.Rng(2), n_el)


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


te_b, cb = timed(lambda: base.encrypt_batch(m, r, True))
te_r, cr = timed(lambda: rns.encrypt_batch(m, r, True))
same_c = bool(torch.equal(cb, cr))
bad_c = int((cb != cr).any(dim=1).sum())
td_b, mb = timed(lambda: base.decrypt_batch(cb, True))
td_r, mr = timed(lambda: rns.decrypt_batch(cb, True))
print(json.dumps(dict(n=n_el, enc_equal=same_c, enc_bad_rows=bad_c, dec_equal=bool(torch.equal(mb, mr)),
                      dec_roundtrip=bool(torch.equal(mb, m)),
                      enc_base_per_s=n_el / te_b, enc_rns_per_s=n_el / te_r,
                      dec_base_per_s=n_el / td_b, dec_rns_per_s=n_el / td_r)), flush=True)
