"""Timing experiment for the streaming RNS core: PCB_RNSX_DBG=0 (full), 1 (tensor + W stream
only), 2 (CUDA-core work only), 3 (W stream only), 4 (MMAs only).  Prints Enc/s for a 2048- or 3072-bit CRT Enc batch."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["PCB_RNSX"] = "1"
from paper_2601_14980_b200 import paillier as P  # noqa: E402

bits, n_el = int(sys.argv[1]), int(sys.argv[2])
pub_mode = len(sys.argv) > 3 and sys.argv[3] == "pub"  # public-key Enc at n^2 (K = 144 for 2048-bit keys)
if pub_mode:
    os.environ["PCB_RNSX_PUB"] = "1"
if bits == 3072:
    rng = P.Rng(3072)
    while True:
        p, q = P.random_prime(rng, 1536), P.random_prime(rng, 1536)
        if p != q and (p * q).bit_length() == 3072:
            kp = P.keypair_from_primes(p, q)
            break
else:
    kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), bits)
ph = P.Paillier(P.PublicKey(kp.n, kp.key_bits)) if pub_mode else P.Paillier(kp)
g = np.random.default_rng(5)
m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = P.Paillier(kp).sample_r_batch(P.Rng(2), n_el)
out = {}
for dbg in ("0", "1", "2", "3", "4"):
    os.environ["PCB_RNSX_DBG"] = dbg
    ph.encrypt_batch(m, r, not pub_mode)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ph.encrypt_batch(m, r, not pub_mode)
    torch.cuda.synchronize()
    out[dbg] = round(n_el / (time.perf_counter() - t0))
print(json.dumps(dict(bits=bits, n=n_el, pub=pub_mode, spin=os.environ.get("PCB_RNSX_SPIN"), enc_per_s=out)))
