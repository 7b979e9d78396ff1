"""ncu target: one 2048-bit CRT Dec batch (two rnsx_kernel<Cfg<72,2>> launches, exponent p-1) of
n elements (default 4 tile pairs per SM), preceded by the Enc that produces the ciphertexts."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 148 * 256 * 4
kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
ph = P.Paillier(kp)
g = np.random.default_rng(5)
m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = ph.sample_r_batch(P.Rng(2), n_el)
c = ph.encrypt_batch(m, r, True)
torch.cuda.synchronize()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    d = ph.decrypt_batch(c, True)
torch.cuda.synchronize()
print("roundtrip", bool(torch.equal(d, m)))
