"""Development probe: one c x c hom_matvec at n^2 (for ncu launch lists)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

c_ = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
ph = P.Paillier(kp)
edge = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
rng = np.random.default_rng(1)
q_b = torch.from_numpy(rng.integers(0, 2**50, (c_, c_), dtype=np.int64)).cuda()
m = torch.zeros((c_, ph.L), dtype=torch.int32, device="cuda")
r = ph.sample_r_batch(P.Rng(3), 2 * c_)
alpha = ph.encrypt_batch(m, r[:c_], True)
zc = ph.encrypt_batch(m, r[c_:], True)
torch.cuda.synchronize()
import time
out = edge.hom_matvec_batch(alpha, q_b, zc, 6)
torch.cuda.synchronize()
t0 = time.perf_counter()
out = edge.hom_matvec_batch(alpha, q_b, zc, 6)
torch.cuda.synchronize()
print("matvec", c_, "x", c_, "s:", round(time.perf_counter() - t0, 4), out.shape)
