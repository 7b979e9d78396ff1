"""ncu target: one CRT Enc + Dec batch (2048-bit key, K = 72 rnsx) and one public-key Enc batch at
n^2 (K = 144 rnsx), each on a full-GPU batch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 37888
kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
ph = P.Paillier(kp)
pub = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
g = np.random.default_rng(5)
m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = ph.sample_r_batch(P.Rng(2), n_el)
c = ph.encrypt_batch(m, r, True)
d = ph.decrypt_batch(c, True)
c2 = pub.encrypt_batch(m[: n_el // 2], r[: n_el // 2], False)
torch.cuda.synchronize()
print("roundtrip", bool(torch.equal(d, m)))
