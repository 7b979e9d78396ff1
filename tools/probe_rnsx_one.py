"""ncu helper: one CRT Enc + Dec batch through the streaming RNS core (PCB_RNSX=1)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["PCB_RNSX"] = "1"
from paper_2601_14980_b200 import paillier as P  # noqa: E402

bits, n_el = int(sys.argv[1]), int(sys.argv[2])
kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), bits)
ph = P.Paillier(kp)
rng = np.random.default_rng(5)
m = torch.from_numpy(rng.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = ph.sample_r_batch(P.Rng(2), n_el)
c = ph.encrypt_batch(m, r, True)
d = ph.decrypt_batch(c, True)
torch.cuda.synchronize()
print("roundtrip", bool(torch.equal(d, m)))
