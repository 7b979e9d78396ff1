"""racecheck target: the smallest launches of the RNS core (rnsx_kernel<Cfg<40>> split stage 1 and
rnsx_kernel<Cfg<72>> stage 2 + Dec) -- a handful of elements, one tile per CTA."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import _lib as L  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402

kp = P.keygen(P.Rng(2048), 2048)
ph = P.Paillier(kp)
m = torch.from_numpy(L.ints_to_limbs([5, 6], ph.L).view(np.int32)).cuda()
r = ph.sample_r_batch(P.Rng(2), 2)
c = ph.encrypt_batch(m, r)
assert torch.equal(ph.decrypt_batch(c), m)
torch.cuda.synchronize()
print("rnsx racecheck probe ok")
