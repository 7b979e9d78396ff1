"""Debug probe: public-key encryption at n^2 (2048-bit key) on the streaming RNS core vs radix."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import _lib as L  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402

kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
pub = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
rng = np.random.default_rng(1)
m = rng.integers(0, 2**32, (n, pub.L), dtype=np.uint64).astype(np.uint32)
m[:, pub.L - 1] = 0
r = np.ascontiguousarray(rng.integers(1, 2**32, (n, pub.L), dtype=np.uint64).astype(np.uint32))
r[:, pub.L - 1] = 1
c0 = pub.encrypt_batch(m, r, use_crt=False)
os.environ["PCB_RNSX_PUB"] = "1"
c1 = pub.encrypt_batch(m, r, use_crt=False)
bad = (c0 != c1).any(axis=1)
print("rows", n, "mismatch", int(bad.sum()))
if bad.any():
    i = int(np.argmax(bad))
    a, b = L.limbs_to_ints(c0[i:i + 1])[0], L.limbs_to_ints(c1[i:i + 1])[0]
    print("row", i, "radix", hex(a)[:40], "rnsx", hex(b)[:40], "rnsx<n2", b < kp.n2)
