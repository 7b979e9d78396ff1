"""Debug probe: hom_matvec at 2048-bit keys (n^2 on the streaming RNS core) vs Python ints."""
import os
import random
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import _lib as L  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402

kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
pub = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
n2 = kp.n2
for rows, cols, bits in [(1, 1, 1), (1, 1, 6), (2, 1, 12), (3, 2, 20), (9, 40, 50)]:
    rnd = random.Random(rows * 100 + cols)
    alpha = [rnd.randrange(1, n2) for _ in range(rows)]
    zv = [rnd.randrange(1, n2) for _ in range(cols)]
    expo = [[rnd.getrandbits(bits) for _ in range(cols)] for _ in range(rows)]
    E = np.array(expo, np.uint64)
    out = pub.hom_matvec_batch(L.ints_to_limbs(alpha, 2 * pub.L), E, L.ints_to_limbs(zv, 2 * pub.L))
    got = L.limbs_to_ints(out)
    res = []
    for i in range(rows):
        want = alpha[i]
        for j in range(cols):
            want = want * pow(zv[j], expo[i][j], n2) % n2
        if os.environ.get("PCB_RNSX_MVDBG") == "1":
            want = alpha[i]
        if os.environ.get("PCB_RNSX_MVDBG") == "2":
            want = zv[0] if i == 0 else -1
        if os.environ.get("PCB_RNSX_MVDBG") == "3":
            want = zv[i] * zv[i] % n2 if i < cols else -1
        tag = "ok" if got[i] == want else ("zero" if got[i] == 0 else ("alpha" if got[i] == alpha[i] else "bad"))
        res.append(tag)
    print(rows, cols, bits, res[:12], flush=True)
