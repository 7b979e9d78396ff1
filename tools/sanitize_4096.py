"""Small launches of the 4096-bit paths for compute-sanitizer: CRT Enc (split stage on
rnsx_kernel<72>, halves on <144>, garner<128>), public Enc at n^2 = 8192 bits (radix core), CRT Dec
(dec_finish<128>), hom_add / scalar_mul / aggregate on wide_kernel<27,304,8>, sample_r at L = 128."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import _lib as L  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402

kp = P.keygen(P.Rng(4096), 4096)
ph = P.Paillier(kp)
edge = P.Paillier(P.PublicKey(kp.n, 4096))
n = 20
ms = list(range(1, n + 1))
M = L.ints_to_limbs(ms, ph.L)
R = ph.sample_r_batch(P.Rng(2), n).cpu().numpy().view(np.uint32)
c = ph.encrypt_batch(M, np.ascontiguousarray(R), use_crt=True)
c2 = ph.encrypt_batch(M, np.ascontiguousarray(R), use_crt=False)
assert np.array_equal(c, c2)
assert L.limbs_to_ints(ph.decrypt_batch(c)) == ms
s = edge.hom_add_batch(c[:10].copy(), c[10:].copy())
k = edge.hom_scalar_mul_batch(np.arange(1, 11, dtype=np.uint64), c[:10].copy())
a = edge.aggregate_batch(c)
print("4096 ok", L.limbs_to_ints(ph.decrypt_batch(a.reshape(1, -1)))[0] == sum(ms))
