import sys
sys.path.insert(0, '.')
from paper_2601_14980_b200 import paillier as P
from paper_2601_14980_b200 import _lib as L
for seed in (20260825, 1 ^ 0x6B657967656E2E2E):
    kp = P.keygen(P.Rng(seed), 2048)
    ph = P.Paillier(kp)
    print(seed, kp.n.bit_length(), kp.p.bit_length(), kp.q.bit_length(), (kp.p**2).bit_length(), (kp.q**2).bit_length(), L.lib().pcb_ctx_engine(ph._ctx), flush=True)
