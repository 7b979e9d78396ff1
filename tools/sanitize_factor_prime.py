"""Small launches of the round-2 additions for compute-sanitizer: node factors (tile_kernel,
potrf_kernel, mirror), device Miller-Rabin (mr_pow_kernel), the pooled split encryption
(pcb_finish_split_encrypt_rn) and the session with pooled randomness."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import admm as ADMM  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402

g = np.random.default_rng(1)
a = torch.as_tensor(g.standard_normal((70, 150)), device="cuda")
y = torch.as_tensor(g.standard_normal(70), device="cuda")
f = ADMM.node_factors(a, y, [1, 63, 64, 22], 1.0, 4)
torch.cuda.synchronize()
print("node_factors ok", float(f[2][0].abs().max()))
r = P.Rng(9)
p = P.random_prime(r, 512, device=0)
print("device prime ok", p.bit_length())
kp = P.keygen(P.Rng(77), 2048)
ph = P.Paillier(kp)
M = np.ascontiguousarray(g.integers(0, 2**31, (40, 1)).astype(np.uint32))
R = ph.sample_r_batch(P.Rng(3), 40).cpu().numpy().view(np.uint32)
rn = ph.encrypt_batch(np.zeros((40, 1), np.uint32), R, use_crt=True)
G = np.ascontiguousarray(g.integers(0, 2**32, (40, 2 * ph.L)).astype(np.uint32))
G[:, -1] = 0
c = ph.finish_split_encrypt_rn_batch(M, G, rn)
print("finish_split_encrypt_rn ok", int(c[0, 0]))
