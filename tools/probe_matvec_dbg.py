"""Timing split of hom_matvec at n^2 (rnsx_kernel<144> step programs; phase B dominates) under the
rnsx timing modes: PCB_RNSX_DBG=0 normal, 1 tensor + W stream only, 2 CUDA-core phases only,
3 W stream only, 4 MMAs only (results are garbage for modes != 0).  One c x c block, CUDA events."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

c_ = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048, device=0)
ph = P.Paillier(kp)
edge = P.Paillier(P.PublicKey(kp.n, kp.key_bits))
rng = np.random.default_rng(1)
q_b = torch.from_numpy(rng.integers(0, 2**50, (c_, c_), dtype=np.int64)).cuda()
m = torch.zeros((c_, ph.L), dtype=torch.int32, device="cuda")
r = ph.sample_r_batch(P.Rng(3), 2 * c_)
alpha = ph.encrypt_batch(m, r[:c_], True)
zc = ph.encrypt_batch(m, r[c_:], True)
torch.cuda.synchronize()
for mode in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2", "3", "4", "0"]):
    os.environ["PCB_RNSX_DBG"] = mode
    best = 1e30
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        edge.hom_matvec_batch(alpha, q_b, zc, 6)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"dbg={mode}: hom_matvec {c_} x {c_} in {best:.2f} ms", flush=True)
