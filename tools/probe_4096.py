"""Paillier-4096 CRT Enc + Dec throughput on one B200 (CUDA events, best of 3), bit-exact round
trip: the reference keygen's largest key size on the device path (rnsx_kernel<72> split stage,
rnsx_kernel<144> halves)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 148 * 128 * 4
kp = P.keygen(P.Rng(4096), 4096, device=0)
ph = P.Paillier(kp)
g = np.random.default_rng(5)
m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = ph.sample_r_batch(P.Rng(2), n_el)
st = torch.zeros(n_el, dtype=torch.int32, device="cuda")


def best(fn):
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), out


te, c = best(lambda: ph.encrypt_batch(m, r, True, status=st))
td, d = best(lambda: ph.decrypt_batch(c, True, status=st))
print(f"4096-bit: {n_el} values  Enc {te:.1f} ms ({n_el / te * 1e3:.0f}/s)  Dec {td:.1f} ms ({n_el / td * 1e3:.0f}/s)  "
      f"pairs/s {n_el / (te + td) * 1e3:.0f}  exact={bool(torch.equal(d, m))}")
