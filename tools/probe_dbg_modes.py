"""Timing split of the K = 72 RNS kernel: PCB_RNSX_DBG=0 (normal), 1 (tensor + W stream only, no
compute handshakes), 2 (CUDA-core phases only, no tensor waits; results are garbage).  One CRT Dec
batch (two rnsx_kernel<72> launches, exponent p - 1) per mode, CUDA-event timed."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 148 * 256 * 4
kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), int(sys.argv[2]) if len(sys.argv) > 2 else 2048)
ph = P.Paillier(kp)
g = np.random.default_rng(5)
m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
m[:, ph.L - 1] = 0
r = ph.sample_r_batch(P.Rng(2), n_el)
c = ph.encrypt_batch(m, r, True)
torch.cuda.synchronize()
st = torch.zeros(n_el, dtype=torch.int32, device="cuda")
for mode in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1", "2", "0"]):
    os.environ["PCB_RNSX_DBG"] = mode
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d = ph.decrypt_batch(c, True, status=st)
        b.record()
        torch.cuda.synchronize()
    ok = bool(torch.equal(d, m))
    print(f"dbg={mode}: Dec {n_el} in {a.elapsed_time(b):.2f} ms -> {n_el / a.elapsed_time(b) * 1e3:.0f}/s  exact={ok}", flush=True)
os.environ["PCB_RNSX_DBG"] = "0"
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    c2 = ph.encrypt_batch(m, r, True, status=st)
    b.record()
    torch.cuda.synchronize()
print(f"Enc {n_el} in {a.elapsed_time(b):.2f} ms -> {n_el / a.elapsed_time(b) * 1e3:.0f}/s exact={bool(torch.equal(c2, c))}")
