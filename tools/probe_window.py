"""Sliding-window width A/B for the fixed-exponent RNS core (PCB_WINDOW, read once per process).
Runs itself once per width in a child process: CRT Enc and CRT Dec of n 2048-bit values, CUDA-event
timed (best of 3), and a digest of the ciphertexts so every width is checked bit-identical.
usage: python tools/probe_window.py [n] [w,w,...]"""
import hashlib
import os
import subprocess
import sys
from pathlib import Path

if os.environ.get("_PW_CHILD"):
    import numpy as np
    import torch

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2601_14980_b200 import paillier as P

    n_el = int(sys.argv[1])
    kp = P.keygen(P.Rng(1 ^ 0x6B657967656E2E2E), 2048)
    ph = P.Paillier(kp)
    g = np.random.default_rng(5)
    m = torch.from_numpy(g.integers(0, 2**32, (n_el, ph.L), dtype=np.uint64).astype(np.uint32).view(np.int32)).cuda()
    m[:, ph.L - 1] = 0
    r = ph.sample_r_batch(P.Rng(2), n_el)
    st = torch.zeros(n_el, dtype=torch.int32, device="cuda")

    def timed(fn):
        best, out = 1e30, None
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = fn()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        return best, out

    te, c = timed(lambda: ph.encrypt_batch(m, r, True, status=st))
    td, d = timed(lambda: ph.decrypt_batch(c, True, status=st))
    dig = hashlib.sha256(c.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"w={os.environ['PCB_WINDOW']}: Enc {te:.2f} ms ({n_el / te * 1e3:.0f}/s)  Dec {td:.2f} ms "
          f"({n_el / td * 1e3:.0f}/s)  roundtrip={bool(torch.equal(d, m))}  enc_digest={dig}", flush=True)
else:
    n = sys.argv[1] if len(sys.argv) > 1 else str(148 * 256 * 4)
    for w in (sys.argv[2] if len(sys.argv) > 2 else "5,4,3,6,5").split(","):
        env = dict(os.environ, _PW_CHILD="1", PCB_WINDOW=w)
        subprocess.run([sys.executable, __file__, n], env=env, check=True)
