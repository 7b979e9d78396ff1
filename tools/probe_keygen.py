"""Where device keygen's time goes: random_prime at 1024 / 2048 bits (the primes of 2048- / 4096-bit
keys) on the serial host search, the batched search with host pow, and the batched search with
the device pow (mr_pow_kernel)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import paillier as P  # noqa: E402

P.random_prime(P.Rng(1), 512, device=0)  # warm-up (context, module load)
for bits in (1024, 2048):
    seeds = range(100, 104) if bits == 1024 else range(100, 102)
    for name, dev in (("host serial", None), ("batched, host pow", -1), ("batched, device pow", 0)):
        t0 = time.perf_counter()
        for s in seeds:
            P.random_prime(P.Rng(s), bits, device=dev)
        print(f"{bits}-bit prime, {name}: {(time.perf_counter() - t0) / len(seeds):.3f} s", flush=True)
