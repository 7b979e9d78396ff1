"""Dev probe: modexp throughput/correctness, old (32-bit carry-chain) vs radix-2^28 core."""
import os, random, sys, time, json, ctypes as C
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import _lib as L
lib = L.lib()
rnd = random.Random(7)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
for bits in (1024, 2048):
    limbs = bits // 32
    m = rnd.getrandbits(bits) | (1 << (bits - 1)) | 1
    e = rnd.getrandbits(bits) | (1 << (bits - 1))
    xs = [rnd.getrandbits(bits) for _ in range(n)]
    X = torch.from_numpy(L.ints_to_limbs(xs, limbs).view(np.int32)).cuda()
    Y = torch.zeros_like(X)
    M, E = L.int_to_limbs(m, limbs), L.int_to_limbs(e, limbs)
    lib.pcb_modexp_batch(L.ptr(M), limbs, L.ptr(E), limbs, L.ptr(X), 512, L.ptr(Y), None)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rc = lib.pcb_modexp_batch(L.ptr(M), limbs, L.ptr(E), limbs, L.ptr(X), n, L.ptr(Y), None)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    ys = L.limbs_to_ints(Y.cpu().numpy().view(np.uint32))
    bad = sum(1 for i in range(0, n, max(1, n // 200)) if ys[i] != pow(xs[i], e, m))
    S = limbs; mm = 2 * S * S + S
    print(json.dumps(dict(core=os.environ.get("PCB_CORE28", "0"), bits=bits, rc=rc, per_s=n / dt, bad_of_200=bad,
                          canon_tmac=n * (bits + bits // 4) * mm / dt / 1e12)), flush=True)
