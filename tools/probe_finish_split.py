"""Localise pcb_finish_split_encrypt on small keys / random generators against Python integers."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import _lib as L  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402


def run(kp, g):
    ph = P.Paillier(kp)
    n, n2 = kp.n, kp.n * kp.n
    p2, q2 = kp.p ** 2, kp.q ** 2
    if g != n + 1:
        gl = L.ints_to_limbs([g], 2 * ph.L)
        assert L.lib().pcb_ctx_set_generator(ph._ctx, gl.ctypes.data, 2 * ph.L) == 0
    bad = 0
    for m, r in [(0, 2), (3, 2), (7, 17), (20, 3), (34 % n, 5)]:
        m %= n
        gp = pow(g % p2, m % (p2 - kp.p), p2)
        want = pow(g, m, n2) * pow(r, n, n2) % n2
        M, G, R = L.ints_to_limbs([m], ph.L), L.ints_to_limbs([gp], 2 * ph.L), L.ints_to_limbs([r], ph.L)
        c = np.zeros((1, 2 * ph.L), np.uint32)
        st = np.zeros(1, np.int32)
        rc = L.lib().pcb_finish_split_encrypt(ph._ctx, M.ctypes.data, ph.L, G.ctypes.data, 2 * ph.L, R.ctypes.data, 1,
                                             c.ctypes.data, st.ctypes.data, None)
        got = L.limbs_to_ints(c)[0]
        ok = rc == 0 and got == want
        bad += not ok
        print(f"  bits={kp.key_bits} g={'n+1' if g == n + 1 else 'rand'} m={m} r={r}: rc={rc} st={st[0]} ok={ok}"
              + ("" if ok else f" got={got} want={want} gq={pow(g, m, q2) * pow(r, n, q2) % q2} cp={gp * pow(r, n, p2) % p2}"))
    return bad


toy = P.keypair_from_primes(5, 7)
k64 = P.keygen(P.Rng(77), 64)
k2048 = P.keygen(P.Rng(77), 2048)
tot = 0
for kp in (toy, k64, k2048):
    tot += run(kp, kp.n + 1)
    g = 3 if kp.n > 100 else 11
    tot += run(kp, g)
print("failures", tot)
