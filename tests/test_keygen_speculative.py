"""Batched Miller-Rabin key generation (pcb_keygen_speculative / pcb_random_prime_speculative,
host/hbn.cpp random_prime_batched) consumes the splitmix64 stream exactly like the reference's
serial random_prime / keygen (bignat.cpp:458-515, paillier.cpp:106-123): same primes, same keys,
same Rng state after.  CPU: the batches evaluated by the host pow (device = -1) against the host
search pcb_random_prime / pcb_keygen and the reference's golden keys; GPU: the same on the device."""
import ctypes as C
import time

import numpy as np
import pytest

from conftest import golden
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import paillier as P


def _prime_spec(seed, bits, device):
    st = C.c_uint64(seed)
    out = np.zeros((bits + 31) // 32, np.uint32)
    rc = L.lib().pcb_random_prime_speculative(C.byref(st), bits, device, out.ctypes.data_as(L._u32p))
    assert rc == 0
    return L.limbs_to_int(out), st.value


@pytest.mark.parametrize("seed,bits", [(1, 65), (2, 96), (3, 128), (4, 200), (5, 256), (6, 512), (0xC0FFEE, 384)])
def test_speculative_prime_search_consumes_the_stream_like_the_serial_one(seed, bits):
    r = P.Rng(seed)
    want = P.random_prime(r, bits)
    got, state = _prime_spec(seed, bits, -1)
    assert got == want and state == r.state


@pytest.mark.parametrize("idx", [0, 1])
def test_speculative_keygen_matches_the_golden_keys(idx):
    k = golden("keys.json")[idx]
    r = P.Rng(k["seed"])
    kp = P.keygen(r, k["bits"], device=-1)
    assert (kp.n, kp.p, kp.q) == (int(k["n"], 16), int(k["p"], 16), int(k["q"], 16))
    r2 = P.Rng(k["seed"])
    P.keygen(r2, k["bits"])
    assert r.state == r2.state


def test_many_seeds_small_primes():
    """Marches with several survivors, composites that pass a first round (small widths make the
    strong-liar case reachable), redraws: 200 seeds at 66..80 bits."""
    for seed in range(200):
        bits = 66 + seed % 15
        r = P.Rng(seed * 7919 + 1)
        want = P.random_prime(r, bits)
        got, state = _prime_spec(seed * 7919 + 1, bits, -1)
        assert (got, state) == (want, r.state), seed


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [1024, 2048])
def test_device_keygen_equals_host_keygen(bits):
    for seed in (11, 12):
        r1, r2 = P.Rng(seed), P.Rng(seed)
        t0 = time.perf_counter()
        k1 = P.keygen(r1, bits)
        t1 = time.perf_counter()
        k2 = P.keygen(r2, bits, device=0)
        t2 = time.perf_counter()
        assert (k1.n, k1.p, k1.q, r1.state) == (k2.n, k2.p, k2.q, r2.state)
        print(f"keygen {bits}: host {t1 - t0:.3f} s, device {t2 - t1:.3f} s")


@pytest.mark.gpu
def test_device_random_prime_1536_and_golden_2048_key():
    r1, r2 = P.Rng(3072), P.Rng(3072)
    assert P.random_prime(r1, 1536) == P.random_prime(r2, 1536, device=0) and r1.state == r2.state
    k = golden("keys.json")[2]
    kp = P.keygen(P.Rng(k["seed"]), k["bits"], device=0)
    assert (kp.n, kp.p, kp.q) == (int(k["n"], 16), int(k["p"], 16), int(k["q"], 16))
