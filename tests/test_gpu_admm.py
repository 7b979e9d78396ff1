"""GPU encrypted ADMM session (paper_2601_14980_b200/admm.py) vs the reference's integer shadow
pipeline (acceptance.cpp:214-281): given the same node factors and QuantSpec, every decrypted
update equals combined_quantized_update and every x/z/v iterate is BIT-IDENTICAL (acceptance [5]).
With node factors computed on the GPU the trajectory matches the plaintext split recurrence to
FP tolerance (test_protocol.cpp:125-155)."""
import numpy as np
import pytest

import admm_oracle as AO
from paper_2601_14980_b200 import admm as ADMM
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu


def factors_for(a, y, sizes, rho=1.0):
    f, at = [], 0
    for c in sizes:
        f.append(AO.node_factor(a[:, at:at + c], y, rho, len(sizes)))
        at += c
    return f


@pytest.mark.parametrize("bits,m,n,k,iters,seed", [(64, 20, 30, 3, 5, 1), (64, 16, 31, 4, 4, 2),
                                                   (1024, 128, 256, 4, 3, 1)])
def test_session_bit_exact_vs_shadow(bits, m, n, k, iters, seed):
    a, y, _ = AO.gen_gaussian_problem(m, n, 0.1, seed)
    sizes = AO.split_columns(n, k)
    fac = factors_for(a, y, sizes)
    delta = 5e7 if bits == 64 else 1e15  # toy keys cap the update magnitude (acceptance.cpp:306)
    spec = AO.session_bounds(a, y, 1.0, 1.0, iters, sizes, 1.5, delta, fac)
    keys = P.keygen(P.Rng(5 if bits == 64 else 1 ^ 0x6B657967656E2E2E), bits)
    cfg = ADMM.SessionConfig(nodes=k, iters=iters)
    res = ADMM.EncryptedSession(keys, cfg).run(a, y, factors=fac, spec=spec)
    trace, z, v = AO.shadow_session(fac, sizes, spec, 1.0, 1.0, iters)
    for t in range(iters):
        assert res.x_trace[t].tolist() == trace[t], f"iteration {t}"
    assert res.z.tolist() == z and res.v.tolist() == v


def test_session_gpu_factors_track_plaintext():
    a, y, _ = AO.gen_gaussian_problem(40, 60, 0.1, 3)
    sizes = AO.split_columns(60, 3)
    keys = P.keygen(P.Rng(5), 64)
    cfg = ADMM.SessionConfig(nodes=3, iters=8, delta=1e8)  # test_protocol.cpp:128
    res = ADMM.EncryptedSession(keys, cfg).run(a, y)
    xs, _, _, objs = AO.lasso_admm_split(a, y, 1.0, 1.0, 8, sizes)
    for t in range(8):
        assert np.mean((res.x_trace[t] - xs[t]) ** 2) < 1e-10
    assert abs(res.objective[-1] - objs[-1]) / objs[-1] < 1e-5  # test_protocol.cpp:150-152
