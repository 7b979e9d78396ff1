"""Host logic of the session surface (CPU): SessionConfig defaults and argument errors
(protocol.hpp:24-41, protocol.cpp:86-88, 384) and the vectorised mask stream at every width
against the serial draw_mask (protocol.cpp:86-93)."""
import pytest

from paper_2601_14980_b200 import admm as ADMM
from paper_2601_14980_b200.paillier import Rng


def test_defaults_follow_the_reference():
    c = ADMM.SessionConfig()
    assert (c.nodes, c.iters, c.rho, c.lam, c.seed, c.window) == (3, 100, 1.0, 1.0, 1, 6)
    assert (c.r_mode, c.pool_size, c.mask_bits, c.use_crt, c.engine) == ("fresh", 16, 64, True, "packed")
    c.validate()


@pytest.mark.parametrize("kw,msg", [({"r_mode": "pooled", "pool_size": 0}, "pool size below 1"),
                                    ({"mask_bits": 65}, "mask width above 64"),
                                    ({"engine": "x"}, "unknown engine"),
                                    ({"variant": "x"}, "unknown protocol variant"),
                                    ({"r_mode": "x"}, "unknown randomness mode")])
def test_argument_errors(kw, msg):
    with pytest.raises(ValueError, match=msg):
        ADMM.SessionConfig(**kw).validate()
    ADMM.SessionConfig(r_mode="fresh", pool_size=0).validate()  # the pool size only matters pooled


@pytest.mark.parametrize("bits", [64, 63, 32, 16, 8, 3, 1])
def test_draw_masks_equals_serial_draw_mask(bits):
    r1, r2 = Rng(0xABCDEF), Rng(0xABCDEF)
    v = ADMM.draw_masks(r1, 4000, bits)
    s = [ADMM.draw_mask(r2, bits) for _ in range(4000)]
    assert [int(x) for x in v] == s and r1.state == r2.state
    assert all(0 < x < (1 << bits) for x in s)


def test_mask_width_zero_draws_nothing():
    r = Rng(5)
    assert ADMM.draw_mask(r, 0) == 0 and r.state == 5
    assert not ADMM.draw_masks(r, 10, 0).any() and r.state == 5
    with pytest.raises(ValueError, match="mask width above 64"):
        ADMM.draw_mask(r, 65)


@pytest.mark.parametrize("m,n,k,iters", [(20, 30, 3, 10), (40, 64, 4, 25), (30, 50, 7, 6), (12, 8, 3, 5)])
def test_batched_session_bounds_follow_the_restated_rehearsal(m, n, k, iters):
    """session_bounds (protocol.cpp:29-70) advances every block at once over the zero-padded stack
    of node factors; the QuantSpec equals the per-block restatement (oracle/admm_oracle.py)."""
    import numpy as np
    import torch

    import admm_oracle as AO

    a, y, _ = AO.gen_gaussian_problem(m, n, 0.1, 3)
    sizes = AO.split_columns(n, k)
    fac, at = [], 0
    for c in sizes:
        fac.append(AO.node_factor(a[:, at:at + c], y, 1.0, k))
        at += c
    want = AO.session_bounds(a, y, 1.0, 1.0, iters, sizes, 1.5, 1e15, fac)
    got = ADMM.session_bounds([(torch.as_tensor(b), torch.as_tensor(al)) for b, al in fac], sizes, 1.0, 1.0, iters,
                              1.5, 1e15)
    assert np.allclose(got, want, rtol=1e-12, atol=0)


@pytest.mark.parametrize("kw,msg", [({"nodes": 0}, "need at least one node"),
                                    ({"iters": 0}, "need at least one iteration")])
def test_session_counts_validated(kw, msg):  # protocol.cpp:533-534, test_protocol.cpp:371-392
    with pytest.raises(ValueError, match=msg):
        ADMM.SessionConfig(**kw).validate()


@pytest.mark.parametrize("spec", [(1.0, 1.0, 1e6), (2.0, 1.0, 1e6), (float("nan"), 1.0, 1e6), (-1.0, 1.0, 0.5),
                                  (-1.0, 1.0, 1e16)])
def test_quant_spec_validated(spec):  # quantize.cpp:8-15, protocol.cpp:535-536
    with pytest.raises(ValueError):
        ADMM.check_spec(spec)
    ADMM.check_spec((-1.0, 1.0, 1e15))
    with pytest.raises(ValueError):
        ADMM.split_columns(8, 9)  # more nodes than columns (test_protocol.cpp:388-391)


def test_session_bounds_cover_the_rehearsal_extremes():  # test_protocol.cpp:97-123
    import torch

    import admm_oracle as AO

    a, y, _ = AO.gen_gaussian_problem(30, 24, 0.2, 11)
    sizes = AO.split_columns(24, 3)
    fac, at = [], 0
    for c in sizes:
        fac.append(AO.node_factor(a[:, at:at + c], y, 1.0, 3))
        at += c
    tf = [(torch.as_tensor(b), torch.as_tensor(al)) for b, al in fac]
    lo, hi, d = ADMM.session_bounds(tf, sizes, 1.0, 1.0, 20, 1.5, 1e6)
    assert lo < 0.0 < hi and d == 1e6
    assert all(lo <= float(v) <= hi for _, al in fac for v in al)
    lo3, hi3, _ = ADMM.session_bounds(tf, sizes, 1.0, 1.0, 20, 3.0, 1e6)
    assert lo3 < lo and hi3 > hi
