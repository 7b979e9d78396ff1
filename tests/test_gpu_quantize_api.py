"""The Python quantizer mirror (paper_2601_14980_b200/quantize.py, quantize.hpp:13-71) on the GPU:
the closed values, clamp counts and errors of the reference's test_quantize.cpp, and bit-equality
with the restated quantizers (oracle/pcadmm_oracle.py, pinned by the compiled reference's golden
vectors) on random inputs."""
import random

import pytest

import pcadmm_oracle as O
from paper_2601_14980_b200 import quantize as Q

pytestmark = pytest.mark.gpu


def test_closed_values_ties_away_from_zero():  # test_quantize.cpp:11-34
    s = Q.QuantSpec(0.0, 1.0, 10.0)
    assert Q.gamma2_vec([0.0, 1.0, 0.44, 0.45, 0.05, 0.25], s) == [0, 10, 4, 5, 1, 3]
    assert Q.gamma1_vec([0.0, 1.0, 0.445, 0.07], s) == [0, 100, 45, 7]
    top = Q.gamma1(6.0, Q.QuantSpec(-6.0, 6.0, 1e15))
    assert top > 1 << 90 and abs(float(top) - 1e30 / 12.0) <= 1e-12 * 1e30 / 12.0


def test_clamps_counted_and_errors():  # test_quantize.cpp:36-57
    s = Q.QuantSpec(-1.0, 1.0, 100.0)
    c = Q.ClampStats()
    assert Q.gamma2(-3.5, s, c) == 0 and Q.gamma2(2.0, s, c) == 100 and Q.gamma1(-9.0, s, c) == 0
    assert (c.low, c.high, c.total()) == (2, 1, 3)
    assert Q.gamma2(0.5, s, c) == 75 and c.total() == 3
    for bad in (float("nan"), float("inf")):
        with pytest.raises(ValueError):
            Q.gamma2(bad, s)
    for spec in ((1.0, 1.0, 10.0), (2.0, 1.0, 10.0), (0.0, 1.0, 0.5), (0.0, 1.0, 1e16)):
        with pytest.raises(ValueError):
            Q.gamma2(0.5, Q.QuantSpec(*spec))


def test_vector_forms_equal_the_restated_quantizers():
    rnd = random.Random(3)
    s = Q.QuantSpec(-6.0, 6.0, 1e15)
    vals = [rnd.uniform(-7.0, 7.0) for _ in range(2000)] + [-6.0, 6.0, 0.0]
    assert Q.gamma2_vec(vals, s) == [O.gamma2(v, -6.0, 6.0, 1e15) for v in vals]
    assert Q.gamma1_vec(vals, s) == [O.gamma1(v, -6.0, 6.0, 1e15) for v in vals]
    q2 = Q.gamma2_vec(vals[:50], s)
    assert [Q.degamma2(q, s) for q in q2] == [O.degamma2(q, -6.0, 6.0, 1e15) for q in q2]
    d = Q.QuantSpec(-2.0, 2.0, float(1 << 20))  # dyadic: exact round trips (test_quantize.cpp:83-94)
    ks = [rnd.randrange(0, (1 << 20) + 1) for _ in range(500)]
    vs = [d.z_min + k * (d.range() / d.delta) for k in ks]
    assert Q.gamma2_vec(vs, d) == ks and [Q.degamma2(k, d) for k in ks] == vs


def test_combined_update_and_inverse_equal_the_restatement():
    rnd = random.Random(5)
    s = Q.QuantSpec(-3.0, 3.0, 1e6)
    rows, cols = 7, 5
    qa = [rnd.getrandbits(100) for _ in range(rows)]
    qb = [[rnd.getrandbits(40) for _ in range(cols)] for _ in range(rows)]
    qz = [rnd.getrandbits(20) for _ in range(cols)]
    qn = [rnd.getrandbits(20) for _ in range(cols)]
    got = Q.combined_quantized_update(qa, qb, qz, qn)
    assert got == O.combined_quantized_update(qa, qb, qz, qn)
    rs = [sum(r) for r in qb]
    assert Q.inverse_quantize_x(got, rs, qz, qn, s) == O.inverse_quantize_x(got, rs, qz, qn, -3.0, 3.0, 1e6)
    with pytest.raises(ValueError):
        Q.combined_quantized_update(qa, qb, qz, qn[:-1])
    w = Q.widen_bounds(-1.0, 2.0, 1.5, 1e6)
    assert (w.z_min, w.z_max) == O.widen_bounds(-1.0, 2.0, 1.5, 1e6)
    with pytest.raises(ValueError):
        Q.widen_bounds(1.0, 0.0, 1.5, 1e6)
