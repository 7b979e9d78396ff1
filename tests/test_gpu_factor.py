"""Node factors on the device (admm.cpp:63-75) against the restated
node_factor (oracle/admm_oracle.py: LAPACK solves of the same normal matrix).  FP64 with a
different factorisation and summation order than the reference's Eigen LDLT, so the bar is a
tolerance: max-abs error <= 1e-11 x max |entry| (the normal matrices here have condition
numbers below 1e4; the session is then bit-pinned on whatever factors it is handed).
Shapes cover ragged blocks (1, 63, 64, 65, 130 columns ...), more columns than rows, both
YScaling modes and rho != 1; errors follow check_inputs (admm.cpp:8-16)."""
import numpy as np
import pytest

import admm_oracle as AO
from paper_2601_14980_b200 import admm as ADMM

pytestmark = pytest.mark.gpu
TOL = 1e-11


def _check(a, y, sizes, rho, k_total, over_k):
    import torch

    at = torch.as_tensor(a, device="cuda")
    yt = torch.as_tensor(y, device="cuda")
    got = ADMM.node_factors(at, yt, sizes, rho, k_total, over_k)
    o = 0
    for (b, al), c in zip(got, sizes):
        b_ref, al_ref = AO.node_factor(a[:, o:o + c], y, rho, k_total, over_k)
        b, al = b.cpu().numpy(), al.cpu().numpy()
        assert np.array_equal(b, b.T), "B_k must come back exactly symmetric"
        assert np.abs(b - b_ref).max() <= TOL * np.abs(b_ref).max(), (c, np.abs(b - b_ref).max())
        assert np.abs(al - al_ref).max() <= TOL * max(np.abs(al_ref).max(), 1e-300), (c, np.abs(al - al_ref).max())
        o += c


@pytest.mark.parametrize("rows,sizes,rho,over_k", [
    (300, [1, 5, 63, 64, 65, 130, 200], 1.0, False),
    (300, [1, 5, 63, 64, 65, 130, 200], 0.37, True),
    (50, [96, 33], 2.5, False),      # more columns than rows: rho I carries the rank
    (1000, [256, 256, 256, 256], 1.0, False),
])
def test_node_factors_match_the_restated_solve(rows, sizes, rho, over_k):
    rng = np.random.default_rng(rows + len(sizes))
    a = rng.standard_normal((rows, sum(sizes)))
    y = rng.standard_normal(rows)
    _check(a, y, sizes, rho, len(sizes), over_k)


def test_cfg5_block_shape():
    """1024-column blocks over 10000 rows (cfg5's block shape), four of them."""
    rng = np.random.default_rng(5)
    a = rng.standard_normal((10000, 4096))
    y = rng.standard_normal(10000)
    _check(a, y, [1024] * 4, 1.0, 64, False)


def test_strided_rows_and_single_block_api():
    import torch

    rng = np.random.default_rng(9)
    big = rng.standard_normal((120, 90))
    a = big[:, 10:80]  # a column window of a wider matrix: row stride 90
    y = rng.standard_normal(120)
    got = ADMM.node_factors(torch.as_tensor(big, device="cuda")[:, 10:80], torch.as_tensor(y, device="cuda"), [30, 40],
                            1.0, 2)
    b1, al1 = ADMM.node_factor(torch.as_tensor(np.ascontiguousarray(a[:, 30:]), device="cuda"),
                               torch.as_tensor(y, device="cuda"), 1.0, 2)
    b_ref, al_ref = AO.node_factor(a[:, 30:], y, 1.0, 2)
    for b, al in [(got[1][0], got[1][1]), (b1, al1)]:
        assert np.abs(b.cpu().numpy() - b_ref).max() <= TOL * np.abs(b_ref).max()
        assert np.abs(al.cpu().numpy() - al_ref).max() <= TOL * np.abs(al_ref).max()


def test_argument_errors():
    import torch

    a = torch.randn(20, 10, dtype=torch.float64, device="cuda")
    y = torch.randn(20, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        ADMM.node_factors(a, y, [5, 5], 0.0, 2)  # rho must be positive
    with pytest.raises(ValueError):
        ADMM.node_factors(a, y, [5, 4], 1.0, 2)  # split does not cover the columns
    with pytest.raises(ValueError):
        ADMM.node_factors(a, y, [5, 5], 1.0, 0)  # node count below 1
    a[3, 2] = float("nan")
    with pytest.raises(ValueError):
        ADMM.node_factors(a, y, [5, 5], 1.0, 2)  # not positive definite


def test_node_factor_closed_form_for_orthonormal_columns():
    """test_admm.cpp:112-130: A^T A = I gives B = rho / (1 + rho) I and alpha = A^T y / (1 + rho);
    YScaling::over_k divides y by K first."""
    import torch

    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((60, 40)))
    y = rng.standard_normal(60)
    rho = 0.5
    for over_k, k in ((False, 4), (True, 4)):
        got = ADMM.node_factors(torch.as_tensor(q, device="cuda"), torch.as_tensor(y, device="cuda"), [40], rho, k,
                                over_k)
        b, al = got[0][0].cpu().numpy(), got[0][1].cpu().numpy()
        ys = y / k if over_k else y
        assert np.abs(b - rho / (1 + rho) * np.eye(40)).max() < 1e-13
        assert np.abs(al - q.T @ ys / (1 + rho)).max() < 1e-13
