"""ADMM-level restatement (oracle/admm_oracle.py) sanity, and the integer shadow pipeline vs the
plaintext split recurrence (the reference's session ~ plaintext check, test_protocol.cpp:125-155).
CPU only."""
import numpy as np

import admm_oracle as A
import pcadmm_oracle as O


def test_split_columns():
    assert A.split_columns(900, 3) == [300, 300, 300]
    assert A.split_columns(10, 3) == [4, 3, 3]


def test_generator_support_and_shape():
    a, y, x = A.gen_gaussian_problem(12, 30, 0.1, 1)
    assert a.shape == (12, 30) and y.shape == (12,)
    assert int((x != 0).sum()) == 3
    assert np.allclose(a @ x, y)


def test_single_block_split_equals_centralized():
    # test_admm.cpp:94-110: one block == centralized ADMM (x = (A^T A + rho I)^-1 (A^T y + rho (z - v)))
    a, y, _ = A.gen_gaussian_problem(20, 15, 0.2, 3)
    xs, z, v, _ = A.lasso_admm_split(a, y, 1.0, 1.0, 30, [15])
    n = 15
    inv = np.linalg.inv(a.T @ a + np.eye(n))
    xc, zc, vc = np.zeros(n), np.zeros(n), np.zeros(n)
    for _ in range(30):
        xc = inv @ (a.T @ y + (zc - vc))
        xv = xc + vc
        zc = np.sign(xv) * np.maximum(np.abs(xv) - 1.0, 0.0)
        vc = vc + (xc - zc)
    assert np.mean((xs[-1] - xc) ** 2) < 1e-18


def test_shadow_pipeline_tracks_plaintext():
    a, y, _ = A.gen_gaussian_problem(16, 24, 0.2, 2)
    sizes = A.split_columns(24, 3)
    factors, at = [], 0
    for c in sizes:
        factors.append(A.node_factor(a[:, at:at + c], y, 1.0, 3))
        at += c
    spec = A.session_bounds(a, y, 1.0, 1.0, 10, sizes, 1.5, 1e15, factors)
    trace, z, v = A.shadow_session(factors, sizes, spec, 1.0, 1.0, 10)
    xs, zp, vp, _ = A.lasso_admm_split(a, y, 1.0, 1.0, 10, sizes, factors)
    for t in range(10):
        assert np.mean((np.array(trace[t]) - xs[t]) ** 2) < 1e-20  # quantization loss ~ 1/Delta^2
