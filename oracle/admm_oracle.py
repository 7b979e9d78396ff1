"""CPU restatement of the reference's ADMM layer — TEST INFRASTRUCTURE ONLY.

The reference's admm.cpp / protocol.cpp / experiments.cpp need Eigen3, which is absent here, so
they cannot be compiled.  This module restates them in numpy (FP64):

  gen_gaussian_problem  experiments.cpp:324-348  (splitmix64 Box-Muller A, partial shuffle support)
  split_columns         admm.cpp:77-83
  node_factor           admm.cpp:63-75          (B = rho (A^T A + rho I)^-1, alpha = (A^T A + rho I)^-1 A^T y)
  lasso_admm_split      admm.cpp:85-125
  lasso_objective       admm.cpp:31-34
  session_bounds        protocol.cpp:29-70       (+ widen_bounds, quantize.cpp:114-129)
  shadow_session        acceptance.cpp:214-281   (the crypto-free integer pipeline)

Parity status: node_factor / lasso_admm_split / session_bounds are FP-tolerance parity with the
reference (Eigen's LDLT rounding is pinned only to 1e-12..1e-18 by test_admm.cpp:94-130).
Downstream of identical node factors and QuantSpec, shadow_session is BIT-EXACT restatement of
the reference's integer pipeline (it uses pcadmm_oracle's gamma/combined/inverse, which are pinned
to the compiled reference by tests/golden/quantize.json) — that is the trajectory the encrypted
session must reproduce exactly (acceptance.cpp [5]).
"""
from __future__ import annotations

import math

import numpy as np

import pcadmm_oracle as O


def gen_gaussian_problem(m: int, n: int, sparsity: float, seed: int):  # experiments.cpp:324-348
    rng = O.Rng(seed)
    a = np.empty((m, n))
    for i in range(m):
        for j in range(n):
            a[i, j] = rng.gaussian()
    nnz = int(math.ceil(sparsity * n))
    idx = list(range(n))
    for i in range(nnz):
        k = i + rng.below(n - i)
        idx[i], idx[k] = idx[k], idx[i]
    x = np.zeros(n)
    for i in range(nnz):
        x[idx[i]] = rng.gaussian()
    return a, a @ x, x


def split_columns(cols: int, k: int):  # admm.cpp:77-83
    if cols < 1 or k < 1 or k > cols:
        raise ValueError("cannot split columns across nodes")
    sizes = [cols // k] * k
    for i in range(cols % k):
        sizes[i] += 1
    return sizes


def node_factor(a_k, y, rho: float, k_total: int, over_k: bool = False):  # admm.cpp:63-75
    n = a_k.shape[1]
    normal = a_k.T @ a_k + rho * np.eye(n)
    y_s = y / float(k_total) if over_k else y
    b_bar = rho * np.linalg.solve(normal, np.eye(n))
    alpha = np.linalg.solve(normal, a_k.T @ y_s)
    return b_bar, alpha


def lasso_objective(a, y, z, lam):  # admm.cpp:31-34
    r = a @ z - y
    return 0.5 * float(r @ r) + lam * float(np.abs(z).sum())


def lasso_admm_split(a, y, rho, lam, iters, sizes, factors=None):  # admm.cpp:85-125
    k_total = len(sizes)
    if factors is None:
        factors, at = [], 0
        for c in sizes:
            factors.append(node_factor(a[:, at:at + c], y, rho, k_total))
            at += c
    n = a.shape[1]
    x, z, v = np.zeros(n), np.zeros(n), np.zeros(n)
    xs, objs = [], []
    kappa = lam / rho
    for _ in range(iters):
        at = 0
        for (b_bar, alpha), c in zip(factors, sizes):
            sl = slice(at, at + c)
            x[sl] = alpha + b_bar @ (z[sl] - v[sl])
            xv = x[sl] + v[sl]
            z[sl] = np.sign(xv) * np.maximum(np.abs(xv) - kappa, 0.0)
            v[sl] = v[sl] + (x[sl] - z[sl])  # Eigen: vk += xk - zk
            at += c
        xs.append(x.copy())
        objs.append(lasso_objective(a, y, z, lam))
    return xs, z, v, objs


def session_bounds(a, y, rho, lam, iters, sizes, margin, delta, factors=None):  # protocol.cpp:29-70
    k_total = len(sizes)
    lo = hi = 0.0
    if factors is None:
        factors, at = [], 0
        for c in sizes:
            factors.append(node_factor(a[:, at:at + c], y, rho, k_total))
            at += c
    for b_bar, alpha in factors:
        lo = min(lo, float(alpha.min()), float(b_bar.min()))
        hi = max(hi, float(alpha.max()), float(b_bar.max()))
    n = a.shape[1]
    z, v = np.zeros(n), np.zeros(n)
    kappa = lam / rho
    for _ in range(iters):
        at = 0
        for (b_bar, alpha), c in zip(factors, sizes):
            sl = slice(at, at + c)
            xk = alpha + b_bar @ (z[sl] - v[sl])
            xv = xk + v[sl]
            zk = np.array([O.soft_threshold(t, kappa) for t in xv])
            v[sl] = v[sl] + (xk - zk)  # Eigen: vk += xk - zk
            z[sl] = zk
            lo = min(lo, float(zk.min()), float((-v[sl]).min()))
            hi = max(hi, float(zk.max()), float((-v[sl]).max()))
            at += c
    return (*O.widen_bounds(lo, hi, margin, delta), delta)


def shadow_session(factors, sizes, spec, rho, lam, iters):
    """acceptance.cpp:214-281: the integer pipeline without cryptography, given node factors."""
    zmin, zmax, delta = spec
    blks = []
    at = 0
    for (b_bar, alpha), c in zip(factors, sizes):
        q_alpha = [O.gamma1(float(x), zmin, zmax, delta) for x in alpha]
        q_b = [[O.gamma2(float(b_bar[i, j]), zmin, zmax, delta) for j in range(c)] for i in range(c)]
        blks.append((at, c, q_alpha, q_b, [sum(r) for r in q_b]))
        at += c
    n = at
    x, z, v = [0.0] * n, [0.0] * n, [0.0] * n
    kappa = lam / rho
    trace = []
    for _ in range(iters):
        for off, c, q_alpha, q_b, rowsum in blks:
            q_z = [O.gamma2(z[off + i], zmin, zmax, delta) for i in range(c)]
            q_nv = [O.gamma2(-v[off + i], zmin, zmax, delta) for i in range(c)]
            q = O.combined_quantized_update(q_alpha, q_b, q_z, q_nv)
            xk = O.inverse_quantize_x(q, rowsum, q_z, q_nv, zmin, zmax, delta)
            for i in range(c):
                g = off + i
                x[g] = xk[i]
                xv = xk[i] + v[g]
                zz = O.soft_threshold(xv, kappa)
                z[g] = zz
                v[g] = xv - zz
        trace.append(list(x))
    return trace, z, v


def shadow_session_ref(factors, sizes, spec, rho, lam, iters, capture_q: bool = False):
    """shadow_session with the per-element integer work done by the COMPILED reference
    (oracle/_ref/libpcref.so through refbind: gamma1/gamma2 quantize.cpp:31-41,
    combined_quantized_update quantize.cpp:66-82, inverse_quantize_x quantize.cpp:84-112), so the
    headline shapes (N_k = 512, 1024) finish in seconds.  The float glue (soft threshold and the
    v update, protocol.cpp:504-511, admm.cpp:18-22) is elementwise IEEE arithmetic in numpy, the
    same operations in the same order as the scalar restatement above.  capture_q: also return, per
    iteration, the quantized (q_z, q_nv) of every block in block order (what the master encrypts)."""
    import refbind as RB

    zmin, zmax, delta = spec
    blks, at = [], 0
    for (b_bar, alpha), c in zip(factors, sizes):
        qa, _, rc = RB.gamma1(np.asarray(alpha, np.float64), zmin, zmax, delta)
        assert rc == 0
        qb, _, rc = RB.gamma2(np.asarray(b_bar, np.float64).reshape(-1), zmin, zmax, delta)
        assert rc == 0
        qb = qb.reshape(c, c)
        rowsum = qb.sum(axis=1, dtype=np.uint64)  # < c * 2^50: exact in u64
        blks.append((at, c, np.ascontiguousarray(qa), np.ascontiguousarray(qb), np.ascontiguousarray(rowsum)))
        at += c
    n = at
    x, z, v = np.zeros(n), np.zeros(n), np.zeros(n)
    kappa = lam / rho
    trace, qtrace = [], []
    lib = RB.lib()
    for _ in range(iters):
        qs = []
        for off, c, qa, qb, rowsum in blks:
            sl = slice(off, off + c)
            q_z, _, _ = RB.gamma2(z[sl].copy(), zmin, zmax, delta)
            q_nv, _, _ = RB.gamma2(-v[sl], zmin, zmax, delta)
            qs.append((q_z, q_nv))
            q = np.zeros(2 * c, np.uint64)
            lib.pcref_combined_update(RB.a(qa), RB.a(qb), RB.a(q_z), RB.a(q_nv), c, c, RB.a(q))
            xk = np.zeros(c)
            lib.pcref_inverse_quantize_x(RB.a(q), RB.a(rowsum), RB.a(q_z), RB.a(q_nv), c, c, zmin, zmax, delta,
                                         RB.a(xk))
            x[sl] = xk
            xv = xk + v[sl]
            zz = np.where(xv > kappa, xv - kappa, np.where(xv < -kappa, xv + kappa, 0.0))
            z[sl] = zz
            v[sl] = xv - zz
        trace.append(x.copy())
        qtrace.append(qs)
    if capture_q:
        return trace, z, v, qtrace
    return trace, z, v
