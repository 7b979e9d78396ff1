"""Python mirror of the reference's quantizer API (/root/reference/proj/include/pcadmm/quantize.hpp:
13-71) over the C ABI: every vector form runs on the GPU (pcb_quantize, pcb_combined_update,
pcb_inverse_quantize_x); the scalar forms are one-element batches.  Same names, argument meaning
and errors (invalid_argument -> ValueError) as quantize.cpp:8-129.  Plaintext integers are Python
ints (u64 for Gamma2, u128 for Gamma1 and the combined update)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .paillier import _raise_for


@dataclass
class QuantSpec:
    """QuantSpec (quantize.hpp:13-21): the window [z_min, z_max] and the resolution delta."""

    z_min: float
    z_max: float
    delta: float

    def range(self) -> float:
        return self.z_max - self.z_min

    def step(self) -> float:
        return (self.z_max - self.z_min) / self.delta


@dataclass
class ClampStats:
    """ClampStats (quantize.hpp:23-27): values clamped below z_min / above z_max."""

    low: int = 0
    high: int = 0

    def total(self) -> int:
        return self.low + self.high


def check_spec(s: QuantSpec) -> None:
    """quantize.cpp:8-15."""
    if not (math.isfinite(s.z_min) and math.isfinite(s.z_max)) or s.z_max <= s.z_min:
        raise ValueError("quantization window is empty or non-finite")
    if not (s.delta >= 1.0) or s.delta > 9.0e15:
        raise ValueError("delta outside [1, 9e15]")


def _quantize(values, s: QuantSpec, fine: bool, clamps: ClampStats | None) -> list[int]:
    check_spec(s)
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(-1))
    if v.size == 0:
        return []
    q = np.zeros((v.size, 2) if fine else v.size, np.uint64)
    cl = (C.c_uint64 * 2)()
    _raise_for(L.lib().pcb_quantize(v.ctypes.data, v.size, s.z_min, s.z_max, s.delta, 1 if fine else 0,
                                    q.ctypes.data, cl, None), "quantize")
    if clamps is not None:
        clamps.low += cl[0]
        clamps.high += cl[1]
    if fine:
        return [int(lo) | (int(hi) << 64) for lo, hi in q]
    return [int(x) for x in q]


def gamma2_vec(values, s: QuantSpec, clamps: ClampStats | None = None) -> list[int]:
    """gamma2_vec (quantize.cpp:52-57): round(delta (clamp(v) - z_min) / range), ties away from zero."""
    return _quantize(values, s, False, clamps)


def gamma1_vec(values, s: QuantSpec, clamps: ClampStats | None = None) -> list[int]:
    """gamma1_vec (quantize.cpp:59-64): the fine quantizer, delta^2 resolution (u128)."""
    return _quantize(values, s, True, clamps)


def gamma2(v: float, s: QuantSpec, clamps: ClampStats | None = None) -> int:
    return gamma2_vec([v], s, clamps)[0]


def gamma1(v: float, s: QuantSpec, clamps: ClampStats | None = None) -> int:
    return gamma1_vec([v], s, clamps)[0]


def degamma2(q: int, s: QuantSpec) -> float:
    """degamma2 (quantize.cpp:43-45)."""
    return s.z_min + float(q) * ((s.z_max - s.z_min) / s.delta)


def degamma1(q: int, s: QuantSpec) -> float:
    """degamma1 (quantize.cpp:47-50)."""
    step = (s.z_max - s.z_min) / s.delta
    return s.z_min + float(q) * (step * step)


def combined_quantized_update(q_alpha, q_b, q_z, q_negv) -> list[int]:
    """combined_quantized_update (quantize.cpp:66-82): q_i = q_alpha_i + sum_j q_b_ij (q_z_j + q_negv_j)
    in u128, on the device.  q_alpha: u128 ints, q_b: rows x cols u64, q_z / q_negv: u64."""
    rows, cols = len(q_alpha), len(q_z)
    if len(q_negv) != cols or any(len(r) != cols for r in q_b) or len(q_b) != rows:
        raise ValueError("shape mismatch")
    if rows == 0:
        return []
    qa = np.array([[x & (2**64 - 1), x >> 64] for x in q_alpha], np.uint64)
    qb = np.ascontiguousarray(np.asarray(q_b, np.uint64).reshape(rows, cols))
    qz, qn = np.asarray(q_z, np.uint64), np.asarray(q_negv, np.uint64)
    out = np.zeros((rows, 2), np.uint64)
    _raise_for(L.lib().pcb_combined_update(qa.ctypes.data, qb.ctypes.data, qz.ctypes.data, qn.ctypes.data, rows,
                                           cols, out.ctypes.data, None), "combined_quantized_update")
    return [int(lo) | (int(hi) << 64) for lo, hi in out]


def inverse_quantize_x(q, q_b_rowsum, q_z, q_negv, s: QuantSpec) -> list[float]:
    """inverse_quantize_x (quantize.cpp:84-112) on the device, the reference's FP64 operation order."""
    check_spec(s)
    rows, cols = len(q), len(q_z)
    if len(q_b_rowsum) != rows or len(q_negv) != cols:
        raise ValueError("shape mismatch")
    if rows == 0:
        return []
    qq = np.array([[x & (2**64 - 1), x >> 64] for x in q], np.uint64)
    rs, qz, qn = (np.asarray(a, np.uint64) for a in (q_b_rowsum, q_z, q_negv))
    x = np.zeros(rows, np.float64)
    _raise_for(L.lib().pcb_inverse_quantize_x(qq.ctypes.data, rs.ctypes.data, qz.ctypes.data, qn.ctypes.data, rows,
                                              cols, s.z_min, s.z_max, s.delta, x.ctypes.data, None),
               "inverse_quantize_x")
    return x.tolist()


def widen_bounds(lo: float, hi: float, margin: float, delta: float) -> QuantSpec:
    """widen_bounds (quantize.cpp:114-129): pad [lo, hi] by (margin - 1) / 2 of its width each side."""
    if not (math.isfinite(lo) and math.isfinite(hi)) or hi < lo:
        raise ValueError("bad value extremes")
    if margin < 1.0:
        raise ValueError("margin below 1")
    if hi - lo < 1e-12:
        lo -= 0.5
        hi += 0.5
    pad = (margin - 1.0) * (hi - lo) / 2.0
    s = QuantSpec(lo - pad, hi + pad, delta)
    check_spec(s)
    return s
