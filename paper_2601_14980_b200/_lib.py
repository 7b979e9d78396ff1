"""ctypes binding of the C ABI (include/pcb200.h) exported by libpcb200.so.

The library is the product: there is no Python or CPU fallback.  Loading fails loudly if the
shared object is missing; compute calls return PCB_E_CUDA without a GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["PCB_LIB"]) if os.environ.get("PCB_LIB") else _PKG / "libpcb200.so"

STATUS = {
    0: "PCB_OK",
    1: "PCB_E_PLAINTEXT_RANGE",
    2: "PCB_E_RANDOMNESS_RANGE",
    3: "PCB_E_CIPHER_RANGE",
    4: "PCB_E_NOT_UNIT",
    5: "PCB_E_OVERFLOW",
    6: "PCB_E_NO_PRIVATE",
    7: "PCB_E_SHAPE",
    8: "PCB_E_UNSUPPORTED",
    9: "PCB_E_CUDA",
    10: "PCB_E_ALLOC",
    11: "PCB_E_RANGE_UPDATE",
}
PCB_OK = 0
PCB_E_PLAINTEXT_RANGE = 1
PCB_E_RANDOMNESS_RANGE = 2
PCB_E_CIPHER_RANGE = 3
PCB_E_NOT_UNIT = 4
PCB_E_OVERFLOW = 5
PCB_E_NO_PRIVATE = 6
PCB_E_SHAPE = 7
PCB_E_UNSUPPORTED = 8
PCB_E_CUDA = 9
PCB_E_ALLOC = 10
PCB_E_RANGE_UPDATE = 11

_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p

# name -> (restype, argtypes); the authoritative list of exported symbols (tests check it
# against include/pcb200.h).
SIGNATURES = {
    "pcb_keygen": (C.c_int, [_u64p, C.c_uint32, _u32p, _u32p, _u32p]),
    "pcb_random_prime": (C.c_int, [_u64p, C.c_uint32, _u32p]),
    "pcb_keygen_speculative": (C.c_int, [_u64p, C.c_uint32, C.c_int, _u32p, _u32p, _u32p]),
    "pcb_random_prime_speculative": (C.c_int, [_u64p, C.c_uint32, C.c_int, _u32p]),
    "pcb_ctx_create": (C.c_int, [C.POINTER(_vp), C.c_int, _u32p, C.c_uint32, _u32p, _u32p, C.c_uint32]),
    "pcb_ctx_destroy": (None, [_vp]),
    "pcb_ctx_set_generator": (C.c_int, [_vp, _vp, C.c_uint32]),
    "pcb_ctx_n_limbs": (C.c_uint32, [_vp]),
    "pcb_ctx_n_bits": (C.c_uint32, [_vp]),
    "pcb_ctx_has_private": (C.c_int, [_vp]),
    "pcb_ctx_engine": (C.c_int, [_vp]),
    "pcb_ctx_set_priority": (C.c_int, [_vp, C.c_int]),
    "pcb_ctx_get_n": (C.c_int, [_vp, _u32p, _u32p]),
    "pcb_ctx_counters": (None, [_vp, _u64p, _u64p]),
    "pcb_ctx_reset_counters": (None, [_vp]),
    "pcb_sample_r": (C.c_int, [_vp, _u64p, C.c_size_t, _vp, _vp]),
    "pcb_encrypt": (C.c_int, [_vp, _vp, C.c_uint32, _vp, C.c_size_t, _vp, C.c_int, _vp, _vp]),
    "pcb_encrypt_rn": (C.c_int, [_vp, _vp, C.c_uint32, _vp, C.c_size_t, _vp, _vp, _vp]),
    "pcb_decrypt": (C.c_int, [_vp, _vp, C.c_size_t, _vp, C.c_int, _vp, _vp]),
    "pcb_decrypt_with_half": (C.c_int, [_vp, _vp, _vp, C.c_uint32, C.c_size_t, _vp, _vp, _vp]),
    "pcb_share_create": (C.c_int, [C.POINTER(_vp), C.c_int, _vp, C.c_uint32, _vp, C.c_uint32]),
    "pcb_share_destroy": (None, [_vp]),
    "pcb_delegated_power": (C.c_int, [_vp, _vp, C.c_uint32, _vp, C.c_uint32, C.c_size_t, _vp, _vp]),
    "pcb_delegated_power_binomial": (C.c_int, [_vp, _vp, C.c_uint32, _vp, C.c_uint32, C.c_size_t, _vp, _vp]),
    "pcb_node_factors": (C.c_int, [_vp, C.c_size_t, C.c_size_t, C.c_size_t, _vp, C.c_size_t, _vp, C.c_double,
                                   C.c_uint32, C.c_int, _vp, _vp, _vp]),
    "pcb_finish_split_encrypt": (C.c_int, [_vp, _vp, C.c_uint32, _vp, C.c_uint32, _vp, C.c_size_t, _vp, _vp, _vp]),
    "pcb_finish_split_encrypt_rn": (C.c_int, [_vp, _vp, C.c_uint32, _vp, C.c_uint32, _vp, C.c_size_t, _vp, _vp, _vp]),
    "pcb_hom_add": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _vp, _vp]),
    "pcb_hom_scalar_mul": (C.c_int, [_vp, _vp, _vp, C.c_size_t, _vp, _vp]),
    "pcb_hom_matvec": (C.c_int, [_vp, _vp, _vp, _vp, C.c_size_t, C.c_size_t, C.c_uint32, _vp, _vp]),
    "pcb_edge_step": (C.c_int, [_vp, _vp, _vp, _vp, _vp, C.c_size_t, C.c_uint32, _vp, _vp]),
    "pcb_edge_step_blocks": (C.c_int, [_vp, C.c_size_t, _vp, _vp, _vp, _vp, _vp, C.c_uint32, _vp, _vp]),
    "pcb_aggregate": (C.c_int, [_vp, _vp, C.c_size_t, _vp, _vp]),
    "pcb_quantize_encrypt": (C.c_int, [_vp, _vp, C.c_size_t, C.c_double, C.c_double, C.c_double, C.c_int, _vp,
                                       C.c_int, _vp, _vp, _u64p, _vp]),
    "pcb_quantize": (C.c_int, [_vp, C.c_size_t, C.c_double, C.c_double, C.c_double, C.c_int, _vp, _u64p, _vp]),
    "pcb_decrypt_update": (C.c_int, [_vp, _vp, C.c_size_t, _vp, _vp, _vp, C.c_double, C.c_double, C.c_double,
                                     C.c_double, _vp, _vp, _vp, _vp, _vp]),
    "pcb_decrypt_update_blocks": (C.c_int, [_vp, C.c_size_t, _vp, _vp, _vp, _vp, _vp, C.c_double, C.c_double,
                                            C.c_double, C.c_double, _vp, _vp, _vp, _vp, _vp]),
    "pcb_decrypt_update_blocks_half": (C.c_int, [_vp, C.c_size_t, _vp, _vp, _vp, _vp, _vp, _vp, C.c_double,
                                                 C.c_double, C.c_double, C.c_double, _vp, _vp, _vp, _vp, _vp]),
    "pcb_wire_put_cipher_vec": (C.c_int, [_vp, C.c_uint32, _vp, C.c_size_t, _vp, C.c_size_t,
                                          C.POINTER(C.c_size_t), _vp]),
    "pcb_wire_get_cipher_vec": (C.c_int, [_vp, C.c_size_t, C.POINTER(C.c_size_t), C.c_uint32, C.c_size_t,
                                          C.POINTER(C.c_size_t), _vp, _vp, _vp]),
    "pcb_encode_envelope": (C.c_int, [C.c_uint8, C.c_uint16, C.c_uint32, _vp, C.c_size_t, _vp, C.c_size_t,
                                      C.POINTER(C.c_size_t), _vp]),
    "pcb_obfuscate_exponent": (C.c_int, [_vp, C.c_uint32, _vp, _vp, C.c_uint32, C.c_size_t, _vp, C.c_uint32, _vp]),
    "pcb_combined_update": (C.c_int, [_vp, _vp, _vp, _vp, C.c_size_t, C.c_size_t, _vp, _vp]),
    "pcb_inverse_quantize_x": (C.c_int, [_vp, _vp, _vp, _vp, C.c_size_t, C.c_size_t, C.c_double, C.c_double,
                                         C.c_double, _vp, _vp]),
    "pcb_quantize_async": (C.c_int, [_vp, C.c_size_t, C.c_double, C.c_double, C.c_double, C.c_int, _vp, _vp, _vp,
                                     _vp]),
    "pcb_edge_step_blocks_async": (C.c_int, [_vp, C.c_size_t, _vp, _vp, _vp, C.c_uint32, _vp, _vp, C.c_uint32, _vp,
                                             _vp, _vp]),
    "pcb_decrypt_update_blocks_async": (C.c_int, [_vp, C.c_size_t, _vp, _vp, _vp, _vp, _vp, C.c_double, C.c_double,
                                                  C.c_double, C.c_double, _vp, _vp, _vp, _vp, _vp]),
    "pcb_delegated_power_fermat": (C.c_int, [_vp, _vp, C.c_uint32, _vp, C.c_size_t, _vp, _vp]),
    "pcb_decrypt_half_q": (C.c_int, [_vp, _vp, C.c_size_t, _vp, _vp]),
    "pcb_decrypt_update_blocks_half_async": (C.c_int, [_vp, C.c_size_t, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                                       C.c_double, C.c_double, C.c_double, C.c_double, _vp, _vp,
                                                       _vp, _vp, _vp]),
    "pcb_modexp_batch": (C.c_int, [_vp, C.c_uint32, _vp, C.c_uint32, _vp, C.c_size_t, _vp, _vp]),
    "pcb_imad_peak": (C.c_double, [C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "pcb_launch_count": (C.c_uint64, []),
    "pcb_profile_begin": (None, []),
    "pcb_profile_end": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.POINTER(C.c_double)]),
    "pcb_profile_int8_macs": (C.c_double, []),
    "pcb_status_str": (C.c_char_p, [C.c_int]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libpcb200.so (building it first if this is a source checkout without one)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if os.environ.get("PCB_NO_AUTOBUILD"):
            raise RuntimeError(f"{LIB_PATH} missing (run python -m paper_2601_14980_b200.build)")
        from . import build as _build

        _build.build()
    L = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        f = getattr(L, name)  # AttributeError == missing export: fail loudly
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class PcbError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"{STATUS.get(code, code)}{': ' + what if what else ''}")


def check(code: int, what: str = "") -> None:
    if code != PCB_OK:
        raise PcbError(code, what)


# ---- limb helpers ------------------------------------------------------------------------
def int_to_limbs(v: int, n: int) -> np.ndarray:
    if v < 0 or v.bit_length() > 32 * n:
        raise ValueError("value does not fit the limb width")
    return np.frombuffer(v.to_bytes(4 * n, "little"), dtype=np.uint32).copy()


def limbs_to_int(a: np.ndarray) -> int:
    return int.from_bytes(np.ascontiguousarray(a, dtype=np.uint32).tobytes(), "little")


def ints_to_limbs(vals, n: int) -> np.ndarray:
    out = np.zeros((len(vals), n), dtype=np.uint32)
    for i, v in enumerate(vals):
        out[i] = int_to_limbs(int(v), n)
    return out


def limbs_to_ints(a: np.ndarray) -> list[int]:
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return [int.from_bytes(row.tobytes(), "little") for row in a]


def ptr(a) -> C.c_void_p | None:
    """Raw pointer of a numpy array (host) or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return C.c_void_p(a.ctypes.data)
    # torch tensor
    assert a.is_contiguous()
    return C.c_void_p(a.data_ptr())
