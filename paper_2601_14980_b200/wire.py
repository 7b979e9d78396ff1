"""Reference wire frames for GPU ciphertexts (wire.cpp:125-173, protocol.cpp:471-476, 273-275), built
and parsed on the device by csrc/wire.cu: a B200 master or edge can exchange enc_state / enc_update
frames with a reference SimCarrier / TcpCarrier peer byte for byte."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .paillier import _raise_for

ENC_STATE, ENC_UPDATE = 3, 4  # MsgType (wire.hpp:16-24)


def _torch():
    import torch

    return torch


def put_cipher_vec(c, plain_bits=None, stream=None):
    """put_cipher_vec of a (count, W) int32 limb tensor -> uint8 device tensor."""
    torch = _torch()
    n = C.c_size_t()
    W = c.shape[1]
    _raise_for(L.lib().pcb_wire_put_cipher_vec(L.ptr(c), W, L.ptr(plain_bits), c.shape[0], None, 0, C.byref(n),
                                               stream), "put_cipher_vec")
    out = torch.empty(n.value, dtype=torch.uint8, device=c.device)
    _raise_for(L.lib().pcb_wire_put_cipher_vec(L.ptr(c), W, L.ptr(plain_bits), c.shape[0], L.ptr(out), n.value,
                                               C.byref(n), stream), "put_cipher_vec")
    return out


def envelope(msg_type: int, session: int, iteration: int, payload, stream=None):
    """encode_envelope around a uint8 payload tensor -> uint8 tensor (same device)."""
    torch = _torch()
    n = C.c_size_t()
    out = torch.empty(payload.numel() + 11, dtype=torch.uint8, device=payload.device)
    _raise_for(L.lib().pcb_encode_envelope(msg_type, session, iteration, L.ptr(payload), payload.numel(), L.ptr(out),
                                           out.numel(), C.byref(n), stream), "encode_envelope")
    return out


def enc_state_frame(zc, vc, session: int, iteration: int, z_bits=None, v_bits=None):
    """The master's enc_state frame of one block (protocol.cpp:471-476)."""
    torch = _torch()
    return envelope(ENC_STATE, session, iteration, torch.cat([put_cipher_vec(zc, z_bits), put_cipher_vec(vc, v_bits)]))


def get_cipher_vec(buf, W: int, off: int = 0, max_count: int = 1 << 24):
    """get_cipher_vec from a uint8 tensor / array at byte off -> ((count, W) int32 tensor, plain_bits, new off)."""
    torch = _torch()
    o = C.c_size_t(off)
    cnt = C.c_size_t()
    # the count comes first: parse once for it, then into right-sized buffers
    hdr = bytes(buf[off:off + 4].cpu().numpy() if hasattr(buf, "cpu") else buf[off:off + 4])
    count = int.from_bytes(hdr, "big")
    dev = buf.device if hasattr(buf, "device") else "cpu"
    c = torch.empty((count, W), dtype=torch.int32, device=dev)
    bits = torch.empty(count, dtype=torch.int32, device=dev)
    n = buf.numel() if hasattr(buf, "numel") else len(buf)
    _raise_for(L.lib().pcb_wire_get_cipher_vec(L.ptr(buf), n, C.byref(o), W, max_count, C.byref(cnt), L.ptr(c),
                                               L.ptr(bits), None), "get_cipher_vec")
    return c, bits, o.value


def parse_enc_update(frame, W: int):
    """decode_envelope + get_cipher_vec of an edge's enc_update frame (protocol.cpp:273-275, 478-482)."""
    f = bytes(frame.cpu().numpy()) if hasattr(frame, "cpu") else bytes(frame)
    body = int.from_bytes(f[:4], "big")
    if body < 7 or len(f) - 4 != body or f[4] != ENC_UPDATE:
        raise ValueError("not an enc_update frame")
    session, iteration = int.from_bytes(f[5:7], "big"), int.from_bytes(f[7:11], "big")
    c, bits, _ = get_cipher_vec(np.frombuffer(f, np.uint8).copy(), W, 11)
    return session, iteration, c, bits
