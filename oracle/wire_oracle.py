"""The reference's wire codecs restated in Python -- TEST INFRASTRUCTURE ONLY (never imported by
the product).  /root/reference/proj/src/wire.cpp cannot be compiled here (wire.hpp includes
admm.hpp -> Eigen, absent), so this restatement is the checker for the device packer
(paper_2601_14980_b200/csrc/wire.cu).  It is pinned by the layout checks of the reference's own
tests/test_transport.cpp:68-159 (big-endian fields, empty BigNat = zero length, round trips), which
tests/test_wire_oracle.py replays.

  put_u16 / put_u32 / put_u64   wire.cpp:40-55   big-endian
  wire_put / wire_get           bignat.cpp:414-429  u32 BE byte count + minimal BE magnitude
  put_cipher_vec / get_...      wire.cpp:125-146  u32 BE count; per element wire_put(value), u32 BE plain_bits
  encode_envelope / decode_...  wire.cpp:148-173  u32 BE body length (7 + payload), type, u16 BE session,
                                                  u32 BE iteration, payload; kFrameCap = 256 MiB
"""
from __future__ import annotations

FRAME_CAP = 256 << 20


class WireError(RuntimeError):
    """std::runtime_error of the decoders (truncation, bad length, unknown type)."""


def put_u16(out: bytearray, v: int) -> None:
    out += (v & 0xFFFF).to_bytes(2, "big")


def put_u32(out: bytearray, v: int) -> None:
    out += (v & 0xFFFFFFFF).to_bytes(4, "big")


def put_u64(out: bytearray, v: int) -> None:
    out += (v & (2**64 - 1)).to_bytes(8, "big")


def _need(d: bytes, off: int, n: int) -> None:
    if off + n > len(d):
        raise WireError("truncated frame")


def get_u16(d: bytes, off: int) -> tuple[int, int]:
    _need(d, off, 2)
    return int.from_bytes(d[off:off + 2], "big"), off + 2


def get_u32(d: bytes, off: int) -> tuple[int, int]:
    _need(d, off, 4)
    return int.from_bytes(d[off:off + 4], "big"), off + 4


def get_u64(d: bytes, off: int) -> tuple[int, int]:
    _need(d, off, 8)
    return int.from_bytes(d[off:off + 8], "big"), off + 8


def wire_put(out: bytearray, v: int) -> None:  # bignat.cpp:414-418
    mag = v.to_bytes((v.bit_length() + 7) // 8, "big") if v else b""
    put_u32(out, len(mag))
    out += mag


def wire_get(d: bytes, off: int) -> tuple[int, int]:  # bignat.cpp:420-429
    if off + 4 > len(d):
        raise WireError("truncated integer field")
    n = int.from_bytes(d[off:off + 4], "big")
    off += 4
    if n > len(d) - off:
        raise WireError("truncated integer field")
    return int.from_bytes(d[off:off + n], "big"), off + n


def put_cipher_vec(out: bytearray, cs) -> None:  # wire.cpp:125-132; cs: (value, plain_bits) pairs
    put_u32(out, len(cs))
    for value, bits in cs:
        wire_put(out, value)
        put_u32(out, bits)


def get_cipher_vec(d: bytes, off: int):  # wire.cpp:134-146
    n, off = get_u32(d, off)
    cs = []
    for _ in range(n):
        v, off = wire_get(d, off)
        b, off = get_u32(d, off)
        cs.append((v, b))
    return cs, off


def encode_envelope(msg_type: int, session: int, iteration: int, payload: bytes) -> bytes:  # wire.cpp:148-159
    body = 1 + 2 + 4 + len(payload)
    if body > FRAME_CAP:
        raise OverflowError("frame past the size cap")
    out = bytearray()
    put_u32(out, body)
    out.append(msg_type & 0xFF)
    put_u16(out, session)
    put_u32(out, iteration)
    out += payload
    return bytes(out)


def decode_envelope(frame: bytes):  # wire.cpp:161-173
    body, off = get_u32(frame, 0)
    if body > FRAME_CAP:
        raise WireError("frame past the size cap")
    if body < 7 or len(frame) - 4 != body:
        raise WireError("frame length field mismatch")
    t = frame[off]
    off += 1
    if t < 1 or t > 7:
        raise WireError("unknown message type")
    session, off = get_u16(frame, off)
    iteration, off = get_u32(frame, off)
    return t, session, iteration, bytes(frame[off:])
