"""Wire-format interop: the restated codec (oracle/wire_oracle.py) replays the
reference's own test_transport.cpp layout checks (CPU), and the device packer / parser
(csrc/wire.cu: pcb_wire_put_cipher_vec, pcb_wire_get_cipher_vec, pcb_encode_envelope) produces the
same bytes for real ciphertexts and parses them back (GPU)."""
import ctypes as C
import random

import numpy as np
import pytest

import wire_oracle as WO
from paper_2601_14980_b200 import _lib as L


def test_oracle_codec_replays_reference_layout_checks():
    out = bytearray()  # test_transport.cpp:68-83
    WO.put_u16(out, 0x1234)
    WO.put_u32(out, 0xDEADBEEF)
    WO.put_u64(out, 0x0102030405060708)
    assert out[0] == 0x12 and out[1] == 0x34 and out[2] == 0xDE and out[6] == 0x01
    a, off = WO.get_u16(out, 0)
    b, off = WO.get_u32(out, off)
    c, off = WO.get_u64(out, off)
    assert (a, b, c, off) == (0x1234, 0xDEADBEEF, 0x0102030405060708, len(out))
    with pytest.raises(WO.WireError):
        WO.get_u16(out, off)
    # big integer and ciphertext codecs (test_transport.cpp:141-159)
    xs = [0, 1, 123456789012345678901234567890]
    cs = [(99, 7), (981273498761234, 51)]
    out = bytearray()
    WO.put_u32(out, len(xs))
    for x in xs:
        WO.wire_put(out, x)
    WO.put_cipher_vec(out, cs)
    n, off = WO.get_u32(out, 0)
    bx = []
    for _ in range(n):
        v, off = WO.wire_get(out, off)
        bx.append(v)
    bc, off = WO.get_cipher_vec(out, off)
    assert bx == xs and bc == cs and off == len(out)
    assert out[4:8] == b"\0\0\0\0"  # the empty BigNat is a zero-length field
    # envelope (test_transport.cpp:34-66)
    f = WO.encode_envelope(3, 9, 17, b"abc")
    assert f[:4] == (10).to_bytes(4, "big") and WO.decode_envelope(f) == (3, 9, 17, b"abc")
    with pytest.raises(WO.WireError):
        WO.decode_envelope(f[:-1])
    with pytest.raises(WO.WireError):
        WO.decode_envelope(f[:4] + b"\x08" + f[5:])


@pytest.mark.gpu
def test_device_cipher_vec_and_envelope_match_the_codec():
    import torch

    rnd = random.Random(5)
    W = 128  # 2048-bit keys: 4096-bit ciphertexts
    vals = [0, 1, 255, 256, (1 << 32) - 1, 1 << 32, (1 << 4095) | 12345] + [rnd.getrandbits(rnd.choice([8, 700, 4096]))
                                                                           for _ in range(993)]
    bits = [rnd.getrandbits(12) for _ in vals]
    want = bytearray()
    WO.put_cipher_vec(want, list(zip(vals, bits)))
    lib = L.lib()
    for dev in (False, True):
        c = L.ints_to_limbs(vals, W)
        pb = np.array(bits, np.uint32)
        if dev:
            c, pb = torch.from_numpy(c.view(np.int32)).cuda(), torch.from_numpy(pb.view(np.int32)).cuda()
        n = C.c_size_t()
        assert lib.pcb_wire_put_cipher_vec(L.ptr(c), W, L.ptr(pb), len(vals), None, 0, C.byref(n), None) == 0
        assert n.value == len(want)
        out = np.zeros(n.value, np.uint8)
        if dev:
            out = torch.zeros(n.value, dtype=torch.uint8, device="cuda")
        assert lib.pcb_wire_put_cipher_vec(L.ptr(c), W, L.ptr(pb), len(vals), L.ptr(out), n.value, C.byref(n),
                                           None) == 0
        got = bytes(out.cpu().numpy() if dev else out)
        assert got == bytes(want)
        # parse back (host frame / device frame)
        off = C.c_size_t(0)
        cnt = C.c_size_t()
        back = np.zeros((len(vals), W), np.uint32)
        bb = np.zeros(len(vals), np.uint32)
        src = out if dev else np.frombuffer(got, np.uint8).copy()
        assert lib.pcb_wire_get_cipher_vec(L.ptr(src), len(got), C.byref(off), W, len(vals), C.byref(cnt),
                                           L.ptr(back), L.ptr(bb), None) == 0
        assert cnt.value == len(vals) and off.value == len(got)
        assert L.limbs_to_ints(back) == vals and bb.tolist() == bits
        # truncated frame -> PCB_E_SHAPE (runtime_error)
        off = C.c_size_t(0)
        assert lib.pcb_wire_get_cipher_vec(L.ptr(src), len(got) - 1, C.byref(off), W, len(vals), C.byref(cnt),
                                           L.ptr(back), L.ptr(bb), None) == L.PCB_E_SHAPE
    # an enc_state frame (protocol.cpp:471-476): envelope around put_cipher_vec(zc) ++ put_cipher_vec(vc)
    payload = np.frombuffer(bytes(want) + bytes(want), np.uint8).copy()
    n = C.c_size_t()
    frame = np.zeros(len(payload) + 11, np.uint8)
    assert lib.pcb_encode_envelope(3, 1, 42, L.ptr(payload), len(payload), L.ptr(frame), len(frame), C.byref(n),
                                   None) == 0
    assert bytes(frame) == WO.encode_envelope(3, 1, 42, bytes(payload))


@pytest.mark.gpu
def test_session_frames_round_trip():
    """enc_state frame of real ciphertexts from the device, decoded by the restated reference
    decoder; an enc_update frame built by the codec parsed back on the device."""
    import torch

    from paper_2601_14980_b200 import paillier as P
    from paper_2601_14980_b200 import wire as WR

    kp = P.keygen(P.Rng(3), 1024)
    ph = P.Paillier(kp)
    r = ph.sample_r_batch(P.Rng(4), 40)
    m = torch.from_numpy(L.ints_to_limbs(list(range(40)), ph.L).view(np.int32)).cuda()
    c = ph.encrypt_batch(m, r)
    f = WR.enc_state_frame(c[:20], c[20:], session=1, iteration=5)
    t, sid, it, payload = WO.decode_envelope(bytes(f.cpu().numpy()))
    assert (t, sid, it) == (3, 1, 5)
    zc, off = WO.get_cipher_vec(payload, 0)
    vc, off = WO.get_cipher_vec(payload, off)
    ints = L.limbs_to_ints(c.cpu().numpy().view(np.uint32))
    assert [v for v, _ in zc] == ints[:20] and [v for v, _ in vc] == ints[20:] and off == len(payload)
    body = bytearray()
    WO.put_cipher_vec(body, [(v, 9) for v in ints])
    sid, it, back, bits = WR.parse_enc_update(WO.encode_envelope(4, 2, 6, bytes(body)), 2 * ph.L)
    assert (sid, it) == (2, 6) and L.limbs_to_ints(back.cpu().numpy().view(np.uint32)) == ints
    assert bits.tolist() == [9] * 40
