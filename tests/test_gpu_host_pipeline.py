"""Large batches with HOST buffers run chunked, the copies of one chunk beside the compute of the
next (abi.cu, kPipeMin / HostPipe).  The bytes must equal the one-piece device-buffer path, and the
statuses / first-failure result must be those of the whole batch."""
import ctypes as C

import numpy as np
import pytest

from conftest import golden
from paper_2601_14980_b200 import _lib as L
from paper_2601_14980_b200 import paillier as P

pytestmark = pytest.mark.gpu

N = 4 * 148 * 256 + 3001  # above kPipeMin, ragged last chunk


@pytest.fixture(scope="module")
def setup():
    import torch

    k = golden("keys.json")[2]
    kp = P.KeyPair(int(k["n"], 16), int(k["p"], 16), int(k["q"], 16), k["bits"])
    ph = P.Paillier(kp)
    g = np.random.default_rng(3)
    vals = g.uniform(-7.0, 7.0, N)  # some clamps at [-6, 6]
    r = ph.sample_r_batch(P.Rng(77), N)
    torch.cuda.synchronize()
    return kp, ph, vals, r


def test_quantize_encrypt_host_output_equals_device(setup):
    import torch

    kp, ph, vals, r = setup
    lib = L.lib()
    W = 2 * ph.L
    # device output, one piece
    vd = torch.from_numpy(vals).cuda()
    cd = torch.empty((N, W), dtype=torch.int32, device="cuda")
    cl_d = (C.c_uint64 * 2)()
    assert lib.pcb_quantize_encrypt(ph._ctx, L.ptr(vd), N, -6.0, 6.0, 1e15, 0, L.ptr(r), 1, L.ptr(cd), None, cl_d,
                                    None) == 0
    # host input and output (pinned and pageable), chunked
    for pin in (True, False):
        hv = torch.from_numpy(vals.copy())
        hc = torch.zeros((N, W), dtype=torch.int32)
        hq = torch.zeros(N, dtype=torch.int64)
        if pin:
            hv, hc, hq = hv.pin_memory(), hc.pin_memory(), hq.pin_memory()
        cl_h = (C.c_uint64 * 2)()
        assert lib.pcb_quantize_encrypt(ph._ctx, L.ptr(hv), N, -6.0, 6.0, 1e15, 0, L.ptr(r), 1, L.ptr(hc), L.ptr(hq),
                                        cl_h, None) == 0
        assert torch.equal(hc, cd.cpu()), pin
        assert (cl_h[0], cl_h[1]) == (cl_d[0], cl_d[1]) and cl_h[0] > 0 and cl_h[1] > 0
        # Gamma2 values match the plaintexts the device path decrypts to
        if pin:
            m = ph.decrypt_batch(cd)
            assert torch.equal(m[:, 0].cpu().view(torch.int32), hq.view(torch.int32)[0::2])


def test_decrypt_host_buffers_equal_device_and_report_first_failure(setup):
    import torch

    kp, ph, vals, r = setup
    lib = L.lib()
    W = 2 * ph.L
    m0 = torch.zeros((N, ph.L), dtype=torch.int32, device="cuda")
    m0[:, 0] = torch.arange(N, dtype=torch.int32, device="cuda")
    c = ph.encrypt_batch(m0, r)
    md = ph.decrypt_batch(c)
    assert torch.equal(md, m0)
    for pin in (True, False):
        hc = c.cpu()
        hm = torch.zeros((N, ph.L), dtype=torch.int32)
        if pin:
            hc, hm = hc.pin_memory(), hm.pin_memory()
        st = torch.zeros(N, dtype=torch.int32)
        assert lib.pcb_decrypt(ph._ctx, L.ptr(hc), N, L.ptr(hm), 1, L.ptr(st), None) == 0
        assert torch.equal(hm, md.cpu()) and int(st.abs().sum()) == 0
    # a ciphertext >= n^2 in the third chunk, another in the fourth: statuses per element, and the
    # status-less call returns the earliest failure's code (PCB_E_CIPHER_RANGE)
    n2 = L.int_to_limbs(kp.n * kp.n, W).view(np.int32)
    hc = c.cpu()
    bad = [2 * (N // 4) + 17, N - 5]
    for i in bad:
        hc[i] = torch.from_numpy(n2.copy())
    hm = torch.zeros((N, ph.L), dtype=torch.int32)
    st = torch.zeros(N, dtype=torch.int32)
    assert lib.pcb_decrypt(ph._ctx, L.ptr(hc), N, L.ptr(hm), 1, L.ptr(st), None) == 0
    assert sorted(np.nonzero(st.numpy())[0].tolist()) == bad
    rc = lib.pcb_decrypt(ph._ctx, L.ptr(hc), N, L.ptr(hm), 1, None, None)
    assert rc == int(st[bad[0]]) and rc != 0
    ok = np.ones(N, bool)
    ok[bad] = False
    assert torch.equal(hm[torch.from_numpy(ok)], md.cpu()[torch.from_numpy(ok)])


def test_encrypt_host_buffers_equal_device_and_report_first_failure(setup):
    """pcb_encrypt with host m / r / c (chunked) == the device path; a plaintext >= n in the second
    chunk and an r = 0 in the fourth are reported per element, the status-less call returns the
    earlier one's code."""
    import torch

    kp, ph, vals, r = setup
    lib = L.lib()
    W = 2 * ph.L
    g = np.random.default_rng(8)
    m = torch.zeros((N, ph.L), dtype=torch.int32)
    m[:, 0] = torch.from_numpy(g.integers(0, 2**31, N).astype(np.int32))
    m[:, 1] = torch.from_numpy(g.integers(0, 2**20, N).astype(np.int32))
    cd = torch.empty((N, W), dtype=torch.int32, device="cuda")
    assert lib.pcb_encrypt(ph._ctx, L.ptr(m.cuda()), ph.L, L.ptr(r), N, L.ptr(cd), 1, None, None) == 0
    rh = r.cpu()
    for pin in (True, False):
        mh, rr, hc = m.clone(), rh.clone(), torch.zeros((N, W), dtype=torch.int32)
        if pin:
            mh, rr, hc = mh.pin_memory(), rr.pin_memory(), hc.pin_memory()
        st = torch.zeros(N, dtype=torch.int32)
        assert lib.pcb_encrypt(ph._ctx, L.ptr(mh), ph.L, L.ptr(rr), N, L.ptr(hc), 1, L.ptr(st), None) == 0
        assert torch.equal(hc, cd.cpu()) and int(st.abs().sum()) == 0, pin
    bad_m, bad_r = N // 4 + 11, 3 * (N // 4) + 101
    mh, rr, hc = m.clone(), rh.clone(), torch.zeros((N, W), dtype=torch.int32)
    mh[bad_m] = torch.from_numpy(L.int_to_limbs(kp.n, ph.L).view(np.int32).copy())
    rr[bad_r] = 0
    st = torch.zeros(N, dtype=torch.int32)
    assert lib.pcb_encrypt(ph._ctx, L.ptr(mh), ph.L, L.ptr(rr), N, L.ptr(hc), 1, L.ptr(st), None) == 0
    assert sorted(np.nonzero(st.numpy())[0].tolist()) == [bad_m, bad_r]
    rc = lib.pcb_encrypt(ph._ctx, L.ptr(mh), ph.L, L.ptr(rr), N, L.ptr(hc), 1, None, None)
    assert rc == int(st[bad_m]) and rc != 0 and int(st[bad_r]) != 0
