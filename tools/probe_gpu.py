"""Development probe: IMAD roofline, modexp core, CRT Enc/Dec correctness + throughput.

Run on a B200 via gpurun:  python tools/probe_gpu.py [--n 16384]
Prints one JSON object per measurement.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import random
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2601_14980_b200 import _lib as L  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


def dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--skip-imad", action="store_true")
    a = ap.parse_args()
    lib = L.lib()
    torch.cuda.init()
    emit(gpu=torch.cuda.get_device_name(0))
    if not a.skip_imad:
        for kind, name in ((0, "imad_wide"), (1, "imad_lohi")):
            ms = C.c_float(0)
            r = lib.pcb_imad_peak(kind, 2000, C.byref(ms))
            emit(probe=name, mac32_per_s=r, ms=ms.value)

    rnd = random.Random(1)
    # ---- modexp core ------------------------------------------------------------------------
    for bits in (1024, 2048):
        limbs = bits // 32
        m = rnd.getrandbits(bits) | (1 << (bits - 1)) | 1
        e = rnd.getrandbits(bits) | (1 << (bits - 1))
        n = a.n
        xs = [rnd.getrandbits(bits) for _ in range(n)]
        X = dev(L.ints_to_limbs(xs, limbs))
        Y = torch.zeros_like(X)
        M = L.int_to_limbs(m, limbs)
        E = L.int_to_limbs(e, limbs)
        # warm
        rc = lib.pcb_modexp_batch(L.ptr(M), limbs, L.ptr(E), limbs, L.ptr(X), 256, L.ptr(Y), None)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = lib.pcb_modexp_batch(L.ptr(M), limbs, L.ptr(E), limbs, L.ptr(X), n, L.ptr(Y), None)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ys = L.limbs_to_ints(Y.cpu().numpy())
        bad = sum(1 for i in range(0, n, max(1, n // 64)) if ys[i] != pow(xs[i], e, m))
        S = limbs
        mm = 2 * S * S + S
        exp_macs = (bits + (bits + 3) // 4) * mm
        emit(probe="modexp", bits=bits, n=n, rc=rc, seconds=dt, per_s=n / dt, bad_of_64=bad,
             canonical_mac32_per_s=n * exp_macs / dt)

    # ---- CRT Enc/Dec at 2048 -----------------------------------------------------------------
    for bits in (1024, 2048):
        st = C.c_uint64(1)
        nl = bits // 32
        nn = np.zeros(nl, np.uint32)
        pp = np.zeros(nl // 2, np.uint32)
        qq = np.zeros(nl // 2, np.uint32)
        L.check(lib.pcb_keygen(C.byref(st), bits, nn.ctypes.data_as(L._u32p), pp.ctypes.data_as(L._u32p),
                               qq.ctypes.data_as(L._u32p)))
        N = L.limbs_to_int(nn)
        ctx = C.c_void_p()
        L.check(lib.pcb_ctx_create(C.byref(ctx), 0, nn.ctypes.data_as(L._u32p), nl, pp.ctypes.data_as(L._u32p),
                                   qq.ctypes.data_as(L._u32p), nl // 2))
        n = a.n
        ms = [rnd.getrandbits(50) for _ in range(n)]
        rs = [rnd.randrange(1, N) for _ in range(n)]
        Md = dev(L.ints_to_limbs(ms, 2))
        Rd = dev(L.ints_to_limbs(rs, nl))
        Cd = torch.zeros((n, 2 * nl), dtype=torch.int32, device="cuda")
        Sd = torch.zeros(n, dtype=torch.int32, device="cuda")
        L.check(lib.pcb_encrypt(ctx, L.ptr(Md), 2, L.ptr(Rd), 64, L.ptr(Cd), 1, L.ptr(Sd), None))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc = lib.pcb_encrypt(ctx, L.ptr(Md), 2, L.ptr(Rd), n, L.ptr(Cd), 1, L.ptr(Sd), None)
        torch.cuda.synchronize()
        te = time.perf_counter() - t0
        cs = L.limbs_to_ints(Cd.cpu().numpy().view(np.uint32))
        n2 = N * N
        badc = 0
        for i in range(0, n, max(1, n // 32)):
            want = (1 + ms[i] * N) * pow(rs[i], N, n2) % n2
            badc += cs[i] != want
        Md2 = torch.zeros((n, nl), dtype=torch.int32, device="cuda")
        L.check(lib.pcb_decrypt(ctx, L.ptr(Cd), 64, L.ptr(Md2), 1, L.ptr(Sd), None))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rc2 = lib.pcb_decrypt(ctx, L.ptr(Cd), n, L.ptr(Md2), 1, L.ptr(Sd), None)
        torch.cuda.synchronize()
        td = time.perf_counter() - t0
        back = L.limbs_to_ints(Md2.cpu().numpy().view(np.uint32))
        badm = sum(1 for i in range(n) if back[i] != ms[i])
        stat = Sd.cpu().numpy()
        emit(probe="crt_encdec", bits=bits, n=n, rc=[rc, rc2], enc_per_s=n / te, dec_per_s=n / td,
             bad_c_of_32=badc, bad_m=badm, status_nonzero=int((stat != 0).sum()))
        lib.pcb_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
