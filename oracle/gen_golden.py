"""Generate tests/golden/*.json from the COMPILED REFERENCE (oracle/_ref/libpcref.so).

    make -C oracle && python oracle/gen_golden.py

Test infrastructure only.  Every vector below is produced by the reference's own code
(pcadmm::keygen, Paillier::sample_r / crt_encrypt_with_r / encrypt_with_r / decrypt /
crt_decrypt / hom_add / hom_scalar_mul / hom_matvec, gamma1 / gamma2 /
combined_quantized_update / inverse_quantize_x), so the fixtures pin both the GPU path and the
Python restatement (oracle/pcadmm_oracle.py) to the reference without needing /root/reference at
test time.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import refbind as R  # noqa: E402

OUT = HERE.parent / "tests" / "golden"

# key seeds: test_paillier.cpp:261 (64-bit, Rng(42)), :324 (1024-bit, Rng(20260825)),
# experiments.cpp:61-64 (seed ^ 0x6b657967656e2e2e, seed 1) for 2048 bits
KEYS = [(42, 64), (20260825, 1024), (1 ^ 0x6B657967656E2E2E, 2048)]


def hx(v: int) -> str:
    return format(int(v), "x")


def keyrec(k: R.RefKey, seed: int, bits: int) -> dict:
    return dict(seed=seed, bits=bits, n=hx(k.n), p=hx(k.p), q=hx(k.q), eps=hx(k.get(3)), mu=hx(k.get(4)),
                rng_state_after=k.rng_state_after, record=k.serialize().hex())


def main() -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    rnd = np.random.default_rng(12345)
    keys, sample, enc, dec = [], [], [], []
    for seed, bits in KEYS:
        k = R.RefKey.keygen(seed, bits)
        keys.append(keyrec(k, seed, bits))
        n, L = k.n, k.L
        # sample_r stream on Rng(2) (BASELINE.md cfg2 r stream)
        r, st = k.sample_r(2, 16)
        rs = R.ints(r)
        sample.append(dict(bits=bits, seed=2, count=16, r=[hx(v) for v in rs], state_after=st))
        # plaintexts: edge cases + Gamma-sized + full-width
        ms = [0, 1, n - 1, (1 << 50) - 1, 10**15]
        ms += [int(rnd.integers(0, 2**62)) for _ in range(5)]
        ms += [int.from_bytes(rnd.bytes(4 * L), "little") % n for _ in range(4)]
        rr = rs[: len(ms) - 2] + [1, n - 1]
        M, RR = R.limbs(ms, L), R.limbs(rr, L)
        c_crt, st_crt = k.encrypt(M, RR, crt=True)
        c_dir, st_dir = k.encrypt(M, RR, crt=False)
        assert (c_crt == c_dir).all() and (st_crt == 0).all() and (st_dir == 0).all()
        # error cases: m = n, r = 0, r = n (paillier.cpp:242, 322-323)
        bad_m = [n, 5, 5]
        bad_r = [rs[0], 0, n]
        cb, stb = k.encrypt(R.limbs(bad_m, L), R.limbs(bad_r, L), crt=True)
        enc.append(dict(bits=bits, m=[hx(v) for v in ms], r=[hx(v) for v in rr], c=[hx(v) for v in R.ints(c_crt)],
                        bad_m=[hx(v) for v in bad_m], bad_r=[hx(v) for v in bad_r], bad_status=stb.tolist()))
        # decryption incl. error cases: 0, n, k*p (non-units), n^2 (range)
        cs = R.ints(c_crt)
        n2 = n * n
        extra = [0, n, 3 * k.p, n2, n2 + 5]
        C = R.limbs(cs + extra, 2 * L)
        m_crt, sd_crt = k.decrypt(C, crt=True)
        m_dir, sd_dir = k.decrypt(C, crt=False)
        assert (m_crt == m_dir).all() and (sd_crt == sd_dir).all()
        dec.append(dict(bits=bits, c=[hx(v) for v in cs + extra], m=[hx(v) for v in R.ints(m_crt)],
                        status=sd_crt.tolist()))
    (OUT / "keys.json").write_text(json.dumps(keys, indent=1))
    (OUT / "sample_r.json").write_text(json.dumps(sample, indent=1))
    (OUT / "encrypt.json").write_text(json.dumps(enc, indent=1))
    (OUT / "decrypt.json").write_text(json.dumps(dec, indent=1))

    # toy key p=5, q=7 (test_paillier.cpp:23-61): every plaintext with the listed units
    toy = R.RefKey.from_primes(5, 7)
    units = [1, 2, 4, 11, 23, 34]
    ms = [m for m in range(35) for _ in units]
    rs = [r for _ in range(35) for r in units]
    ct, stt = toy.encrypt(R.limbs(ms, 1), R.limbs(rs, 1), crt=True)
    assert (stt == 0).all()
    (OUT / "toy.json").write_text(json.dumps(dict(p=5, q=7, m=ms, r=rs, c=[int(v) for v in R.ints(ct)])))

    # quantizers (quantize.cpp:31-41) on U[-6, 6] from Rng(1).unit() + edges
    sys.path.insert(0, str(HERE))
    import pcadmm_oracle as O
    rng = O.Rng(1)
    vals = [-6.0 + 12.0 * rng.unit() for _ in range(64)]
    vals += [-6.0, 6.0, 0.0, -7.5, 9.25, -6.0 + 12.0 * 0.5, 1e-300, -1e-300]
    z0, z1, delta = -6.0, 6.0, 1e15
    g2, cl2, _ = R.gamma2(vals, z0, z1, delta)
    g1, cl1, _ = R.gamma1(vals, z0, z1, delta)
    quant = dict(zmin=z0, zmax=z1, delta=delta, v=[v.hex() for v in vals], g2=[int(x) for x in g2],
                 g1=[int(lo) | (int(hi) << 64) for lo, hi in g1], clamps2=cl2.tolist(), clamps1=cl1.tolist())
    # combined update + inverse on a small random block (quantize.cpp:66-112)
    rows = cols = 6
    qa = [int(rnd.integers(0, 2**62)) << 30 for _ in range(rows)]
    qb = [[int(rnd.integers(0, 10**15)) for _ in range(cols)] for _ in range(rows)]
    qz = [int(rnd.integers(0, 10**15)) for _ in range(cols)]
    qn = [int(rnd.integers(0, 10**15)) for _ in range(cols)]
    QA = np.array([[v & (2**64 - 1), v >> 64] for v in qa], np.uint64)
    QB = np.array(qb, np.uint64)
    QZ, QN = np.array(qz, np.uint64), np.array(qn, np.uint64)
    out = np.zeros(2 * rows, np.uint64)
    R.lib().pcref_combined_update(R.a(QA), R.a(QB), R.a(QZ), R.a(QN), rows, cols, R.a(out))
    comb = [int(out[2 * i]) | (int(out[2 * i + 1]) << 64) for i in range(rows)]
    rowsum = np.array([sum(r) for r in qb], np.uint64)
    xs = np.zeros(rows, np.float64)
    R.lib().pcref_inverse_quantize_x(R.a(out), R.a(rowsum), R.a(QZ), R.a(QN), rows, cols, -1.5, 2.25, 1e15, R.a(xs))
    quant.update(comb_alpha=[str(v) for v in qa], comb_b=qb, comb_z=qz, comb_nv=qn, comb_out=[str(v) for v in comb],
                 inv_zmin=-1.5, inv_zmax=2.25, inv_delta=1e15, inv_x=[float(x).hex() for x in xs])
    (OUT / "quantize.json").write_text(json.dumps(quant, indent=1))
    print("wrote", sorted(p.name for p in OUT.glob("*.json")))


if __name__ == "__main__":
    main()
