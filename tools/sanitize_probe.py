"""compute-sanitizer target: one small call of every kernel family of libpcb200.so (RNS core
Enc/Dec incl. split stage 1, carry core, public-key n^2 path, homomorphic add / scalar / matvec /
aggregate, sample_r, quantizers, async ADMM entries, collaborative entries, wire codec)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2601_14980_b200 import _lib as L  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402
from paper_2601_14980_b200 import wire as WR  # noqa: E402

lib = L.lib()
n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 300
for bits in (1024, 2048):
    kp = P.keygen(P.Rng(bits), bits)
    ph, pub = P.Paillier(kp), P.Paillier(P.PublicKey(kp.n, bits))
    m = torch.from_numpy(L.ints_to_limbs([i * 7919 for i in range(n_el)], ph.L).view(np.int32)).cuda()
    r = ph.sample_r_batch(P.Rng(2), n_el)
    c = ph.encrypt_batch(m, r)
    assert torch.equal(ph.decrypt_batch(c), m)
    c2 = pub.encrypt_batch(m, r, use_crt=False)
    assert torch.equal(c, c2)
    a = pub.hom_add_batch(c, c2)
    k = torch.arange(n_el, dtype=torch.int64, device="cuda")
    s = pub.hom_scalar_mul_batch(k, c)
    agg = pub.aggregate_batch(c)
    E = np.random.default_rng(1).integers(0, 2**50, (16, 16), dtype=np.uint64)
    mv = pub.hom_matvec_batch(c[:16].cpu().numpy().view(np.uint32), E, c[16:32].cpu().numpy().view(np.uint32))
    f = WR.put_cipher_vec(c)
    back, _, _ = WR.get_cipher_vec(f, 2 * ph.L)
    assert torch.equal(back, c)
    if bits == 2048:
        share = P.crt_share(kp)
        g = torch.from_numpy(np.tile(L.int_to_limbs(kp.n + 1, 2 * share.S).view(np.int32), (n_el, 1))).cuda()
        ob = torch.from_numpy(L.ints_to_limbs([i * 3 + kp.n for i in range(n_el)], 2 * ph.L + 3).view(np.int32)).cuda()
        gp = share.delegated_power_tensor(g, ob)
        v = torch.linspace(-1, 1, n_el, dtype=torch.float64, device="cuda")
        cq, q, _ = ph.quantize_encrypt_batch(v, -2.0, 2.0, 1e15, r)
    torch.cuda.synchronize()
print("sanitize probe ok")
