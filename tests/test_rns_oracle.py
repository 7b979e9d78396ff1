"""CPU: the RNS Montgomery restatement (oracle/rns_oracle.py) that the streaming RNS core
(rnsx.cu) implements -- both the two-REDC GEMM-1 epilogue and the fused one (W1' = M_i C3_j,
r' = REDC(t' C2 + V')) -- gives exact modular exponentiation against Python integers, and every
intermediate stays in its lazy range (asserted inside RnsCtx.mm)."""
import random

import pytest

import rns_oracle as R


@pytest.mark.parametrize("bits,k", [(2048, 72), (1024, 40)])
def test_rns_pow_fused_and_unfused_exact(bits, k):
    rnd = random.Random(bits)
    N = rnd.getrandbits(bits) | (1 << (bits - 1)) | 1
    ctx = R.RnsCtx(N, k)
    for _ in range(2):
        b, e = rnd.randrange(N), rnd.getrandbits(40)
        want = pow(b, e, N)
        ctx.fused = True
        assert ctx.pow(b, e) == want
        ctx.fused = False
        assert ctx.pow(b, e) == want
