"""Development probe: cfg3 encrypted ADMM session (N=4096, K=8, 2048-bit), `iters` iterations.
Run under ncu (--metrics gpu__time_duration.sum) for the per-kernel breakdown of an iteration."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2601_14980_b200 import admm as ADMM  # noqa: E402
from paper_2601_14980_b200 import paillier as P  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
a, y = bench.gen_problem_fast(512, 4096, 0.1, 1)
keys = P.keygen(P.Rng(bench.KEY_SEED), 2048)
sess = ADMM.EncryptedSession(keys, ADMM.SessionConfig(nodes=8, iters=iters))
t0 = time.perf_counter()
res = sess.run(a, y, record_trace=False)
print("iter_seconds", res.iter_seconds, "wall", time.perf_counter() - t0)
