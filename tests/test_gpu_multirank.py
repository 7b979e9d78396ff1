"""Multi-rank encrypted sessions on ONE GPU (gpurun has one device): ranks are processes sharing
cuda:0 with the gloo backend (gloo moves CUDA tensors through host memory), which exercises the
sharded EncryptedSession -- including a rank that owns no block (world > nodes) -- and
the faithful-trust FaithfulDriver with the CUDA backend, against the single-rank trajectory."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ITERS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    import admm_oracle as AO

    a, y, _ = AO.gen_gaussian_problem(32, 48, 0.1, 5)
    sizes = AO.split_columns(48, 2)
    fac, at = [], 0
    for c in sizes:
        fac.append(AO.node_factor(a[:, at:at + c], y, 1.0, 2))
        at += c
    spec = AO.session_bounds(a, y, 1.0, 1.0, ITERS, sizes, 1.5, 1e15, fac)
    return a, y, fac, spec


def _worker(rank, world, port, mode, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle")]
    import torch
    import torch.distributed as dist

    from paper_2601_14980_b200 import admm as ADMM
    from paper_2601_14980_b200 import paillier as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    a, y, fac, spec = _problem()
    keys = P.keygen(P.Rng(9), 1024)
    cfg = ADMM.SessionConfig(nodes=2, iters=ITERS)
    if mode == "sharded":
        res = ADMM.EncryptedSession(keys, cfg, device=0, rank=rank, world=world, group=dist.group.WORLD).run(
            a, y, factors=fac, spec=spec)
        out = [t.tolist() for t in res.x_trace]
    elif mode == "sharded_pooled":
        cfg = ADMM.SessionConfig(nodes=2, iters=ITERS, r_mode="pooled", pool_size=3)
        sess = ADMM.EncryptedSession(keys, cfg, device=0, rank=rank, world=world, group=dist.group.WORLD)
        sess.capture = {"iters": ITERS}
        res = sess.run(a, y, factors=fac, spec=spec)
        cts = [c.cpu().numpy().tolist() for c in sess.capture.get("ct", [])]
        out = ([t.tolist() for t in res.x_trace], cts, sess.mine)
    else:
        dev = torch.device("cuda:0")
        drv = ADMM.FaithfulDriver(ADMM.FaithfulGpuBackend(keys, rank, 0), cfg, rank=rank, world=world,
                                  group=dist.group.WORLD)
        res = drv.run(torch.as_tensor(a, device=dev), torch.as_tensor(y, device=dev),
                      [(torch.as_tensor(b, device=dev), torch.as_tensor(al, device=dev)) for b, al in fac], spec)
        out = [t.tolist() for t in res.x_trace]
    q.put((rank, out))
    dist.destroy_process_group()


def _run(world, mode):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=600) for _ in range(world))
    for p in ps:
        p.join(timeout=120)
    return out


def test_sharded_session_with_an_empty_rank_matches_single_rank():
    from paper_2601_14980_b200 import admm as ADMM
    from paper_2601_14980_b200 import paillier as P

    a, y, fac, spec = _problem()
    single = ADMM.EncryptedSession(P.keygen(P.Rng(9), 1024), ADMM.SessionConfig(nodes=2, iters=ITERS)).run(
        a, y, factors=fac, spec=spec)
    want = [t.tolist() for t in single.x_trace]
    out = _run(3, "sharded")  # 3 ranks, 2 blocks: rank 2 owns nothing
    for rank, tr in out:
        assert tr == want, rank


def test_faithful_driver_two_ranks_cuda_backend():
    from paper_2601_14980_b200 import admm as ADMM
    from paper_2601_14980_b200 import paillier as P

    a, y, fac, spec = _problem()
    single = ADMM.EncryptedSession(P.keygen(P.Rng(9), 1024), ADMM.SessionConfig(nodes=2, iters=ITERS)).run(
        a, y, factors=fac, spec=spec)
    want = [t.tolist() for t in single.x_trace]
    out = _run(2, "faithful")
    assert out[0][1] == want and out[1][1] == []


def test_sharded_pooled_session_slices_the_pool_like_one_rank():
    """Pooled randomness over 3 ranks (one owns nothing): every rank indexes the shared pool at the
    reference's stream positions, so its enc_state rows equal the single-rank session's."""
    from paper_2601_14980_b200 import admm as ADMM
    from paper_2601_14980_b200 import paillier as P

    a, y, fac, spec = _problem()
    sess = ADMM.EncryptedSession(P.keygen(P.Rng(9), 1024),
                                 ADMM.SessionConfig(nodes=2, iters=ITERS, r_mode="pooled", pool_size=3))
    sess.capture = {"iters": ITERS}
    single = sess.run(a, y, factors=fac, spec=spec)
    want = [t.tolist() for t in single.x_trace]
    sizes, n = sess.sizes, sum(sess.sizes)
    offs = [0, sizes[0]]
    out = _run(3, "sharded_pooled")
    for rank, (tr, cts, mine) in out:
        assert tr == want, rank
        if not mine:
            assert cts == []
            continue
        for t in range(ITERS):
            full = sess.capture["ct"][t].cpu().numpy()
            rows = [full[offs[k]:offs[k] + sizes[k]] for k in mine] + \
                   [full[n + offs[k]:n + offs[k] + sizes[k]] for k in mine]
            assert np.array_equal(np.array(cts[t]), np.concatenate(rows)), (rank, t)
