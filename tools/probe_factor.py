"""Times the device node factors (pcb_node_factors) on cfg5's shape -- 64 blocks of 1024 columns
over 10000 rows -- against the torch.linalg library path (cuBLAS Gram + cuSOLVER solve), and
prints the per-launch breakdown from the CUDA-event profile of the tile kernel launches."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2601_14980_b200 import admm as ADMM  # noqa: E402


def torch_path(a, y, sizes):
    out, o = [], 0
    for c in sizes:
        ak = a[:, o:o + c]
        normal = ak.T @ ak + torch.eye(c, dtype=torch.float64, device=a.device)
        b = torch.linalg.solve(normal, torch.eye(c, dtype=torch.float64, device=a.device))
        al = torch.linalg.solve(normal, ak.T @ y)
        out.append((b, al))
        o += c
    return out


def timed(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts), r


def main():
    nblk = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    rows, c = 10000, 1024
    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(rows, nblk * c, dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn(rows, dtype=torch.float64, device="cuda", generator=g)
    sizes = [c] * nblk
    ADMM.node_factors(a[:, :2 * c], y, [c, c], 1.0, nblk)  # warm-up (module load, pools)
    t_dev, f_dev = timed(lambda: ADMM.node_factors(a, y, sizes, 1.0, nblk))
    t_lib, f_lib = timed(lambda: torch_path(a, y, sizes), reps=2)
    err_b = max(float((b1 - b2).abs().max() / b2.abs().max()) for (b1, _), (b2, _) in zip(f_dev, f_lib))
    err_a = max(float((a1 - a2).abs().max() / a2.abs().max()) for (_, a1), (_, a2) in zip(f_dev, f_lib))
    gram = nblk * rows * c * (c + 64) * 1.0  # lower tiles only: FMAs (x2 for FLOPs)
    chol = nblk * c ** 3 / 3 * 3  # potrf + trtri + lauum FMAs (~n^3/3 each)
    print(json.dumps({"blocks": nblk, "rows": rows, "cols_per_block": c, "device_s": t_dev, "torch_linalg_s": t_lib,
                      "speedup": t_lib / t_dev, "gram_fp64_tflops": 2 * gram / t_dev / 1e12,
                      "all_fp64_tflops": 2 * (gram + chol) / t_dev / 1e12,
                      "max_rel_diff_b": err_b, "max_rel_diff_alpha": err_a}))


if __name__ == "__main__":
    main()
