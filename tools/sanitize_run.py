"""Small invocations of every kernel family for compute-sanitizer (one tool per run):
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
fp32 tcgen05 + PDL path (b = 32; swizzled TMA Gram, TMEM-A update, and the round-1 variants), FFMA fallback,
b = 8/16 kernels, virtual shards, ragged and tall shapes, Alg. 4 RRQR, the sec. 3.4 V formation, the AUTO
fp32 QR-SVD branch, step-level entry points."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2209_04626_b200 as mp  # noqa: E402
import testmat  # noqa: E402


def dev(a):
    return torch.from_numpy(np.asfortranarray(a)).cuda().t().contiguous().t()


def main():
    torch.cuda.set_device(0)
    cases = [("C1", 192, {}), ("C2", 130, {"block_cols": 16}), ("C5", 128, {"block_cols": 8}),
             ("C1", 128, {"fp32_tensor_cores": 0}), ("C3", 128, {"virtual_shards": 2}),
             ("C1", 160, {"mp_rrqr": 1}), ("C1", 96, {"pdl_overlap": 0}),
             ("C3", 128, {"refine_v": 1}), ("C1", 128, {"path": 1, "tol_alg": 1e-3}),
             ("C2", 160, {"gram_tma": 1}), ("C2", 160, {"gram_tma": 0}), ("C1", 192, {"update_variant": 0}),
             ("C3", 128, {"switch_u": 0})]
    for name, n, opts in cases:
        a = testmat.config_matrix(name, n)
        U, S, V, st = mp.factor(dev(a), **opts)
        torch.cuda.synchronize()
        print(name, n, opts, "sweeps", st["sweeps32"], st["sweeps64"], "rc", st["rc"], flush=True)
    rng = np.random.default_rng(1)
    a = rng.standard_normal((300, 70))
    U, S, V, st = mp.factor(dev(a))
    torch.cuda.synchronize()
    print("tall", st["rc"], flush=True)
    g = torch.from_numpy(rng.standard_normal((3, 40, 40))).cuda()
    g = g @ g.transpose(1, 2)
    mp.inner_solve(g, 1e-12)
    mp.qr(dev(rng.standard_normal((200, 120))), pivot=1)
    mp.qr(dev(rng.standard_normal((200, 120))), pivot=3)
    torch.cuda.synchronize()
    print("sanitize run ok", flush=True)


if __name__ == "__main__":
    main()
