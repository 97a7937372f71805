"""Per-round cost of the 2b x 2b inner solve (k_inner_solve_batch, same device code as k_pair_solve):
time `count` independent solves capped at S inner sweeps; (t(S2) - t(S1)) / ((S2 - S1) * 63) is the cost
of one inner round (w = 64)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_04626_b200 as mp  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    count, w = 128, 64
    for dtype in (torch.float32, torch.float64):
        x = torch.from_numpy(rng.standard_normal((count, 512, w))).to(dtype).cuda()
        g = (x.transpose(1, 2) @ x).contiguous()
        h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream)
        res = {}
        for s in (1, 2, 4, 8):
            for _ in range(3):
                mp.inner_solve(g, 1e-30, max_inner=s, handle=h)        # warm-up (tol tiny: every pair rotates)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = 20
            for _ in range(reps):
                mp.inner_solve(g, 1e-30, max_inner=s, handle=h)
            torch.cuda.synchronize()
            res[s] = (time.perf_counter() - t0) / reps * 1e6
        per_round = (res[8] - res[2]) / (6 * 63)
        print(f"{dtype}: launch us {', '.join(f'S={k}: {v:.1f}' for k, v in res.items())}; per inner round {per_round:.3f} us",
              flush=True)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def phases():
    """Per-warp-group end clocks of an inner round (diag_timing bit 8): critical warps, rotation warp, slowest
    other G warp, slowest E warp, cycles from the round start (the round ends at the CTA barrier after all)."""
    rng = np.random.default_rng(0)
    count, w = 128, 64
    for dtype in (torch.float32, torch.float64):
        x = torch.from_numpy(rng.standard_normal((count, 512, w))).to(dtype).cuda()
        g = (x.transpose(1, 2) @ x).contiguous()
        h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream, diag_timing=8)
        mp.inner_solve(g, 1e-30, max_inner=2, handle=h)
        torch.cuda.synchronize()


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "phases":
    phases()
