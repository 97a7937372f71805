"""Time the blocked Householder QR (mpjsvd_qr, pivot = 0) on an n x n random matrix; tools only.
usage: python tools/bench_qr.py [n] [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_04626_b200 as mp

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g).t()
h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream)
mp.qr(a, pivot=0, handle=h)
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    mp.qr(a, pivot=0, handle=h)
    e1.record()
    torch.cuda.synchronize()
    print(f"qr n={n}: {e0.elapsed_time(e1):.2f} ms (includes a {n}x{n} clone)")
h.close()
