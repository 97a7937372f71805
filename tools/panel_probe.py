import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2209_04626_b200 as mp
h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream)
for m in (8192, 2048):
    for n in (16, 32, 64, 128, 256):
        a = torch.randn(n, m, dtype=torch.float64, device="cuda").t()
        mp.qr(a, pivot=0, handle=h)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): mp.qr(a, pivot=0, handle=h)
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 5
        print(f"m={m} n={n}: {t*1000:.0f} us, {t*1000/n:.2f} us/col")
