"""Time the hand-written fp32 QR SVD step (mpjsvd_qrsvd32) at several n on the GPU (CUDA events)."""
import sys
import os
import json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_04626_b200 as mp
import testmat

out = {}
h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream)
for n in [int(x) for x in (sys.argv[1:] or ["512", "1024", "2048", "4096"])]:
    a = testmat.config_matrix("C3", n)
    x = torch.from_numpy(np.ascontiguousarray((a / np.abs(a).max()).astype(np.float32).T)).t().cuda()
    mp.qrsvd32(x, handle=h)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    U, S = mp.qrsvd32(x, handle=h)
    e1.record()
    torch.cuda.synchronize()
    out[n] = e0.elapsed_time(e1)
    print(n, round(out[n], 2), "ms", flush=True)
print(json.dumps(out))
