"""Time the library DMMA GEMM (mpjsvd_gemm_f64) at the path's shapes: TF/s vs the DMMA peak."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_04626_b200 as mp
import ctypes as C

h = mp.Handle(stream=torch.cuda.current_stream().cuda_stream)
L = mp.lib()
for (M, N, K, ta) in [(8192, 8192, 256, 0), (8192, 8192, 256, 1), (8192, 8192, 8192, 0), (4096, 4096, 256, 0),
                      (8192, 256, 8192, 1), (8192, 8192, 64, 0)]:
    A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda").t().contiguous().t() if False else None
    A = torch.randn(M * K, dtype=torch.float64, device="cuda")
    B = torch.randn(K * N, dtype=torch.float64, device="cuda")
    Cm = torch.zeros(M * N, dtype=torch.float64, device="cuda")
    lda = K if ta else M
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        rc = L.mpjsvd_gemm_f64(h.ptr, ta, 0, M, N, K, 1.0, C.c_void_p(A.data_ptr()), lda, C.c_void_p(B.data_ptr()), K,
                               0.0, C.c_void_p(Cm.data_ptr()), M)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"M={M} N={N} K={K} ta={ta}: {ms:.3f} ms  {2.0 * M * N * K / ms / 1e9:.1f} TF/s  rc={rc}", flush=True)
