"""Probe fixed overhead vs per-k-block cost of the tcgen05 GEMM on the recurrent shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_11199_b200 import _lib

def t(M, N, K, amn=0, bmn=0, reps=50):
    A = (torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")).to(torch.bfloat16)
    B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda")
    f = lambda: _lib.check(_lib.lib().adpsgd_gemm(1, M, N, K, A.data_ptr(), A.stride(0), amn, B.data_ptr(), B.stride(0), bmn,
                                               C.data_ptr(), C.stride(0), 0, 1.0, 0, None, torch.cuda.current_stream().cuda_stream))
    for _ in range(3): f()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay(); torch.cuda.synchronize(); e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000

mode = os.environ.get("ADPSGD_NO_PAIR", "0")
for (M, N) in [(1024, 4096), (1024, 1024), (2048, 4096), (8192, 8192)]:
    row = []
    for K in [256, 1024, 3072, 6144]:
        us = t(M, N, K)
        row.append(f"K={K}: {us:7.1f}us {2*M*N*K/us/1e6:6.0f}TF")
    print(f"pair_off={mode} M={M} N={N} | " + " | ".join(row), flush=True)
