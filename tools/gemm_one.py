"""Run one GEMM shape a few times (for ncu). Usage: gemm_one.py M N K amn bmn cbf16"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_11199_b200 import _lib
M, N, K, amn, bmn, cb = map(int, sys.argv[1:7])
A = (torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")).to(torch.bfloat16)
B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if cb else torch.float32)
for _ in range(3):
    _lib.check(_lib.lib().adpsgd_gemm(1, M, N, K, A.data_ptr(), A.stride(0), amn, B.data_ptr(), B.stride(0), bmn,
                                      C.data_ptr(), C.stride(0), cb, 1.0, 0, None, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
