"""Weight-gradient GEMM (both operands MN-major, K = 21504) at 256- vs 512-wide CTA-pair tiles:
dW_ih-like [4096 x 2048] (ADPSGD_FORCE_EXT=1 takes the one-wave 512-wide path)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_11199_b200 import _lib
M, N, K = 4096, 2048, 21504
A = torch.randn(K, M, device="cuda").to(torch.bfloat16)
B = torch.randn(K, N, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.float32)
s = torch.cuda.current_stream().cuda_stream
f = lambda: _lib.check(_lib.lib().adpsgd_gemm(1, M, N, K, A.data_ptr(), A.stride(0), 1, B.data_ptr(), B.stride(0), 1,
                                           C.data_ptr(), C.stride(0), 0, 1.0, 0, None, s))
for _ in range(3): f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(10): f()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
ref = (A.float().t() @ B.float())
err = ((C - ref).norm() / ref.norm()).item()
print(f"force_ext={os.environ.get('ADPSGD_FORCE_EXT', '0')}: {ms*1000:.1f} us {2.0*M*N*K/ms/1e9:.1f} TF/s rel err {err:.2e}")
