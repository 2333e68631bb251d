"""Microbenchmark of the tcgen05 GEMM (adpsgd_gemm) across shapes and operand majorness,
against torch.matmul (cuBLAS) on the same shapes, CUDA-event timed."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_11199_b200 import _lib

def run(M, N, K, amn, bmn, cbf16=0, reps=20):
    A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if amn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if bmn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if cbf16 else torch.float32)
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.check(_lib.lib().adpsgd_gemm(1, M, N, K, A.data_ptr(), A.stride(0), amn, B.data_ptr(), B.stride(0), bmn,
                                               C.data_ptr(), C.stride(0), cbf16, 1.0, 0, None, s))
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    a = A.t() if amn else A
    b = B if bmn else B.t()
    for _ in range(3): torch.matmul(a, b)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): torch.matmul(a, b)
    e1.record(); torch.cuda.synchronize()
    cms = e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * K / ms / 1e9
    print(f"M={M:6d} N={N:6d} K={K:6d} amn={amn} bmn={bmn} c_bf16={cbf16}: {ms*1000:9.1f} us {tf:7.1f} TF/s | cuBLAS {cms*1000:9.1f} us {2.0*M*N*K/cms/1e9:7.1f} TF/s", flush=True)

for amn, bmn in [(0,0),(0,1),(1,0),(1,1)]:
    run(8192, 8192, 8192, amn, bmn)
for amn, bmn in [(0,0),(0,1),(1,1)]:
    run(1024, 4096, 3072, amn, bmn)
    run(1024, 1024, 4096, amn, bmn)
run(21504, 8192, 2048, 0, 0)
run(21504, 2048, 8192, 0, 1)
run(4096, 2048, 21504, 1, 1)
run(21504, 32000, 256, 0, 0)
run(21504, 32000, 256, 0, 0, cbf16=1)
