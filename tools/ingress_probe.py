"""Per-SM operand ingress probe: the same 256x256 CTA-pair tile mainloop timed with 1..74 pairs
busy (M = 256 * pairs, N = 256, long K). If the time per tile grows with the number of busy
SMs, the limit is the chip-wide L2 throughput; if it stays flat, it is per SM."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ADPSGD_FORCE_BN"] = "256"
os.environ["ADPSGD_NO_STREAMK"] = "1"
import torch
from paper_2110_11199_b200 import _lib
K = 32768
CFGS = [tuple(int(c) for c in x) for x in os.environ.get("PROBE_CFGS", "01,11").split(",")]
PAIRS = [int(x) for x in os.environ.get("PROBE_PAIRS", "2,16,38,64,74").split(",")]
for amn, bmn in CFGS:
    for pairs in PAIRS:
        M, N = 256 * pairs, 256
        A = (torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")).to(torch.bfloat16)
        B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.float32)
        s = torch.cuda.current_stream().cuda_stream
        f = lambda: _lib.check(_lib.lib().adpsgd_gemm(1, M, N, K, A.data_ptr(), A.stride(0), amn, B.data_ptr(), B.stride(0), bmn,
                                                   C.data_ptr(), C.stride(0), 0, 1.0, 0, None, s))
        for _ in range(3): f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        kb = K // 64
        per_sm = 32 * 1024 * kb / (ms * 1e-3) / 1e9  # A 16 KB + B 16 KB per k-block per CTA
        print(f"amn={amn} bmn={bmn} pairs={pairs:3d}: {ms*1000:8.1f} us  {2.0*M*N*K/ms/1e9:7.1f} TF/s  "
              f"per-SM ingress {per_sm:6.1f} GB/s  chip {per_sm*2*pairs/1000:6.2f} TB/s", flush=True)
