"""cuBLAS (torch bf16) calibration of the learner-step GEMM shapes: what a library GEMM reaches
on the exact per-time-step / per-layer shapes (CUDA-event timed, warm L2 for small shapes)."""
import torch

def t(f, reps=30):
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

bf = torch.bfloat16
def case(name, b, M, N, K):
    A = torch.randn(b, M, K, device="cuda", dtype=bf); B = torch.randn(b, K, N, device="cuda", dtype=bf)
    ms = t(lambda: torch.bmm(A, B))
    print(f"{name:28s} b={b} M={M:6d} N={N:6d} K={K:6d}: {ms*1000:8.1f} us {2.0*b*M*N*K/ms/1e9:7.1f} TF/s", flush=True)

case("rec fwd [x|h][Wih|Whh]^T", 2, 1024, 4096, 3072)
case("rec fwd h Whh^T only", 2, 1024, 4096, 1024)
case("rec bwd dz Whh", 2, 1024, 1024, 4096)
case("input proj hoisted", 1, 21504, 8192, 2048)
case("input proj per dir", 2, 21504, 4096, 2048)
case("dgrad_x", 1, 21504, 2048, 8192)
case("wgrad dW_ih per dir", 2, 4096, 2048, 21504)
case("wgrad dW_hh per dir", 2, 4096, 1024, 20480)
case("CE logits", 1, 21504, 32000, 256)
case("dY = dl W_out", 1, 21504, 256, 32000)
case("dW_out", 1, 32000, 256, 21504)
case("dW_out+1", 1, 32000, 257, 21504)
