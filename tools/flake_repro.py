"""Reproducer hunt: alternate large and small contexts in one process; the small one's first-step
loss must always equal the oracle-checked value 4.5725398 (diagnosis)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig
small = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=64, classes=96, unroll=7)
rng = np.random.default_rng(9)
f, l = rng.normal(size=(64, 7, 40)).astype(np.float32), rng.integers(0, 96, size=(64, 7)).astype(np.int32)
PREC = Precision.FP32 if os.environ.get("REPRO_FP32") else Precision.BF16
def small_loss():
    g = LearnerGroup(small, StrategyConfig(learners=1, batch=64, seed=4), precision=PREC)
    v = float(g.step_host_batch(0.1, f, l)[0]); g.close(); return v
REF = small_loss()
print("ref", REF, flush=True)
big_models = [ModelDesc(layers=2, hidden=1024, bidirectional=True, input_dim=260, proj=256, classes=32000, unroll=21),
              ModelDesc(layers=1, hidden=512, bidirectional=True, input_dim=40, proj=256, classes=64, unroll=21),
              ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=260, proj=256, classes=520, unroll=11)]
bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    bm = big_models[it % len(big_models)]
    M = 256
    g = LearnerGroup(bm, StrategyConfig(learners=1, batch=M, seed=3), precision=Precision.BF16)
    r = np.random.default_rng(it)
    g.set_dataset(r.normal(size=(300, bm.unroll, bm.input_dim)).astype(np.float32),
                  r.integers(0, bm.classes, size=(300, bm.unroll)).astype(np.int32), 300)
    g.gradient(g.weights(0), r.integers(0, 300, size=M).astype(np.int32))
    g.close()
    v = [small_loss() for _ in range(3)]
    ok = all(x == REF for x in v)
    bad += not ok
    print(it, type(bm).__name__, bm.hidden, v, "OK" if ok else "BAD", flush=True)
print("bad", bad)

# direct GEMM check (the projection GEMM's shape) after big contexts
import torch
from paper_2110_11199_b200 import _lib
def proj_gemm(seed=0):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    A = torch.randn(448, 256, generator=gen, device="cuda").to(torch.bfloat16)
    B = torch.randn(64, 256, generator=gen, device="cuda").to(torch.bfloat16)
    bias = torch.randn(64, generator=gen, device="cuda")
    C = torch.zeros(448, 64, device="cuda", dtype=torch.bfloat16)
    _lib.check(_lib.lib().adpsgd_gemm(1, 448, 64, 256, A.data_ptr(), 256, 0, B.data_ptr(), 256, 0, C.data_ptr(), 64, 1, 1.0, 0,
                                      bias.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ref = (A.float() @ B.float().t() + bias).to(torch.bfloat16)
    return (C.float() - ref.float()).abs().max().item()
bad2 = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    bm = big_models[it % len(big_models)]
    g = LearnerGroup(bm, StrategyConfig(learners=1, batch=256, seed=3), precision=Precision.BF16)
    r = np.random.default_rng(it)
    g.set_dataset(r.normal(size=(300, bm.unroll, bm.input_dim)).astype(np.float32),
                  r.integers(0, bm.classes, size=(300, bm.unroll)).astype(np.int32), 300)
    g.gradient(g.weights(0), r.integers(0, 300, size=256).astype(np.int32))
    g.close()
    errs = [proj_gemm(s) for s in range(3)]
    bad2 += max(errs) > 0.1
    print("gemm", it, errs, flush=True)
print("gemm bad", bad2)
