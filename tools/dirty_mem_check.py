"""Read-before-write check: fill (and free) device memory with garbage before creating the
engine context; the step results must not change (diagnosis). Usage: dirty_mem_check.py [fill]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig
m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=64, classes=96, unroll=7)
rng = np.random.default_rng(9)
batches = [(rng.normal(size=(64, m.unroll, m.input_dim)).astype(np.float32),
            rng.integers(0, m.classes, size=(64, m.unroll)).astype(np.int32)) for _ in range(3)]
def run():
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=64, seed=4), precision=Precision.BF16)
    out = [float(g.step_host_batch(0.1, f, l)[0]) for f, l in batches]
    w = g.weights(0).copy(); g.close()
    return out, w
clean = run()
for fill in (float("nan"), 3.0, -1e30):
    x = torch.empty(int(6e9) // 4, device="cuda", dtype=torch.float32).fill_(fill)
    torch.cuda.synchronize(); del x; torch.cuda.empty_cache()
    d = run()
    print(f"fill {fill}: losses {d[0]} vs clean {clean[0]}; weights equal {np.array_equal(d[1], clean[1])}", flush=True)
