"""Repeat the prefetch/no-prefetch comparison; report the first diverging step (diagnosis)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig
m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=64, classes=96, unroll=7)
rng = np.random.default_rng(9)
batches = [(rng.normal(size=(64, m.unroll, m.input_dim)).astype(np.float32),
            rng.integers(0, m.classes, size=(64, m.unroll)).astype(np.int32)) for _ in range(5)]
def run(prefetch):
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=64, seed=4), precision=Precision.BF16)
    out = []
    if prefetch: g.prefetch_host_batch(*batches[0])
    for i, (f, l) in enumerate(batches):
        if prefetch and i + 1 < len(batches) and i != 2: g.prefetch_host_batch(*batches[i + 1])
        if prefetch and i == 3: g.prefetch_host_batch(*batches[0])
        out.append((float(g.step_host_batch(0.1, f, l)[0]), g.weights(0).copy()))
    g.close()
    return out
ref = run(False)
bad = 0
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    for pf in (False, True):
        o = run(pf)
        d = [i for i in range(5) if o[i][0] != ref[i][0] or not np.array_equal(o[i][1], ref[i][1])]
        if d:
            bad += 1
            i = d[0]
            print(f"rep {rep} prefetch={pf}: first diverging step {i}: loss {o[i][0]} vs {ref[i][0]}, "
                  f"max |dw| {np.abs(o[i][1]-ref[i][1]).max():.3e}", flush=True)
print("diverging runs:", bad)
