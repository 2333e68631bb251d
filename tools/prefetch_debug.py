import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig
m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=64, classes=96, unroll=7)
rng = np.random.default_rng(9)
batches = [(rng.normal(size=(64, m.unroll, m.input_dim)).astype(np.float32),
            rng.integers(0, m.classes, size=(64, m.unroll)).astype(np.int32)) for _ in range(5)]
def run(prefetch, graphs=True):
    os.environ["ADPSGD_NO_GRAPHS"] = "0" if graphs else "1"
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=64, seed=4), precision=Precision.BF16)
    out = []
    if prefetch: g.prefetch_host_batch(*batches[0])
    for i, (f, l) in enumerate(batches):
        if prefetch and i + 1 < len(batches): g.prefetch_host_batch(*batches[i + 1])
        loss = g.step_host_batch(0.1, f, l)[0]
        out.append((loss, g.weights(0).copy()))
    g.close()
    return out
A = run(False); B = run(True); E = run(False, graphs=False); E2 = run(False, graphs=False)
for name, X in (("prefetch", B), ("eager", E), ("eager2", E2)):
    print(name, [ (float(a[0]) == float(b[0]), bool(np.array_equal(a[1], b[1]))) for a, b in zip(A, X)])
def run_test_pattern():
    os.environ["ADPSGD_NO_GRAPHS"] = "0"
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=64, seed=4), precision=Precision.BF16)
    out = []
    g.prefetch_host_batch(*batches[0])
    for i, (f, l) in enumerate(batches):
        if i + 1 < len(batches) and i != 2:
            g.prefetch_host_batch(*batches[i + 1])
        if i == 3:
            g.prefetch_host_batch(*batches[0])
        out.append((g.step_host_batch(0.1, f, l)[0], g.weights(0).copy()))
    g.close()
    return out
for rep in range(2):
    T_ = run_test_pattern()
    print("test-pattern", [(float(a[0]) == float(b[0]), bool(np.array_equal(a[1], b[1]))) for a, b in zip(A, T_)])
    A2 = run(False)
    print("plain-again", [(float(a[0]) == float(b[0]), bool(np.array_equal(a[1], b[1]))) for a, b in zip(A, A2)])
