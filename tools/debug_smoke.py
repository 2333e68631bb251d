"""Debug: which variant of the smoke configuration produces non-finite weights (GPU)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, Strategy, StrategyConfig

m = ModelDesc(layers=int(os.environ.get("DL", 2)), hidden=int(os.environ.get("DH", 32)), bidirectional=True,
              input_dim=int(os.environ.get("DI", 20)), proj=int(os.environ.get("DP", 16)), classes=int(os.environ.get("DC", 24)), unroll=int(os.environ.get("DT", 6)))
rng = np.random.default_rng(0)
feats = rng.normal(size=(64, m.unroll, m.input_dim)).astype(np.float32)
labels = rng.integers(0, m.classes, size=(64, m.unroll)).astype(np.int32)
B = int(os.environ.get('DB', 4))
for L in (1,):
    cfg = StrategyConfig(strategy=Strategy.ADPSGD_FM if L == 3 else Strategy.SDPSGD, learners=L, batch=B, seed=5)
    g = LearnerGroup(m, cfg, precision=Precision.BF16)
    g.set_dataset(feats, labels, 60)
    w0 = g.weights(0)
    loss, grad = g.gradient(w0, np.arange(B, dtype=np.int32))
    print("L", L, "gradient(): loss", loss, "grad finite", np.all(np.isfinite(grad)), "nonfinite idx", np.flatnonzero(~np.isfinite(grad))[:10])
    loss = g.step(0.1)
    w = g.weights(0)
    bad = np.flatnonzero(~np.isfinite(w))
    print("L", L, "step(): loss", loss, "nonfinite weights", bad.size, bad[:10])
    g.close()
