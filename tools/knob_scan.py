import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig
m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=64, classes=96, unroll=7)
rng = np.random.default_rng(9)
f, l = rng.normal(size=(64, m.unroll, m.input_dim)).astype(np.float32), rng.integers(0, m.classes, size=(64, m.unroll)).astype(np.int32)
for kv in ["", "ADPSGD_NO_FUSED", "ADPSGD_NO_PAIR", "ADPSGD_NO_WIDE", "ADPSGD_NO_SPLITK", "ADPSGD_NO_PERSIST", "ADPSGD_NO_PERSIST_FWD",
           "ADPSGD_NO_STREAMK", "ADPSGD_NO_XTRA", "ADPSGD_FORCE_EXT", "ADPSGD_NO_WIDE_GEMM", "ADPSGD_NO_FOLD_BIAS", "ADPSGD_FORCE_BN"]:
    for k in list(os.environ):
        if k.startswith("ADPSGD_"): del os.environ[k]
    if kv: os.environ[kv] = "256" if kv == "ADPSGD_FORCE_BN" else "1"
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=64, seed=4), precision=Precision.BF16)
    print(kv or "default", float(g.step_host_batch(0.1, f, l)[0]), flush=True)
    g.close()
