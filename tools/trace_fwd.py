"""Device timeline (globaltimer, us) of one CTA-pair tensor-core launch inside a real step.
Usage: trace_fwd.py <n> : trace the n-th pair-kernel launch of the step (1-based).
Events per CTA: 4*i+0 MMA starts tile i (accumulator free), +1 first stage landed,
+2 last MMA committed, +3 epilogue of tile i done; 30 kernel start, 31 kernel end."""
import sys, os, ctypes as C
os.environ["ADPSGD_NO_GRAPHS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, StrategyConfig, Precision, _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = LearnerGroup(ModelDesc(), StrategyConfig(learners=1, batch=1024, seed=1), precision=Precision.BF16)
g.synth_dataset(4096, 4096, 3)
g.step(0.1)
buf = (C.c_uint64 * (160 * 32))()
L = _lib.lib()
L.adpsgd_debug_trace(n, None, 0)
g.step(0.1)
L.adpsgd_debug_trace(0, buf, 160 * 32)
a = np.array(buf, dtype=np.uint64).reshape(160, 32).astype(np.int64)
t0 = a[a > 0].min()
print("launch", n, "span us", (a.max() - t0) / 1000.0)
for cta in list(range(0, 148, 10)) + [146, 147]:
    row = a[cta]
    ev = [(i, (row[i] - t0) / 1000.0) for i in range(32) if row[i] > 0]
    print(cta, " ".join(f"{i}:{t:.1f}" for i, t in ev))
