"""Which forward buffer differs between a correct and a wrong first step (diagnosis)."""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig, _lib
small = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=64, classes=96, unroll=7)
rng = np.random.default_rng(9)
f, l = rng.normal(size=(64, 7, 40)).astype(np.float32), rng.integers(0, 96, size=(64, 7)).astype(np.int32)
NAMES = {0: "X0", 1: "H0", 2: "H1", 100: "Y", 101: "row_loss", 102: "shadow", 200: "c0", 201: "c1", 300: "gates0", 301: "gates1"}
def small_run():
    g = LearnerGroup(small, StrategyConfig(learners=1, batch=64, seed=4), precision=Precision.BF16)
    bufs = {}
    # shadow before the step (the step's update rewrites it)
    sh = np.zeros(40_000_000, dtype=np.uint8)
    _lib.check(_lib.lib().adpsgd_debug_buffer(g.handle, 102, sh.ctypes.data, sh.nbytes))
    bufs["shadow0"] = sh[: 2 * g.D].copy()
    v = float(g.step_host_batch(0.1, f, l)[0])
    for w, n in NAMES.items():
        if w == 102: continue
        b = np.zeros(8_000_000, dtype=np.uint8)
        _lib.check(_lib.lib().adpsgd_debug_buffer(g.handle, w, b.ctypes.data, b.nbytes))
        bufs[n] = b
    g.close()
    return v, bufs
ref_v, ref = small_run()
bigs = [ModelDesc(layers=2, hidden=1024, bidirectional=True, input_dim=260, proj=256, classes=32000, unroll=21),
        ModelDesc(layers=1, hidden=512, bidirectional=True, input_dim=40, proj=256, classes=64, unroll=21),
        ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=260, proj=256, classes=520, unroll=11)]
for it in range(18):
    big = bigs[it % 3]
    g = LearnerGroup(big, StrategyConfig(learners=1, batch=256, seed=3), precision=Precision.BF16)
    r = np.random.default_rng(it)
    g.set_dataset(r.normal(size=(300, big.unroll, big.input_dim)).astype(np.float32),
                  r.integers(0, big.classes, size=(300, big.unroll)).astype(np.int32), 300)
    g.gradient(g.weights(0), r.integers(0, 300, size=256).astype(np.int32))
    g.close()
    v, b = small_run()
    if v != ref_v:
        diff = [k for k in ref if not np.array_equal(ref[k], b[k])]
        print(it, "BAD", v, "differs:", diff, flush=True)
        for k in diff:
            x, y = ref[k], b[k]
            idx = np.nonzero(x != y)[0]
            print("   ", k, "bytes differ", len(idx), "first", idx[:8], "last", idx[-4:], flush=True)
        break
    print(it, "ok", flush=True)
