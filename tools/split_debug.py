import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig
H=512; L=1; T=21; M=256; C=64
m = ModelDesc(layers=L, hidden=H, bidirectional=True, input_dim=40, proj=256, classes=C, unroll=T)
rng = np.random.default_rng(1)
feats = rng.normal(size=(300, T, 40)).astype(np.float32); labels = rng.integers(0, C, size=(300, T)).astype(np.int32)
idx = rng.integers(0, 300, size=M).astype(np.int32)
out = {}
w = None
for smax in sys.argv[1:]:
    os.environ["ADPSGD_SPLIT_MAX"] = smax
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=3), precision=Precision.BF16)
    g.set_dataset(feats, labels, 300)
    if w is None: w = g.weights(0)
    out[smax] = g.gradient(w, idx)[1]; g.close()
off = 0
for l in range(L):
    I = 40 if l == 0 else 2*H
    off += 2*(4*H*I + 4*H*H + 4*H)
Wp = slice(off, off + 256*2*H)
a = out[sys.argv[1]][Wp].reshape(256, 2*H); 
for s in sys.argv[2:]:
    b = out[s][Wp].reshape(256, 2*H)
    print("S", s, "total rel", np.linalg.norm(b-a)/np.linalg.norm(a))
    for n in range(2*H//256):
        errs = []
        for c in range(8):
            sl_ = (slice(None), slice(n*256+32*c, n*256+32*c+32))
            errs.append(np.linalg.norm(b[sl_]-a[sl_])/max(np.linalg.norm(a[sl_]),1e-30))
        print(" tile", n, " ".join(f"{e:.2e}" for e in errs))
    rows = [np.linalg.norm(b[r*32:(r+1)*32]-a[r*32:(r+1)*32])/np.linalg.norm(a[r*32:(r+1)*32]) for r in range(8)]
    print(" row blocks", " ".join(f"{e:.2e}" for e in rows))
