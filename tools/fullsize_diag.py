"""Full-size bf16 vs fp32 engine gradient, per parameter block (diagnosis). Usage: fullsize_diag.py [M] [H] [L] [T]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig
M = int(sys.argv[1]) if len(sys.argv) > 1 else 256
H = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
L = int(sys.argv[3]) if len(sys.argv) > 3 else 6
T = int(sys.argv[4]) if len(sys.argv) > 4 else 21
C = int(sys.argv[5]) if len(sys.argv) > 5 else 32000
m = ModelDesc(layers=L, hidden=H, bidirectional=True, input_dim=260, proj=256, classes=C, unroll=T)
rng = np.random.default_rng(101)
n_seg = 512
feats = rng.normal(size=(n_seg, T, 260)).astype(np.float32)
labels = rng.integers(0, C, size=(n_seg, T)).astype(np.int32)
idx = rng.integers(0, n_seg, size=M).astype(np.int32)
out = {}
w = None
for prec in (Precision.BF16, Precision.FP32):
    g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=3), precision=prec)
    g.set_dataset(feats, labels, n_seg)
    if w is None:
        w = g.weights(0)
    out[prec] = g.gradient(w, idx)
    g.close()
(lb, gb), (lf, gf) = out[Precision.BF16], out[Precision.FP32]
print(f"M={M} H={H} L={L} T={T} C={C}: loss bf16 {lb:.6f} fp32 {lf:.6f}  total rel {np.linalg.norm(gb-gf)/np.linalg.norm(gf):.3e}")
# block layout: per layer, per dir: W_ih [4H x I], W_hh [4H x H], b [4H]; then W_proj [256 x 2H], b_proj, W_out [C x 256], b_out
off = 0
names = []
for l in range(L):
    I = 260 if l == 0 else 2 * H
    for d in range(2):
        for nm, n in (("W_ih", 4 * H * I), ("W_hh", 4 * H * H), ("b", 4 * H)):
            names.append((f"L{l}d{d}.{nm}", off, off + n)); off += n
for nm, n in (("W_proj", 256 * 2 * H), ("b_proj", 256), ("W_out", C * 256), ("b_out", C)):
    names.append((nm, off, off + n)); off += n
assert off == gb.size, (off, gb.size)
for nm, a, b in names:
    x, y = gb[a:b], gf[a:b]
    ny = np.linalg.norm(y)
    print(f"{nm:12s} |g| {ny:10.3e}  rel {np.linalg.norm(x - y) / max(ny, 1e-30):9.3e}")
