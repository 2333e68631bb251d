"""Sensitivity of the fp32 engine gradient to a bf16-sized weight perturbation (conditioning check)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, StrategyConfig
M, H, L, T, C = [int(a) for a in sys.argv[1:6]] if len(sys.argv) > 5 else (256, 1024, 6, 21, 32000)
m = ModelDesc(layers=L, hidden=H, bidirectional=True, input_dim=260, proj=256, classes=C, unroll=T)
rng = np.random.default_rng(101)
n_seg = 512
feats = rng.normal(size=(n_seg, T, 260)).astype(np.float32)
labels = rng.integers(0, C, size=(n_seg, T)).astype(np.int32)
idx = rng.integers(0, n_seg, size=M).astype(np.int32)
g = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=3), precision=Precision.FP32)
g.set_dataset(feats, labels, n_seg)
w = g.weights(0).copy()
wr = torch.from_numpy(w).to(torch.bfloat16).float().numpy()
l0, g0 = g.gradient(w, idx)
l1, g1 = g.gradient(wr, idx)
print(f"weights |w| {np.linalg.norm(w):.3e} max {np.abs(w).max():.3e}")
print(f"fp32(w) vs fp32(bf16(w)): loss {l0:.6f} {l1:.6f} grad rel {np.linalg.norm(g1-g0)/np.linalg.norm(g0):.3e}")
gb = LearnerGroup(m, StrategyConfig(learners=1, batch=M, seed=3), precision=Precision.BF16)
gb.set_dataset(feats, labels, n_seg)
l2, g2 = gb.gradient(w, idx)
l3, g3 = gb.gradient(wr, idx)
print(f"bf16(w) vs fp32(bf16 w): grad rel {np.linalg.norm(g3-g1)/np.linalg.norm(g1):.3e}; bf16 run-to-run(w,wr) {np.linalg.norm(g3-g2)/np.linalg.norm(g2):.3e}")
