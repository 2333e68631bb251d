"""One small bf16 learner step that runs the persistent recurrent kernels (64-unit FwdPersistT /
BwdPersistTraits<2> forced with ADPSGD_NO_FWD_U32 / ADPSGD_NO_BWD_U32), the fused CE and the
generic tcgen05 GEMMs -- the target of the compute-sanitizer runs (memcheck / initcheck /
racecheck / synccheck) recorded in profiles/. Prints the kernel variants that ran."""
import os
import sys

os.environ.setdefault("ADPSGD_NO_FWD_U32", "1")
os.environ.setdefault("ADPSGD_NO_BWD_U32", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2110_11199_b200 import LearnerGroup, ModelDesc, Precision, Strategy, StrategyConfig, _lib  # noqa: E402

m = ModelDesc(layers=2, hidden=128, bidirectional=True, input_dim=40, proj=32, classes=64, unroll=int(sys.argv[1]) if len(sys.argv) > 1 else 4)
rng = np.random.default_rng(0)
n = 512
feats = rng.normal(size=(n, m.unroll, m.input_dim)).astype(np.float32)
labels = rng.integers(0, m.classes, size=(n, m.unroll)).astype(np.int32)
g = LearnerGroup(m, StrategyConfig(strategy=Strategy.ADPSGD_D1D, learners=1, batch=256, seed=3), precision=Precision.BF16)
g.set_dataset(feats, labels, n)
_lib.kernel_variants(reset=True)
for _ in range(2):
    loss = g.step(0.1)
print("loss", loss.tolist())
w = g.weights(0)
print("weights_sha", __import__("hashlib").sha256(w.tobytes()).hexdigest(), "finite", bool(np.isfinite(w).all()))
print("variants", sorted(_lib.kernel_variants(reset=True)))
import ctypes as C  # noqa: E402
for which, name in [(200, "c_state[l0]"), (201, "c_state[l1]"), (300, "gates[l0]"), (301, "gates[l1]"),
                    (400, "dH_a"), (401, "dH_b"), (1, "H_out[l0]"), (2, "H_out[l1]")]:
    a, n = C.c_uint64(), C.c_uint64()
    _lib.check(_lib.lib().adpsgd_debug_buffer_range(g.handle, which, C.byref(a), C.byref(n)))
    print(f"buffer {name:12s} 0x{a.value:x} .. 0x{a.value + n.value:x}")
g.close()
