"""Device timeline (globaltimer, us) of CTA-pair tensor-core launches inside a real step.
Usage: trace_fwd.py <n> [<n> ...] : trace the n-th pair-kernel launch of the step (1-based).
Events per CTA: 4*i+0 MMA starts tile i (accumulator free), +1 first stage landed,
+2 last MMA committed, +3 epilogue of tile i done; 30 kernel start, 31 kernel end.
Prints, per launch, the median over CTAs of each event (relative to the earliest start)."""
import sys, os, ctypes as C
os.environ["ADPSGD_NO_GRAPHS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, StrategyConfig, Precision, _lib
ns = [int(x) for x in sys.argv[1:]] or [1]
H = int(os.environ.get("TRACE_H", "1024"))  # model width (shape P: 512)
g = LearnerGroup(ModelDesc(hidden=H), StrategyConfig(learners=1, batch=1024, seed=1), precision=Precision.BF16)
g.synth_dataset(4096, 4096, 3)
g.step(0.1)
L = _lib.lib()
names = {0: "mma_start", 1: "first_stage", 2: "last_mma", 3: "epi_done"}
for n in ns:
    buf = (C.c_uint64 * (160 * 48))()
    L.adpsgd_debug_trace(n, None, 0)
    g.step(0.1)
    L.adpsgd_debug_trace(0, buf, 160 * 48)
    a = np.array(buf, dtype=np.uint64).reshape(160, 48).astype(np.int64)
    ctas = int((a[:, 46] > 0).sum())
    t0 = a[a > 0].min()
    rel = np.where(a > 0, (a - t0) / 1000.0, np.nan)
    print(f"launch {n}: ctas {ctas} span {(a.max() - t0) / 1000.0:.1f} us")
    parts = [f"start {np.nanmedian(rel[:, 46]):.1f}", f"end {np.nanmedian(rel[:, 47]):.1f} (max {np.nanmax(rel[:, 47]):.1f})"]
    for i in range(10):
        for k in range(4):
            col = rel[:, 4 * i + k]
            if np.isfinite(col).any():
                parts.append(f"t{i}.{names[k]} {np.nanmedian(col):.1f}")
    for i in list(range(12, 40)) + [40, 41, 42, 43]:
        col = rel[:, i]
        if np.isfinite(col).any() and (i >= 40 or not np.isfinite(rel[:, 4 * (i // 4)]).any()):
            parts.append(f"ev{i} {np.nanmedian(col):.1f}")
    print("   ", " | ".join(parts))
L.adpsgd_debug_trace(0, None, 0)
