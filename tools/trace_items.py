"""Per-item device timeline of one CTA-pair launch inside a real learner step (tc_core.cuh
trace_item): for every work item, the median over CTAs (and the spread max - min) of
  reach  producer reaches the item (before its cross-CTA dependency wait)
  load0  first TMA load issued          dep   mid-item (k-block 32) load issued
  loadN  last TMA load issued           mma0  first stage landed at the MMA warp
  mmaN   last MMA committed             acc   epilogue sees the accumulator   epi  epilogue done
Usage: trace_items.py <n> [<n> ...]   (n = 1-based pair-kernel launch within the step)
Env: TRACE_H (model width, default 1024), TRACE_ITEMS (items to print, default 12)."""
import sys, os, ctypes as C
os.environ["ADPSGD_NO_GRAPHS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2110_11199_b200 import LearnerGroup, ModelDesc, StrategyConfig, Precision, _lib

CTAS, EV, ITEMS, IEV = 160, 48, 64, 12
NAMES = ["load0", "dep", "loadN", "mma0", "mmaN", "acc", "epi", "reach"]
ORDER = [7, 0, 1, 2, 3, 4, 5, 6]


def main():
    ns = [int(x) for x in sys.argv[1:]] or [3]
    H = int(os.environ.get("TRACE_H", "1024"))
    show = int(os.environ.get("TRACE_ITEMS", "12"))
    g = LearnerGroup(ModelDesc(hidden=H), StrategyConfig(learners=1, batch=1024, seed=1), precision=Precision.BF16)
    g.synth_dataset(4096, 4096, 3)
    g.step(0.1)
    L = _lib.lib()
    DI, DK = 8, 64
    words = CTAS * EV + CTAS * ITEMS * IEV + 2 * DI * DK * 3
    for n in ns:
        buf = (C.c_uint64 * words)()
        L.adpsgd_debug_trace(n, None, 0)
        g.step(0.1)
        L.adpsgd_debug_trace(0, buf, words)
        a = np.array(buf, dtype=np.uint64).astype(np.int64)
        it = a[CTAS * EV:CTAS * EV + CTAS * ITEMS * IEV].reshape(CTAS, ITEMS, IEV)
        det = a[CTAS * EV + CTAS * ITEMS * IEV:].reshape(2, DI, DK, 3)
        ctas = int((a[:CTAS * EV].reshape(CTAS, EV)[:, 46] > 0).sum())
        valid = it[:, :, :8] > 0
        if not valid.any():
            print(f"launch {n}: no item stamps")
            continue
        t0 = it[:, :, :8][valid].min()
        rel = np.where(valid, (it[:, :, :8] - t0) / 1000.0, np.nan)
        nitems = int(np.isfinite(rel[:, :, 4]).any(axis=0).sum())
        end = np.nanmax(rel)
        print(f"launch {n}: ctas {ctas} items {nitems} span {end:.1f} us ({end / max(nitems, 1):.2f} us per item)")
        print("  item " + " ".join(f"{NAMES[e]:>13s}" for e in ORDER) + "   mma(N-0)  dep-wait")
        for i in list(range(min(show, nitems))) + ([nitems - 1] if nitems > show else []):
            cells = []
            for e in ORDER:
                col = rel[:, i, e]
                if np.isfinite(col).any():
                    cells.append(f"{np.nanmedian(col):7.1f}±{np.nanmax(col) - np.nanmin(col):5.1f}")
                else:
                    cells.append(f"{'-':>13s}")
            mma = np.nanmedian(rel[:, i, 4] - rel[:, i, 3]) if np.isfinite(rel[:, i, 3]).any() else float("nan")
            dw = np.nanmedian(rel[:, i, 0] - rel[:, i, 7]) if np.isfinite(rel[:, i, 7]).any() else float("nan")
            ck = it[:, i, 11] - it[:, i, 10]
            okc = (it[:, i, 10] > 0) & (it[:, i, 11] > 0)
            clk = f"  {np.median(ck[okc]):9.0f} clk" if okc.any() else ""
            print(f"  {i:4d} " + " ".join(cells) + f"   {mma:7.2f}  {dw:7.2f}{clk}")
        stamps = a[:CTAS * EV].reshape(CTAS, EV).astype(np.int64)
        for ev in (40, 41, 42, 43, 44, 45):
            col = stamps[:, ev]
            if (col > 0).any():
                print(f"  stamp ev{ev}: median {np.median((col[col > 0] - t0) / 1000.0):.2f} us")
        # steady-state averages over items 4 .. n-2
        if nitems > 8:
            sl = slice(4, nitems - 2)
            d = lambda x, y: np.nanmedian(rel[:, sl, x] - rel[:, sl, y])
            step = np.nanmedian(np.diff(np.nanmedian(rel[:, :nitems, 4], axis=0))[4:nitems - 2])
            print(f"  steady state: item period {step:.2f} us; mma0->mmaN {d(4, 3):.2f}; load0->loadN {d(2, 0):.2f}; "
                  f"reach->load0 (dependency wait) {d(0, 7):.2f}; mmaN->epi {d(6, 4):.2f}; acc->epi {d(6, 5):.2f}")
            fw = np.nanmedian(np.where(it[:, sl, 8] > 0, it[:, sl, 8] / 1000.0, np.nan))
            ew = np.nanmedian(np.where(it[:, sl, 9] > 0, it[:, sl, 9] / 1000.0, np.nan))
            print(f"  per item: MMA warp waiting for full stages {fw:.2f} us; producer waiting for empty stages {ew:.2f} us")
            clk = it[:, sl, 11] - it[:, sl, 10]
            ns = it[:, sl, 4] - it[:, sl, 3]
            ok = (it[:, sl, 10] > 0) & (it[:, sl, 11] > 0) & (ns > 0)
            if ok.any():
                print(f"  SM clock during the MMA phase: {np.median(clk[ok] / ns[ok]) * 1000:.0f} MHz")
        if os.environ.get("TRACE_DETAIL"):
            item = int(os.environ["TRACE_DETAIL"])
            d0 = det[0, item]
            base = d0[d0 > 0].min() if (d0 > 0).any() else 0
            print(f"  detail item {item} (CTA 0 / CTA 1 issue, CTA 0 stage full), us from first issue:")
            for kb in range(DK):
                i0, f0, i1, g0 = det[0, item, kb, 0], det[0, item, kb, 1], det[1, item, kb, 0], det[0, item, kb, 2]
                if i0 == 0 and f0 == 0:
                    continue
                f = lambda x: f"{(x - base) / 1000.0:7.2f}" if x > 0 else "      -"
                print(f"    kb {kb:2d}: got-empty {f(g0)} issued {f(i0)} (issue took {(i0 - g0) / 1000.0 if g0 and i0 else float('nan'):5.2f}) / CTA1 {f(i1)}  full {f(f0)}  latency {(f0 - max(i0, i1)) / 1000.0 if f0 and i0 and i1 else float('nan'):6.2f}")
    L.adpsgd_debug_trace(0, None, 0)


if __name__ == "__main__":
    main()
