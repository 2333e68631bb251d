"""Summarise tools/tensor_counters.sh output per kernel class: UTCHMMA bf16 math ops (ncu counts
2 per MAC: it equals the algorithmic FLOPs of the forward launch to 0.4 %), the ops rate over the
kernel's duration, and ncu's own percentages. Usage: tensor_counters.py <tag>_tensor.csv [out.md]"""
import collections
import csv
import sys

OPS = "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum"
PCT = OPS + ".pct_of_peak_sustained_elapsed"
PIPE = "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"
HMMA = "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"
CLK = "sm__cycles_elapsed.avg.per_second"
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "ms": 1e3, "msecond": 1e3}


def load(path):
    rows = collections.OrderedDict()
    for r in csv.DictReader([ln for ln in open(path) if ln.startswith('"')]):
        d = rows.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        if r["Metric Name"] == "gpu__time_duration.sum":
            v *= SCALE.get(r["Metric Unit"], 1e-3)
        d[r["Metric Name"]] = v
    return rows


def short(name):
    s = name.split("(")[0].replace("void ", "").replace("tc::", "").replace("unnamed>::", "")
    return s.replace("persistent_kernel_2cta<", "pair<").split(", FwdPParams")[0].split(", BwdPParams")[0][:72]


def main():
    rows = load(sys.argv[1])
    agg = collections.OrderedDict()
    for d in rows.values():
        if d.get(OPS, 0) <= 0:
            continue
        a = agg.setdefault(short(d["name"]), collections.defaultdict(float))
        us = d["gpu__time_duration.sum"]
        a["n"] += 1
        a["us"] += us
        a["ops"] += d[OPS]
        for m in (PCT, PIPE, HMMA, CLK):  # duration-weighted means
            a[m] += d.get(m, 0.0) * us
    out = ["| kernel | launches | µs / launch | UTCHMMA GFLOP / launch | counter TFLOP/s | ops % of ncu peak "
           "| pipe_tensor realtime % | hmma subpipe % | SM MHz |", "|---|---|---|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        us = a["us"]
        out.append(f"| `{k}` | {int(a['n'])} | {us / a['n']:.1f} | {a['ops'] / a['n'] / 1e9:.1f} | "
                   f"{a['ops'] / us / 1e6:.0f} | {a[PCT] / us:.1f} | {a[PIPE] / us:.1f} | {a[HMMA] / us:.1f} | "
                   f"{a[CLK] / us / 1e6:.0f} |")
    tot_ops = sum(a["ops"] for a in agg.values())
    tot_us = sum(a["us"] for a in agg.values())
    out.append(f"\nAll tcgen05 kernels: {tot_ops / tot_us / 1e6:.0f} TFLOP/s by the UTCHMMA counter over their "
               f"summed ncu durations ({tot_ops / 1e12:.2f} TFLOP in {tot_us / 1e3:.1f} ms).")
    text = "\n".join(out)
    print(text)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text + "\n")


if __name__ == "__main__":
    main()
