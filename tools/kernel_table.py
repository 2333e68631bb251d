"""Per-kernel evidence table (markdown) from ncu --set full reports: duration, tensor-pipe and
TMEM activity, DRAM traffic and bandwidth, L2 throughput, plus algorithmic TFLOP/s or GB/s where
the launch's work is known. Usage: kernel_table.py out.md name=report.ncu-rep[:flops|:bytes=N] ..."""
import csv, io, subprocess, sys

KEYS = {
    "dur_us": "gpu__time_duration.sum",
    "tensor_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "tmem_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "grid": "launch__grid_size",
    "ops": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum",
    "ops_pct": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum.pct_of_peak_sustained_elapsed",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
        "nsecond": 1e-3}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    res = []
    for v in r[2:]:
        d = {"name": v[h.index("Kernel Name")]}
        for k, m in KEYS.items():
            if m in h:
                i = h.index(m)
                try:
                    x = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = x * UNIT.get(u[i], 1) if k in ("dur_us", "dram_rd", "dram_wr") else x
        res.append(d)
    return res


def main():
    if len(sys.argv) < 3 or not sys.argv[1].endswith(".md") or "=" not in sys.argv[2]:
        sys.exit(__doc__)
    out = sys.argv[1]
    lines = ["| kernel | launch | µs | tensor pipe % | UTCHMMA TFLOP/s | dense tensor % | TMEM % | DRAM rd+wr (MB) "
             "| DRAM GB/s | L2 % | algorithmic |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for spec in sys.argv[2:]:
        name, rest = spec.split("=", 1)
        parts = rest.split(":")
        path, work = parts[0], (parts[1] if len(parts) > 1 else "")
        for i, d in enumerate(rows(path)):
            us = d.get("dur_us", 0.0)
            dram = d.get("dram_rd", 0.0) + d.get("dram_wr", 0.0)
            alg = ""
            if work.startswith("flops="):
                alg = f"{float(work[6:]) / (us * 1e-6) / 1e12:.0f} TFLOP/s"
            elif work.startswith("bytes="):
                alg = f"{float(work[6:]) / (us * 1e-6) / 1e9:.0f} GB/s"
            ops = d.get("ops", 0.0)
            lines.append(f"| {name} | {i} (grid {int(d.get('grid', 0))}) | {us:.1f} | {d.get('tensor_pct', 0):.1f} | "
                         f"{ops / (us * 1e-6) / 1e12:.0f} | {2 * d.get('ops_pct', 0):.1f} | "
                         f"{d.get('tmem_pct', 0):.1f} | {dram / 1e6:.0f} | {dram / (us * 1e-6) / 1e9:.0f} | "
                         f"{d.get('l2_pct', 0):.1f} | {alg} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
