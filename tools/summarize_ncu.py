"""Summarise ncu reports / launch lists into profiles/ (tracked). Usage:
  python tools/summarize_ncu.py <tag> <report.ncu-rep>... [--launches launches.csv]"""
import csv, io, json, subprocess, sys, collections

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "gpc__cycles_elapsed.max",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]

def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = r[i] + (f" {units[i]}" if units[i] else "")
        res.append(d)
    return res

def launches(path):
    agg = collections.defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:80]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    return {"total_us": tot, "kernels": sorted(([k, n, round(us, 1), round(100 * us / tot, 2)] for k, (n, us) in agg.items()),
                                               key=lambda x: -x[2])}

if __name__ == "__main__":
    tag = sys.argv[1]
    out = {"tag": tag, "reports": {}, "launch_list": None}
    args = sys.argv[2:]
    if "--launches" in args:
        i = args.index("--launches")
        out["launch_list"] = launches(args[i + 1])
        args = args[:i] + args[i + 2:]
    for p in args:
        out["reports"][p.split("/")[-1]] = report(p)
    json.dump(out, open(f"profiles/{tag}_ncu_summary.json", "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])
