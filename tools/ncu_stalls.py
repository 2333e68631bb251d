"""Top stall reasons + top stalled SASS lines of an ncu report (reads it with the local ncu)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw))); h, v = r[0], r[2]
get = lambda k: v[h.index(k)] if k in h else "?"
print("duration", get("gpu__time_duration.sum"), "regs", get("launch__registers_per_thread"),
      "inst", get("smsp__inst_executed.sum"))
st = []
for i, k in enumerate(h):
    if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"):
        try: st.append((float(v[i]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError: pass
print("stalls:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]; data = rows[2:]
iS = hh.index("Warp Stall Sampling (All Samples)"); iE = hh.index("Instructions Executed")
tot = sum(float(x[iS] or 0) for x in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
top = sorted(range(len(data)), key=lambda i: -float(data[i][iS] or 0))[:n]
for i in sorted(top):
    print(f"{i:5d} {data[i][1][:60]:60s} {100*float(data[i][iS] or 0)/tot:5.1f}% exec {data[i][iE]}")
