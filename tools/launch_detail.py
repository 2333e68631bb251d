"""Per-launch detail of one learner step from an ncu launch list (gpu__time_duration.sum +
launch__grid_size): prints the step's launches in order with grid and duration, and per-class
totals. Usage: launch_detail.py launches.csv [first_launch_id] [count]"""
import csv, sys, collections
path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = collections.OrderedDict()
for r in csv.DictReader(lines):
    k = int(r["ID"])
    d = rows.setdefault(k, {"name": r["Kernel Name"]})
    v = float(r["Metric Value"].replace(",", ""))
    if r["Metric Name"] == "gpu__time_duration.sum":
        scale = {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
        d["us"] = v * scale
    else:
        d[r["Metric Name"]] = v
ids = list(rows)
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else len(ids)
tot = collections.defaultdict(float)
for k in ids[first:first + count]:
    d = rows[k]
    n = d["name"]
    short = n.split("(")[0].replace("void ", "").replace("ab::", "").replace("<unnamed>::", "").replace("tc::", "")[:90]
    grid = int(d.get("launch__grid_size", 0))
    tot[short] += d.get("us", 0)
    if d.get("us", 0) > 20 or "Gen" in short:
        print(f"{k:5d} {d.get('us', 0):9.1f} us grid {grid:4d} {short}")
print("---- totals (us) ----")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} {k}")
print("sum", sum(tot.values()))
