"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(ln for ln in open(sys.argv[1]) if not ln.startswith("=="))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    nm = r["Kernel Name"].split("(")[0][:64]
    agg[nm][0] += 1
    agg[nm][1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
tot = sum(a[1] for a in agg.values())
print(f"{len(rows)} launches, {tot:.1f} us total")
for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{nm:64s} {c:6d} {t:10.1f} us {t / c:8.2f} us/launch {100 * t / tot:5.1f}%")
