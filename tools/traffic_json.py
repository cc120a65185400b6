"""Turn an ncu DRAM capture of tools/capture_traffic.py into bench.py's
profiles/r02_sweep_<workload>_<precision>.json (tools only).

    python tools/traffic_json.py gpurun_out/traffic_cfg3_fp64
reads <prefix>.csv (ncu --csv log) and <prefix>.json (the program's line);
the middle sweeps' DRAM read + write bytes are averaged per launch.
"""
import csv
import json
import os
import subprocess
import sys
import time

prefix = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
meta = json.loads(open(prefix + ".json").read().strip().splitlines()[-1])
per, dur, names = {}, {}, {}
with open(prefix + ".csv") as fh:
    for r in csv.DictReader(ln for ln in fh if not ln.startswith("==")):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(r["Metric Unit"], 1.0)
        v = float(r["Metric Value"].replace(",", "")) * scale
        names[r["ID"]] = r["Kernel Name"]
        if r["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[r["ID"]] = per.get(r["ID"], 0.0) + v
        elif r["Metric Name"] == "gpu__time_duration.sum":
            dur[r["ID"]] = v
def mode_of(name):
    """template arguments <T, G, VPL, MODE, PERM>: MODE 1 = a middle order"""
    t = name[name.index("sweep_kernel<") + len("sweep_kernel<"):]
    args = t[:t.index(">")].split(",")
    return int(args[3].strip()) if len(args) >= 5 else -1


mid = [i for i in per if mode_of(names[i]) == 1]
ids = mid or list(per)
commit = subprocess.run(["git", "-C", root, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                        text=True).stdout.strip()
out = dict(meta)
out.update({"dram_bytes_per_launch": sum(per[i] for i in ids) / len(ids),
            "ncu_ms_per_launch": 1e3 * sum(dur.get(i, 0.0) for i in ids) / len(ids),
            "launches": len(ids), "ncu_kernel_names": sorted({names[i] for i in ids}),
            "commit": commit, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
            "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                   "--clock-control none -k regex:sweep_kernel (cold-cache, serialised launches)"})
dst = os.path.join(root, "profiles", f"r02_sweep_{meta['workload']}_{meta['precision']}.json")
with open(dst, "w") as fh:
    json.dump(out, fh, indent=1)
print(dst, out["dram_bytes_per_launch"])
