"""Per-basic-block instruction and stall-sample shares from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.split("\n", 1)[1]
r = list(csv.reader(out.splitlines()))
h = r[0]
ci = {n: i for i, n in enumerate(h)}
rows = r[1:]
ie = [int(x[ci["Instructions Executed"]] or 0) for x in rows]
st = [float(x[ci["Warp Stall Sampling (All Samples)"]] or 0) for x in rows]
tot, ts = sum(ie), sum(st)
print(f"warp instructions {tot}, stall samples {ts:.0f}")
blocks, cur = [], None
for i, (x, n, s) in enumerate(zip(rows, ie, st)):
    if cur is None or n != cur[1]:
        cur = [i, n, collections.Counter(), 0.0]
        blocks.append(cur)
    src = x[ci["Source"]].strip()
    op = (src.split()[1] if src.startswith("@") else src.split()[0]) if src else "?"
    cur[2][op.split(".")[0]] += 1
    cur[3] += s
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
for b0, n, c, s in blocks:
    share = n * sum(c.values()) / tot
    if share > thr or s / ts > thr:
        print(f"@{b0:5d} x{n:9d} instr {100 * share:5.1f}% stall {100 * s / ts:5.1f}%  {dict(c.most_common(6))}")

# per-reason stall samples inside the blocks listed on the command line (start indices)
if len(sys.argv) > 3:
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    starts = [int(v) for v in sys.argv[3].split(",")]
    for b0, n, c, s in blocks:
        if b0 in starts:
            end = b0 + sum(c.values())
            agg = {rn: sum(float(x[ci[rn]] or 0) for x in rows[b0:end]) for rn in reasons}
            tt = sum(agg.values())
            print(f"@{b0}: " + ", ".join(f"{k[6:]} {100 * v / tt:.0f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:7]))
