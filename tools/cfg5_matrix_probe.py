"""Run bench.py's configs[4] matrix alone and print each cell (tools only).

    python tools/cfg5_matrix_probe.py [--steps 4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
a = ap.parse_args()
m = bench.run_dynamic_cfg5_matrix(0, steps=a.steps)
for c in m["cells"]:
    print(json.dumps(c), flush=True)
for c in m.get("quality", {}).get("cells", []):
    print(json.dumps(c), flush=True)
