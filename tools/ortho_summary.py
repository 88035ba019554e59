"""Summarises the c4ortho bench line and its ncu launch list (tools/ortho_run.sh)."""
import csv
import json
import sys
from collections import defaultdict

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
lines = [x for x in open(f"{out}/ortho_bench.log") if x.startswith("{")]
if lines:
    d = json.loads(lines[-1])
    print("step ms", d["ms_per_step"], "frac", d["roofline"]["frac"], d["config"]["parity"][:60], "e2e ms", d["e2e"]["ms_per_step"])
rows = list(csv.DictReader(x for x in open(f"{out}/ortho_launches.csv") if x.startswith('"')))
by = defaultdict(dict)
for r in rows:
    by[(int(r["ID"]), r["Kernel Name"][:40])][r["Metric Name"]] = r["Metric Value"]
items = sorted(by.items())
last = [it for it in items if it[0][0] >= items[-1][0][0] - 40]
tot = 0.0
for (i, k), m in last:
    t = float(m["gpu__time_duration.sum"]) / 1e3
    byt = (float(m["dram__bytes_read.sum"]) + float(m["dram__bytes_write.sum"])) / 1e6
    print(f"{i:4d} {k:42s} {t:9.1f} us {byt:9.1f} MB {byt / t if t else 0:6.2f} TB/s")
